// ntt_str14: the forward 16384-word block transform as TWO STREAMS per thread.
//
// Why: in ntt_grp14 the 16 warps of the CTA move through
// the block in lockstep, so while they exchange words through shared memory
// (about 30% of a block) nobody computes, although the hardware overlaps the
// FP64 pipe and the shared-memory path perfectly. After the forward's first
// stage (index bit 13) the block is two independent 8192-word transforms, A
// (bit 13 clear) and B. Here every thread carries 16 words of each and
// alternates between them: while one stream's words are in flight through
// shared memory the thread runs the other stream's stages, so the data
// movement hides behind arithmetic of the same warp and no barrier is waited
// on with nothing to do.
//
// Passes (block-local index j, S = j13 the stream; t = 32 w + l):
//   P1  bits 13..9 on 32 words, as ntt_grp14 (thread bits j0..j8: jt1): stage
//       13 on all 16 pairs, then stages 12..9 per stream
//   e1  CTA-wide exchange of each stream, in place in its half of the staging
//       buffer (after every warp has read its P1 words): P1's register bits
//       j9..j12 become warp bits, thread bits j5..j8 become registers
//   Q2  bits 8..5 on 16 words per stream; lanes j0..j4, warps j9..j12 (the
//       twiddles are warp-uniform)
//   e2  warp-local exchange (warp bits unchanged: only __syncwarp) through the
//       warp's 4 KiB of E: registers j5..j8 <-> lane bits, j1..j4 become registers
//   Q3  bits 4..1; lanes (j0, j5..j8), warps j9..j12
//   sh  lane pairs (l, l ^ 1) swap half their words by shuffle: j0 becomes a
//       register bit, j1 the lane bit
//   Q4  bit 0; then the canonical words of the stream go out: the warp's 512
//       words are contiguous in memory, written as a 4 KiB 128B-swizzled image
//       (the same 4 KiB of E) and stored by one bulk tensor store
// Both exchanges use 8-byte accesses with the 16-byte-chunk XOR swizzles
// derived below (conflict free on both sides; tests/test_str_layout.py).
//
// Twiddles: P1 and Q2 read the reference-order table (broadcast loads), Q3 and
// Q4 a table in (stream, entry, thread) order: entry 0 = stage bit 4, 1..2 =
// bit 3, 3..6 = bit 2, 7..14 = bit 1, 15..22 = bit 0 (kStrEntries = 23), so a
// warp's 32 loads are 32 consecutive entries. The butterflies, their order
// and the twiddles are the reference's (ntt.hpp:363-394): every arithmetic
// policy keeps its exactness argument.
#pragma once
#include "ntt_grp.cuh"

namespace nk {

constexpr int kStrEntries = 23;
constexpr uint32_t kStrTableWords = 2u * kStrEntries * 512u;  // per limb (and 16384-word block)

// thread index bits of each pass (block-local j without the stream bit)
struct StrMap {
  __host__ __device__ static constexpr uint32_t jt1(uint32_t w, uint32_t l) { return GrpMap<true>::jt1(w, l); }
  __host__ __device__ static constexpr uint32_t jt2(uint32_t w, uint32_t l) { return l | (w << 9); }
  __host__ __device__ static constexpr uint32_t jt3(uint32_t w, uint32_t l) {
    return (l & 1u) | ((l >> 1) << 5) | (w << 9);
  }
};

// table index (reference order, relative to the limb's table) of entry e of
// thread t in stream S, for a block at offset boff of a row of length n
__host__ __device__ constexpr uint64_t str_tw_index(uint64_t n, uint64_t boff, uint32_t S, int e, uint32_t t) {
  const uint32_t w = t >> 5, l = t & 31u;
  const uint64_t jb = boff + (static_cast<uint64_t>(S) << 13);
  if (e < 15) {
    // Q3 stage bit b, hi = the register bits above b
    const int b = e == 0 ? 4 : (e < 3 ? 3 : (e < 7 ? 2 : 1));
    const int hi = e == 0 ? 0 : (e < 3 ? e - 1 : (e < 7 ? e - 3 : e - 7));
    const uint64_t j = jb + StrMap::jt3(w, l) + (static_cast<uint64_t>(hi) << (b + 1));
    return (n + j) >> (b + 1);
  }
  // Q4: bit 0; registers (j2, j3, j4) = hi, lane bit 0 = j1
  const int hi = e - 15;
  const uint64_t j = jb + (StrMap::jt3(w, l) & ~1u) + ((l & 1u) << 1) + (static_cast<uint64_t>(hi) << 2);
  return (n + j) >> 1;
}

template <class A>
__device__ __forceinline__ const typename A::Tw* twq_of(const NttArgs& a, uint32_t limb) {
  const uint64_t per_limb = (a.n >> kB14) * kStrTableWords;
  if constexpr (std::is_same_v<typename A::Tw, uint64_t>) return a.twq8 + limb * per_limb;
  else return a.twq + limb * per_limb;
}

// [1 KiB align][staging 128 KiB][E 64 KiB][limb constants x2][mbarriers: full, P1 reads, e1 A, e1 B][counter]
constexpr size_t kStrSmemBytes = 1024 + kStageBytes + kGrpExBytes + 2 * sizeof(LimbConst) + 8 * 8;

namespace str {

// K stages (forward order: bit LO + K - 1 first) on the 16 registers x[0..15]
// whose index bits are j_LO .. j_{LO+3}; the twiddle of stage bit b, position
// hi (the register bits above b) comes from `twf(i, hi)`, i = b - LO.
// GS0: the first stage's number from the block's first stage (fwd_skip14).
template <class A, int NST, int GS0, class F>
__device__ __forceinline__ void pass16(uint64_t* x, const LimbConst& c, F&& twf) {
#pragma unroll
  for (int s = 0; s < NST; ++s) {
    const int i = 3 - s;
#pragma unroll
    for (int hi = 0; hi < (16 >> (i + 1)); ++hi) {
      const typename A::Tw w = twf(i, hi);
#pragma unroll
      for (int lo = 0; lo < (1 << i); ++lo) {
        const int r0 = (hi << (i + 1)) | lo, r1 = r0 | (1 << i);
        if (fwd_skip14<A>(false, GS0 + s, 1 << 30)) A::template fwd<true>(x[r0], x[r1], w, c);
        else A::template fwd<false>(x[r0], x[r1], w, c);
      }
    }
  }
}

// The inverse's stages (bit LO first) on 16 registers; twiddles as in pass16.
template <class A, class F>
__device__ __forceinline__ void pass16i(uint64_t* x, const LimbConst& c, F&& twf) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int hi = 0; hi < (16 >> (i + 1)); ++hi) {
      const typename A::Tw w = twf(i, hi);
#pragma unroll
      for (int lo = 0; lo < (1 << i); ++lo) {
        const int r0 = (hi << (i + 1)) | lo, r1 = r0 | (1 << i);
        // canonical-only policies: both inputs are products of stage i - 1 when that stage's
        // register bit is set: their sum needs no reduction (kInvSkipTT, modmath.cuh)
        if (inv_skip_tt<A>() && i > 0 && ((lo >> (i - 1)) & 1)) A::template inv<true>(x[r0], x[r1], w, c);
        else A::template inv<false>(x[r0], x[r1], w, c);
      }
    }
  }
}

// the same stages on both streams at once (x and x + 16), stage by stage: 16 independent butterflies per stage
template <class A, int NST, int GS0, class FA, class FB>
__device__ __forceinline__ void pass16x2(uint64_t* x, const LimbConst& c, FA&& twa, FB&& twb) {
#pragma unroll
  for (int s = 0; s < NST; ++s) {
    const int i = 3 - s;
#pragma unroll
    for (int hi = 0; hi < (16 >> (i + 1)); ++hi) {
      const typename A::Tw wa = twa(i, hi);
      const typename A::Tw wb = twb(i, hi);
#pragma unroll
      for (int lo = 0; lo < (1 << i); ++lo) {
        const int r0 = (hi << (i + 1)) | lo, r1 = r0 | (1 << i);
        if (fwd_skip14<A>(false, GS0 + s, 1 << 30)) {
          A::template fwd<true>(x[r0], x[r1], wa, c);
          A::template fwd<true>(x[16 + r0], x[16 + r1], wb, c);
        } else {
          A::template fwd<false>(x[r0], x[r1], wa, c);
          A::template fwd<false>(x[16 + r0], x[16 + r1], wb, c);
        }
      }
    }
  }
}

}  // namespace str

namespace str {

// The stamps of an NK_DBG_TIMELINE build (NK_GTS, ntt_grp.cuh) use `a`, `l`, `w`, `it_` of the caller.

// Forward core: from the block in the staging buffer (bar_full waited by the
// caller) to the Q4 results: v[16 S + 2 hi + j0] of stream S, with lane bit 0 =
// j1, lane bits 1..4 = j5..j8, warp = j9..j12, before the final reduction.
// `par_rd` / `par_w`: parities of bar_rd / bar_w for this transform; `before_e2` runs before
// the warp's 4 KiB buffer is first written (e.g. waits for a store that still
// reads it); `consumed` once this warp has read its last staging word.
template <class A, bool ILTM0, class FPRE, class FCONS>
__device__ __forceinline__ void fwd_core(uint64_t (&v)[32], uint8_t* St, uint8_t* Ew, const LimbConst& c,
                                         const NttArgs& a, const typename A::Tw* __restrict__ tw,
                                         const typename A::Tw* __restrict__ twq, uint64_t xbase, uint32_t w,
                                         uint32_t l, uint64_t* bar_rd, uint64_t* bar_w, uint32_t par_rd,
                                         uint32_t par_w, uint32_t it_, FPRE&& before_e2, FCONS&& consumed) {
  using P1 = PassD<9, 5, -1>;
  using Tw = typename A::Tw;
  (void)it_;
  // ---- thread-constant byte offsets ----
  const uint32_t jt1 = StrMap::jt1(w, l);
  // e1, write side: stream word j' = jt1 | r << 9 at chunk-swizzled position
  //   phys(j') = j' ^ (((j' >> 4) & 7) << 1): the half-warp's lanes (j0, j4, j5, j6) hit 16 distinct 8-byte slots
  const uint32_t e1w = (jt1 ^ (((jt1 >> 4) & 7u) << 1)) << 3;  // + r * 4096 + S * 65536
  // e1, read side: j' = l | r << 5 | w << 9 (lanes j0..j4): (base ^ ((r & 3) << 5)) + r * 256
  const uint32_t e1r = ((l ^ ((l >> 4) << 1)) << 3) + (w << 12);
  // e2 (warp-local, word m = j & 511 at m ^ (((m >> 5) & 7) << 1)): write (l << 3 ^ (r & 7) << 4) + r * 256,
  // read tb ^ (r3 << 4)
  const uint32_t e2w = l << 3;
  const uint32_t e2r = ((l & 1u) << 3) | (((l >> 1) & 7u) << 4) | ((l >> 1) << 8);

  // ---- P1: words from the staging buffer, stage 13, then stages 12..9 per stream ----
  grp::p1_read<A, true>(v, St, jt1);
  __syncwarp();
  if (l == 0) mbar_arrive_local(bar_rd);
  NK_GTS(2);
  stages14<A, true, P1, ILTM0, 0, 1>(v, tw, tw, a.n, xbase + jt1, c);
  stages14<A, true, P1, ILTM0, 1, 5, 0>(v, tw, tw, a.n, xbase + jt1, c);
  NK_GTS(3);
  // e1 of stream A: in place in the lower half of the staging buffer
  mbar_wait(bar_rd, par_rd);
#pragma unroll
  for (int r = 0; r < 16; ++r) *reinterpret_cast<uint64_t*>(St + e1w + r * 4096) = v[r];
  __syncwarp();
  if (l == 0) mbar_arrive_local(bar_w);
  NK_GTS(4);
  stages14<A, true, P1, ILTM0, 1, 5, 1>(v, tw, tw, a.n, xbase + jt1, c);
#pragma unroll
  for (int r = 0; r < 16; ++r) *reinterpret_cast<uint64_t*>(St + 65536 + e1w + r * 4096) = v[16 + r];
  __syncwarp();
  if (l == 0) mbar_arrive_local(bar_w + 1);
  NK_GTS(5);

  // Twiddles. Q2: (N + j) >> (b + 1), b = 5 + i, j = w << 9 | S << 13 (+ r << 5): warp-uniform loads of
  // the reference-order table; Q3 / Q4: the (stream, entry, thread) table. The twiddles of a pass's
  // first two stages (3 values) are loaded ahead of the data movement in front of the pass (`pre`),
  // so that no pass starts by waiting for L2.
  auto q2addr = [&](uint32_t S, int i, int hi) {
    const uint64_t js = xbase + (static_cast<uint64_t>(w) << 9) + (static_cast<uint64_t>(S) << 13);
    return tw + (js >> (6 + i)) + hi;
  };
  auto q3addr = [&](uint32_t S, int i, int hi) {
#ifdef NK_STR_NOTW  // timing experiment (wrong results): every low-stage twiddle from one address
    return twq + 0 * (S + i + hi);
#else
    return twq + S * (kStrEntries * 512u) + ((i == 3 ? 0 : (i == 2 ? 1 : (i == 1 ? 3 : 7))) + hi) * 512;
#endif
  };
  Tw pa[3], pb[3];
  pa[0] = ldtw(q2addr(0, 3, 0)), pa[1] = ldtw(q2addr(0, 2, 0)), pa[2] = ldtw(q2addr(0, 2, 1));
  pb[0] = ldtw(q2addr(1, 3, 0)), pb[1] = ldtw(q2addr(1, 2, 0)), pb[2] = ldtw(q2addr(1, 2, 1));
  auto q2tw = [&](uint32_t S, const Tw* pre) {
    return [=](int i, int hi) { return i >= 2 ? pre[i == 3 ? 0 : 1 + hi] : ldtw(q2addr(S, i, hi)); };
  };
  auto q3tw = [&](uint32_t S, const Tw* pre) {
    return [=](int i, int hi) { return i >= 2 ? pre[i == 3 ? 0 : 1 + hi] : ldtw(q3addr(S, i, hi)); };
  };

  // ---- Q2 of stream A first: the wait for B (every warp through P1) comes after it, when the
  // slower warps have caught up ----
  mbar_wait(bar_w, par_w);
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = *reinterpret_cast<const uint64_t*>(St + ((e1r ^ ((r & 3) << 5)) + r * 256));
  NK_GTS(6);
  pass16<A, 4, 5>(v, c, q2tw(0, pa));
  pa[0] = ldtw(q3addr(0, 3, 0)), pa[1] = ldtw(q3addr(0, 2, 0)), pa[2] = ldtw(q3addr(0, 2, 1));  // A's Q3
  mbar_wait(bar_w + 1, par_w);
#pragma unroll
  for (int r = 0; r < 16; ++r)
    v[16 + r] = *reinterpret_cast<const uint64_t*>(St + 65536 + ((e1r ^ ((r & 3) << 5)) + r * 256));
  consumed();  // the staging buffer is consumed by this warp
  before_e2();
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 16; ++r) *reinterpret_cast<uint64_t*>(Ew + ((e2w ^ ((r & 7) << 4)) + r * 256)) = v[r];
  __syncwarp();
  NK_GTS(7);
  pass16<A, 4, 5>(v + 16, c, q2tw(1, pb));
  pb[0] = ldtw(q3addr(1, 3, 0)), pb[1] = ldtw(q3addr(1, 2, 0)), pb[2] = ldtw(q3addr(1, 2, 1));  // B's Q3
  NK_GTS(8);
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = *reinterpret_cast<const uint64_t*>(Ew + (e2r ^ (r << 4)));
  __syncwarp();  // A's words are in registers: the buffer takes B's
#pragma unroll
  for (int r = 0; r < 16; ++r) *reinterpret_cast<uint64_t*>(Ew + ((e2w ^ ((r & 7) << 4)) + r * 256)) = v[16 + r];
  __syncwarp();
  NK_GTS(9);

  // ---- Q3 of both streams together (B's words read back first), shuffle, Q4 ----
#pragma unroll
  for (int r = 0; r < 16; ++r) v[16 + r] = *reinterpret_cast<const uint64_t*>(Ew + (e2r ^ (r << 4)));
  pass16x2<A, 4, 9>(v, c, q3tw(0, pa), q3tw(1, pb));
  const bool odd = (l & 1u) != 0;
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    // lane pairs swap: this lane keeps j1 = its bit 0 and gets both j0
    // (registers r3 = j1 | hi << 1: own words (j0 = lane bit) with j1 = 0 / 1)
    const uint64_t own0 = v[2 * q], own1 = v[2 * q + 1];
    const uint64_t recv = __shfl_xor_sync(0xffffffffu, odd ? own0 : own1, 1);
    v[2 * q] = odd ? recv : own0;      // j0 = 0, j1 = lane bit
    v[2 * q + 1] = odd ? own1 : recv;  // j0 = 1
  }
  // Q4: bit 0, twiddle entries 15 + hi
#pragma unroll
  for (int hi = 0; hi < 8; ++hi) {
#ifdef NK_STR_NOTW
    const Tw wa = ldtw(twq), wb = ldtw(twq + 512);
#else
    const Tw wa = ldtw(twq + (15 + hi) * 512);
    const Tw wb = ldtw(twq + (kStrEntries + 15 + hi) * 512);
#endif
    if (fwd_skip14<A>(false, 13, 1 << 30)) {
      A::template fwd<true>(v[2 * hi], v[2 * hi + 1], wa, c);
      A::template fwd<true>(v[16 + 2 * hi], v[16 + 2 * hi + 1], wb, c);
    } else {
      A::template fwd<false>(v[2 * hi], v[2 * hi + 1], wa, c);
      A::template fwd<false>(v[16 + 2 * hi], v[16 + 2 * hi + 1], wb, c);
    }
  }
  __syncwarp();  // every lane has read B's e2 words: the buffer is free
  NK_GTS(10);
}

// Inverse core: from v[16 S + 2 hi + j0] (the forward core's output layout,
// in the policy's representation) through Q4', Q3', Q2' and P1' of both
// streams; the caller runs the last stage (bit 13) on v[r], v[r + 16], whose
// word index is l | w << 5 | r << 9. `ta`: stream A's first twiddles (8 Q4'
// entries, and with 8-byte tables the 8 entries of Q3''s first stage), loaded
// by the caller ahead of its wait for the block; `inputs_read` runs before the
// staging halves are first written (waits until every warp has its input);
// `consumed` once this warp has read its last word of the staging buffer;
// `before_e2` before the warp's 4 KiB of E is first written.
template <class A, bool ILTM0, class FPRE, class FRD, class FCONS>
__device__ __forceinline__ void inv_core(uint64_t (&v)[32], uint8_t* St, uint8_t* Ew, const LimbConst& c,
                                         const NttArgs& a, const typename A::Tw* __restrict__ tw,
                                         const typename A::Tw* __restrict__ twq, uint64_t xbase, uint32_t w,
                                         uint32_t l, typename A::Tw* ta, uint64_t* bar_w, uint32_t par, uint32_t it_,
                                         FPRE&& before_e2, FRD&& inputs_read, FCONS&& consumed) {
  using Tw = typename A::Tw;
  (void)it_;
  constexpr bool kPre16 = sizeof(Tw) == 8;
  const uint32_t e2w = l << 3;
  const uint32_t e2r = ((l & 1u) << 3) | (((l >> 1) & 7u) << 4) | ((l >> 1) << 8);
  const uint32_t e1w = (l << 3) + (w << 12);  // Q2' map: word l | r << 5 | w << 9
  const uint32_t e1r = (l << 3) + (w << 8);   // P1' map: word l | w << 5 | r << 9
  auto q3addr = [&](uint32_t S, int i, int hi) {
    return twq + S * (kStrEntries * 512u) + ((i == 3 ? 0 : (i == 2 ? 1 : (i == 1 ? 3 : 7))) + hi) * 512;
  };
  auto q2tw = [&](uint32_t S) {
    const uint64_t js = xbase + (static_cast<uint64_t>(w) << 9) + (static_cast<uint64_t>(S) << 13);
    return [=](int i, int hi) { return ldtw(tw + (js >> (6 + i)) + hi); };
  };
  auto p1tw = [&](uint32_t S) {
    const uint64_t js = xbase + (static_cast<uint64_t>(S) << 13);
    return [=](int i, int hi) { return ldtw(tw + (js >> (10 + i)) + hi); };
  };
  const bool odd = (l & 1u) != 0;
  // Q4' (bit 0), j0 back to the lane, Q3' (bits 1..4) of stream S; tq: its first twiddles
  auto low_passes = [&](uint32_t S, const Tw* tq) {
    uint64_t* x = v + 16 * S;
#pragma unroll
    for (int hi = 0; hi < 8; ++hi) {
      if (ILTM0) A::template inv<true>(x[2 * hi], x[2 * hi + 1], tq[hi], c);
      else A::template inv<false>(x[2 * hi], x[2 * hi + 1], tq[hi], c);
    }
    // this lane keeps j0 = its bit 0 and gets both j1
#pragma unroll
    for (int hi = 0; hi < 8; ++hi) {
      const uint64_t y0 = x[2 * hi], y1 = x[2 * hi + 1];
      const uint64_t recv = __shfl_xor_sync(0xffffffffu, odd ? y0 : y1, 1);
      x[2 * hi] = odd ? recv : y0;      // j1 = 0
      x[2 * hi + 1] = odd ? y1 : recv;  // j1 = 1
    }
    pass16i<A>(x, c, [=](int i, int hi) { return (kPre16 && i == 0) ? tq[kPre16 ? 8 + hi : 0] : ldtw(q3addr(S, i, hi)); });
  };

  low_passes(0, ta);
  before_e2();  // e.g. the previous block's output stores have read this warp's 4 KiB
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 16; ++r) *reinterpret_cast<uint64_t*>(Ew + (e2r ^ (r << 4))) = v[r];
  __syncwarp();
  NK_GTS(3);
#pragma unroll
  for (int hi = 0; hi < 8; ++hi) {
    ta[hi] = ldtw(twq + (kStrEntries + 15 + hi) * 512);
    if constexpr (kPre16) ta[8 + hi] = ldtw(q3addr(1, 0, hi));
  }
  low_passes(1, ta);
  NK_GTS(4);
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = *reinterpret_cast<const uint64_t*>(Ew + ((e2w ^ ((r & 7) << 4)) + r * 256));
  __syncwarp();  // A's words are in registers: the buffer takes B's
#pragma unroll
  for (int r = 0; r < 16; ++r) *reinterpret_cast<uint64_t*>(Ew + (e2r ^ (r << 4))) = v[16 + r];
  __syncwarp();
  NK_GTS(5);

  // ---- Q2' of A; B's words back; e1' of A ----
  pass16i<A>(v, c, q2tw(0));
#pragma unroll
  for (int r = 0; r < 16; ++r)
    v[16 + r] = *reinterpret_cast<const uint64_t*>(Ew + ((e2w ^ ((r & 7) << 4)) + r * 256));
  NK_GTS(6);
  inputs_read();  // every warp has its input: the staging halves take the streams
#pragma unroll
  for (int r = 0; r < 16; ++r) *reinterpret_cast<uint64_t*>(St + e1w + r * 256) = v[r];
  __syncwarp();
  if (l == 0) mbar_arrive_local(bar_w);
  pass16i<A>(v + 16, c, q2tw(1));
#pragma unroll
  for (int r = 0; r < 16; ++r) *reinterpret_cast<uint64_t*>(St + 65536 + e1w + r * 256) = v[16 + r];
  __syncwarp();
  if (l == 0) mbar_arrive_local(bar_w + 1);
  NK_GTS(7);

  // ---- P1': bits 9..12 per stream ----
  mbar_wait(bar_w, par);
  NK_GTS(8);
#pragma unroll
  for (int r = 0; r < 16; ++r) v[r] = *reinterpret_cast<const uint64_t*>(St + e1r + r * 4096);
  pass16i<A>(v, c, p1tw(0));
  NK_GTS(9);
  mbar_wait(bar_w + 1, par);
#pragma unroll
  for (int r = 0; r < 16; ++r) v[16 + r] = *reinterpret_cast<const uint64_t*>(St + 65536 + e1r + r * 4096);
  consumed();
  pass16i<A>(v + 16, c, p1tw(1));
  NK_GTS(10);
}

// stream A's first inverse twiddles (see inv_core)
template <class A>
__device__ __forceinline__ void inv_first_twiddles(typename A::Tw* ta, const typename A::Tw* __restrict__ twq) {
#pragma unroll
  for (int hi = 0; hi < 8; ++hi) {
    ta[hi] = ldtw(twq + (15 + hi) * 512);
    if constexpr (sizeof(typename A::Tw) == 8) ta[8 + hi] = ldtw(twq + (7 + hi) * 512);
  }
}

// The inverse's result words out by TMA. Thread (w, l) holds word l | w << 5 | r << 9 in v[r]:
// for a fixed r the warp's 32 words are 256 contiguous bytes, so 8 values of r are an
// 8-row x 256-byte box of the output seen as [words / 512][512] (kStriOutMap). Half h
// (pairs r = 8h .. 8h + 7 of the last stage, i.e. rows 8h.. and 16 + 8h..) goes through the
// warp's 4 KiB of E as two 2 KiB images and two bulk tensor stores; the caller computes
// half 1's words while half 0's stores read their images. y0 = the block's first row
// ((row n + block offset) / 512).
__device__ __forceinline__ void out_half_tma(const CUtensorMap* tout, uint8_t* Ew, uint32_t w, uint32_t l,
                                             int32_t y0, const uint64_t (&v)[32], int h) {
  if (h == 1) {
    if (l == 0) bulk_wait_read();  // half 0's stores have read the images
    __syncwarp();
  }
#pragma unroll
  for (int rr = 0; rr < 8; ++rr) {
    *reinterpret_cast<uint64_t*>(Ew + rr * 256 + l * 8) = v[8 * h + rr];
    *reinterpret_cast<uint64_t*>(Ew + 2048 + rr * 256 + l * 8) = v[16 + 8 * h + rr];
  }
  fence_proxy_async();
  __syncwarp();
  if (l == 0) {
#pragma unroll
    for (int q = 0; q < 2; ++q)
      asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                       reinterpret_cast<uint64_t>(tout)),
                   "r"(static_cast<int32_t>(w << 5)), "r"(y0 + 8 * h + 16 * q), "r"(smem_u32(Ew + 2048 * q))
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
}

}  // namespace str

template <class A, bool ILTM0>
__global__ void __launch_bounds__(512, 1)
    ntt_str14(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, NttArgs a,
              uint32_t nitems) {
  using Tw = typename A::Tw;
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* St = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);  // staging (TMA, 128B-swizzled), then e1
  uint8_t* E = St + kStageBytes;                                         // per warp 4 KiB: e2, then the output image
  const LimbConst* Cs = reinterpret_cast<const LimbConst*>(E + kGrpExBytes);
  uint64_t* bar_full = reinterpret_cast<uint64_t*>(E + kGrpExBytes + 2 * sizeof(LimbConst));
  uint64_t* bar_rd = bar_full + 1;  // every warp has read its P1 words
  uint64_t* bar_w = bar_full + 2;   // [2] every warp has written its e1 words of stream S
  uint32_t* cnt = reinterpret_cast<uint32_t*>(bar_full + 4);
  const uint32_t t = threadIdx.x, l = t & 31u, w = t >> 5;
  const uint32_t lognb = a.logn - kB14;
  const uint64_t rowwords16 = a.n >> 4;

  auto item_row = [&](uint32_t k, uint64_t& row, uint64_t& blk) {
    row = (static_cast<uint64_t>(k) >> lognb) * a.row_mul + a.row_add;
    blk = static_cast<uint64_t>(k) & ((uint64_t{1} << lognb) - 1);
  };
  auto issue = [&](uint32_t k, uint32_t slot) {
    uint64_t row, blk;
    item_row(k, row, blk);
    const int32_t y0 = static_cast<int32_t>(row * rowwords16 + (blk << (kB14 - 4)));
    const uint32_t limb = a.limb0 + static_cast<uint32_t>(row % a.nlimbs);
    mbar_expect_tx(bar_full, kStageBytes + static_cast<uint32_t>(sizeof(LimbConst)));
#pragma unroll
    for (int q = 0; q < 4; ++q) tma_load_2d(St + q * 32768, &tin, 0, y0 + q * 256, bar_full);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(Cs + slot)),
                 "l"(a.lc + limb), "r"(static_cast<uint32_t>(sizeof(LimbConst))), "r"(smem_u32(bar_full))
                 : "memory");
  };

  if (t == 0) {
    mbar_init(bar_full, 1);
    mbar_init(bar_rd, 16);
    mbar_init(bar_w, 16);
    mbar_init(bar_w + 1, 16);
    *cnt = 0;
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tin)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tout)) : "memory");
  }
  __syncthreads();
  if (t == 0 && blockIdx.x < nitems) issue(blockIdx.x, 0);

  uint8_t* Ew = E + (w << 12);
  uint32_t phase = 0;
  uint32_t it_ = 0;
  (void)it_;
  for (uint32_t k = blockIdx.x; k < nitems; k += gridDim.x) {
    uint64_t row, blk;
    item_row(k, row, blk);
    NK_GTS(0);
    const uint32_t limb = a.limb0 + static_cast<uint32_t>(row % a.nlimbs);
    const Tw* __restrict__ tw = tw_of<A>(a, limb);
    const Tw* __restrict__ twq = twq_of<A>(a, limb) + blk * kStrTableWords + t;
    const uint64_t boff = blk << kB14;
    uint64_t v[32];

    mbar_wait(bar_full, phase);
    const LimbConst& c = Cs[phase];
    NK_GTS(1);
    str::fwd_core<A, ILTM0>(
        v, St, Ew, c, a, tw, twq, a.n + boff, w, l, bar_rd, bar_w, phase, phase, it_,
        [&] {
          if (l == 0) bulk_wait_read();  // the previous block's last output store has read this warp's 4 KiB
        },
        [&] {
          grp::staging_consumed(cnt, l, [&] {  // the last of the 16 warps refills the staging buffer
            if (k + gridDim.x < nitems) {
              fence_proxy_async();
              issue(k + gridDim.x, phase ^ 1);
            }
          });
        });

    // ---- canonical words out: per stream a 4 KiB image and one bulk tensor store ----
    const int32_t orow16 = static_cast<int32_t>((row * a.n + boff + (static_cast<uint64_t>(w) << 9)) >> 4);
#pragma unroll
    for (uint32_t S = 0; S < 2; ++S) {
      uint64_t* y = v + 16 * S;
#pragma unroll
      for (int i = 0; i < 16; ++i) y[i] = fwd_out<A>(y[i], c, a.fout);
      // image: word m = j0 | j1 << 1 | hi << 2 | (l >> 1) << 5 at row m >> 4, chunk ((m >> 1) & 7) ^ (row & 7)
      if (S == 1) {
        if (l == 0) bulk_wait_read();  // A's store has read the image
        __syncwarp();
      }
#pragma unroll
      for (int hi = 0; hi < 8; ++hi) {
        const uint32_t rowi = (hi >> 2) + 2 * (l >> 1);
        const uint32_t chunk = ((l & 1u) | ((hi & 3) << 1)) ^ (rowi & 7u);
        *reinterpret_cast<ulonglong2*>(Ew + (rowi << 7) + (chunk << 4)) = make_ulonglong2(y[2 * hi], y[2 * hi + 1]);
      }
      fence_proxy_async();
      __syncwarp();
      if (l == 0) {
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                         reinterpret_cast<uint64_t>(&tout)),
                     "r"(0), "r"(orow16 + static_cast<int32_t>(S << 9)), "r"(smem_u32(Ew))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    NK_GTS(11);
    phase ^= 1;
    ++it_;
  }
  if (l == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---------------------------------------------------------------------------
// ntt_stri14: the inverse as two streams per thread, the mirror image of
// ntt_str14. The inverse's stages 0..12 stay inside the two 8192-word halves;
// only the last one (bit 13) pairs them, in a thread's own registers.
//   in   each warp reads the 512 consecutive words of its two streams from the
//        staging buffer (the TMA's 128B-swizzled lines are the forward's
//        output image): registers (j0; j2, j3, j4), lane bit 0 = j1
//   Q4'  bit 0; sh: j0 back to the lane; Q3' bits 1..4; e2' warp-local;
//   Q2'  bits 5..8; e1' CTA-wide, in place in the stream's staging half (after
//        every warp has read its input), plain layout: both sides have lanes
//        j0..j4;  P1' bits 9..12 per stream (lanes j0..j4, warps j5..j8), then
//        bit 13 on both (n^-1 folded in for canonical outputs); the words
//        leave by bulk tensor stores (str::out_half_tma)
// ---------------------------------------------------------------------------
template <class A, bool ILTM0, bool LONG = false>
__global__ void __launch_bounds__(512, 1)
    ntt_stri14(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, NttArgs a,
               uint32_t nitems) {
  using Tw = typename A::Tw;
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* St = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  uint8_t* E = St + kStageBytes;
  const LimbConst* Cs = reinterpret_cast<const LimbConst*>(E + kGrpExBytes);
  uint64_t* bar_full = reinterpret_cast<uint64_t*>(E + kGrpExBytes + 2 * sizeof(LimbConst));
  uint64_t* bar_rd = bar_full + 1;  // every warp has read its input words
  uint64_t* bar_w = bar_full + 2;   // [2] every warp has written its e1' words of stream S
  uint32_t* cnt = reinterpret_cast<uint32_t*>(bar_full + 4);
  const uint32_t t = threadIdx.x, l = t & 31u, w = t >> 5;
  const uint32_t lognb = a.logn - kB14;
  const uint64_t rowwords16 = a.n >> 4;

  // (a 16384-word block's row number fits 32 bits -- 2^32 rows would be 2^49 bytes -- so the
  // limb of a row is a 32-bit remainder here, not a call to the 64-bit division routine;
  // measured: cfg4 inverse 338 -> 329 us, while the same change cost the forward 6 us and the
  // CTA-pair kernel 35%, so those keep the call)
  auto item_row = [&](uint32_t k, uint64_t& row, uint64_t& blk) {
    row = (static_cast<uint64_t>(k) >> lognb) * a.row_mul + a.row_add;
    blk = static_cast<uint64_t>(k) & ((uint64_t{1} << lognb) - 1);
  };
  auto issue = [&](uint32_t k, uint32_t slot) {
    uint64_t row, blk;
    item_row(k, row, blk);
    const int32_t y0 = static_cast<int32_t>(row * rowwords16 + (blk << (kB14 - 4)));
    const uint32_t limb = a.limb0 + static_cast<uint32_t>(row) % a.nlimbs;
    mbar_expect_tx(bar_full, kStageBytes + static_cast<uint32_t>(sizeof(LimbConst)));
#pragma unroll
    for (int q = 0; q < 4; ++q) tma_load_2d(St + q * 32768, &tin, 0, y0 + q * 256, bar_full);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(Cs + slot)),
                 "l"(a.lc + limb), "r"(static_cast<uint32_t>(sizeof(LimbConst))), "r"(smem_u32(bar_full))
                 : "memory");
  };

  if (t == 0) {
    mbar_init(bar_full, 1);
    mbar_init(bar_rd, 16);
    mbar_init(bar_w, 16);
    mbar_init(bar_w + 1, 16);
    *cnt = 0;
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tin)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tout)) : "memory");
  }
  __syncthreads();
  if (t == 0 && blockIdx.x < nitems) issue(blockIdx.x, 0);

  uint8_t* Ew = E + (w << 12);
  uint32_t phase = 0;
  uint32_t it_ = 0;
  (void)it_;

  for (uint32_t k = blockIdx.x; k < nitems; k += gridDim.x) {
    uint64_t row, blk;
    item_row(k, row, blk);
    const uint32_t limb = a.limb0 + static_cast<uint32_t>(row) % a.nlimbs;
    const Tw* __restrict__ tw = tw_of<A>(a, limb);
    const Tw* __restrict__ twq = twq_of<A>(a, limb) + blk * kStrTableWords + t;
    const uint64_t boff = blk << kB14;
    const uint64_t xbase = a.n + boff;
    uint64_t v[32];

    // the first two stages' twiddles of stream A are loaded before the wait for the block, B's while
    // A computes: the block does not start by waiting for L2
    Tw ta[sizeof(Tw) == 8 ? 16 : 8];
    str::inv_first_twiddles<A>(ta, twq);
    NK_GTS(0);
    // ---- input: both streams' words, (j0 = 0, 1) pairs (the forward's output image) ----
    mbar_wait(bar_full, phase);
    const LimbConst& c = Cs[phase];
    NK_GTS(1);
#pragma unroll
    for (uint32_t S = 0; S < 2; ++S)
#pragma unroll
      for (int hi = 0; hi < 8; ++hi) {
        const uint32_t rowi = (hi >> 2) + 2 * (l >> 1);
        const uint32_t chunk = ((l & 1u) | ((hi & 3) << 1)) ^ (rowi & 7u);
        const ulonglong2 p =
            *reinterpret_cast<const ulonglong2*>(St + (S << 16) + (w << 12) + (rowi << 7) + (chunk << 4));
        v[16 * S + 2 * hi] = A::load(p.x);
        v[16 * S + 2 * hi + 1] = A::load(p.y);
      }
    __syncwarp();
    if (l == 0) mbar_arrive_local(bar_rd);
    NK_GTS(2);

    str::inv_core<A, ILTM0>(
        v, St, Ew, c, a, tw, twq, xbase, w, l, ta, bar_w, phase, it_,
        [&] {
          if (l == 0) bulk_wait_read();  // the previous block's output stores have read this warp's 4 KiB
        },
        [&] { mbar_wait(bar_rd, phase); },
        [&] {
          grp::staging_consumed(cnt, l, [&] {
            if (k + gridDim.x < nitems) {
              fence_proxy_async();
              issue(k + gridDim.x, phase ^ 1);
            }
          });
        });

    // ---- bit 13 (n^-1 folded in for canonical results); result words out by TMA, in two
    // halves of 8 pairs (plain stores from here cost the inverse 12%: 32 STG.64 per thread
    // through the LSU against four bulk tensor stores per warp) ----
    constexpr bool kFoldLast = A::kSigned && !LONG;
    const int32_t y0 = static_cast<int32_t>((row * a.n + boff) >> 9);
    Tw w13{};
    if constexpr (!kFoldLast) w13 = ldtw(tw + (xbase >> 14));
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int r = 8 * h; r < 8 * h + 8; ++r) {
        if constexpr (kFoldLast) {
          A::inv_fold(v[r], v[r + 16], c);
        } else {
          A::template inv<false>(v[r], v[r + 16], w13, c);
          if constexpr (LONG) {
            v[r] = A::store(v[r]);  // intermediate of a long row
            v[r + 16] = A::store(v[r + 16]);
          } else {
            v[r] = inv_out<A>(v[r], c, a.fout);
            v[r + 16] = inv_out<A>(v[r + 16], c, a.fout);
          }
        }
      }
      str::out_half_tma(&tout, Ew, w, l, y0, v, h);
    }
    NK_GTS(11);
    phase ^= 1;
    ++it_;
  }
  if (l == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace nk
