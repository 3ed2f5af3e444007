// Negacyclic NTT kernels for sm_100a.
//
// Algorithm = the reference's, stage for stage (so lazy outputs match bit for
// bit): radix-2 Cooley-Tukey forward over psi powers in bit-reversed order
// (ntt.hpp:363-394), Gentleman-Sande inverse (ntt.hpp:396-433) with the
// standalone n^-1 Shoup pass (ntt.hpp:429-432), Harvey lazy butterflies.
//
// Index algebra used throughout. With N the row length and j an element index,
// the butterfly of stage "bit b" pairs j and j + 2^b (bit b of j clear) and
// uses the twiddle at table index (N + j) >> (b + 1) in BOTH directions:
//   forward, stage m = N >> (b+1), t = 2^b: w_arr[m + (j >> (b+1))]  (ntt.hpp:384-386)
//   inverse, h = N >> (b+1), t = 2^b:        w_arr[h + (j >> (b+1))]  (ntt.hpp:416-420)
// The forward runs b = logN-1 .. 0, the inverse b = 0 .. logN-1.
//
// Kernels (A = arithmetic policy, modmath.cuh: Arith52S / Arith52P on the FP64
// pipe for beta = 2^52, ArithIntL / ArithInt<64> on the integer pipes for
// beta = 2^64; capi.cu: ntt_dispatch_aligned picks one per call):
//  * ntt_pair14<A, FWD, ILTM0> (ntt_pair.cuh): the forward's 16384-word block
//    kernel, one block per CTA pair (cluster of 2), two pairs per SM.
//  * ntt_grp14<A, FWD, ILTM0> (ntt_grp.cuh): the inverse's. Persistent, one
//    512-thread CTA per SM, walks 16384-word blocks (a whole row at N = 16384,
//    or the low 14 bits of a longer row); each block arrives by TMA
//    (cp.async.bulk.tensor, 128B swizzle) into a staging buffer while the
//    previous block is still being transformed; three register passes of
//    5/4(+1)/5 stages with exchanges inside 4-warp groups.
//  * ntt_block<LOGB, LOGV, A, FWD, ILTM0>: same register passes for
//    2^10..2^13-word rows, loads straight from global; ntt_block_lat: the
//    same for batches smaller than the SM count, twiddle row staged in shared
//    memory before griddepcontrol.wait (programmatic dependent launch).
//  * ntt_global_pass<K, A, FWD>: K stages on bits [lo, lo+K) of long rows
//    (N > 2^14), one column of 2^K words per thread, coalesced.
//  * ntt_small<A, FWD>: any N <= 2^9, stage by stage in shared memory.
#pragma once
#include <cuda.h>

#include <cstdint>
#include <type_traits>

#include "modmath.cuh"

namespace nk {

using LimbConst = LimbConstDev;

struct NttArgs {
  uint64_t* out;
  const uint64_t* in;
  const ulonglong2* tw;   // [limb][N] {w, w'} of the plan (fwd or inv table)
  const ulonglong2* twl;  // [limb][N] the same entries for bits 0..4, lane-contiguous (see low_index)
  const LimbConst* lc;    // [limb]
  uint64_t n;            // row length
  uint64_t rows;         // launched rows
  uint32_t limb0, nlimbs;     // row r (after remapping) holds limb limb0 + r % nlimbs
  uint32_t row_mul, row_add;  // launched row i is row i * row_mul + row_add
  uint32_t logn;
  int32_t fin, fout;
  uint64_t* dbg;  // debug: per-warp phase timestamps of an NK_DBG_TIMELINE build (tools/timeline.py)
  const uint64_t* mulb;  // forward (CTA-pair kernel, fout == 1): multiply the canonical
                         // result by these canonical words (same layout) before storing
  const uint64_t* tw8;   // [limb][N] w only (double bits), same order as tw: Arith52S
  const uint64_t* twl8;  // [limb][N] the same entries in the low-table order of twl
  // the low tables in the group-exchange kernels' thread order (entry (b, d, t)
  // = low-table entry (b, d, jhi of thread t's low pass), GrpMap in ntt_grp.cuh):
  // a warp's 32 loads of one (stage, d) are 32 consecutive entries
  const ulonglong2* twg;
  const uint64_t* twg8;
  // the two-stream forward's low-stage twiddles in (stream, entry, thread) order (ntt_str.cuh)
  const ulonglong2* twq;
  const uint64_t* twq8;
};

__device__ __forceinline__ ulonglong2 ldtw(const ulonglong2* p) { return __ldg(p); }
__device__ __forceinline__ uint64_t ldtw(const uint64_t* p) { return __ldg(p); }

// c consecutive table entries in one non-coherent vector load of up to 32
// bytes (c = 1, 2 or 4 for 8-byte entries, 1 or 2 for 16-byte entries; p
// aligned to c entries). c is a constant after unrolling.
__device__ __forceinline__ void ldtw_vec(uint64_t (&w)[4], const uint64_t* p, int c) {
  if (c == 4) {
    asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]) : "l"(p));
  } else if (c == 2) {
    const ulonglong2 t = __ldg(reinterpret_cast<const ulonglong2*>(p));
    w[0] = t.x;
    w[1] = t.y;
  } else {
    w[0] = __ldg(p);
  }
}
__device__ __forceinline__ void ldtw_vec(ulonglong2 (&w)[2], const ulonglong2* p, int c) {
  if (c == 2) {
    asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(w[0].x), "=l"(w[0].y), "=l"(w[1].x), "=l"(w[1].y) : "l"(p));
  } else {
    w[0] = __ldg(p);
  }
}

// four consecutive row words by one 32-byte access (a thread's contiguous run in the block
// kernels' first inverse / last forward pass: one full sector per lane instead of two halves)
__device__ __forceinline__ void ld_words4(uint64_t (&w)[4], const uint64_t* p) {
  asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]) : "l"(p) : "memory");
}
__device__ __forceinline__ void st_words4(uint64_t* p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}

// the twiddle tables of a policy (entries of type A::Tw), offset to limb `limb`
template <class A>
__device__ __forceinline__ const typename A::Tw* tw_of(const NttArgs& a, uint32_t limb) {
  if constexpr (std::is_same_v<typename A::Tw, uint64_t>) return a.tw8 + static_cast<uint64_t>(limb) * a.n;
  else return a.tw + static_cast<uint64_t>(limb) * a.n;
}
template <class A>
__device__ __forceinline__ const typename A::Tw* twl_of(const NttArgs& a, uint32_t limb) {
  if constexpr (std::is_same_v<typename A::Tw, uint64_t>) return a.twl8 + static_cast<uint64_t>(limb) * a.n;
  else return a.twl + static_cast<uint64_t>(limb) * a.n;
}

template <class A>
__device__ __forceinline__ const typename A::Tw* twg_of(const NttArgs& a, uint32_t limb) {
  if constexpr (std::is_same_v<typename A::Tw, uint64_t>) return a.twg8 + static_cast<uint64_t>(limb) * a.n;
  else return a.twg + static_cast<uint64_t>(limb) * a.n;
}

// Padded shared-memory image index: additive over disjoint bit fields, so every
// shared address is a per-thread base plus an immediate, and all exchange
// patterns below (lane strides 1, 16, 32, ..., 512 words) are conflict free.
__host__ __device__ constexpr uint32_t smem_phys(uint32_t j) {
  return j + (j >> 4) + (j >> 8) + (j >> 12);
}

// ---------------------------------------------------------------------------
// compile-time pass schedule of the block kernels
// ---------------------------------------------------------------------------
template <int LOGB, int LOGV>
struct Sched {
  static constexpr int LOGT = LOGB - LOGV;
  static constexpr int T = 1 << LOGT;
  static constexpr int V = 1 << LOGV;
  static constexpr int NP = (LOGB + LOGV - 1) / LOGV;
  // passes in top-down (forward) order: sizes as even as possible, larger first
  __host__ __device__ static constexpr int k(int p) { return LOGB / NP + (p < LOGB % NP ? 1 : 0); }
  __host__ __device__ static constexpr int lo(int p) {
    int s = LOGB;
    for (int i = 0; i <= p; ++i) s -= k(i);
    return s;
  }
  // place outer-index bits o into the positions outside [lo, lo+k)
  __host__ __device__ static constexpr uint32_t scatter(uint32_t o, int lo_, int k_) {
    return (o & ((1u << lo_) - 1u)) | ((o >> lo_) << (lo_ + k_));
  }
  // group g's contribution to the index in pass (lo_, k_)
  __host__ __device__ static constexpr uint32_t jg(int g, int lo_, int k_) {
    return scatter(static_cast<uint32_t>(g) << LOGT, lo_, k_);
  }
};

// P-th pass in processing order.
template <int LOGB, int LOGV, bool FWD>
struct PassOf {
  using S = Sched<LOGB, LOGV>;
  __host__ __device__ static constexpr int td(int p) { return FWD ? p : (S::NP - 1 - p); }
  __host__ __device__ static constexpr int lo(int p) { return S::lo(td(p)); }
  __host__ __device__ static constexpr int k(int p) { return S::k(td(p)); }
};

// Does forward stage `gs` of a whole-row or 16384-word-block transform (0 = its
// first stage; s_local = the stage's position in its pass, iltm0 only on the
// first pass of a transform with canonical input) skip the pre-reduction of
// x0? The signed FP64 policy reduces on even stages only, the loose integer
// policy on odd ones (modmath.cuh, Arith52S::fwd_skip, ArithIntL::fwd_skip);
// the exact policies skip their first kIltmFwd stages at fin = 1, like the
// reference.
template <class A>
__host__ __device__ constexpr bool fwd_skip_stage(bool iltm0, int gs, int s_local) {
  if constexpr (A::kSigned || A::kLoose) return A::fwd_skip(iltm0, gs);
  else return iltm0 && s_local < A::kIltmFwd;
}
// Inverse: may the sum of two products of the stage before skip its reduction?
template <class A>
__host__ __device__ constexpr bool inv_skip_tt() {
  if constexpr (A::kSigned || A::kLoose) return A::kInvSkipTT;
  else return false;
}

// One register pass: K butterfly bits [LO, LO+K) over G = V / 2^K independent
// groups held in v[g * 2^K + r]. xt = N + block offset + this thread's index
// bits (outside the pass). ILTM0: first stage with InputLessThanMod.
// TWS: tw points at a copy of the twiddle row in shared memory (ntt_block_lat).
template <class A, bool FWD, int LOGB, int LOGV, int LO, int K, bool ILTM0, bool TWS = false>
__device__ __forceinline__ void do_pass(uint64_t (&v)[1 << LOGV], const typename A::Tw* __restrict__ tw,
                                        uint64_t xt, const LimbConst& c, bool fold = false) {
  using S = Sched<LOGB, LOGV>;
  constexpr int R = 1 << K;
  constexpr int G = (1 << LOGV) / R;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    const int i = FWD ? (K - 1 - s) : s;  // bit within the pass
    const int b = LO + i;                 // bit of the block index
    // canonical inverse of a whole row: its last stage (bit LOGB - 1, the single twiddle w_1)
    // takes the n^-1 factor and leaves canonical words (A::inv_fold; the caller skips inv_out)
    if (!FWD && s == K - 1 && fold) {
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int r0 = 0; r0 < R / 2; ++r0) A::inv_fold(v[g * R + r0], v[g * R + r0 + R / 2], c);
      break;
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint64_t base = (xt + S::jg(g, LO, K)) >> (b + 1);
      // the stage's R >> (i + 1) twiddles of this group are consecutive table entries
      // (aligned to their count): vector loads of up to 32 bytes
      constexpr int CMAX = 32 / sizeof(typename A::Tw);
      const int H = R >> (i + 1);
      const int C = H < CMAX ? H : CMAX;
      typename A::Tw wv[CMAX];
#pragma unroll
      for (int hi = 0; hi < H; ++hi) {
        if (!TWS && (hi % C) == 0) ldtw_vec(wv, tw + base + hi, C);
        const typename A::Tw w = TWS ? tw[base + hi] : wv[hi % C];
#pragma unroll
        for (int l = 0; l < (1 << i); ++l) {
          const int r0 = (hi << (i + 1)) | l;
          const int r1 = r0 | (1 << i);
          uint64_t& x0 = v[g * R + r0];
          uint64_t& x1 = v[g * R + r1];
          if (FWD) {
            // LOGB - 1 - b: the stage's number from the row's first stage (whole rows only)
            if (fwd_skip_stage<A>(ILTM0, LOGB - 1 - b, s)) A::template fwd<true>(x0, x1, w, c);
            else A::template fwd<false>(x0, x1, w, c);
          } else {
            // canonical-only policies: both inputs are products of the stage before (its bit is a
            // register bit of this pass): their sum needs no reduction (kInvSkipTT, modmath.cuh)
            if ((ILTM0 && s == 0) || (inv_skip_tt<A>() && i > 0 && ((l >> (i - 1)) & 1)))
              A::template inv<true>(x0, x1, w, c);
            else A::template inv<false>(x0, x1, w, c);
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// ntt_block: register passes with full padded shared exchanges (2^10..2^13)
// ---------------------------------------------------------------------------
template <int LOGB, int LOGV, class A, bool FWD, int P, bool ILTM0, bool TWS = false>
__device__ __forceinline__ void run_passes(uint64_t (&v)[1 << LOGV], uint64_t* sm,
                                           const typename A::Tw* __restrict__ tw, uint32_t t,
                                           uint64_t xbase, const LimbConst& c, bool fold = false) {
  using S = Sched<LOGB, LOGV>;
  using PO = PassOf<LOGB, LOGV, FWD>;
  constexpr int LO = PO::lo(P), K = PO::k(P);
  constexpr int R = 1 << K, G = S::V / R;
  const uint32_t jt = S::scatter(t, LO, K);
  if constexpr (P > 0) {
    __syncthreads();  // pass P-1 wrote its image
    const uint32_t bt = smem_phys(jt);
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int r = 0; r < R; ++r) v[g * R + r] = sm[bt + smem_phys(S::jg(g, LO, K) | (r << LO))];
  }
  // fold: inverse only, in the last pass (its last stage is the row's last: bit LOGB - 1)
  do_pass<A, FWD, LOGB, LOGV, LO, K, ILTM0 && P == 0, TWS>(v, tw, xbase + jt, c,
                                                           !FWD && P + 1 == S::NP && fold);
  if constexpr (P + 1 < S::NP) {
    __syncthreads();  // every thread has read the previous image
    const uint32_t bt = smem_phys(jt);
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int r = 0; r < R; ++r) sm[bt + smem_phys(S::jg(g, LO, K) | (r << LO))] = v[g * R + r];
    run_passes<LOGB, LOGV, A, FWD, P + 1, ILTM0, TWS>(v, sm, tw, t, xbase, c, fold);
  }
}

// 512-thread CTAs (N = 8192 at 16 words per thread) are held to 64 registers: two per SM
// (0 = no occupancy target: an explicit 1 makes ptxas spend 128-168 registers where 72-106 do)
template <int LOGB, int LOGV, class A, bool FWD, bool ILTM0>
__global__ void __launch_bounds__(1 << (LOGB - LOGV), (LOGB - LOGV) == 9 ? 2 : 0) ntt_block(NttArgs a) {
  using S = Sched<LOGB, LOGV>;
  using PO = PassOf<LOGB, LOGV, FWD>;
  extern __shared__ uint64_t sm[];
  const uint32_t t = threadIdx.x;
  const uint32_t lognb = a.logn - LOGB;  // log2 of blocks per row
  const uint64_t row = (static_cast<uint64_t>(blockIdx.x) >> lognb) * a.row_mul + a.row_add;
  const uint64_t blk = static_cast<uint64_t>(blockIdx.x) & ((uint64_t{1} << lognb) - 1);
  const uint32_t limb = a.limb0 + static_cast<uint32_t>(row % a.nlimbs);
  const LimbConst c = a.lc[limb];
  const typename A::Tw* __restrict__ tw = tw_of<A>(a, limb);
  const uint64_t boff = blk << LOGB;
  const uint64_t* __restrict__ src = a.in + row * a.n + boff;
  uint64_t* __restrict__ dst = a.out + row * a.n + boff;
  const bool whole = (lognb == 0);

  uint64_t v[S::V];
  {
    constexpr int LO = PO::lo(0), K = PO::k(0);
    constexpr int R = 1 << K, G = S::V / R;
    const uint32_t jt = S::scatter(t, LO, K);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t jg = S::jg(g, LO, K);
      if constexpr (LO == 0 && R >= 4) {
#pragma unroll
        for (int r = 0; r < R; r += 4) {
          uint64_t w4[4];
          ld_words4(w4, src + jt + jg + r);
#pragma unroll
          for (int k = 0; k < 4; ++k) v[g * R + r + k] = A::load(w4[k]);
        }
      } else if constexpr (LO == 0 && R >= 2) {
#pragma unroll
        for (int r = 0; r < R; r += 2) {
          const ulonglong2 p = *reinterpret_cast<const ulonglong2*>(src + jt + jg + r);
          v[g * R + r] = A::load(p.x);
          v[g * R + r + 1] = A::load(p.y);
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) v[g * R + r] = A::load(src[jt + jg + (r << LO)]);
      }
    }
  }
  // canonical inverse: n^-1 folded into the last stage (A::inv_fold), no separate n^-1 pass
  // (not in the 64-register FP64 instances of N = 8192, where the second copy of the last
  // stage costs more than the saved product: 209 -> 221 us per 2^25 coefficients)
  const bool fold = !FWD && A::kFold && a.fout == 1 && !(A::kFP && (LOGB - LOGV) == 9);
  run_passes<LOGB, LOGV, A, FWD, 0, ILTM0>(v, sm, tw, t, a.n + boff, c, fold);

  constexpr int PL = S::NP - 1;
  constexpr int LO = PO::lo(PL), K = PO::k(PL);
  constexpr int R = 1 << K, G = S::V / R;
  // ntt_block always transforms whole rows: final words
  if (!fold) {
#pragma unroll
    for (int i = 0; i < S::V; ++i) v[i] = FWD ? fwd_out<A>(v[i], c, a.fout) : inv_out<A>(v[i], c, a.fout);
  }
  const uint32_t jt = S::scatter(t, LO, K);
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const uint32_t jg = S::jg(g, LO, K);
    if constexpr (LO == 0 && R >= 4) {
#pragma unroll
      for (int r = 0; r < R; r += 4)
        st_words4(dst + jt + jg + r, v[g * R + r], v[g * R + r + 1], v[g * R + r + 2], v[g * R + r + 3]);
    } else if constexpr (LO == 0 && R >= 2) {
#pragma unroll
      for (int r = 0; r < R; r += 2)
        *reinterpret_cast<ulonglong2*>(dst + jt + jg + r) =
            make_ulonglong2(v[g * R + r], v[g * R + r + 1]);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) dst[jt + jg + (r << LO)] = v[g * R + r];
    }
  }
}

template <int LOGB, int LOGV>
constexpr size_t block_smem_bytes() {
  return Sched<LOGB, LOGV>::NP > 1 ? (smem_phys((1u << LOGB) - 1) + 1) * sizeof(uint64_t) : 0;
}

// ---------------------------------------------------------------------------
// TMA / mbarrier primitives (sm_90+ PTX, sm_100a SASS: UTMALDG, SYNCS.*)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Byte offset of word j in a 128B-swizzled staging tile ([rows][16 words],
// 16-byte chunk c of row r stored at chunk c ^ (r & 7)), as TMA writes it.
__device__ __forceinline__ uint32_t swz_off(uint32_t j) {
  const uint32_t row = j >> 4, col = j & 15;
  return (row << 7) + ((((col >> 1) ^ (row & 7))) << 4) + ((col & 1) << 3);
}

// ---------------------------------------------------------------------------
// ntt_block_lat: whole rows of 2^10..2^13 words for batches smaller than the
// SM count (cfg1: one row), where a transform's latency is the metric. Same
// passes as ntt_block, plus:
//  * the row's twiddle table (plan data, read-only since plan creation) is
//    copied into shared memory by one bulk copy BEFORE griddepcontrol.wait, so
//    under programmatic dependent launch it lands while the previous kernel in
//    the stream is still running, and every pass reads its twiddles from
//    shared memory instead of waiting on L2;
//  * griddepcontrol.launch_dependents right away, so the next transform can
//    stage its own table during this one.
// Inputs are read and outputs written only after griddepcontrol.wait.
// ---------------------------------------------------------------------------
template <int LOGB, int LOGV>
constexpr size_t lat_smem_bytes() {
  return ((block_smem_bytes<LOGB, LOGV>() + 15) & ~size_t{15}) + (size_t{16} << LOGB) + 16;
}

template <int LOGB, int LOGV, class A, bool FWD, bool ILTM0>
__global__ void __launch_bounds__(1 << (LOGB - LOGV)) ntt_block_lat(NttArgs a) {
  using S = Sched<LOGB, LOGV>;
  using PO = PassOf<LOGB, LOGV, FWD>;
  extern __shared__ __align__(16) uint64_t sm[];
  constexpr size_t kImgWords = ((block_smem_bytes<LOGB, LOGV>() + 15) & ~size_t{15}) / 8;
  using Tw = typename A::Tw;
  Tw* tws = reinterpret_cast<Tw*>(sm + kImgWords);
  uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(tws) + (size_t{16} << LOGB));
  const uint32_t t = threadIdx.x;
  const uint64_t row = static_cast<uint64_t>(blockIdx.x) * a.row_mul + a.row_add;
  const uint32_t limb = a.limb0 + static_cast<uint32_t>(row % a.nlimbs);
  if (t == 0) {
    mbar_init(bar, 1);
    constexpr uint32_t kBytes = static_cast<uint32_t>(sizeof(Tw)) << LOGB;
    mbar_expect_tx(bar, kBytes);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(tws)),
        "l"(tw_of<A>(a, limb)), "r"(kBytes), "r"(smem_u32(bar))
        : "memory");
  }
  asm volatile("griddepcontrol.launch_dependents;" :::);
  const LimbConst c = a.lc[limb];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint64_t* __restrict__ src = a.in + row * a.n;
  uint64_t* __restrict__ dst = a.out + row * a.n;

  uint64_t v[S::V];
  {
    constexpr int LO = PO::lo(0), K = PO::k(0);
    constexpr int R = 1 << K, G = S::V / R;
    const uint32_t jt = S::scatter(t, LO, K);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t jg = S::jg(g, LO, K);
      if constexpr (LO == 0 && R >= 4) {
#pragma unroll
        for (int r = 0; r < R; r += 4) {
          uint64_t w4[4];
          ld_words4(w4, src + jt + jg + r);
#pragma unroll
          for (int k = 0; k < 4; ++k) v[g * R + r + k] = A::load(w4[k]);
        }
      } else if constexpr (LO == 0 && R >= 2) {
#pragma unroll
        for (int r = 0; r < R; r += 2) {
          const ulonglong2 p = *reinterpret_cast<const ulonglong2*>(src + jt + jg + r);
          v[g * R + r] = A::load(p.x);
          v[g * R + r + 1] = A::load(p.y);
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) v[g * R + r] = A::load(src[jt + jg + (r << LO)]);
      }
    }
  }
  __syncthreads();  // the barrier's initialisation is visible to every thread
  mbar_wait(bar, 0);
  // canonical inverse: n^-1 folded into the last stage (A::inv_fold)
  const bool fold = !FWD && A::kFold && a.fout == 1;
  run_passes<LOGB, LOGV, A, FWD, 0, ILTM0, true>(v, sm, tws, t, a.n, c, fold);

  constexpr int PL = S::NP - 1;
  constexpr int LO = PO::lo(PL), K = PO::k(PL);
  constexpr int R = 1 << K, G = S::V / R;
  if (!fold) {
#pragma unroll
    for (int i = 0; i < S::V; ++i) v[i] = FWD ? fwd_out<A>(v[i], c, a.fout) : inv_out<A>(v[i], c, a.fout);
  }
  const uint32_t jt = S::scatter(t, LO, K);
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const uint32_t jg = S::jg(g, LO, K);
    if constexpr (LO == 0 && R >= 4) {
#pragma unroll
      for (int r = 0; r < R; r += 4)
        st_words4(dst + jt + jg + r, v[g * R + r], v[g * R + r + 1], v[g * R + r + 2], v[g * R + r + 3]);
    } else if constexpr (LO == 0 && R >= 2) {
#pragma unroll
      for (int r = 0; r < R; r += 2)
        *reinterpret_cast<ulonglong2*>(dst + jt + jg + r) = make_ulonglong2(v[g * R + r], v[g * R + r + 1]);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) dst[jt + jg + (r << LO)] = v[g * R + r];
    }
  }
}

// 16384-word blocks (the transforms' block kernels: ntt_pair14 in
// ntt_pair.cuh, ntt_grp14 in ntt_grp.cuh): one register pass = 4 or 5
// butterfly bits over 32 words per thread; PassD below describes a pass, pass14
// runs it.
// ---------------------------------------------------------------------------
constexpr int kB14 = 14;
constexpr uint32_t kStageBytes = (1u << kB14) * 8;  // 128 KiB: one block

// deposit the low bits of t into the set bits of MASK (ascending), like PDEP
template <uint32_t MASK>
__host__ __device__ __forceinline__ constexpr uint32_t pdep(uint32_t t) {
  uint32_t res = 0;
  int src = 0;
#pragma unroll
  for (int b = 0; b < 32;) {
    if (!((MASK >> b) & 1u)) { ++b; continue; }
    int len = 0;
    while (b + len < 32 && ((MASK >> (b + len)) & 1u)) ++len;
    res |= ((t >> src) & ((len == 32) ? ~0u : ((1u << len) - 1u))) << b;
    src += len;
    b += len;
  }
  return res;
}

// remove bit X from a 14-bit index (half-image index for a split on X)
template <int X>
__host__ __device__ __forceinline__ constexpr uint32_t squeeze(uint32_t j) {
  return (j & ((1u << X) - 1u)) | ((j >> (X + 1)) << X);
}

// Low table (per 16384-word block, blocks contiguous per limb): for stage bit
// b < 5, entry (d, jhi) with d < 2^(4-b), jhi < 512 (block-local j >> 5) holds
// psi_rev[(N >> (b+1)) + ((boff >> 5) + jhi) * 2^(4-b) + d]; segment b starts at
// 16384 - (16384 >> b). Offsets are compile-time constants in the kernel.
__host__ __device__ constexpr uint32_t low_index(int b, int d, uint32_t jhi) {
  return (16384u - (16384u >> b)) + static_cast<uint32_t>(d) * 512u + jhi;
}

template <int LO_, int K_, int X_>
struct PassD {
  static constexpr int LO = LO_, K = K_, X = X_;
  static constexpr int R = 1 << K;
  static constexpr int G = 32 / R;
  static constexpr uint32_t bmask = ((1u << K) - 1u) << LO;
  static constexpr uint32_t xmask = (X >= 0) ? (1u << X) : 0u;
  static constexpr uint32_t tmask = ((1u << kB14) - 1u) & ~(bmask | xmask);
  __device__ __forceinline__ static uint32_t jt(uint32_t t) { return pdep<tmask>(t); }
  __host__ __device__ static constexpr uint32_t jc(int g, int r) {
    return (g ? xmask : 0u) | (static_cast<uint32_t>(r) << LO);
  }
};


template <class A>
__host__ __device__ constexpr bool fwd_skip14(bool iltm0, int gs, int s_local) {
  return fwd_skip_stage<A>(iltm0, gs, s_local);
}

// Stages [S0, S1) (processing order) of the register pass PD, on all 32 words
// or on one half of them (HALF = 0 / 1: registers 16 HALF .. 16 HALF + 15;
// only for stages whose butterflies stay inside a half: every stage of a
// K = 4 pass, whose halves are its two groups, and the stages below register
// bit 4 of a K = 5 pass). The kernels use the halves to overlap an exchange
// round of one half with the arithmetic of the other.
template <class A, bool FWD, class PD, bool ILTM0, int S0, int S1, int HALF = -1>
__device__ __forceinline__ void stages14(uint64_t (&v)[32], const typename A::Tw* __restrict__ tw,
                                         const typename A::Tw* __restrict__ twl, uint64_t n,
                                         uint64_t xt, const LimbConst& c) {
  constexpr int K = PD::K, R = PD::R, G = PD::G;
  // the pass over bits 0..4 reads the transposed low table (twl points at this
  // block's segment plus this thread's position): loads of one (stage, d) are
  // lane-contiguous and their offsets are immediates
  constexpr bool kLow = (PD::LO == 0 && PD::K == 5);
  // a passenger bit below the pass's bits does not reach the twiddle index
  // ((N + j) >> (b+1) with b > X): both groups share each twiddle
  constexpr bool kShared = (G == 2) && (PD::X >= 0) && (PD::X < PD::LO);
  constexpr int GL = kShared ? 1 : G;  // groups with their own twiddles
#pragma unroll
  for (int s = S0; s < S1; ++s) {
    const int i = FWD ? (K - 1 - s) : s;
    const int b = PD::LO + i;
#pragma unroll
    for (int gl = 0; gl < GL; ++gl) {
      if (HALF >= 0 && G == 2 && !kShared && gl != HALF) continue;
      const uint64_t base = (xt + PD::jc(gl, 0)) >> (b + 1);
#pragma unroll
      for (int hi = 0; hi < (R >> (i + 1)); ++hi) {
        if (HALF >= 0 && G == 1 && (((hi << (i + 1)) >> 4) & 1) != HALF) continue;
        const typename A::Tw w = kLow ? ldtw(twl + low_index(b, hi, 0)) : ldtw(tw + base + hi);
#pragma unroll
        for (int gg = 0; gg < G / GL; ++gg) {
          if (HALF >= 0 && kShared && gg != HALF) continue;
#pragma unroll
          for (int l = 0; l < (1 << i); ++l) {
            const int g = kShared ? gg : gl;
            const int r0 = (hi << (i + 1)) | l;
            const int r1 = r0 | (1 << i);
            uint64_t& x0 = v[g * R + r0];
            uint64_t& x1 = v[g * R + r1];
            if (FWD) {
              // kB14 - 1 - b: the stage's number from the block's first stage (index bit 13)
              if (fwd_skip14<A>(ILTM0, kB14 - 1 - b, s)) A::template fwd<true>(x0, x1, w, c);
              else A::template fwd<false>(x0, x1, w, c);
            } else {
              if ((ILTM0 && s == 0) || (inv_skip_tt<A>() && i > 0 && ((l >> (i - 1)) & 1)))
                A::template inv<true>(x0, x1, w, c);
              else A::template inv<false>(x0, x1, w, c);
            }
          }
        }
      }
    }
  }
}

// One register pass over the bits of PD (stage order by direction).
// SKIP_LAST: leave the pass's last stage to the caller (the folded n^-1 stage
// of the canonical inverses).
template <class A, bool FWD, class PD, bool ILTM0, int SKIP_LAST = 0>
__device__ __forceinline__ void pass14(uint64_t (&v)[32], const typename A::Tw* __restrict__ tw,
                                       const typename A::Tw* __restrict__ twl, uint64_t n,
                                       uint64_t xt, const LimbConst& c) {
  stages14<A, FWD, PD, ILTM0, 0, PD::K - SKIP_LAST>(v, tw, twl, n, xt, c);
}

// ---------------------------------------------------------------------------
// K stages over bits [lo, lo+K) of long rows; one column per thread.
// first_iltm: forward with fin == 1 at the top stage. last: inverse final pass
// (apply n^-1 and the fout reduction).
// ---------------------------------------------------------------------------
template <int K, class A, bool FWD>
__global__ void __launch_bounds__(256) ntt_global_pass(NttArgs a, uint32_t lo, int first_iltm,
                                                       int last) {
  constexpr int R = 1 << K;
  const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t logcols = a.logn - K;
  if (gid >= (a.rows << logcols)) return;
  const uint64_t row = (gid >> logcols) * a.row_mul + a.row_add;
  const uint64_t o = gid & ((uint64_t{1} << logcols) - 1);
  const uint32_t limb = a.limb0 + static_cast<uint32_t>(row % a.nlimbs);
  const LimbConst c = a.lc[limb];
  const typename A::Tw* __restrict__ tw = tw_of<A>(a, limb);
  const uint64_t j0 = (o & ((uint64_t{1} << lo) - 1)) | ((o >> lo) << (lo + K));
  const uint64_t* src = a.in + row * a.n;
  uint64_t* dst = a.out + row * a.n;
  uint64_t v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = A::load(src[j0 + (static_cast<uint64_t>(r) << lo)]);
  const uint64_t xt = a.n + j0;
  // canonical inverse: the last stage (bit logn - 1, one twiddle) takes the
  // n^-1 factor (A::inv_fold) and stores canonical words directly
  const bool fold = !FWD && A::kFold && last && a.fout == 1;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    const int i = FWD ? (K - 1 - s) : s;
    const uint32_t b = lo + i;
    const uint64_t base = xt >> (b + 1);
    if (!FWD && s == K - 1 && fold) {
#pragma unroll
      for (int r0 = 0; r0 < R / 2; ++r0) A::inv_fold(v[r0], v[r0 + R / 2], c);
      break;
    }
#pragma unroll
    for (int hi = 0; hi < (R >> (i + 1)); ++hi) {
      const typename A::Tw w = ldtw(tw + base + hi);
#pragma unroll
      for (int l = 0; l < (1 << i); ++l) {
        const int r0 = (hi << (i + 1)) | l, r1 = r0 | (1 << i);
        if (FWD) {
          if (s == 0 && first_iltm) A::template fwd<true>(v[r0], v[r1], w, c);
          else A::template fwd<false>(v[r0], v[r1], w, c);
        } else {
          A::template inv<false>(v[r0], v[r1], w, c);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
    dst[j0 + (static_cast<uint64_t>(r) << lo)] =
        fold ? v[r] : ((!FWD && last) ? inv_out<A>(v[r], c, a.fout) : A::store(v[r]));
}

// ---------------------------------------------------------------------------
// Any N <= 2^9: one CTA per row, whole row in shared memory, one stage at a
// time. Used for the small sizes of the reference's tests.
// ---------------------------------------------------------------------------
template <class A, bool FWD>
__global__ void __launch_bounds__(256) ntt_small(NttArgs a) {
  extern __shared__ uint64_t smw[];
  const uint64_t row = static_cast<uint64_t>(blockIdx.x) * a.row_mul + a.row_add;
  const uint32_t limb = a.limb0 + static_cast<uint32_t>(row % a.nlimbs);
  const LimbConst c = a.lc[limb];
  const typename A::Tw* __restrict__ tw = tw_of<A>(a, limb);
  const uint32_t n = static_cast<uint32_t>(a.n);
  for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) smw[j] = A::load(a.in[row * a.n + j]);
  __syncthreads();
  for (uint32_t s = 0; s < a.logn; ++s) {
    const uint32_t b = FWD ? (a.logn - 1 - s) : s;
    const bool iltm = (s == 0) && (a.fin == 1);
    for (uint32_t p = threadIdx.x; p < n / 2; p += blockDim.x) {
      const uint32_t j = ((p >> b) << (b + 1)) | (p & ((1u << b) - 1u));
      const typename A::Tw w = ldtw(tw + ((a.n + j) >> (b + 1)));
      uint64_t x0 = smw[j], x1 = smw[j + (1u << b)];
      if (FWD) {
        if (iltm) A::template fwd<true>(x0, x1, w, c);
        else A::template fwd<false>(x0, x1, w, c);
      } else {
        if (iltm) A::template inv<true>(x0, x1, w, c);
        else A::template inv<false>(x0, x1, w, c);
      }
      smw[j] = x0;
      smw[j + (1u << b)] = x1;
    }
    __syncthreads();
  }
  for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) {
    a.out[row * a.n + j] = FWD ? fwd_out<A>(smw[j], c, a.fout) : inv_out<A>(smw[j], c, a.fout);
  }
}

}  // namespace nk

namespace nk {

// warp-image position of a word (index bits 0..3 and 5..9; bit 4 is the
// round): 512 words + 2 words of padding per 16, conflict-free for both sides
// of the warp-local exchanges (ntt_pair14)
__host__ __device__ constexpr uint32_t wimg(uint32_t j) {
  const uint32_t idx = (j & 15u) | (((j >> 5) & 31u) << 4);
  return idx + 2u * (idx >> 4);
}

}  // namespace nk
