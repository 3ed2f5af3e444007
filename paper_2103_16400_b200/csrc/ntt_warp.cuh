// ntt_warp14: the 16384-word negacyclic transform with NO block-level
// synchronisation: every warp is an independent worker.
//
// A row j = 128 a + b (a, b in [0, 128)) is transformed in two phases of 7
// stages (the reference's radix-2 butterflies, ntt.hpp:363-433, unchanged):
//   forward: phase 0 = stages 13..7 on the columns (bits of a) of 8 adjacent
//            columns (1024 words per warp item), phase 1 = stages 6..0 on
//            8 adjacent 128-word rows (1024 contiguous words);
//   inverse: phase 0 = stages 0..6 on 8 rows, phase 1 = stages 7..13 on 8
//            columns (then the n^-1 pass).
// Each item holds 32 words per lane in registers (5 index bits), runs 5
// stages, swaps index bits between registers and lanes through a private
// 8.25 KiB shared-memory image (warp-local, __syncwarp only), runs 2 stages.
// Phase 0 writes its result in place into the output row (an L2-resident
// intermediate); phase 1 items of a row wait on a per-row counter that the 16
// phase-0 items of that row increment (release / acquire at gpu scope).
//
// Work order: one global sequence of items, phase-0 items running `lag` rows
// ahead of phase-1 items; warp w takes positions w, w + W, w + 2W, ... Every
// wait is on items at EARLIER positions, and all warps are resident
// (persistent grid), so the smallest waiting position always progresses: no
// deadlock. A bounded spin turns any bug into wrong numbers, not a hang.
#pragma once
#include "ntt_kernels.cuh"

namespace nk {

constexpr uint32_t kWImgWords = 1056;  // per-warp exchange image (words)
constexpr int kWarpsPerCta = 8;
constexpr size_t kWarpSmemBytes = kWarpsPerCta * kWImgWords * 8;

struct WarpNttArgs {
  NttArgs a;
  uint32_t* cnt;  // [rows] phase-0 completions per launched row (zeroed per call)
  uint32_t* err;  // set to 1 when a wait times out
  uint32_t lag;   // rows of phase-0 items issued ahead of phase-1 items
};

// column image: word (a, b_lo) of an 8-column item; 8 words of padding per
// 256 so the two exchange patterns are conflict free
__device__ __forceinline__ uint32_t cidx(uint32_t a, uint32_t blo) { return 8 * a + blo + 8 * (a >> 5); }
// row image: word (a_lo, b) of an 8-row item; rows 132 words apart, 16-byte
// chunks XOR-swizzled on chunk bit 3 (conflict-free 16-byte reads by lane)
__device__ __forceinline__ uint32_t ridx(uint32_t alo, uint32_t b) {
  const uint32_t ch = b >> 1;
  return 132 * alo + 2 * (ch ^ ((ch >> 3) & 1)) + (b & 1);
}

// L2 cache policies: the intermediate is kept (evict_last) until phase 1 reads
// it; streamed input and final output are evict_first
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_hint(uint64_t* p, uint64_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t ld_hint(const uint64_t* p, uint64_t pol) {
  uint64_t v;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint64_t ld_cg_hint(const uint64_t* p, uint64_t pol) {
  uint64_t v;
  asm volatile("ld.global.cg.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}
__device__ __forceinline__ uint64_t ld_cg(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void ld_v4(const uint64_t* p, uint64_t& a, uint64_t& b, uint64_t& c, uint64_t& d) {
  asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}
__device__ __forceinline__ void st_v4(uint64_t* p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  asm volatile("st.global.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__device__ __forceinline__ void st_v4_hint(uint64_t* p, uint64_t a, uint64_t b, uint64_t c, uint64_t d,
                                           uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.u64 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void ld_v4_hint(const uint64_t* p, uint64_t& a, uint64_t& b, uint64_t& c, uint64_t& d,
                                           uint64_t pol) {
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v4.u64 {%0,%1,%2,%3}, [%4], %5;"
               : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
               : "l"(p), "l"(pol));
}
__device__ __forceinline__ void red_release_gpu(uint32_t* p) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// One radix-2 stage over register bit I of 32 registers; tw_of(hi) gives the
// twiddle of the butterflies whose registers agree above bit I (hi = r >> (I+1)).
template <class A, bool FWD, bool ILTM, int I, class TwF>
__device__ __forceinline__ void stage32(uint64_t (&v)[32], const LimbConst& c, TwF tw_of) {
#pragma unroll
  for (int hi = 0; hi < (32 >> (I + 1)); ++hi) {
    const ulonglong2 w = tw_of(hi);
#pragma unroll
    for (int l = 0; l < (1 << I); ++l) {
      const int r0 = (hi << (I + 1)) | l, r1 = r0 | (1 << I);
      if (FWD) A::template fwd<ILTM>(v[r0], v[r1], w, c);
      else A::template inv<ILTM>(v[r0], v[r1], w, c);
    }
  }
}

// global item sequence -> (phase, launched row, sub-block 0..15)
__device__ __forceinline__ void warp_item(uint32_t p, uint32_t rows, uint32_t lag, int& phase, uint32_t& rl,
                                          uint32_t& sub) {
  const uint32_t L = lag < rows ? lag : rows;
  sub = p & 15u;
  if (p < 16 * L) {
    phase = 0;
    rl = p >> 4;
    return;
  }
  const uint32_t q = p - 16 * L, mid = rows - L;
  if (q < 32 * mid) {
    const uint32_t k = q >> 5;
    phase = (q & 16u) ? 0 : 1;
    rl = phase ? k : L + k;
    return;
  }
  phase = 1;
  rl = mid + ((q - 32 * mid) >> 4);
}

template <class A, bool FWD, bool ILTM0>
__global__ void __launch_bounds__(256, 2) ntt_warp14(WarpNttArgs wa) {
  extern __shared__ uint64_t wsm[];
  const NttArgs& a = wa.a;
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  uint64_t* img = wsm + wid * kWImgWords;
  const uint32_t nw = gridDim.x * kWarpsPerCta;
  const uint32_t rows = static_cast<uint32_t>(a.rows);
  const uint32_t total = rows * 32u;
  // lane roles: column items (b_lo = lane & 7, two a bits = lane >> 3),
  // row items (b01 = lane & 3, a_lo = lane >> 2; after the swap b >> 2 = lane)
  const uint32_t blo = lane & 7u, g = lane >> 3, b01 = lane & 3u, alo = lane >> 2;

  const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
  // a finished phase-0 item is announced late (after the next item's loads
  // have landed), so the release fence rarely waits on its stores; always
  // before this warp waits on any counter (no self-deadlock)
  uint32_t pending = ~0u;
  // release without __threadfence(): that one also invalidates L1
  // (CCTL.IVALL), which would send every later twiddle load to L2
  auto publish = [&]() {
    if (pending != ~0u) {
      __syncwarp();  // orders the warp's stores before lane 0's release
      if (lane == 0) red_release_gpu(wa.cnt + pending);
      pending = ~0u;
    }
  };

  for (uint32_t p = blockIdx.x * kWarpsPerCta + wid; p < total; p += nw) {
    int phase;
    uint32_t rl, sub;
    warp_item(p, rows, wa.lag, phase, rl, sub);
    {  // L2 prefetch of this warp's next item when it streams from HBM (phase 0)
      int ph2;
      uint32_t rl2, sub2;
      if (p + nw < total) {
        warp_item(p + nw, rows, wa.lag, ph2, rl2, sub2);
        if (ph2 == 0) {
          const uint64_t* s2 = a.in + (static_cast<uint64_t>(rl2) * a.row_mul + a.row_add) * 16384u;
          if (FWD) {
#pragma unroll
            for (int k = 0; k < 4; ++k) prefetch_l2(s2 + 128u * (lane + 32u * k) + 8u * sub2);
          } else {
#pragma unroll
            for (int k = 0; k < 2; ++k) prefetch_l2(s2 + 1024u * sub2 + 16u * (lane + 32u * k));
          }
        }
      }
    }
    const uint64_t row = static_cast<uint64_t>(rl) * a.row_mul + a.row_add;
    const uint32_t limb = a.limb0 + static_cast<uint32_t>(row % a.nlimbs);
    const LimbConst c = a.lc[limb];
    const ulonglong2* __restrict__ tw = a.tw + static_cast<uint64_t>(limb) * 16384u;
    uint64_t* __restrict__ dst = a.out + row * 16384u;
    uint64_t v[32];
    const bool cols = (phase == 0) == FWD;  // this item works on columns

    if (phase == 1) {  // wait for the 16 phase-0 items of this row
      publish();
      if (lane == 0) {
        uint32_t spins = 0;
        while (ld_relaxed_gpu(wa.cnt + rl) < 16u) {
          __nanosleep(128);
          if (++spins > (1u << 23)) {  // ~1 s: give up (wrong result, no hang)
            atomicOr(wa.err, 1u);
            break;
          }
        }
        // no acquire fence (it would invalidate L1): every read of the
        // intermediate below is an L2 (.cg) load issued after this wait
      }
      __syncwarp();
    }

    if (cols) {
      const uint32_t m = sub;  // columns 8m .. 8m+7
      if (FWD) {
        // ---- forward phase 0: stages 13..9 (a bits 6..2 in registers) ----
        const uint64_t* __restrict__ src = a.in + row * 16384u;
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = A::load(ld_hint(src + 128u * (4u * r + g) + 8u * m + blo, pol_stream));
        {
          auto t = [&](int i, int hi) { return ldtw(tw + (16 >> i) + hi); };
          stage32<A, true, ILTM0, 4>(v, c, [&](int hi) { return t(4, hi); });
          publish();
          stage32<A, true, false, 3>(v, c, [&](int hi) { return t(3, hi); });
          stage32<A, true, false, 2>(v, c, [&](int hi) { return t(2, hi); });
          stage32<A, true, false, 1>(v, c, [&](int hi) { return t(1, hi); });
          stage32<A, true, false, 0>(v, c, [&](int hi) { return t(0, hi); });
        }
        // ---- registers <- a bits 0..4, lanes <- a bits 5, 6 ----
#pragma unroll
        for (int r = 0; r < 32; ++r) img[cidx(4u * r + g, blo)] = v[r];
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = img[cidx(r + 32u * g, blo)];
        __syncwarp();
        // ---- stages 8, 7 ----
        {
          auto t = [&](int i, int hi) { return ldtw(tw + (64 >> i) + hi + (g << (4 - i))); };
          stage32<A, true, false, 1>(v, c, [&](int hi) { return t(1, hi); });
          stage32<A, true, false, 0>(v, c, [&](int hi) { return t(0, hi); });
        }
#pragma unroll
        for (int r = 0; r < 32; ++r) st_hint(dst + 128u * (r + 32u * g) + 8u * m + blo, v[r], pol_keep);  // intermediate
      } else {
        // ---- inverse phase 1: stages 7, 8 (a bits 0..4 in registers) ----
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = ld_cg_hint(dst + 128u * (r + 32u * g) + 8u * m + blo, pol_stream);
        {
          auto t = [&](int i, int hi) { return ldtw(tw + (64 >> i) + hi + (g << (4 - i))); };
          stage32<A, false, false, 0>(v, c, [&](int hi) { return t(0, hi); });
          stage32<A, false, false, 1>(v, c, [&](int hi) { return t(1, hi); });
        }
#pragma unroll
        for (int r = 0; r < 32; ++r) img[cidx(r + 32u * g, blo)] = v[r];
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = img[cidx(4u * r + g, blo)];
        __syncwarp();
        // ---- stages 9..13 (a bits 2..6 in registers), then n^-1 ----
        {
          auto t = [&](int i, int hi) { return ldtw(tw + (16 >> i) + hi); };
          stage32<A, false, false, 0>(v, c, [&](int hi) { return t(0, hi); });
          stage32<A, false, false, 1>(v, c, [&](int hi) { return t(1, hi); });
          stage32<A, false, false, 2>(v, c, [&](int hi) { return t(2, hi); });
          stage32<A, false, false, 3>(v, c, [&](int hi) { return t(3, hi); });
          stage32<A, false, false, 4>(v, c, [&](int hi) { return t(4, hi); });
        }
#pragma unroll
        for (int r = 0; r < 32; ++r) dst[128u * (4u * r + g) + 8u * m + blo] = inv_out<A>(v[r], c, a.fout);
      }
    } else {
      const uint32_t ab = 8u * sub;  // rows ab .. ab+7
      if (FWD) {
        // ---- forward phase 1: stages 6..2 (b bits 2..6 in registers) ----
        const uint32_t arow = ab + alo;
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = ld_cg_hint(dst + 128u * arow + 4u * r + b01, pol_stream);
        {
          auto t = [&](int i, int hi) { return ldtw(tw + (2048 >> i) + (arow << (4 - i)) + hi); };
          stage32<A, true, false, 4>(v, c, [&](int hi) { return t(4, hi); });
          stage32<A, true, false, 3>(v, c, [&](int hi) { return t(3, hi); });
          stage32<A, true, false, 2>(v, c, [&](int hi) { return t(2, hi); });
          stage32<A, true, false, 1>(v, c, [&](int hi) { return t(1, hi); });
          stage32<A, true, false, 0>(v, c, [&](int hi) { return t(0, hi); });
        }
        // ---- registers <- (b0, b1, a_lo), lanes <- b bits 2..6 ----
#pragma unroll
        for (int r = 0; r < 32; ++r) img[ridx(alo, 4u * r + b01)] = v[r];
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const ulonglong2 p2 = *reinterpret_cast<const ulonglong2*>(img + ridx(q, 4u * lane + 2 * h));
            v[4 * q + 2 * h] = p2.x;
            v[4 * q + 2 * h + 1] = p2.y;
          }
        __syncwarp();
        // ---- stages 1, 0; canonical words; 32-byte coalesced stores ----
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t ar = ab + q;
          const ulonglong2 w1 = ldtw(tw + 4096u + 32u * ar + lane);
          A::template fwd<false>(v[4 * q + 0], v[4 * q + 2], w1, c);
          A::template fwd<false>(v[4 * q + 1], v[4 * q + 3], w1, c);
          const ulonglong2 w0a = ldtw(tw + 8192u + 64u * ar + 2u * lane);
          const ulonglong2 w0b = ldtw(tw + 8192u + 64u * ar + 2u * lane + 1u);
          A::template fwd<false>(v[4 * q + 0], v[4 * q + 1], w0a, c);
          A::template fwd<false>(v[4 * q + 2], v[4 * q + 3], w0b, c);
          st_v4(dst + 128u * ar + 4u * lane, fwd_out<A>(v[4 * q], c, a.fout), fwd_out<A>(v[4 * q + 1], c, a.fout),
                fwd_out<A>(v[4 * q + 2], c, a.fout), fwd_out<A>(v[4 * q + 3], c, a.fout));
        }
      } else {
        // ---- inverse phase 0: stages 0, 1 ((b0, b1, a_lo) in registers) ----
        const uint64_t* __restrict__ src = a.in + row * 16384u;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t ar = ab + q;
          uint64_t x0, x1, x2, x3;
          ld_v4_hint(src + 128u * ar + 4u * lane, x0, x1, x2, x3, pol_stream);
          x0 = A::load(x0);
          x1 = A::load(x1);
          x2 = A::load(x2);
          x3 = A::load(x3);
          const ulonglong2 w0a = ldtw(tw + 8192u + 64u * ar + 2u * lane);
          const ulonglong2 w0b = ldtw(tw + 8192u + 64u * ar + 2u * lane + 1u);
          A::template inv<ILTM0>(x0, x1, w0a, c);
          A::template inv<ILTM0>(x2, x3, w0b, c);
          const ulonglong2 w1 = ldtw(tw + 4096u + 32u * ar + lane);
          A::template inv<false>(x0, x2, w1, c);
          A::template inv<false>(x1, x3, w1, c);
          *reinterpret_cast<ulonglong2*>(img + ridx(q, 4u * lane)) = make_ulonglong2(x0, x1);
          *reinterpret_cast<ulonglong2*>(img + ridx(q, 4u * lane + 2)) = make_ulonglong2(x2, x3);
        }
        publish();
        __syncwarp();
        // ---- registers <- b bits 2..6, lanes <- (b01, a_lo) ----
        const uint32_t arow = ab + alo;
#pragma unroll
        for (int r = 0; r < 32; ++r) v[r] = img[ridx(alo, 4u * r + b01)];
        __syncwarp();
        // ---- stages 2..6 ----
        {
          auto t = [&](int i, int hi) { return ldtw(tw + (2048 >> i) + (arow << (4 - i)) + hi); };
          stage32<A, false, false, 0>(v, c, [&](int hi) { return t(0, hi); });
          stage32<A, false, false, 1>(v, c, [&](int hi) { return t(1, hi); });
          stage32<A, false, false, 2>(v, c, [&](int hi) { return t(2, hi); });
          stage32<A, false, false, 3>(v, c, [&](int hi) { return t(3, hi); });
          stage32<A, false, false, 4>(v, c, [&](int hi) { return t(4, hi); });
        }
#pragma unroll
        for (int r = 0; r < 32; ++r) st_hint(dst + 128u * arow + 4u * r + b01, v[r], pol_keep);  // intermediate
      }
    }

    if (phase == 0) pending = rl;  // announced by publish() later
  }
  publish();
}

}  // namespace nk

namespace nk {

// ---------------------------------------------------------------------------
// ntt_warp14s: the forward warp-per-item transform with asynchronous staging.
// Each warp owns a 12.4 KiB shared region: an item image (the TMA / bulk-copy
// landing zone, reused as the exchange image) and the phase-1 items' twiddle
// segments. The next item's data is requested as soon as the current item's
// exchange has been read, so the copy overlaps the last two stages, the
// stores and the other warps' work; phase-0 input is also prefetched into L2
// one item ahead. A phase-1 item's copy is only issued once the row counter
// shows all 16 phase-0 items of the row published; if it is not ready at the
// exchange, the warp finishes and publishes its own item first, so a waiting
// warp never holds unpublished work (no cycle of waits).
// ---------------------------------------------------------------------------
constexpr uint32_t kWSWords = 1056;                    // image (8448 B)
constexpr uint32_t kWRegionBytes = 8448 + 4096 + 128;  // + twiddles (4 KiB) + mbarrier
constexpr size_t kWarpSSmemBytes = 128 + kWarpsPerCta * kWRegionBytes;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// twiddle segment of part-1 stage i (index bit 2 + i) inside the region
__host__ __device__ constexpr uint32_t twseg(int i) {
  return i == 4 ? 0 : (i == 3 ? 8 : (i == 2 ? 24 : (i == 1 ? 56 : 120)));
}

template <class A, bool ILTM0_UNUSED>
__global__ void __launch_bounds__(256, 2)
    ntt_warp14s(const __grid_constant__ CUtensorMap tin_cols, WarpNttArgs wa) {
  extern __shared__ __align__(128) uint8_t wraw[];
  const NttArgs& a = wa.a;
  const uint32_t lane = threadIdx.x & 31u, wid = threadIdx.x >> 5;
  uint8_t* region = wraw + ((128u - (smem_u32(wraw) & 127u)) & 127u) + wid * kWRegionBytes;
  uint64_t* SW = reinterpret_cast<uint64_t*>(region);
  ulonglong2* TWB = reinterpret_cast<ulonglong2*>(region + 8448);
  uint64_t* bar = reinterpret_cast<uint64_t*>(region + 8448 + 4096);
  const uint32_t nw = gridDim.x * kWarpsPerCta;
  const uint32_t rows = static_cast<uint32_t>(a.rows);
  const uint32_t total = rows * 32u;
  const uint32_t blo = lane & 7u, g = lane >> 3, b01 = lane & 3u, alo = lane >> 2;
  const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();

  auto row_of = [&](uint32_t rl) { return static_cast<uint64_t>(rl) * a.row_mul + a.row_add; };
  auto limb_of = [&](uint64_t row) { return a.limb0 + static_cast<uint32_t>(row % a.nlimbs); };
  // lane 0 only: is the row's phase 0 complete (non-blocking / blocking)
  auto row_ready = [&](uint32_t rl) { return ld_relaxed_gpu(wa.cnt + rl) >= 16u; };
  auto wait_row = [&](uint32_t rl) {
    uint32_t spins = 0;
    while (!row_ready(rl)) {
      __nanosleep(64);
      if (++spins > (1u << 24)) {  // give up (wrong result, no hang)
        atomicOr(wa.err, 1u);
        break;
      }
    }
  };
  // lane 0 only: request item p's data into this warp's region
  auto issue = [&](uint32_t p) {
    int ph;
    uint32_t rl, sub;
    warp_item(p, rows, wa.lag, ph, rl, sub);
    const uint64_t row = row_of(rl);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (ph == 0) {
      mbar_expect_tx(bar, 8192);
      tma_load_2d(SW, &tin_cols, static_cast<int32_t>(8 * sub), static_cast<int32_t>(row * 128), bar);
    } else {
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const ulonglong2* tw = a.tw + static_cast<uint64_t>(limb_of(row)) * 16384u;
      const uint32_t ab = 8 * sub;
      mbar_expect_tx(bar, 8192 + 248 * 16);
      for (int q = 0; q < 8; ++q)
        bulk_g2s(SW + 132 * q, a.out + row * 16384u + 128u * (ab + q), 1024, bar);
      for (int i = 4; i >= 0; --i)
        bulk_g2s(TWB + twseg(i), tw + (2048 >> i) + (ab << (4 - i)), (8u << (4 - i)) * 16u, bar);
    }
  };
  auto prefetch_in = [&](uint32_t p) {  // L2 prefetch of a phase-0 item's input
    int ph;
    uint32_t rl, sub;
    warp_item(p, rows, wa.lag, ph, rl, sub);
    if (ph != 0) return;
    const uint64_t* s2 = a.in + row_of(rl) * 16384u;
#pragma unroll
    for (int k = 0; k < 4; ++k) prefetch_l2(s2 + 128u * (lane + 32u * k) + 8u * sub);
  };

  uint32_t pending = ~0u;
  auto publish = [&]() {
    if (pending != ~0u) {
      __syncwarp();
      if (lane == 0) red_release_gpu(wa.cnt + pending);
      pending = ~0u;
    }
  };

  const uint32_t p0 = blockIdx.x * kWarpsPerCta + wid;
  if (lane == 0) mbar_init(bar, 1);
  __syncwarp();
  // the first request: phase-0 items at once; a phase-1 first item (small
  // batches, rows < lag) goes through the deferred path (wait for its row)
  bool loaded = false;
  if (p0 < total) {
    int ph;
    uint32_t rl0, sub0;
    warp_item(p0, rows, wa.lag, ph, rl0, sub0);
    loaded = (ph == 0);
    if (loaded && lane == 0) issue(p0);
  }
  uint32_t parity = 0;

  for (uint32_t p = p0; p < total; p += nw) {
    int phase;
    uint32_t rl, sub;
    warp_item(p, rows, wa.lag, phase, rl, sub);
    const uint64_t row = row_of(rl);
    const uint32_t limb = limb_of(row);
    const LimbConst c = a.lc[limb];
    const ulonglong2* __restrict__ tw = a.tw + static_cast<uint64_t>(limb) * 16384u;
    uint64_t* __restrict__ dst = a.out + row * 16384u;
    const uint32_t pn = p + nw;
    if (!loaded) {  // deferred request (the row was not ready at the last exchange)
      if (lane == 0) {
        int ph;
        uint32_t rl2, sub2;
        warp_item(p, rows, wa.lag, ph, rl2, sub2);
        if (ph == 1) wait_row(rl2);
        issue(p);
      }
      __syncwarp();
    }
    if (pn < total) prefetch_in(pn);
    mbar_wait(bar, parity);
    parity ^= 1;
    uint64_t v[32];
    bool next_issued = false;
    auto request_next = [&]() {  // after the exchange reads: the region is free
      __syncwarp();
      bool ok = true;
      if (lane == 0 && pn < total) {
        int ph;
        uint32_t rl2, sub2;
        warp_item(pn, rows, wa.lag, ph, rl2, sub2);
        ok = (ph == 0) || row_ready(rl2);
        if (ok) issue(pn);
      }
      next_issued = __shfl_sync(0xffffffffu, ok ? 1 : 0, 0) != 0;
    };

    if (phase == 0) {
      // ---- columns: stages 13..9, a bits 6..2 in registers ----
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = A::load(SW[32 * r + lane]);
      {
        auto t = [&](int i, int hi) { return ldtw(tw + (16 >> i) + hi); };
        stage32<A, true, false, 4>(v, c, [&](int hi) { return t(4, hi); });
        publish();  // the previous item's stores have had a stage to drain
        stage32<A, true, false, 3>(v, c, [&](int hi) { return t(3, hi); });
        stage32<A, true, false, 2>(v, c, [&](int hi) { return t(2, hi); });
        stage32<A, true, false, 1>(v, c, [&](int hi) { return t(1, hi); });
        stage32<A, true, false, 0>(v, c, [&](int hi) { return t(0, hi); });
      }
      __syncwarp();  // every lane has read the landing image
#pragma unroll
      for (int r = 0; r < 32; ++r) SW[cidx(4u * r + g, blo)] = v[r];
      __syncwarp();
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = SW[cidx(r + 32u * g, blo)];
      request_next();
      {
        auto t = [&](int i, int hi) { return ldtw(tw + (64 >> i) + hi + (g << (4 - i))); };
        stage32<A, true, false, 1>(v, c, [&](int hi) { return t(1, hi); });
        stage32<A, true, false, 0>(v, c, [&](int hi) { return t(0, hi); });
      }
#pragma unroll
      for (int r = 0; r < 32; ++r) st_hint(dst + 128u * (r + 32u * g) + 8u * sub + blo, v[r], pol_keep);
      pending = rl;
    } else {
      // ---- rows: stages 6..2, b bits 2..6 in registers; twiddles staged ----
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = SW[132 * alo + 4 * r + b01];
      {
        auto t = [&](int i, int hi) { return TWB[twseg(i) + (alo << (4 - i)) + hi]; };
        stage32<A, true, false, 4>(v, c, [&](int hi) { return t(4, hi); });
        publish();  // the previous item's stores have had a stage to drain
        stage32<A, true, false, 3>(v, c, [&](int hi) { return t(3, hi); });
        stage32<A, true, false, 2>(v, c, [&](int hi) { return t(2, hi); });
        stage32<A, true, false, 1>(v, c, [&](int hi) { return t(1, hi); });
        stage32<A, true, false, 0>(v, c, [&](int hi) { return t(0, hi); });
      }
      __syncwarp();
#pragma unroll
      for (int r = 0; r < 32; ++r) SW[ridx(alo, 4u * r + b01)] = v[r];
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const ulonglong2 p2 = *reinterpret_cast<const ulonglong2*>(SW + ridx(q, 4u * lane + 2 * h));
          v[4 * q + 2 * h] = p2.x;
          v[4 * q + 2 * h + 1] = p2.y;
        }
      request_next();
      const uint32_t ab = 8u * sub;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t ar = ab + q;
        const ulonglong2 w1 = ldtw(tw + 4096u + 32u * ar + lane);
        A::template fwd<false>(v[4 * q + 0], v[4 * q + 2], w1, c);
        A::template fwd<false>(v[4 * q + 1], v[4 * q + 3], w1, c);
        const ulonglong2 w0a = ldtw(tw + 8192u + 64u * ar + 2u * lane);
        const ulonglong2 w0b = ldtw(tw + 8192u + 64u * ar + 2u * lane + 1u);
        A::template fwd<false>(v[4 * q + 0], v[4 * q + 1], w0a, c);
        A::template fwd<false>(v[4 * q + 2], v[4 * q + 3], w0b, c);
        st_v4(dst + 128u * ar + 4u * lane, fwd_out<A>(v[4 * q], c, a.fout), fwd_out<A>(v[4 * q + 1], c, a.fout),
              fwd_out<A>(v[4 * q + 2], c, a.fout), fwd_out<A>(v[4 * q + 3], c, a.fout));
      }
    }
    loaded = next_issued;
    if (!loaded) publish();  // nothing of ours may be pending while we wait for a row
  }
  publish();
}

}  // namespace nk
