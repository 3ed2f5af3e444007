// ntt_pair14: the 16384-word block transform on a CTA PAIR (thread-block
// cluster of 2), two pairs resident per SM.
//
// Why: one 16384-word block fills half the register file (32 words x 512
// threads). With one CTA per SM every exchange phase idles the FP64 pipe for
// the whole SM. Here a block is split over the two CTAs of a cluster (8192
// words each, 256 threads x 32 words), so an SM hosts halves of two
// independent blocks and one half computes while the other exchanges or waits.
//
// Index bits of a block word j (14 bits) in each register pass
// (regs = the 5 bits a thread holds in registers; X = a passenger bit):
//
//   forward (stages 13..0)        inverse (stages 0..13)
//   P1 regs 13..9                 P1 regs 0..4
//      thread 0..7, CTA 8            lanes 5..9, warps 10..12, CTA 13
//   -- DSMEM exchange --          -- warp-local exchange (2 rounds on bit 4) --
//   P2 regs 8..5 + X=4            P2 regs 8..5 + X=4
//      lanes 0..3,9 warps 10..12     lanes 0..3,9 warps 10..12, CTA 13
//      CTA 13                     -- DSMEM exchange --
//   -- warp-local exchange --     P3 regs 13..9
//   P3 regs 4..0                     thread 0..7, CTA 8
//      lanes 5..9, warps 10..12, CTA 13
//
// DSMEM exchange: every thread stores each register into the image of the
// CTA that owns it in the next pass (st.shared::cluster for the peer), a
// cluster barrier, then local reads. The image is the CTA's TMA staging
// buffer, so the next block's TMA is issued right after the image is read.
// The warp-local exchange uses a per-warp 4.5 KiB image (two rounds split on
// bit 4, which is a register bit on both sides) under __syncwarp only.
// Butterfly arithmetic, twiddle addressing and the low (lane-contiguous)
// twiddle table are those of pass14 (ntt_kernels.cuh).
#pragma once
#include "ntt_kernels.cuh"

namespace nk {

constexpr uint32_t kPairHalfWords = 8192;
constexpr uint32_t kPairStageBytes = kPairHalfWords * 8;  // 64 KiB
constexpr uint32_t kWarpImgWords = 640;                   // 512 + 2 * 32 pad, rounded to 1 KiB (TMA-store swizzle atoms)
// barriers: full (TMA), x (exchange landed), free_mine / free_peer (staging
// consumed by this CTA's / the peer's warps), sfree (image read: TMA may refill)
constexpr size_t kPairSmemBytes = 1024 + kPairStageBytes + 8 * kWarpImgWords * 8 + 5 * 8;

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t ncluster_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_peer(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_cluster_u64(uint32_t addr, uint64_t v) {
  asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
// st.async: 8-byte store into the peer CTA's shared memory that signals the
// peer's mbarrier (complete_tx) when it lands; no cluster barrier needed.
__device__ __forceinline__ void st_async_u64(uint32_t addr, uint64_t v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(addr),
               "l"(v), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_local(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// relaxed arrive: used only where data dependence already orders the
// preceding shared loads (their values have been consumed)
__device__ __forceinline__ void mbar_arrive_relaxed_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_relaxed_remote(uint32_t rbar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
}
// try_wait with a back-off between polls: a warp that waits (for the TMA, the
// exchange or the peer) leaves the issue slots to the other resident CTA,
// which is usually computing. 64 ns: forward 242 -> 240 us, cfg5 763 -> 756 us
// (32-256 ns measured alike; the spin loops were 21% of issued instructions).
#ifndef NK_WAIT_BACKOFF
#define NK_WAIT_BACKOFF 64
#endif
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t phase) {
#if NK_WAIT_BACKOFF > 0
  uint32_t done;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  while (!done) {
    __nanosleep(NK_WAIT_BACKOFF);
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
#else
  mbar_wait(bar, phase);
#endif
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            int32_t c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2,
                                             const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}


#if defined(NK_DBG_TIMELINE)  // perf experiment: per-warp phase timestamps into a.dbg
#define NK_TS(id)                                                                            \
  do {                                                                                       \
    if (a.dbg && l == 0 && it_ < 32)                                                         \
      a.dbg[((static_cast<uint64_t>(blockIdx.x) * 8 + w) * 32 + it_) * 16 + (id)] = clock64(); \
  } while (0)
#else
#define NK_TS(id) ((void)0)
#endif

// tout (forward): 3D view [words/32][2][16] of the result, boxes 16 x 1 x 32
// with 128B swizzle = one warp's output round straight from its image.
// MULB: the fused poly_mult_mod forward (dyadic product in the store; a
// separate instance so the plain transform carries none of its registers)
template <class A, bool FWD, bool ILTM0, bool MULB = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 2)
    ntt_pair14(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, NttArgs a,
               uint32_t nitems) {
  using P1 = typename std::conditional<FWD, PassD<9, 5, -1>, PassD<0, 5, -1>>::type;
  using P2 = PassD<5, 4, 4>;
  using P3 = typename std::conditional<FWD, PassD<0, 5, -1>, PassD<9, 5, -1>>::type;
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* Sb = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  uint64_t* S = reinterpret_cast<uint64_t*>(Sb);  // staging / DSMEM image (8192 words)
  const uint32_t t = threadIdx.x, l = t & 31u, w = t >> 5;
  uint64_t* W = S + kPairHalfWords + w * kWarpImgWords;  // this warp's image
  uint64_t* bar = S + kPairHalfWords + 8 * kWarpImgWords;
  uint64_t* bar_x = bar + 1;
  uint64_t* bar_free_mine = bar + 2;
  uint64_t* bar_free_peer = bar + 3;
  uint64_t* bar_sfree = bar + 4;
  const uint32_t c = cluster_ctarank();
  const uint32_t peer = c ^ 1u;
  const uint32_t s_peer = mapa_peer(smem_u32(S), peer);
  const uint32_t x_peer = mapa_peer(smem_u32(bar_x), peer);
  const uint32_t free_peer_remote = mapa_peer(smem_u32(bar_free_peer), peer);
  const uint32_t lognb = a.logn - kB14;

  auto item_row = [&](uint32_t k, uint64_t& row, uint64_t& blk) {
    row = (static_cast<uint64_t>(k) >> lognb) * a.row_mul + a.row_add;
    blk = static_cast<uint64_t>(k) & ((uint64_t{1} << lognb) - 1);
  };
  // this CTA's half of block k: forward = the words with index bit 8 == c
  // (3D map [superline of 512][32 lines][16 words], box 16 x 16 x 32 at line
  // 16c), inverse = the words with bit 13 == c (2D swizzled lines, 2 boxes)
  auto issue = [&](uint32_t k) {
    uint64_t row, blk;
    item_row(k, row, blk);
    const uint64_t word0 = row * a.n + (blk << kB14);
    mbar_expect_tx(bar, kPairStageBytes);
    if (FWD) {
      tma_load_3d(S, &tin, 0, static_cast<int32_t>(16 * c), static_cast<int32_t>(word0 >> 9), bar);
    } else {
      const int32_t line0 = static_cast<int32_t>((word0 >> 4) + 512 * c);
      tma_load_2d(Sb, &tin, 0, line0, bar);
      tma_load_2d(Sb + 32768, &tin, 0, line0 + 256, bar);
    }
  };

  // the same boxes as issue(), prefetched into L2 only: the real TMA (which
  // must wait until the staging buffer is free) then reads from L2
  auto prefetch_l2 = [&](uint32_t k) {
    uint64_t row, blk;
    item_row(k, row, blk);
    const uint64_t word0 = row * a.n + (blk << kB14);
    if (FWD) {
      asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                       reinterpret_cast<uint64_t>(&tin)),
                   "r"(0), "r"(static_cast<int32_t>(16 * c)), "r"(static_cast<int32_t>(word0 >> 9))
                   : "memory");
    } else {
      const int32_t line0 = static_cast<int32_t>((word0 >> 4) + 512 * c);
      asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                       reinterpret_cast<uint64_t>(&tin)),
                   "r"(0), "r"(line0)
                   : "memory");
      asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(
                       reinterpret_cast<uint64_t>(&tin)),
                   "r"(0), "r"(line0 + 256)
                   : "memory");
    }
  };

  const uint32_t k0 = cluster_id_x(), kstep = ncluster_x();
  if (t == 0) {
    mbar_init(bar, 1);
    mbar_init(bar_x, 256);
    mbar_init(bar_free_mine, 8);
    mbar_init(bar_free_peer, 8);
    mbar_init(bar_sfree, 8);
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tin)) : "memory");
  }
  // the peer's barriers must be initialised before any remote arrive / st.async
  cluster_arrive();
  cluster_wait();
  if (t == 0 && k0 < nitems) issue(k0);
  uint32_t phase = 0;  // parity of every per-item barrier

  // thread index bits of each pass (block-local j), see the header table
  const uint32_t jt_p2 = (l & 15u) | ((l >> 4) << 9) | (w << 10) | (c << 13);
  const uint32_t jt_low = (l << 5) | (w << 10) | (c << 13);  // fwd P3 / inv P1
  const uint32_t jt_hi = t | (c << 8);                        // fwd P1 / inv P3
  const uint32_t jt1 = FWD ? jt_hi : jt_low;
  const uint32_t jt3 = FWD ? jt_low : jt_hi;

  uint32_t it_ = 0;
  (void)it_;
  for (uint32_t k = k0; k < nitems; k += kstep) {
    uint64_t row, blk;
    item_row(k, row, blk);
    NK_TS(0);
    const uint32_t limb = a.limb0 + static_cast<uint32_t>(row % a.nlimbs);
    const LimbConst cst = a.lc[limb];
    const typename A::Tw* __restrict__ tw = tw_of<A>(a, limb);
    const typename A::Tw* __restrict__ twl = twl_of<A>(a, limb) + (blk << kB14) + (jt_low >> 5);
    const uint64_t boff = blk << kB14;
    uint64_t* __restrict__ dst = a.out + row * a.n + boff;
    const uint64_t xbase = a.n + boff;
    uint64_t v[32];

    // ---- P1 words from the staging buffer ----
    mbar_wait_backoff(bar, phase);
    if (FWD && t == 0 && k + kstep < nitems) prefetch_l2(k + kstep);
    NK_TS(1);
    if (FWD) {
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = A::load(S[t + 256 * r]);  // local = j & 255 | (j >> 9) << 8
    } else {
      const uint32_t jl = jt_low & 0x1FFFu;  // 32 contiguous words, 128B-swizzled lines
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t row16 = (jl >> 4) + h;
        const uint32_t rowoff = row16 << 7, sw = row16 & 7;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc) {
          const ulonglong2 p = *reinterpret_cast<const ulonglong2*>(Sb + rowoff + ((cc ^ sw) << 4));
          v[16 * h + 2 * cc] = A::load(p.x);
          v[16 * h + 2 * cc + 1] = A::load(p.y);
        }
      }
    }

    NK_TS(2);
    pass14<A, FWD, P1, ILTM0>(v, tw, twl, a.n, xbase + jt1, cst);
    NK_TS(3);
    // every P1 word has been consumed: the staging buffer may be overwritten
    __syncwarp();
    if (l == 0) {
      mbar_arrive_relaxed_local(bar_free_mine);
      mbar_arrive_relaxed_remote(free_peer_remote);
    }

    if (FWD) {
      // ---- DSMEM exchange P1 -> P2: word j goes to CTA bit13(j), index j & 0x1FFF ----
      mbar_wait_backoff(bar_free_mine, phase);
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if ((r >> 4) == static_cast<int>(c)) S[t + 256u * c + 512u * (r & 15)] = v[r];
      if (t == 0) mbar_arrive_expect_local(bar_x, kPairStageBytes / 2);
      else mbar_arrive_local(bar_x);
      mbar_wait_backoff(bar_free_peer, phase);
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if ((r >> 4) != static_cast<int>(c)) st_async_u64(s_peer + (t + 256u * c + 512u * (r & 15)) * 8u, v[r], x_peer);
      mbar_wait_backoff(bar_x, phase);  // acquire.cta: st.async data is ordered by complete_tx (no L1 invalidate)
      NK_TS(4);
#pragma unroll
      for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int r = 0; r < 16; ++r) v[16 * g + r] = S[(jt_p2 + (g << 4) + (r << 5)) & 0x1FFFu];
      __syncwarp();
      if (l == 0) mbar_arrive_local(bar_sfree);  // release: the image reads are performed
      if (t == 0) {
        mbar_wait(bar_sfree, phase);
        if (k + kstep < nitems) {
          fence_proxy_async();
          issue(k + kstep);
        }
      }
    } else {
      // ---- warp-local exchange P1 -> P2 (rounds on bit 4) ----
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int m = 0; m < 16; m += 2)
          *reinterpret_cast<ulonglong2*>(W + wimg(jt_low + 16 * h + m)) =
              make_ulonglong2(v[16 * h + m], v[16 * h + m + 1]);
        __syncwarp();
#pragma unroll
        for (int r = 0; r < 16; ++r) v[16 * h + r] = W[wimg(jt_p2 + (r << 5))];
        __syncwarp();
      }
    }

    NK_TS(5);
    pass14<A, FWD, P2, false>(v, tw, twl, a.n, xbase + jt_p2, cst);
    NK_TS(6);

    if (FWD) {
      // ---- warp-local exchange P2 -> P3 (rounds on bit 4) ----
      if (l == 0) bulk_wait_read();  // the last item's output store has read the image
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int r = 0; r < 16; ++r) W[wimg(jt_p2 + (r << 5))] = v[16 * h + r];
        __syncwarp();
#pragma unroll
        for (int m = 0; m < 16; m += 2) {
          const ulonglong2 p = *reinterpret_cast<const ulonglong2*>(W + wimg(jt_low + 16 * h + m));
          v[16 * h + m] = p.x;
          v[16 * h + m + 1] = p.y;
        }
        __syncwarp();
      }
    } else {
      // ---- DSMEM exchange P2 -> P3: word j goes to CTA bit8(j), index (j & 255) | (j >> 9) << 8 ----
      mbar_wait_backoff(bar_free_mine, phase);
#pragma unroll
      for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const uint32_t j = jt_p2 + (g << 4) + (r << 5);
          if (((r >> 3) & 1) == static_cast<int>(c)) S[(j & 255u) | ((j >> 9) << 8)] = v[16 * g + r];
        }
      if (t == 0) mbar_arrive_expect_local(bar_x, kPairStageBytes / 2);
      else mbar_arrive_local(bar_x);
      mbar_wait_backoff(bar_free_peer, phase);
#pragma unroll
      for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const uint32_t j = jt_p2 + (g << 4) + (r << 5);
          if (((r >> 3) & 1) != static_cast<int>(c))
            st_async_u64(s_peer + ((j & 255u) | ((j >> 9) << 8)) * 8u, v[16 * g + r], x_peer);
        }
      mbar_wait_backoff(bar_x, phase);  // acquire.cta: st.async data is ordered by complete_tx (no L1 invalidate)
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = S[t + 256 * r];
      __syncwarp();
      if (l == 0) mbar_arrive_local(bar_sfree);
      if (t == 0) {
        mbar_wait(bar_sfree, phase);
        if (k + kstep < nitems) {
          fence_proxy_async();
          issue(k + kstep);
        }
      }
    }

    NK_TS(7);
    // canonical inverse (Arith52S, whole rows): n^-1 folded into the last stage
    // (bit 13, single twiddle), as in ntt_pair14 / ntt_grp14
    constexpr bool kFoldLast = !FWD && A::kSigned;
    if constexpr (kFoldLast) {
      pass14<A, FWD, P3, false, 1>(v, tw, twl, a.n, xbase + jt3, cst);
#pragma unroll
      for (int r = 0; r < 16; ++r) A::inv_fold(v[r], v[r + 16], cst);
    } else {
      pass14<A, FWD, P3, false>(v, tw, twl, a.n, xbase + jt3, cst);
    }
    NK_TS(8);

    if (FWD) {
      // 32 contiguous words per thread -> coalesced lines through the warp
      // image (32 rows of 16 words, 128B swizzle), one round per bit 4
      uint8_t* Wb = reinterpret_cast<uint8_t*>(W);
      uint64_t* wdst = dst + (w << 10) + (c << 13);
      // Code shape per instance, as measured: the plain Arith52S forward drops
      // the direct-store path entirely (no spills: 241 -> 236 us), while the
      // other plain instances keep it behind a runtime test (the integer
      // forward is scheduled 8% better with it present: 363 vs 391 us).
      constexpr bool kKeepDirect = !A::kSigned;
      const uint64_t* mulb =
          (MULB || (kKeepDirect && a.mulb)) ? a.mulb + row * a.n + boff + (w << 10) + (c << 13) : nullptr;
      // the fused product multiplies the signed words and canonicalises once
      // (mulmod_signed_canon) in the store loop below
      if constexpr (!(A::kSigned && MULB)) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = fwd_out<A>(v[i], cst, a.fout);
      }
      if (!MULB && (!kKeepDirect || !mulb)) {
        // the image rows are the TMA box rows: one bulk tensor store per round
        const int32_t srow = static_cast<int32_t>((row * a.n + boff + (w << 10) + (c << 13)) >> 5);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 1) {
            if (l == 0) bulk_wait_read();
            __syncwarp();
          }
#pragma unroll
          for (int cc = 0; cc < 8; ++cc)
            *reinterpret_cast<ulonglong2*>(Wb + (l << 7) + ((cc ^ (l & 7)) << 4)) =
                make_ulonglong2(v[16 * h + 2 * cc], v[16 * h + 2 * cc + 1]);
          fence_proxy_async();
          __syncwarp();
          if (l == 0) tma_store_3d(&tout, 0, h, srow, Wb);
        }
      } else
#pragma unroll
      for (int h = 0; h < 2; ++h) {
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
          *reinterpret_cast<ulonglong2*>(Wb + (l << 7) + ((cc ^ (l & 7)) << 4)) =
              make_ulonglong2(v[16 * h + 2 * cc], v[16 * h + 2 * cc + 1]);
        // the round's multiplier words in flight across the image round trip,
        // issued once the round's words left their registers (cfg5 736 -> 730 us)
        ulonglong2 gbv[8];
        if constexpr (A::kSigned && MULB) {
#pragma unroll
          for (int s2 = 0; s2 < 8; ++s2)
            gbv[s2] = __ldg(reinterpret_cast<const ulonglong2*>(
                mulb + ((((l >> 3) + 4 * s2) << 5) + (h << 4) + ((l & 7) << 1))));
        }
        __syncwarp();
#pragma unroll
        for (int s2 = 0; s2 < 8; ++s2) {  // 32 rows, 4 per warp instruction
          const uint32_t rw = (l >> 3) + 4 * s2, cc = l & 7;
          ulonglong2 p = *reinterpret_cast<const ulonglong2*>(Wb + (rw << 7) + ((cc ^ (rw & 7)) << 4));
          const uint32_t off = (rw << 5) + (h << 4) + (cc << 1);
          if constexpr (A::kSigned && MULB) {
            {  // fused dyadic product of poly_mult_mod (ring.hpp:39-41)
              const ulonglong2 gb = gbv[s2];
              p.x = mulmod_signed_canon(p.x, gb.x, cst);
              p.y = mulmod_signed_canon(p.y, gb.y, cst);
            }
          }
          *reinterpret_cast<ulonglong2*>(wdst + off) = p;
        }
        __syncwarp();
      }
    } else {
      if (kFoldLast) {
        // already canonical
      } else if (lognb == 0) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = inv_out<A>(v[i], cst, a.fout);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = A::store(v[i]);  // intermediate of a long row
      }
#pragma unroll
      for (int r = 0; r < 32; ++r) dst[jt_hi + 512 * r] = v[r];
    }
    NK_TS(9);
    phase ^= 1;
    ++it_;
  }
  if (FWD && l == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  // no CTA may exit while its peer can still signal or write into it: every
  // remote operation of the last item precedes the peer's wait on bar_x
  cluster_arrive();
  cluster_wait();
}

}  // namespace nk
