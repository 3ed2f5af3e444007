// poly_mul14: poly_mult_mod (ring.hpp:28-43: fwd(f), fwd(g), dyadic product,
// inv) for N = 16384 rows in ONE persistent kernel, the intermediate spectra
// never leaving the SM:
//
//   per (limb, polynomial) row k, on one 512-thread CTA (the ntt_grp14 passes):
//   1. g: TMA load -> forward (three register passes, two group exchanges) ->
//      g^ reduced to |g^| < 2q -> Tensor Memory (tcgen05.st, 128 KiB of the
//      SM's 256 KiB TMEM; each thread its own 64 columns of one lane)
//   2. f: TMA load (issued as soon as g's staging words are consumed) ->
//      forward -> f^ (|f^| < 4q, signed FP64) -> times g^ read back from TMEM
//      (tcgen05.ld): p = mul_recip(csubS(f^), g^), |p| < 1.75q
//   3. p written into the staging buffer as the inverse's input image, the
//      inverse (n^-1 folded into its last stage) -> canonical words -> HBM
//
// HBM traffic: 8 B (f) + 8 B (g) + 8 B (result) per coefficient, against 56 B
// for the three-launch sequence. The arithmetic is Arith52S (q < 2^50, whole
// rows, canonical result): the result is unique, so it equals the
// reference's fwd(1,4) x2 / eltwise_mult_mod(4) / inv(1,1) word for word.
//
// Product bound: csubS gives |f^|, |g^| < 2q, so |f^ g^| < 4q^2 < 2^102 and
// the rounded-reciprocal product of modmath.cuh (mul_recip) applies as for a
// twiddle (its derivation only uses |w v| < 4q^2): |p| < 1.75q, within the
// signed inverse's |x| < 2q input range.
//
// Product image (the inverse's P1 input): word j at line j >> 4, 16-byte chunk
// ((j >> 1) & 7) ^ (line & 7) ^ ((j >> 9) & 7) ^ (j >> 13) (the last term makes the
// inverse's P1 reads conflict free: its eight lanes of a phase differ in j5, j6, j13). Against the TMA layout the
// extra XOR (j9..j11) permutes chunks inside a line only, so every exchange-1
// group keeps its slot set (exchange 1 is in place); it makes the writes
// conflict free (the forward's P3 threads of one 8-lane phase differ exactly
// in j9..j11) while the inverse's P1 reads keep their layout (the key is a
// thread constant there).
#pragma once
#include "ntt_grp.cuh"
#include "ntt_str.cuh"

namespace nk {

struct PolyArgs {
  NttArgs a;             // out, forward tables (tw8 / twg8), lc, n, rows, limbs
  const uint64_t* itw8;  // inverse tables of the plan, same layouts
  const uint64_t* itwg8;
  const uint64_t* itwq8;  // (two-stream kernel: a.twq8 / itwq8)
};

// [grp layout][bar_free][TMEM base address]
constexpr size_t kPolySmemBytes = kGrpSmemBytes + 16;
constexpr uint32_t kPolyTmemCols = 256;  // 128 lanes x 256 columns x 4 B = one 128 KiB spectrum

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint64_t* v8) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16};" ::"r"(taddr),
      "r"(lo32(v8[0])), "r"(hi32(v8[0])), "r"(lo32(v8[1])), "r"(hi32(v8[1])), "r"(lo32(v8[2])), "r"(hi32(v8[2])),
      "r"(lo32(v8[3])), "r"(hi32(v8[3])), "r"(lo32(v8[4])), "r"(hi32(v8[4])), "r"(lo32(v8[5])), "r"(hi32(v8[5])),
      "r"(lo32(v8[6])), "r"(hi32(v8[6])), "r"(lo32(v8[7])), "r"(hi32(v8[7]))
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint64_t* v8) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, "
      "[%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v8[i] = (static_cast<uint64_t>(r[2 * i + 1]) << 32) | r[2 * i];
}

// One forward transform (the ntt_grp14 forward, canonical input) of the row
// in the staging buffer (bar_full phase `fph`); `consumed` runs once this
// warp has read all its staging words. nx: transforms done by the CTA (the
// exchange barriers' parity), incremented.
// threadIdx.x read through a volatile asm: thread-constant addresses derived
// from it are recomputed where they are used instead of being hoisted out of
// the item loop for all three transforms at once (which spills)
__device__ __forceinline__ uint32_t tid_opaque() {
  uint32_t t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return t;
}

template <class A, class F>
__device__ __forceinline__ void poly_forward(uint64_t (&v)[32], uint8_t* St, uint8_t* Eg, const NttArgs& a, uint32_t k,
                                             uint64_t* bar_full, uint32_t fph, uint64_t* bar_r1g, uint64_t* bar_r2g,
                                             uint32_t& nx, F&& consumed) {
  using M = GrpMap<true>;
  const uint32_t t = tid_opaque(), w = t >> 5, l = t & 31u;
  const uint32_t jt1 = M::jt1(w, l), jt2 = M::jt2(w, l), jt3 = M::jt3(w, l);
  const uint32_t limb = a.limb0 + (k % a.nlimbs);
  const LimbConst c = a.lc[limb];
  const uint64_t n = a.n;
  const uint64_t* __restrict__ tw = a.tw8 + static_cast<uint64_t>(limb) * n;
  const uint64_t* __restrict__ twl = a.twg8 + static_cast<uint64_t>(limb) * n + t;
  mbar_wait(bar_full, fph);
  grp::p1_read<A, true>(v, St, jt1);
  __syncwarp();
  if (l == 0) mbar_arrive_local(bar_r1g);
  pass14<A, true, PassD<9, 5, -1>, true>(v, tw, twl, n, n + jt1, c);
  grp::ex1<true>(v, St, jt1, grp::q2_of<true>(jt2), bar_r1g, nx & 1u, w >> 2);
  consumed();
  pass14<A, true, PassD<5, 4, 4>, false>(v, tw, twl, n, n + jt2, c);
  grp::ex2<true>(v, Eg, ex2_off<true>(jt2), ex2_off<true>(jt3), bar_r2g, (nx & 1u) ^ 1u, w & 3u, l);
  pass14<A, true, PassD<0, 5, -1>, false>(v, tw, twl, n, n + jt3, c);
  ++nx;
}

template <class A>
__global__ void __launch_bounds__(512, 1)
    poly_mul14(const __grid_constant__ CUtensorMap tf, const __grid_constant__ CUtensorMap tg, PolyArgs pa,
               uint32_t nitems) {
  static_assert(A::kSigned, "poly_mul14 runs the signed FP64 policy");
  using I1 = PassD<0, 5, -1>;
  using I2 = PassD<5, 4, 13>;
  using I3 = PassD<9, 5, -1>;
  using MF = GrpMap<true>;
  using MI = GrpMap<false>;
  const NttArgs& a = pa.a;
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* St = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  uint8_t* E = St + kStageBytes;
  uint64_t* bar_full = reinterpret_cast<uint64_t*>(E + kGrpExBytes + kGrpOutBytes);
  uint64_t* bar_r1 = bar_full + 1;    // [4] ex1 groups: P1 reads done
  uint64_t* bar_r2 = bar_full + 5;    // [4] ex2 groups: last-round reads done
  uint32_t* cnt = reinterpret_cast<uint32_t*>(bar_full + 9);
  uint64_t* bar_free = bar_full + 10;  // f's P2 reads done (16 warps): the staging buffer takes p
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar_full + 11);
  const uint32_t t = threadIdx.x, l = t & 31u, w = t >> 5;
  const uint32_t g1 = w >> 2, g2 = w & 3u;

  auto issue = [&](const CUtensorMap* map, uint32_t k) {
    const int32_t y0 = static_cast<int32_t>(static_cast<uint64_t>(k) * (a.n >> 4));
    mbar_expect_tx(bar_full, kStageBytes);
#pragma unroll
    for (int q = 0; q < 4; ++q) tma_load_2d(St + q * 32768, map, 0, y0 + q * 256, bar_full);
  };

  if (t == 0) {
    mbar_init(bar_full, 1);
    for (int i = 0; i < 4; ++i) {
      mbar_init(bar_r1 + i, 4);
      mbar_init(bar_r2 + i, 4);
    }
    mbar_init(bar_free, 16);
    *cnt = 0;
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tf)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tg)) : "memory");
  }
  if (w == 0) {  // one warp allocates the TMEM columns (one CTA per SM: never contended by this kernel)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "n"(kPolyTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // this warp's TMEM quarter: lanes 32 (w % 4) .. + 31 (the lanes a warp may
  // access), columns 64 (w / 4) .. + 63: 32 words per thread
  const uint32_t taddr = *tslot + ((32u * (w & 3u)) << 16) + 64u * (w >> 2);
  if (t == 0 && blockIdx.x < nitems) issue(&tg, blockIdx.x);

  uint8_t* Eg = E + (g2 << 14);
  uint32_t nx = 0;  // transforms done by this CTA: parity of the exchange barriers
  uint32_t it = 0;  // items done by this CTA: parity of bar_free

  for (uint32_t k = blockIdx.x; k < nitems; k += gridDim.x) {
    uint64_t v[32];

    // ---- g^ -> TMEM, then f^ (one copy of the forward's code: the kernel
    // body must stay small enough for the instruction caches) ----
#pragma unroll 1
    for (uint32_t ph = 0; ph < 2; ++ph) {
      poly_forward<A>(v, St, Eg, a, k, bar_full, ph, bar_r1 + g1, bar_r2 + g2, nx, [&] {
        if (ph == 0) {
          grp::staging_consumed(cnt, l, [&] {
            fence_proxy_async();
            issue(&tf, k);  // f of the same row
          });
        } else {
          __syncwarp();
          if (l == 0) mbar_arrive_local(bar_free);  // the staging buffer may take the product
        }
      });
      if (ph == 0) {
        const double twoq = a.lc[a.limb0 + (k % a.nlimbs)].twoq_d;
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = as_u(csubS(as_d(v[i]), twoq));
#pragma unroll
        for (int q = 0; q < 4; ++q) tmem_st16(taddr + 16u * q, v + 8 * q);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
    }
    const uint32_t limb = a.limb0 + (k % a.nlimbs);
    {
      const LimbConst c = a.lc[limb];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint64_t gh[8];
        tmem_ld16(taddr + 16u * q, gh);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          v[8 * q + i] = as_u(mul_recip(csubS(as_d(v[8 * q + i]), c.twoq_d), as_d(gh[i]), c.qinv, c.q_d));
      }
    }

    // ---- the product image in the staging buffer (see the header) ----
    mbar_wait(bar_free, it & 1u);  // every warp has read f's staging words
    {
      const uint32_t to = tid_opaque(), jf3 = MF::jt3(to >> 5, to & 31u);
      const uint32_t key = ((jf3 >> 9) & 7u) ^ ((jf3 >> 13) & 1u);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t line = (jf3 >> 4) | static_cast<uint32_t>(h);
        const uint32_t sw = (line & 7u) ^ key;
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
          *reinterpret_cast<ulonglong2*>(St + (line << 7) + ((cc ^ sw) << 4)) =
              make_ulonglong2(v[16 * h + 2 * cc], v[16 * h + 2 * cc + 1]);
      }
    }
    __syncthreads();

    // ---- inverse (n^-1 folded into the last stage), canonical words out ----
    {
      const uint32_t to = tid_opaque(), wo = to >> 5, lo = to & 31u;
      const uint32_t ji1 = MI::jt1(wo, lo), ji2 = MI::jt2(wo, lo), ji3 = MI::jt3(wo, lo);
      const LimbConst c = a.lc[limb];
      const uint64_t* __restrict__ itw = pa.itw8 + static_cast<uint64_t>(limb) * a.n;
      const uint64_t* __restrict__ itwl = pa.itwg8 + static_cast<uint64_t>(limb) * a.n + tid_opaque();
      grp::p1_read<A, false, true>(v, St, ji1, ((ji1 >> 9) & 7u) ^ ((ji1 >> 13) & 1u));
      __syncwarp();
      if (l == 0) mbar_arrive_local(bar_r1 + g1);
      pass14<A, false, I1, false>(v, itw, itwl, a.n, a.n + ji1, c);
      grp::ex1<false>(v, St, ji1, grp::q2_of<false>(ji2), bar_r1 + g1, nx & 1u, g1);
      grp::staging_consumed(cnt, l, [&] {
        if (k + gridDim.x < nitems) {
          fence_proxy_async();
          issue(&tg, k + gridDim.x);  // g of the next row
        }
      });
      pass14<A, false, I2, false>(v, itw, itwl, a.n, a.n + ji2, c);
      grp::ex2<false>(v, Eg, ex2_off<false>(ji2), ex2_off<false>(ji3), bar_r2 + g2, (nx & 1u) ^ 1u, g2, l);
      pass14<A, false, I3, false, 1>(v, itw, itwl, a.n, a.n + ji3, c);
#pragma unroll
      for (int r = 0; r < 16; ++r) A::inv_fold(v[r], v[r + 16], c);
      ++nx;
      uint64_t* __restrict__ dst = a.out + static_cast<uint64_t>(k) * a.n;
#pragma unroll
      for (int r = 0; r < 32; ++r) dst[ji3 | (static_cast<uint32_t>(r) << 9)] = v[r];
    }
    ++it;
  }

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tslot), "n"(kPolyTmemCols)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// poly_str14: the same single-kernel poly_mult_mod on the two-stream cores
// (ntt_str.cuh). The forward core leaves every thread with 16 words of each
// 8192-word half in exactly the layout the inverse core starts from, so g^
// goes to Tensor Memory and comes back in the same thread, the product
// p = f^ g^ is formed in registers, and the inverse starts from them: no
// product image, and the exchanges of both directions overlap the other
// stream's arithmetic.
//   bar_full   g (with the row's limb constants), then f, per row
//   bar_rd     P1 reads done: once per forward
//   bar_w[2]   stream written by every warp: g's forward, f's forward, the inverse
//   bar_free   f's staging words consumed by every warp: the inverse's e1' may use the halves
// ---------------------------------------------------------------------------
constexpr size_t kPolyStrSmemBytes = kStrSmemBytes + 16;

template <class A>
__global__ void __launch_bounds__(512, 1)
    poly_str14(const __grid_constant__ CUtensorMap tf, const __grid_constant__ CUtensorMap tg,
               const __grid_constant__ CUtensorMap tout, PolyArgs pa, uint32_t nitems) {
  static_assert(A::kSigned, "poly_str14 runs the signed FP64 policy");
  using Tw = typename A::Tw;
  const NttArgs& a = pa.a;
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* St = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  uint8_t* E = St + kStageBytes;
  const LimbConst* Cs = reinterpret_cast<const LimbConst*>(E + kGrpExBytes);
  uint64_t* bar_full = reinterpret_cast<uint64_t*>(E + kGrpExBytes + 2 * sizeof(LimbConst));
  uint64_t* bar_rd = bar_full + 1;
  uint64_t* bar_w = bar_full + 2;
  uint32_t* cnt = reinterpret_cast<uint32_t*>(bar_full + 4);
  uint64_t* bar_free = bar_full + 5;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar_full + 6);
  const uint32_t t = threadIdx.x, l = t & 31u, w = t >> 5;

  // cslot >= 0: also fetch row k's limb constants into that slot
  auto issue = [&](const CUtensorMap* map, uint32_t k, int cslot) {
    const int32_t y0 = static_cast<int32_t>(static_cast<uint64_t>(k) * (a.n >> 4));
    mbar_expect_tx(bar_full, kStageBytes + (cslot >= 0 ? static_cast<uint32_t>(sizeof(LimbConst)) : 0u));
#pragma unroll
    for (int q = 0; q < 4; ++q) tma_load_2d(St + q * 32768, map, 0, y0 + q * 256, bar_full);
    if (cslot >= 0)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(Cs + cslot)),
                   "l"(a.lc + (a.limb0 + (k % a.nlimbs))), "r"(static_cast<uint32_t>(sizeof(LimbConst))),
                   "r"(smem_u32(bar_full))
                   : "memory");
  };

  if (t == 0) {
    mbar_init(bar_full, 1);
    mbar_init(bar_rd, 16);
    mbar_init(bar_w, 16);
    mbar_init(bar_w + 1, 16);
    mbar_init(bar_free, 16);
    *cnt = 0;
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tf)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tg)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tout)) : "memory");
  }
  if (w == 0) {  // one warp allocates the TMEM columns (one CTA per SM: never contended by this kernel)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "n"(kPolyTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // this warp's TMEM quarter: lanes 32 (w % 4) .. + 31, columns 64 (w / 4) .. + 63: 32 words per thread
  const uint32_t taddr = *tslot + ((32u * (w & 3u)) << 16) + 64u * (w >> 2);
  if (t == 0 && blockIdx.x < nitems) issue(&tg, blockIdx.x, 0);

  uint32_t it = 0;  // rows done by this CTA

  for (uint32_t k = blockIdx.x; k < nitems; k += gridDim.x) {
    uint64_t v[32];
    const uint32_t limb = a.limb0 + (k % a.nlimbs);
    const LimbConst& c = Cs[it & 1u];  // valid once g's bar_full phase completes

    // ---- g^ -> TMEM, then f^ (one copy of the forward's code) ----
#pragma unroll 1
    for (uint32_t ph = 0; ph < 2; ++ph) {
      const Tw* __restrict__ tw = a.tw8 + static_cast<uint64_t>(limb) * a.n;
      const Tw* __restrict__ twq = a.twq8 + static_cast<uint64_t>(limb) * kStrTableWords + tid_opaque();
      mbar_wait(bar_full, ph);
      // (thread constants from an opaque thread index: recomputed per transform instead of
      // staying live across the whole row)
      const uint32_t to = tid_opaque(), wo = to >> 5, lo = to & 31u;
      str::fwd_core<A, true>(
          v, St, E + (wo << 12), c, a, tw, twq, a.n, wo, lo, bar_rd, bar_w, ph, (it + ph) & 1u, 0u,
          [&] {
            if (lo == 0) bulk_wait_read();  // the previous row's output stores have read this warp's 4 KiB
          },
          [&] {
            if (ph == 0) {
              grp::staging_consumed(cnt, l, [&] {
                fence_proxy_async();
                issue(&tf, k, -1);  // f of the same row
              });
            } else {
              __syncwarp();
              if (l == 0) mbar_arrive_local(bar_free);  // the staging halves may take the inverse's streams
            }
          });
      if (ph == 0) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = as_u(csubS(as_d(v[i]), c.twoq_d));
#pragma unroll
        for (int q = 0; q < 4; ++q) tmem_st16(taddr + 16u * q, v + 8 * q);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
    }
    // ---- p = f^ g^ in registers, the inverse's first twiddles ----
    const Tw* __restrict__ itw = pa.itw8 + static_cast<uint64_t>(limb) * a.n;
    const Tw* __restrict__ itwq = pa.itwq8 + static_cast<uint64_t>(limb) * kStrTableWords + tid_opaque();
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint64_t gh[8];
      tmem_ld16(taddr + 16u * q, gh);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        v[8 * q + i] = as_u(mul_recip(csubS(as_d(v[8 * q + i]), c.twoq_d), as_d(gh[i]), c.qinv, c.q_d));
    }
    Tw ta[16];
    str::inv_first_twiddles<A>(ta, itwq);
    // ---- inverse (n^-1 folded into the last stage), canonical words out ----
    const uint32_t to = tid_opaque(), wo = to >> 5, lo = to & 31u;
    str::inv_core<A, false>(
        v, St, E + (wo << 12), c, a, itw, itwq, a.n, wo, lo, ta, bar_w, it & 1u, 0u, [] {},
        [&] { mbar_wait(bar_free, it & 1u); },
        [&] {
          grp::staging_consumed(cnt, l, [&] {
            if (k + gridDim.x < nitems) {
              fence_proxy_async();
              issue(&tg, k + gridDim.x, static_cast<int>((it + 1u) & 1u));  // g of the next row
            }
          });
        });
    // (result words out by bulk tensor stores, as in ntt_stri14)
    const int32_t y0 = static_cast<int32_t>((static_cast<uint64_t>(k) * a.n) >> 9);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
#pragma unroll
      for (int r = 8 * h; r < 8 * h + 8; ++r) A::inv_fold(v[r], v[r + 16], c);
      str::out_half_tma(&tout, E + (wo << 12), wo, lo, y0, v, h);
    }
    ++it;
  }
  if (l == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");

  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tslot), "n"(kPolyTmemCols)
                 : "memory");
  }
}

}  // namespace nk
