// Single-kernel poly_mult_mod for whole rows of N = 2^10 .. 2^13 words
// (ring.hpp:28-43: forward f, forward g, dyadic product, inverse), one CTA per
// row pair, on the register passes of ntt_block (ntt_kernels.cuh):
//
//   g  -> registers -> forward (passes exchanged through the padded shared
//         image) -> g^ reduced below 2q, parked in a second shared area in
//         the last pass's register layout (each thread reads back only the
//         words it wrote: no barrier, [word][thread] order, conflict free)
//   f  -> registers -> forward -> p = f^ g^ in registers -> inverse, whose
//         first pass is the forward's last one (same register layout) ->
//         n^-1, canonical words -> HBM
//
// HBM traffic: 24 B per coefficient (f, g in, the result out) in one launch,
// against 56 B in four launches for the reference's sequence (g^ and f^
// written, read by the product, its result read by the inverse).
//
// Only the canonical result is observable (ring.hpp:43 reduces it to [0, q)),
// and it is unique, so the canonical-only policies apply as in poly_str14
// (ntt_poly.cuh):
//   Arith52S  (q < 2^50): |f^|, |g^| < 4q after the forward; both reduced
//             below 2q (csubS), p = mul_recip(f^, g^), |p| < 1.75q: inside the
//             |x| < 2q the inverse starts from.
//   ArithIntL (2^50 <= q < 2^60): forward words below 16q, each reduced to
//             [0, q) (red16); p by the plan's Barrett constants for canonical
//             factors (mult_barrett<1>, the element-wise kernel's product):
//             canonical, so the inverse's first stage adds without reducing.
// result may alias f or g: a CTA has read both rows before it writes.
#pragma once
#include "eltwise_kernels.cuh"
#include "ntt_kernels.cuh"

namespace nk {

struct PolyBlkArgs {
  uint64_t* out;
  const uint64_t* f;
  const uint64_t* g;
  NttArgs fw;  // forward tables (tw / tw8), lc, n, logn, limb0, nlimbs
  NttArgs iv;  // inverse tables of the same plan
  const MultConst* mc;  // [limb] Barrett constants, fin = 1 (ArithIntL product)
};

template <int LOGB, int LOGV>
constexpr size_t polyblk_smem_bytes() {
  return block_smem_bytes<LOGB, LOGV>() + (size_t{8} << LOGB);
}

// one row into registers in the first pass's layout (ntt_block's load)
template <int LOGB, int LOGV, class A, bool FWD>
__device__ __forceinline__ void polyblk_load(uint64_t (&v)[1 << LOGV], const uint64_t* __restrict__ src, uint32_t t) {
  using S = Sched<LOGB, LOGV>;
  using PO = PassOf<LOGB, LOGV, FWD>;
  constexpr int LO = PO::lo(0), K = PO::k(0);
  constexpr int R = 1 << K, G = S::V / R;
  const uint32_t jt = S::scatter(t, LO, K);
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const uint32_t jg = S::jg(g, LO, K);
#pragma unroll
    for (int r = 0; r < R; ++r) v[g * R + r] = A::load(__ldcs(src + jt + jg + (r << LO)));
  }
}

// Launch bounds: no occupancy target for N <= 4096 (ptxas then uses 48-88 registers; with an
// explicit target it spends whatever the target allows, 110-128, and fewer CTAs fit). At N =
// 8192 shared memory leaves one CTA per SM anyway, and the explicit target of one CTA
// lets the schedule keep more loads in flight (50-bit limbs: 618 us against 766).
template <int LOGB, int LOGV, class A>
__global__ void __launch_bounds__(1 << (LOGB - LOGV), LOGB == 13 ? 1 : 0) poly_block(PolyBlkArgs a) {
  using S = Sched<LOGB, LOGV>;
  using PI = PassOf<LOGB, LOGV, false>;
  extern __shared__ uint64_t sm[];
  uint64_t* const park = sm + block_smem_bytes<LOGB, LOGV>() / sizeof(uint64_t) + threadIdx.x;
  const uint32_t t = threadIdx.x;
  const uint64_t row = static_cast<uint64_t>(blockIdx.x) * a.fw.row_mul + a.fw.row_add;
  const uint32_t limb = a.fw.limb0 + static_cast<uint32_t>(row % a.fw.nlimbs);
  const LimbConst c = a.fw.lc[limb];
  const typename A::Tw* __restrict__ twf = tw_of<A>(a.fw, limb);
  const typename A::Tw* __restrict__ twi = tw_of<A>(a.iv, limb);
  const uint64_t off = row << LOGB;

  uint64_t v[S::V];
  // ---- g^, then f^: one copy of the forward, run twice ----
#pragma unroll 1
  for (int it = 0; it < 2; ++it) {
    // the thread index and the table pointer are redefined per iteration: the loop-invariant
    // twiddle indices (and the non-coherent twiddle loads) would otherwise be hoisted out of
    // the loop and held in registers (spills)
    uint32_t t_it = t;
    const typename A::Tw* tw_it = twf;
    asm volatile("" : "+r"(t_it), "+l"(tw_it));
    polyblk_load<LOGB, LOGV, A, true>(v, (it ? a.f : a.g) + off, t_it);
    // the exchange image is free again: run_passes' barrier before its first write
    run_passes<LOGB, LOGV, A, true, 0, true>(v, sm, tw_it, t_it, a.fw.n, c);
    if (it == 0) {
#pragma unroll
      for (int i = 0; i < S::V; ++i) {
        if constexpr (A::kSigned) park[i * S::T] = as_u(csubS(as_d(v[i]), c.twoq_d));
        else park[i * S::T] = A::red16(v[i], c);
      }
    }
  }
  // ---- dyadic product in the last pass's register layout ----
  if constexpr (A::kSigned) {
#pragma unroll
    for (int i = 0; i < S::V; ++i)
      v[i] = as_u(mul_recip(csubS(as_d(v[i]), c.twoq_d), as_d(park[i * S::T]), c.qinv, c.q_d));
  } else {
    const MultConst mc = a.mc[limb];
#pragma unroll
    for (int i = 0; i < S::V; ++i) v[i] = mult_barrett<1, true>(A::red16(v[i], c), park[i * S::T], mc);
  }
  // ---- inverse; canonical factors' product is canonical for the integer policy ----
  // (n^-1 folded into its last stage: canonical words out, A::inv_fold)
  run_passes<LOGB, LOGV, A, false, 0, !A::kSigned>(v, sm, twi, t, a.fw.n, c, true);
  constexpr int PL = S::NP - 1;
  constexpr int LO = PI::lo(PL), K = PI::k(PL);
  constexpr int R = 1 << K, G = S::V / R;
  const uint32_t jt = S::scatter(t, LO, K);
  uint64_t* __restrict__ dst = a.out + off;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const uint32_t jg = S::jg(g, LO, K);
#pragma unroll
    for (int r = 0; r < R; ++r) dst[jt + jg + (r << LO)] = v[g * R + r];
  }
}

}  // namespace nk
