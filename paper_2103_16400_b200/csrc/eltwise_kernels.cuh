// Element-wise modular kernels for sm_100a: HBM-bound streaming, 32-byte
// vector loads/stores (four words per access) when aligned, grid-stride.
//
// Outputs are canonical ([0, q)), so any exact algorithm gives the
// reference's words. We follow the reference's integer formulas:
//   eltwise_mult_mod  -> mult_mod_int_loop  eltwise.hpp:74-92 (Barrett, L = 63 + bits)
//                        (the reference's FP64 path, eltwise.hpp:106-125, yields the
//                         same canonical words; eltwise.hpp:177-179)
//   eltwise_fma_mod   -> fma_mod_loop       eltwise.hpp:192-209
//   eltwise_add_mod   ->                    eltwise.hpp:47-57
//   eltwise_neg_mod   ->                    eltwise.hpp:60-70
#pragma once
#include <cstdint>

#include "modmath.cuh"

namespace nk {

struct MultConst {
  uint64_t q, twoq, barrett;
  uint32_t shift;  // bits - 1
  int32_t fin;
};

// x - m if x >= m else x, for x, m < 2^63 (sign test on the high word only)
__device__ __forceinline__ uint64_t csub63(uint64_t x, uint64_t m) {
  const uint64_t d = x - m;
  return (static_cast<int32_t>(hi32(d)) < 0) ? x : d;
}

// mult_mod_int_loop<F> body (eltwise.hpp:82-90). LOOSE (5q < 2^63): the
// Barrett quotient c3 = mulhi(c1, k) takes three of the four 32-bit partial
// products (qhat64_loose, modmath.cuh: floor minus 0..2), so c4 < 5q and one
// more conditional subtraction follows; every intermediate stays below 2^63
// and the sign test on the high word suffices. The canonical product is
// unique, so the words are the reference's.
template <int FIN, bool LOOSE>
__device__ __forceinline__ uint64_t mult_barrett(uint64_t a, uint64_t b, const MultConst& c) {
  const uint64_t x = small_mod(a, c.q, FIN);
  const uint64_t y = small_mod(b, c.q, FIN);
  const uint64_t plo = x * y, phi = __umul64hi(x, y);
  const uint64_t c1 = (plo >> c.shift) | (phi << (64 - c.shift));  // shift in [1, 61]
  const uint64_t c3 = LOOSE ? qhat64_loose(c1, c.barrett) : __umul64hi(c1, c.barrett);
  uint64_t c4 = plo - c3 * c.q;  // true value < 3q (exact) / 5q (loose), wraps exactly
  if (LOOSE) {
    c4 = csub63(c4, c.twoq << 1);
    c4 = csub63(c4, c.twoq);
    c4 = csub63(c4, c.q);
  } else {
    c4 = csub(c4, c.twoq);
    c4 = csub(c4, c.q);
  }
  return c4;
}

// Vector access of VEC consecutive words (VEC = 4: one 256-bit LDG/STG,
// sm_100; 2: 128-bit; 1: scalar), streaming cache hints (each word is touched
// once). The launcher picks VEC from the pointers' alignment.
template <int VEC>
struct WordVec {
  uint64_t w[VEC];
};
template <int VEC>
__device__ __forceinline__ WordVec<VEC> ld_stream(const uint64_t* p) {
  WordVec<VEC> v;
  if constexpr (VEC == 4) {
    asm volatile("ld.global.cs.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(v.w[0]), "=l"(v.w[1]), "=l"(v.w[2]), "=l"(v.w[3])
                 : "l"(p));
  } else if constexpr (VEC == 2) {
    const ulonglong2 t = __ldcs(reinterpret_cast<const ulonglong2*>(p));
    v.w[0] = t.x;
    v.w[1] = t.y;
  } else {
    v.w[0] = __ldcs(p);
  }
  return v;
}
template <int VEC>
__device__ __forceinline__ void st_stream(uint64_t* p, const WordVec<VEC>& v) {
  if constexpr (VEC == 4) {
    asm volatile("st.global.cs.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(v.w[0]), "l"(v.w[1]), "l"(v.w[2]),
                 "l"(v.w[3])
                 : "memory");
  } else if constexpr (VEC == 2) {
    __stcs(reinterpret_cast<ulonglong2*>(p), make_ulonglong2(v.w[0], v.w[1]));
  } else {
    __stcs(p, v.w[0]);
  }
}

// Programmatic dependent launch: the kernels are launched with programmatic
// stream serialisation, so the next kernel's launch overlaps this one's tail;
// each kernel still waits for its predecessor's memory before touching data.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
}

// Rows of `n` = 2^logn words (BATCHED: row r uses consts[r % nlimbs]) or one
// vector under c0. Each thread streams kU chunks of VEC words per iteration
// with all loads issued before any arithmetic; grid-stride beyond a few waves
// of resident CTAs; the last total % VEC words are done by thread 0.
// kU = 1 with ~6 resident CTAs per SM: at 2^20 words a call is ~6 us, and
// more, smaller CTAs start streaming sooner and drain faster than fewer CTAs
// with deeper per-thread batches (tools/elt_probe.cu: 5.6 vs 6.2 us per call).
constexpr int kU = 1;
template <int FIN, bool LOOSE, bool BATCHED, int VEC>
__global__ void __launch_bounds__(256, FIN == 1 ? 6 : 4) eltwise_mult_kernel(uint64_t* __restrict__ r,
                                                           const uint64_t* __restrict__ a,
                                                           const uint64_t* __restrict__ b,
                                                           uint64_t total, uint32_t logn,
                                                           MultConst c0,
                                                           const MultConst* __restrict__ consts,
                                                           uint32_t nlimbs) {
  pdl_enter();
  const uint64_t chunks = total / VEC;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  auto cst = [&](uint64_t word) { return BATCHED ? consts[(word >> logn) % nlimbs] : c0; };
  for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < chunks;
       i0 += kU * stride) {
    WordVec<VEC> x[kU], y[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < chunks) {
        x[u] = ld_stream<VEC>(a + i * VEC);
        y[u] = ld_stream<VEC>(b + i * VEC);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < chunks) {
        WordVec<VEC> o;
        // rows are >= VEC words whenever logn >= log2(VEC): one constant per chunk
        const bool one_row = !BATCHED || (VEC == 1) || ((1u << logn) >= static_cast<uint32_t>(VEC));
        const MultConst c = cst(i * VEC);
#pragma unroll
        for (int k = 0; k < VEC; ++k)
          o.w[k] = mult_barrett<FIN, LOOSE>(x[u].w[k], y[u].w[k], one_row ? c : cst(i * VEC + k));
        st_stream<VEC>(r + i * VEC, o);
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (uint64_t k = chunks * VEC; k < total; ++k) r[k] = mult_barrett<FIN, LOOSE>(a[k], b[k], cst(k));
}

// eltwise_mult_mod_float (eltwise.hpp:158-175, loop 106-125) for q < 2^50 on
// the FP64 pipe: small_mod both inputs, then mulmod_canon (modmath.cuh):
// TwoProduct h + l = x y, quotient round(h / q) through the rounded reciprocal,
// r = (h - k q) + l exact, one correction. The reference takes floor(h u) with
// u = 1/q rounded up and corrects in both directions; the canonical product is
// unique, so the words are the same.
template <int FIN, int VEC>
__global__ void __launch_bounds__(256, 6) eltwise_mult_float_kernel(uint64_t* __restrict__ r,
                                                                    const uint64_t* __restrict__ a,
                                                                    const uint64_t* __restrict__ b,
                                                                    uint64_t total, LimbConstDev c) {
  pdl_enter();
  const uint64_t chunks = total / VEC;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < chunks; i += stride) {
    const WordVec<VEC> x = ld_stream<VEC>(a + i * VEC), y = ld_stream<VEC>(b + i * VEC);
    WordVec<VEC> o;
#pragma unroll
    for (int k = 0; k < VEC; ++k)
      o.w[k] = mulmod_canon(small_mod(x.w[k], c.q, FIN), small_mod(y.w[k], c.q, FIN), c);
    st_stream<VEC>(r + i * VEC, o);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (uint64_t k = chunks * VEC; k < total; ++k)
      r[k] = mulmod_canon(small_mod(a[k], c.q, FIN), small_mod(b[k], c.q, FIN), c);
}

struct FmaConst {
  uint64_t q, y, ybarr;
  int32_t fin, bs;
};

// fma_mod_loop<B, F> body (eltwise.hpp:199-208)
template <int BS, bool HAS_Z, int FIN>
__device__ __forceinline__ uint64_t fma_one(uint64_t a, uint64_t z, const FmaConst& c) {
  // q < 2^61 (eltwise.hpp:243-245): every value below is < 2^63
  const uint64_t x = small_mod(a, c.q, FIN);
  // beta = 2^64 with an addend: the loose quotient (qhat64_loose, floor minus
  // 0..2) leaves v in [0, 4q) < 2^63 for one more conditional subtraction
  // (cfg2 FMA 5.51 -> 5.27 us; the one-stream vector-scalar form measured
  // 4.28 -> 4.36 us with it, so it keeps the exact quotient)
  constexpr bool kLoose = (BS == 64) && HAS_Z;
  const uint64_t qh = (BS == 52) ? qhat52(c.ybarr, x) : (kLoose ? qhat64_loose(c.ybarr, x) : __umul64hi(x, c.ybarr));
  uint64_t v = x * c.y - qh * c.q;  // in [0, 2q) / [0, 4q) (loose)
  if (kLoose) v = csub63(v, 2 * c.q);
  v = csub63(v, c.q);
  if (HAS_Z) {
    v += small_mod(z, c.q, FIN);
    v = csub63(v, c.q);
  }
  return v;
}

// chunks per thread of the FMA kernel: one input stream (vector-scalar
// multiply) keeps two chunks in flight per thread, two streams one
__host__ __device__ constexpr int fma_ku(bool has_z) { return has_z ? 1 : 2; }

template <int BS, bool HAS_Z, int FIN, int VEC>
__global__ void __launch_bounds__(256, HAS_Z ? 6 : 1) eltwise_fma_kernel(uint64_t* __restrict__ r,
                                                          const uint64_t* __restrict__ a,
                                                          const uint64_t* __restrict__ z,
                                                          uint64_t n, FmaConst c) {
  pdl_enter();
  constexpr int KU = fma_ku(HAS_Z);
  const uint64_t chunks = n / VEC;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < chunks;
       i0 += KU * stride) {
    WordVec<VEC> x[KU], zz[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const uint64_t i = i0 + u * stride;
#pragma unroll
      for (int k = 0; k < VEC; ++k) zz[u].w[k] = 0;
      if (i < chunks) {
        x[u] = ld_stream<VEC>(a + i * VEC);
        if (HAS_Z) zz[u] = ld_stream<VEC>(z + i * VEC);
      }
    }
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < chunks) {
        WordVec<VEC> o;
#pragma unroll
        for (int k = 0; k < VEC; ++k) o.w[k] = fma_one<BS, HAS_Z, FIN>(x[u].w[k], zz[u].w[k], c);
        st_stream<VEC>(r + i * VEC, o);
      }
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (uint64_t k = chunks * VEC; k < n; ++k) r[k] = fma_one<BS, HAS_Z, FIN>(a[k], HAS_Z ? z[k] : 0, c);
}

// eltwise_add_mod / eltwise_neg_mod (eltwise.hpp:47-70) for canonical inputs:
// the same streaming shape as the multiply (VEC-word vector accesses, one
// chunk per thread per sweep, the total % VEC tail on thread 0).
__device__ __forceinline__ uint64_t add_one(uint64_t a, uint64_t b, uint64_t q) { return csub(a + b, q); }
__device__ __forceinline__ uint64_t neg_one(uint64_t a, uint64_t q) { return a == 0 ? 0 : q - a; }

template <int VEC>
__global__ void __launch_bounds__(256, 6) eltwise_add_kernel(uint64_t* __restrict__ r,
                                                             const uint64_t* __restrict__ a,
                                                             const uint64_t* __restrict__ b, uint64_t n,
                                                             uint64_t q) {
  pdl_enter();
  const uint64_t chunks = n / VEC;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < chunks; i += stride) {
    const WordVec<VEC> x = ld_stream<VEC>(a + i * VEC), y = ld_stream<VEC>(b + i * VEC);
    WordVec<VEC> o;
#pragma unroll
    for (int k = 0; k < VEC; ++k) o.w[k] = add_one(x.w[k], y.w[k], q);
    st_stream<VEC>(r + i * VEC, o);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (uint64_t k = chunks * VEC; k < n; ++k) r[k] = add_one(a[k], b[k], q);
}

template <int VEC>
__global__ void __launch_bounds__(256, 6) eltwise_neg_kernel(uint64_t* __restrict__ r,
                                                             const uint64_t* __restrict__ a, uint64_t n,
                                                             uint64_t q) {
  pdl_enter();
  const uint64_t chunks = n / VEC;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < chunks; i += stride) {
    const WordVec<VEC> x = ld_stream<VEC>(a + i * VEC);
    WordVec<VEC> o;
#pragma unroll
    for (int k = 0; k < VEC; ++k) o.w[k] = neg_one(x.w[k], q);
    st_stream<VEC>(r + i * VEC, o);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (uint64_t k = chunks * VEC; k < n; ++k) r[k] = neg_one(a[k], q);
}

}  // namespace nk
