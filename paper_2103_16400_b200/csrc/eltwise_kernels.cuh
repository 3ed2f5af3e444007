// Element-wise modular kernels for sm_100a: HBM-bound streaming, 16-byte
// vector loads/stores (two words per access), grid-stride over the vector.
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

// mult_mod_int_loop<F> body (eltwise.hpp:82-90). SMALLQ: q < 2^61, so every
// intermediate of the tail is below 2^63 and the cheaper sign test applies.
template <int FIN, bool SMALLQ>
__device__ __forceinline__ uint64_t mult_barrett(uint64_t a, uint64_t b, const MultConst& c) {
  const uint64_t x = small_mod(a, c.q, FIN);
  const uint64_t y = small_mod(b, c.q, FIN);
  const uint64_t plo = x * y, phi = __umul64hi(x, y);
  const uint64_t c1 = (plo >> c.shift) | (phi << (64 - c.shift));  // shift in [1, 61]
  const uint64_t c3 = __umul64hi(c1, c.barrett);
  uint64_t c4 = plo - c3 * c.q;  // true value < 3q, wraps exactly
  if (SMALLQ) {
    c4 = csub63(c4, c.twoq);
    c4 = csub63(c4, c.q);
  } else {
    c4 = csub(c4, c.twoq);
    c4 = csub(c4, c.q);
  }
  return c4;
}

// Rows of `n` = 2^logn words (BATCHED: row r uses consts[r % nlimbs]) or one
// vector under c0. Each thread streams kU 16-byte chunks per iteration with all
// loads issued before any arithmetic (memory-level parallelism for an
// HBM-bound loop); grid-stride over a few waves of resident CTAs.
constexpr int kU = 4;
template <int FIN, bool SMALLQ, bool BATCHED>
__global__ void __launch_bounds__(256) eltwise_mult_kernel(uint64_t* __restrict__ r,
                                                           const uint64_t* __restrict__ a,
                                                           const uint64_t* __restrict__ b,
                                                           uint64_t total, uint32_t logn,
                                                           MultConst c0,
                                                           const MultConst* __restrict__ consts,
                                                           uint32_t nlimbs) {
  const uint64_t total2 = total >> 1;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const ulonglong2* __restrict__ a2 = reinterpret_cast<const ulonglong2*>(a);
  const ulonglong2* __restrict__ b2 = reinterpret_cast<const ulonglong2*>(b);
  ulonglong2* __restrict__ r2 = reinterpret_cast<ulonglong2*>(r);
  for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < total2;
       i0 += kU * stride) {
    ulonglong2 x[kU], y[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < total2) {
        x[u] = __ldcs(a2 + i);  // streamed once: evict-first
        y[u] = __ldcs(b2 + i);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < total2) {
        MultConst c = c0;
        if (BATCHED) c = consts[((2 * i) >> logn) % nlimbs];  // n even: both words in one row
        ulonglong2 o;
        o.x = mult_barrett<FIN, SMALLQ>(x[u].x, y[u].x, c);
        o.y = mult_barrett<FIN, SMALLQ>(x[u].y, y[u].y, c);
        __stcs(r2 + i, o);
      }
    }
  }
  if (!BATCHED && (total & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const uint64_t k = total - 1;
    r[k] = mult_barrett<FIN, SMALLQ>(a[k], b[k], c0);
  }
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
  const uint64_t qh = (BS == 52) ? qhat52(c.ybarr, x) : __umul64hi(x, c.ybarr);
  uint64_t v = x * c.y - qh * c.q;  // in [0, 2q)
  v = csub63(v, c.q);
  if (HAS_Z) {
    v += small_mod(z, c.q, FIN);
    v = csub63(v, c.q);
  }
  return v;
}

template <int BS, bool HAS_Z, int FIN>
__global__ void __launch_bounds__(256) eltwise_fma_kernel(uint64_t* __restrict__ r,
                                                          const uint64_t* __restrict__ a,
                                                          const uint64_t* __restrict__ z,
                                                          uint64_t n, FmaConst c) {
  const uint64_t n2 = n >> 1;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const ulonglong2* __restrict__ a2 = reinterpret_cast<const ulonglong2*>(a);
  const ulonglong2* __restrict__ z2 = reinterpret_cast<const ulonglong2*>(z);
  ulonglong2* __restrict__ r2 = reinterpret_cast<ulonglong2*>(r);
  for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < n2;
       i0 += kU * stride) {
    ulonglong2 x[kU], zz[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t i = i0 + u * stride;
      zz[u] = make_ulonglong2(0, 0);
      if (i < n2) {
        x[u] = __ldcs(a2 + i);
        if (HAS_Z) zz[u] = __ldcs(z2 + i);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < n2) {
        ulonglong2 o;
        o.x = fma_one<BS, HAS_Z, FIN>(x[u].x, zz[u].x, c);
        o.y = fma_one<BS, HAS_Z, FIN>(x[u].y, zz[u].y, c);
        __stcs(r2 + i, o);
      }
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const uint64_t k = n - 1;
    r[k] = fma_one<BS, HAS_Z, FIN>(a[k], HAS_Z ? z[k] : 0, c);
  }
}

__global__ void __launch_bounds__(256) eltwise_add_kernel(uint64_t* __restrict__ r,
                                                          const uint64_t* __restrict__ a,
                                                          const uint64_t* __restrict__ b,
                                                          uint64_t n, uint64_t q) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride)
    r[i] = csub(a[i] + b[i], q);
}

__global__ void __launch_bounds__(256) eltwise_neg_kernel(uint64_t* __restrict__ r,
                                                          const uint64_t* __restrict__ a,
                                                          uint64_t n, uint64_t q) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const uint64_t x = a[i];
    r[i] = x == 0 ? 0 : q - x;
  }
}

}  // namespace nk
