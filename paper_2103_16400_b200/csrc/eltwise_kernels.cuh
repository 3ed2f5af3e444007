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

// mult_mod_int_loop<F> body (eltwise.hpp:82-90)
__device__ __forceinline__ uint64_t mult_barrett(uint64_t a, uint64_t b, const MultConst& c) {
  const uint64_t x = small_mod(a, c.q, c.fin);
  const uint64_t y = small_mod(b, c.q, c.fin);
  const uint64_t plo = x * y, phi = __umul64hi(x, y);
  const uint64_t c1 = (plo >> c.shift) | (phi << (64 - c.shift));  // shift in [1, 61]
  const uint64_t c3 = __umul64hi(c1, c.barrett);
  uint64_t c4 = plo - c3 * c.q;
  c4 = csub(c4, c.twoq);
  c4 = csub(c4, c.q);
  return c4;
}

// Rows of `n` words; row r uses consts[r % nlimbs], or c0 for every row when consts is NULL.
__global__ void __launch_bounds__(256) eltwise_mult_kernel(uint64_t* __restrict__ r,
                                                           const uint64_t* __restrict__ a,
                                                           const uint64_t* __restrict__ b,
                                                           uint64_t n, uint64_t rows,
                                                           MultConst c0,
                                                           const MultConst* __restrict__ consts,
                                                           uint32_t nlimbs) {
  const uint64_t total2 = (n * rows) >> 1;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const bool one = (consts == nullptr);
  MultConst c = one ? c0 : consts[0];
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total2;
       i += stride) {
    if (!one) c = consts[((2 * i) / n) % nlimbs];  // n even: both words in one row
    const ulonglong2 x = reinterpret_cast<const ulonglong2*>(a)[i];
    const ulonglong2 y = reinterpret_cast<const ulonglong2*>(b)[i];
    ulonglong2 o;
    o.x = mult_barrett(x.x, y.x, c);
    o.y = mult_barrett(x.y, y.y, c);
    reinterpret_cast<ulonglong2*>(r)[i] = o;
  }
  // odd tail (single modulus only; batched rows have even n)
  if (((n * rows) & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const uint64_t k = n * rows - 1;
    r[k] = mult_barrett(a[k], b[k], c0);
  }
}

struct FmaConst {
  uint64_t q, y, ybarr;
  int32_t fin, bs;
};

// fma_mod_loop<B, F> body (eltwise.hpp:199-208)
template <int BS, bool HAS_Z>
__device__ __forceinline__ uint64_t fma_one(uint64_t a, uint64_t z, const FmaConst& c) {
  const uint64_t x = small_mod(a, c.q, c.fin);
  const uint64_t qh = (BS == 52) ? qhat52(c.ybarr, x) : __umul64hi(x, c.ybarr);
  uint64_t v = x * c.y - qh * c.q;  // in [0, 2q)
  v = csub(v, c.q);
  if (HAS_Z) {
    v += small_mod(z, c.q, c.fin);
    v = csub(v, c.q);
  }
  return v;
}

template <int BS, bool HAS_Z>
__global__ void __launch_bounds__(256) eltwise_fma_kernel(uint64_t* __restrict__ r,
                                                          const uint64_t* __restrict__ a,
                                                          const uint64_t* __restrict__ z,
                                                          uint64_t n, FmaConst c) {
  const uint64_t n2 = n >> 1;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n2;
       i += stride) {
    const ulonglong2 x = reinterpret_cast<const ulonglong2*>(a)[i];
    ulonglong2 zz = make_ulonglong2(0, 0);
    if (HAS_Z) zz = reinterpret_cast<const ulonglong2*>(z)[i];
    ulonglong2 o;
    o.x = fma_one<BS, HAS_Z>(x.x, zz.x, c);
    o.y = fma_one<BS, HAS_Z>(x.y, zz.y, c);
    reinterpret_cast<ulonglong2*>(r)[i] = o;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const uint64_t k = n - 1;
    r[k] = fma_one<BS, HAS_Z>(a[k], HAS_Z ? z[k] : 0, c);
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
