// Device-side modular arithmetic for the sm_100a hot path.
//
// Everything here reproduces, bit for bit, the scalar primitives of the
// reference (nttkit, /root/reference/proj/include/nttkit/):
//   mul_factor_lazy<B>   ntt.hpp:97-101      (Shoup/Harvey product, result in [0,2q))
//   fwd_butterfly<B,I>   ntt.hpp:103-113     (CT, [0,4q) in/out)
//   inv_butterfly<B,I>   ntt.hpp:115-130     (GS, [0,2q) in/out)
//   small_mod            modarith.hpp:217-225
// but is written for the B200 integer pipes: 64-bit words are handled as
// 32-bit halves so every partial product is one IMAD / IMAD.WIDE / IMAD.HI.
//
// beta = 2^52 (tables for 4q < 2^52, i.e. every 50-bit limb):
//   qhat = floor(W' * x / 2^52) with W', x < 2^52 is computed exactly as
//     s    = hi32(a0*b0) + a0*b1 + a1*b0            (< 2^54, no overflow)
//     qhat = ((a1 << 12) * b1) + (s >> 20)
//   where W' = a1:a0 and x = b1:b0 (a1, b1 < 2^20). The low 32 bits of a0*b0
//   cannot carry across the 2^52 boundary, so this is the exact floor.
//   The reference then forms (w*x + qhat*(2^52 - q)) mod 2^52; since the true
//   value w*x - qhat*q lies in [0, 2q) (Harvey's bound for x < beta) the same
//   number is obtained modulo 2^64 with -q in two's complement, i.e. the 52-bit
//   mask at ntt.hpp:121-123 / modarith.hpp:161 never changes a value.
// beta = 2^64 (60-bit limbs): qhat = mulhi64(W', x) exactly, same low-word form.
#pragma once
#include <cstdint>

namespace nk {

struct u64x2 {
  uint64_t x, y;
};

__device__ __forceinline__ uint32_t lo32(uint64_t v) { return static_cast<uint32_t>(v); }
__device__ __forceinline__ uint32_t hi32(uint64_t v) { return static_cast<uint32_t>(v >> 32); }

// Wide multiply-add a*b + c (32x32 -> 64 plus a 64-bit addend): one IMAD.WIDE.U32.
__device__ __forceinline__ uint64_t mad_wide(uint32_t a, uint32_t b, uint64_t c) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(c));
  return r;
}

// floor(wp * x / 2^52) for wp, x < 2^52 (the reference's mul_hi<52>, modarith.hpp:133-139).
__device__ __forceinline__ uint64_t qhat52(uint64_t wp, uint64_t x) {
  const uint32_t a0 = lo32(wp), a1 = hi32(wp);
  const uint32_t b0 = lo32(x), b1 = hi32(x);
  uint64_t s = __umulhi(a0, b0);
  s = mad_wide(a0, b1, s);
  s = mad_wide(a1, b0, s);
  return mad_wide(a1 << 12, b1, s >> 20);
}

// floor(wp * x / 2^64) (the reference's mul_hi<64>).
__device__ __forceinline__ uint64_t qhat64(uint64_t wp, uint64_t x) { return __umul64hi(wp, x); }

// (w*x + qhat*negq) mod 2^64, computed from 32-bit partial products.
__device__ __forceinline__ uint64_t lo_sum(uint64_t w, uint64_t x, uint64_t qhat, uint64_t negq) {
  return w * x + qhat * negq;
}

// mul_factor_lazy<B>(x, w, w', -q): w*x - floor(w'x/beta)*q in [0, 2q) for x < beta.
template <int BS>
__device__ __forceinline__ uint64_t mul_lazy(uint64_t x, uint64_t w, uint64_t wp, uint64_t negq) {
  const uint64_t qh = (BS == 52) ? qhat52(wp, x) : qhat64(wp, x);
  return lo_sum(w, x, qh, negq);
}

// min(x, x - m): the reference's branch-free conditional subtraction
// (modarith.hpp:221-223, ntt.hpp:108,126).
__device__ __forceinline__ uint64_t csub(uint64_t x, uint64_t m) {
  const uint64_t d = x - m;
  return d < x ? d : x;  // d wraps above x exactly when x < m
}

__device__ __forceinline__ uint64_t small_mod(uint64_t x, uint64_t q, int factor) {
  if (factor == 8) x = csub(x, 4 * q);
  if (factor >= 4) x = csub(x, 2 * q);
  if (factor >= 2) x = csub(x, q);
  return x;
}

// fwd_butterfly<B, ILTM> (ntt.hpp:103-113). ILTM skips the [0,4q)->[0,2q)
// pre-reduction, a value no-op for inputs below q.
template <int BS, bool ILTM>
__device__ __forceinline__ void fwd_bfly(uint64_t& x0, uint64_t& x1, uint64_t w, uint64_t wp,
                                         uint64_t twoq, uint64_t negq) {
  uint64_t u = x0;
  if (!ILTM) u = csub(u, twoq);
  const uint64_t t = mul_lazy<BS>(x1, w, wp, negq);
  x0 = u + t;
  x1 = u + twoq - t;
}

// inv_butterfly<B, ILTM> (ntt.hpp:115-130). t = x0 - x1 + 2q lies in (0, 4q),
// so the 52-bit mask of ntt.hpp:121-123 is a value no-op and is omitted.
template <int BS, bool ILTM>
__device__ __forceinline__ void inv_bfly(uint64_t& x0, uint64_t& x1, uint64_t w, uint64_t wp,
                                         uint64_t twoq, uint64_t negq) {
  const uint64_t t = x0 + twoq - x1;
  uint64_t s = x0 + x1;
  if (!ILTM) s = csub(s, twoq);
  x0 = s;
  x1 = mul_lazy<BS>(t, w, wp, negq);
}

}  // namespace nk
