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

// ---------------------------------------------------------------------------
// beta = 2^52 on the FP64 pipe.
//
// Measured on B200 (tools/pipe_bench.cu): IMAD 62/clk/SM, IMAD.WIDE 23 and
// IMAD.HI 32/clk/SM, DFMA/DMUL/DADD 60/clk/SM, IADD3/LOP3 ~122/clk/SM.
// The integer Shoup product above costs ~16 fma-pipe slots (6 wide products);
// for beta = 2^52 (every operand < 2^52) the same words come out of 6 exact
// FP64 operations on plain doubles v = x < 2^52:
//   hq = fma_rd(W', v, 2^104)             = 2^104 + floor(W'x/2^52)*2^52
//        (the sum lies in [2^104, 2^105) where the ulp is 2^52, so rounding
//         down IS the reference's mul_hi<52>, modarith.hpp:133-139)
//   qh = hq - 2^104                       (exact: qhat * 2^52)
//   h1 = w*v (rn), l1 = fma(w, v, -h1)    (exact TwoProduct: h1 + l1 = w x)
//   e  = fma(-qh, q*2^-52, h1)            (exact: |h1 - qhat q| < 2^53, integer)
//   T  = e + l1                           (exact: w x - qhat q in [0, 2q))
// T is the reference's mul_factor_lazy<52> result (ntt.hpp:97-101): same
// qhat, same representative.
// ---------------------------------------------------------------------------
constexpr uint64_t kDBias = 0x4330000000000000ull;  // bits of 2^52
constexpr uint64_t kMask52 = (uint64_t{1} << 52) - 1;
constexpr double kC52 = 4503599627370496.0;                   // 2^52
constexpr double kC104 = 20282409603651670423947251286016.0;  // 2^104

__device__ __forceinline__ double as_d(uint64_t b) { return __longlong_as_double(static_cast<long long>(b)); }
__device__ __forceinline__ uint64_t as_u(double d) { return static_cast<uint64_t>(__double_as_longlong(d)); }

// w*v - floor(w'v/2^52)*q as a plain double (exact integer in [0, 2q)) for a
// plain double v < 2^52.
__device__ __forceinline__ double mul_lazy_plain(double v, double w, double wp, double qq) {
  const double hq = __fma_rd(wp, v, kC104);
  const double qh = __dsub_rn(hq, kC104);
  const double h1 = __dmul_rn(w, v);
  const double l1 = __fma_rn(w, v, -h1);
  const double e = __fma_rn(-qh, qq, h1);
  return __dadd_rn(e, l1);
}

// ---------------------------------------------------------------------------
// Arithmetic policies for the transform kernels. Values live in registers and
// shared memory in the policy's representation; load()/store() convert at the
// HBM boundary. Twiddle-table entries are 16 bytes {w, w'} in the policy's
// format (uint64 for the integer policies, the doubles' bit patterns for the
// FP64 ones).
// ---------------------------------------------------------------------------
struct LimbConstDev {
  uint64_t q, twoq, negq, ninv, ninvp;  // integer policies: integers; FP64 policies: ninv/ninvp are double bits
  double qq;                            // q * 2^-52
  double twoq_d;                        // 2q as a double
  int32_t bs;
  int32_t pad;
  double q_d;     // q as a double
  double qinv;    // 1/q rounded (Arith52S canonicalisation)
  double q_bias;  // q + 2^52
  // n^-1 * w_1 mod q and its Shoup quotient (policy encoding like ninv): the
  // last inverse stage's single twiddle (table index 1) times n^-1, for the
  // folded last stage of canonical inverses (inv_fold)
  uint64_t nw, nwp;
  uint64_t fourq;  // 4q (ArithIntL)
  // Arith52S: n^-1 and n^-1 * w_1 as balanced doubles in (-q/2, q/2] (the folded last stage's
  // integer-grid products, inv_fold); 128 bytes: one bulk copy into shared memory (ntt_grp14)
  double ninv_b, nw_b;
};
static_assert(sizeof(LimbConstDev) == 128, "LimbConstDev is copied as one 128-byte bulk transfer");

template <int BS>
struct ArithInt {  // integer Shoup products, beta = 2^BS (52 or 64)
  using Tw = ulonglong2;  // twiddle-table entry {w, w'}
  static constexpr int kIltmFwd = 1;  // forward stages whose pre-reduction is skipped at fin = 1
  static constexpr bool kLoose = false;
  static constexpr bool kFP = false;
  __device__ static uint64_t load(uint64_t x) { return x; }
  __device__ static uint64_t store(uint64_t x) { return x; }
  template <bool ILTM>
  __device__ static void fwd(uint64_t& x0, uint64_t& x1, ulonglong2 w, const LimbConstDev& c) {
    fwd_bfly<BS, ILTM>(x0, x1, w.x, w.y, c.twoq, c.negq);
  }
  template <bool ILTM>
  __device__ static void inv(uint64_t& x0, uint64_t& x1, ulonglong2 w, const LimbConstDev& c) {
    inv_bfly<BS, ILTM>(x0, x1, w.x, w.y, c.twoq, c.negq);
  }
  __device__ static uint64_t scale_ninv(uint64_t x, const LimbConstDev& c) {
    return mul_lazy<BS>(x, c.ninv, c.ninvp, c.negq);
  }
  __device__ static uint64_t csub(uint64_t x, uint64_t m) { return nk::csub(x, m); }
  static constexpr bool kSigned = false;
  __device__ static uint64_t red4(uint64_t x, const LimbConstDev& c) { return nk::csub(nk::csub(x, c.twoq), c.q); }
  __device__ static uint64_t red2(uint64_t x, const LimbConstDev& c) { return nk::csub(x, c.q); }
  // last GS stage (twiddle w_1) with the n^-1 pass folded in, canonical words
  // out: x0 = n^-1 (x0 + x1), x1 = (n^-1 w_1)(x0 - x1), inputs in [0, 2q).
  // Only for fout == 1, where the result is unique (not the reference's
  // operation sequence: two Shoup products per butterfly instead of three).
  static constexpr bool kFold = true;
  __device__ static void inv_fold(uint64_t& x0, uint64_t& x1, const LimbConstDev& c) {
    const uint64_t s = x0 + x1, t = x0 + c.twoq - x1;  // [0, 4q), (0, 4q): below beta
    x0 = nk::csub(mul_lazy<BS>(s, c.ninv, c.ninvp, c.negq), c.q);
    x1 = nk::csub(mul_lazy<BS>(t, c.nw, c.nwp, c.negq), c.q);
  }
};

// ---------------------------------------------------------------------------
// beta = 2^52 on the FP64 pipe, values as plain doubles ("P representation").
//
// The reference's butterflies and representatives (so lazy outputs stay
// bit-exact), with a word carried as the double whose value it is: the Shoup
// product needs no unbiasing and the conditional subtraction is one DADD plus
// a sign test, no 64-bit integer add (which ptxas issues as IADD3 + IMAD.X,
// and IMAD shares issue bandwidth with the FP64 pipe).
// Registers hold the double's bit pattern (uint64_t) so the kernels stay
// policy-agnostic.
// ---------------------------------------------------------------------------
// y >= m ? y - m : y on plain doubles (y, m exact integers below 2^53)
__device__ __forceinline__ double csubP(double y, double m) {
  const double d = __dsub_rn(y, m);
  return (static_cast<int32_t>(hi32(as_u(d))) >= 0) ? d : y;
}

struct Arith52P {
  using Tw = ulonglong2;  // {w, w'} as doubles' bit patterns
  static constexpr int kIltmFwd = 1;  // forward stages whose pre-reduction is skipped at fin = 1
  static constexpr bool kLoose = false;
  static constexpr bool kFP = true;
  __device__ static uint64_t load(uint64_t x) { return as_u(__dsub_rn(as_d(x | kDBias), kC52)); }
  __device__ static uint64_t store(uint64_t x) { return as_u(__dadd_rn(as_d(x), kC52)) & kMask52; }
  template <bool ILTM>
  __device__ static void fwd(uint64_t& x0, uint64_t& x1, ulonglong2 w, const LimbConstDev& c) {
    const double u = ILTM ? as_d(x0) : csubP(as_d(x0), c.twoq_d);
    const double t = mul_lazy_plain(as_d(x1), as_d(w.x), as_d(w.y), c.qq);
    x0 = as_u(__dadd_rn(u, t));
    x1 = as_u(__dsub_rn(__dadd_rn(u, c.twoq_d), t));
  }
  template <bool ILTM>
  __device__ static void inv(uint64_t& x0, uint64_t& x1, ulonglong2 w, const LimbConstDev& c) {
    const double a = as_d(x0), b = as_d(x1);
    const double t = __dadd_rn(__dsub_rn(a, b), c.twoq_d);
    double s = __dadd_rn(a, b);
    if (!ILTM) s = csubP(s, c.twoq_d);
    x0 = as_u(s);
    x1 = as_u(mul_lazy_plain(t, as_d(w.x), as_d(w.y), c.qq));
  }
  __device__ static uint64_t scale_ninv(uint64_t x, const LimbConstDev& c) {
    return as_u(mul_lazy_plain(as_d(x), as_d(c.ninv), as_d(c.ninvp), c.qq));
  }
  static constexpr bool kSigned = false;
  __device__ static uint64_t red4(uint64_t x, const LimbConstDev& c) {
    return as_u(csubP(csubP(as_d(x), c.twoq_d), c.q_d));
  }
  __device__ static uint64_t red2(uint64_t x, const LimbConstDev& c) { return as_u(csubP(as_d(x), c.q_d)); }
  // see ArithInt::inv_fold; plain doubles in [0, 2q) in, stored words out
  static constexpr bool kFold = true;
  __device__ static void inv_fold(uint64_t& x0, uint64_t& x1, const LimbConstDev& c) {
    const double a = as_d(x0), b = as_d(x1);
    const double s = __dadd_rn(a, b), t = __dadd_rn(__dsub_rn(a, b), c.twoq_d);  // exact, < 4q
    x0 = store(as_u(csubP(mul_lazy_plain(s, as_d(c.ninv), as_d(c.ninvp), c.qq), c.q_d)));
    x1 = store(as_u(csubP(mul_lazy_plain(t, as_d(c.nw), as_d(c.nwp), c.qq), c.q_d)));
  }
};

// ---------------------------------------------------------------------------
// beta = 2^52 on the FP64 pipe, SIGNED values (canonical-output transforms
// only: fout == 1). Requires q < 2^50 (so 4q <= 2^52).
//
// Signed product from w alone (8-byte twiddles; the quotient comes from the
// rounded reciprocal qinv = fl(1/q) instead of a Shoup table):
//   h1 = fl(w v), l1 = fma(w, v, -h1)            exact TwoProduct: h1 + l1 = w v
//   k  = fma(h1, qinv, C) - C                    h1 qinv rounded to the grid of C
//   e  = fma(-k, q, h1)                          exact: integer, |e| < 2^53
//   T  = e + l1 = w v - k q                      exact
// Two grids:
//  * mul_recip, C = 1.5*2^53 (even integers), for |w v| < 4 q^2 (|h1 qinv| <
//    2^52 keeps the sum in [2^53, 2^54)): |h1 - wv| <= 2^48, |h1 qinv - h1/q|
//    < 1/2, |h1 qinv - k| <= 1, so |T| < 1.75q. Used where both factors are
//    only known below 2q (the dyadic product of two transform outputs).
//  * mul_recip_fine, C = 1.5*2^52 (integers), for |w v| < 2 q^2 (|h1 qinv| <
//    2^51 keeps the sum in [2^52, 2^53)): |l1| <= 2^-53 |wv| < q (q / 2^52) <
//    q/4, |h1 qinv - h1/q| <= 2q 2^-53 (1 + 2^-52) < 1/4, |h1 qinv - k| <= 1/2,
//    so |T| < q. THE TRANSFORMS' TWIDDLES ARE STORED BALANCED, w in (-q/2, q/2]
//    (w - q for w > q/2: the same residue, capi.cu balanced8), so every
//    butterfly product with |v| < 4q is in this case.
// Signed words drop Harvey's "+2q" (x1' = u - T) and the GS "+2q" (t = x0 - x1):
//   forward: |x| < 4q in; a reducing stage takes u = x0 - 2q sgn(x0) [|x0| >=
//            2q] in (-2q, 2q), x0' = u + T, x1' = u - T in (-3q, 3q); because
//            |T| < q, the NEXT stage may skip the reduction (u = x0): its
//            outputs stay below 4q, the bound a reducing stage starts from. The
//            16384-word kernels reduce on even stages only (fwd_skip below):
//            6 conditional subtractions (one DADD + four ALU operations each)
//            in 14 stages instead of 12. At fin = 1 the first stage skips it
//            too (|x| < q in, < 2q out, < 3q after stage 1).
//   inverse: |x| < 2q in, s = x0 + x1 in (-4q, 4q) -> (-2q, 2q) by the same
//            signed conditional subtraction, x1' = T(x0 - x1) in (-q, q): the
//            sum doubles at every stage, so every stage reduces.
// Representatives differ from the reference's lazy ones; canonical results
// (every value reduced to [0, q) at the end) are identical.
// The n^-1 products of the folded last inverse stage keep the Shoup form
// (mul_signed, constants in LimbConstDev: W' v / 2^52 rounded to an even
// integer via 3*2^104, |T| < 2q for |v| < 4q).
// ---------------------------------------------------------------------------
constexpr double kC104x3 = 60847228810955011271841753858048.0;  // 3 * 2^104

__device__ __forceinline__ double mul_signed(double v, double w, double wp, double qq) {
  const double hq = __fma_rn(wp, v, kC104x3);
  const double qh = __dsub_rn(hq, kC104x3);
  const double h1 = __dmul_rn(w, v);
  const double l1 = __fma_rn(w, v, -h1);
  const double e = __fma_rn(-qh, qq, h1);
  return __dadd_rn(e, l1);
}
constexpr double kC53x15 = 13510798882111488.0;  // 1.5 * 2^53: round-to-even-integer constant
constexpr double kC52x15 = 6755399441055744.0;   // 1.5 * 2^52: round-to-integer constant
__device__ __forceinline__ double mul_recip(double v, double w, double qinv, double q) {
  const double h1 = __dmul_rn(w, v);
  const double l1 = __fma_rn(w, v, -h1);
  const double k = __dsub_rn(__fma_rn(h1, qinv, kC53x15), kC53x15);
  const double e = __fma_rn(-k, q, h1);
  return __dadd_rn(e, l1);
}
// The same product with the integer-grid constant 1.5*2^52 for |v| < 2q:
// |h1 qinv| < 2q < 2^51 keeps the sum in [2^52, 2^53) (ulp 1), so k is the
// nearest integer to h1 qinv and |wv/q - k| <= 1/2 + 2^47/q + 2q 2^-53 < 7/8:
// |T| < 0.875q (used where a canonical result follows: one fix-up instead of
// a full canonicalisation).
__device__ __forceinline__ double mul_recip_fine(double v, double w, double qinv, double q) {
  const double h1 = __dmul_rn(w, v);
  const double l1 = __fma_rn(w, v, -h1);
  const double k = __dsub_rn(__fma_rn(h1, qinv, kC52x15), kC52x15);
  const double e = __fma_rn(-k, q, h1);
  return __dadd_rn(e, l1);
}
// |y| >= m ? y - m sgn(y) : y  (one DADD on |y|, sign copied on the integer pipe)
__device__ __forceinline__ double csubS(double y, double m) {
  const double d = __dsub_rn(fabs(y), m);
  const uint64_t yb = as_u(y), db = as_u(d);
  const uint64_t r = db | (yb & 0x8000000000000000ull);
  return (static_cast<int32_t>(hi32(db)) >= 0) ? as_d(r) : y;
}

struct Arith52S {
  using Tw = uint64_t;  // w as a double's bit pattern (8-byte tables)
  // Forward stages without the conditional subtraction when the input is
  // canonical (fin = 1), for the kernels that reduce at every later stage:
  // |x| < q in, < 2q after stage 1, < 3q after stage 2 (|T| < q), inside the
  // |x| < 4q a reducing stage starts from.
  static constexpr int kIltmFwd = 2;
  // The 16384-word kernels' schedule: stage gs (0 = the block's first stage,
  // index bit 13) skips the reduction when gs is odd -- the stage before it
  // reduced, so |x| < 3q in and < 4q out -- and at gs = 0 when the input is
  // canonical (< q in, < 2q out; stage 1: < 3q out; stage 2 reduces).
  __host__ __device__ static constexpr bool fwd_skip(bool iltm0, int gs) { return (gs & 1) || (iltm0 && gs == 0); }
  static constexpr bool kLoose = false;
  static constexpr bool kFP = true;
  static constexpr bool kSigned = true;
  __device__ static uint64_t load(uint64_t x) { return as_u(__dsub_rn(as_d(x | kDBias), kC52)); }
  // raw bits; the dispatcher never runs this policy where an intermediate
  // (non-canonical) result is written to memory
  __device__ static uint64_t store(uint64_t x) { return x; }
  // canonical integer of a value x in (-8q, 8q): k = round(x/q) (x*qinv is
  // within 2^-49 of x/q), r = x - kq exact in (-q/2 - 1, q/2 + 1); the result
  // is r + q or r, formed in the biased domain (2^52 + r + q, then minus q
  // when that stays >= 2^52), so no signed-zero case can arise.
  __device__ static uint64_t canon(double x, const LimbConstDev& c) {
    const double k = __dsub_rn(__fma_rn(x, c.qinv, kC52x15), kC52x15);
    return canon_small(__fma_rn(-k, c.q_d, x), c);
  }
  // canonical integer of an integer-valued double |r| < q (+1): r + q, minus q
  // when that stays >= q, in the biased domain (2^52 + r + q)
  __device__ static uint64_t canon_small(double r, const LimbConstDev& c) {
    const uint64_t rb = as_u(__dadd_rn(r, c.q_bias));  // 2^52 + r + q
    const uint64_t db = as_u(__dsub_rn(as_d(rb), c.q_d));
    return ((hi32(db) >= 0x43300000u) ? db : rb) & kMask52;
  }
  template <bool ILTM>
  __device__ static void fwd(uint64_t& x0, uint64_t& x1, uint64_t w, const LimbConstDev& c) {
    const double u = ILTM ? as_d(x0) : csubS(as_d(x0), c.twoq_d);
    const double t = mul_recip_fine(as_d(x1), as_d(w), c.qinv, c.q_d);  // balanced w: |w x1| < 2q^2
    x0 = as_u(__dadd_rn(u, t));
    x1 = as_u(__dsub_rn(u, t));
  }
  template <bool ILTM>
  __device__ static void inv(uint64_t& x0, uint64_t& x1, uint64_t w, const LimbConstDev& c) {
    const double a = as_d(x0), b = as_d(x1);
    const double t = __dsub_rn(a, b);
    double s = __dadd_rn(a, b);
    if (!ILTM) s = csubS(s, c.twoq_d);
    x0 = as_u(s);
    x1 = as_u(mul_recip_fine(t, as_d(w), c.qinv, c.q_d));  // balanced w, |t| < 4q
  }
  __device__ static uint64_t scale_ninv(uint64_t x, const LimbConstDev& c) {
    return as_u(mul_signed(as_d(x), as_d(c.ninv), as_d(c.ninvp), c.qq));
  }
  // see ArithInt::inv_fold; signed doubles |x| < 2q in, canonical words out:
  // |a +- b| < 4q times the BALANCED constants n^-1, n^-1 w_1 (|w v| < 2q^2:
  // integer-grid product, |T| < q), then one fix-up to [0, q): 9 FP64
  // operations per word, no conditional subtraction
  static constexpr bool kFold = true;
  __device__ static void inv_fold(uint64_t& x0, uint64_t& x1, const LimbConstDev& c) {
    const double a = as_d(x0), b = as_d(x1);
    const double s = __dadd_rn(a, b), t = __dsub_rn(a, b);
    x0 = canon_small(mul_recip_fine(s, c.ninv_b, c.qinv, c.q_d), c);
    x1 = canon_small(mul_recip_fine(t, c.nw_b, c.qinv, c.q_d), c);
  }
  // An inverse stage on the pair (x0, x1) whose two inputs are BOTH products
  // of the stage before (|x| < q each: T outputs): the sum stays below 2q
  // without the conditional subtraction. Inside a register pass this is known
  // per butterfly (the index bit of the previous stage is a register bit).
  static constexpr bool kInvSkipTT = true;
};

// ---------------------------------------------------------------------------
// ArithIntL: beta = 2^64 limbs with q < 2^60, canonical outputs only (fout ==
// 1, like Arith52S for beta = 2^52).
//
// The Shoup quotient drops the low x low partial product and the carries of
// the two cross products' low halves:
//   qh = a1 b1 + hi32(a1 b0) + hi32(a0 b1)     (w' = a1:a0, x = b1:b0)
// The dropped terms sum to less than 3 * 2^64, so qh = floor(w'x / 2^64) - d
// with d in {0, 1, 2}, and T = w x - qh q (mod 2^64) = T_exact + d q lies in
// [0, 4q). Cost: one IMAD.WIDE and two IMAD.HI instead of four IMAD.WIDE
// (IMAD.WIDE issues at half the IMAD rate).
// The bound holds for every 64-bit x (Shoup: w x - floor(w' x / 2^64) q < q (1 +
// x / 2^64) < 2q), so the multiplicand needs no reduction, and with 16q <= 2^64
// the words have room to skip reductions:
//   forward: a reducing stage takes x < 16q: u = x0 reduced by 8q once ([0,
//            8q)), x0' = u + T, x1' = u + 4q - T, both below 12q; the stage
//            after it may skip the reduction (u = x0 < 12q): outputs below
//            16q. The 16384-word kernels reduce on odd stages only (fwd_skip);
//            inputs are below 4q (fin <= 4) or, after the global passes of a
//            long row (which reduce at every stage but the first), below 12q.
//            Final words below 16q: four conditional subtractions to [0, q).
//   inverse: words in [0, 8q): x0' = x0 + x1 reduced by 8q once, x1' = T(x0 +
//            8q - x1) < 4q; the sum of two products (both inputs T outputs of
//            the stage before) stays below 8q without the reduction
//            (kInvSkipTT: known per butterfly inside a register pass).
// Representatives differ from the reference's lazy ones; canonical results
// are identical (they are unique).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t qhat64_loose(uint64_t wp, uint64_t x) {
  const uint32_t a0 = lo32(wp), a1 = hi32(wp), b0 = lo32(x), b1 = hi32(x);
  const uint64_t cross = static_cast<uint64_t>(__umulhi(a1, b0)) + __umulhi(a0, b1);
  return mad_wide(a1, b1, cross);
}
__device__ __forceinline__ uint64_t mul_loose(uint64_t x, uint64_t w, uint64_t wp, uint64_t negq) {
  return lo_sum(w, x, qhat64_loose(wp, x), negq);
}

struct ArithIntL {
  static constexpr int kIltmFwd = 1;  // forward stages whose pre-reduction is skipped at fin = 1
  using Tw = ulonglong2;  // {w, w'}
  static constexpr bool kFP = false;
  static constexpr bool kSigned = false;
  static constexpr bool kLoose = true;
  __device__ static uint64_t load(uint64_t x) { return x; }
  __device__ static uint64_t store(uint64_t x) { return x; }
  // ILTM: the stage skips its reduction (inputs below 12q; at fin <= 4 the first stage's
  // inputs are below 4q)
  template <bool ILTM>
  __device__ static void fwd(uint64_t& x0, uint64_t& x1, ulonglong2 w, const LimbConstDev& c) {
    const uint64_t u = ILTM ? x0 : nk::csub(x0, c.fourq << 1);
    const uint64_t t = mul_loose(x1, w.x, w.y, c.negq);
    x0 = u + t;
    x1 = u + c.fourq - t;
  }
  // the 16384-word kernels' schedule: stage gs (0 = the block's first stage) skips on even gs
  __host__ __device__ static constexpr bool fwd_skip(bool, int gs) { return (gs & 1) == 0; }
  template <bool ILTM>
  __device__ static void inv(uint64_t& x0, uint64_t& x1, ulonglong2 w, const LimbConstDev& c) {
    const uint64_t eightq = c.fourq << 1;
    const uint64_t t = x0 + eightq - x1;
    uint64_t s = x0 + x1;
    if (!ILTM) s = nk::csub(s, eightq);
    x0 = s;
    x1 = mul_loose(t, w.x, w.y, c.negq);
  }
  static constexpr bool kInvSkipTT = true;
  __device__ static uint64_t scale_ninv(uint64_t x, const LimbConstDev& c) {
    return mul_loose(x, c.ninv, c.ninvp, c.negq);
  }
  // [0, 16q) -> [0, q)
  __device__ static uint64_t red16(uint64_t x, const LimbConstDev& c) {
    return nk::csub(nk::csub(nk::csub(nk::csub(x, c.fourq << 1), c.fourq), c.twoq), c.q);
  }
  // [0, 4q) -> [0, q)
  __device__ static uint64_t red4(uint64_t x, const LimbConstDev& c) {
    return nk::csub(nk::csub(x, c.twoq), c.q);
  }
  static constexpr bool kFold = true;
  __device__ static void inv_fold(uint64_t& x0, uint64_t& x1, const LimbConstDev& c) {
    const uint64_t s = x0 + x1, t = x0 + (c.fourq << 1) - x1;  // both below 16q
    x0 = red4(mul_loose(s, c.ninv, c.ninvp, c.negq), c);
    x1 = red4(mul_loose(t, c.nw, c.nwp, c.negq), c);
  }
};

// a * b mod q, canonical, for canonical integers a, b < q < 2^50 on the FP64
// pipe: h + l = a b exactly (TwoProduct), k = round(h / q) through the
// rounded reciprocal (|h/q - k| <= 0.75), r = h - k q + l exact in
// (-0.76q, 0.76q), one conditional add of q. The product is unique, so this
// equals the reference's eltwise_mult_mod (eltwise.hpp:180-188) result.
__device__ __forceinline__ uint64_t mulmod_canon(uint64_t a, uint64_t b, const LimbConstDev& c) {
  const double x = __dsub_rn(as_d(a | kDBias), kC52), y = __dsub_rn(as_d(b | kDBias), kC52);
  const double h = __dmul_rn(x, y);
  const double l = __fma_rn(x, y, -h);
  const double k = __dsub_rn(__fma_rn(h, c.qinv, kC52x15), kC52x15);
  const double r = __dadd_rn(__fma_rn(-k, c.q_d, h), l);
  const uint64_t rb = as_u(__dadd_rn(r, c.q_bias));  // 2^52 + r + q
  const uint64_t db = as_u(__dsub_rn(as_d(rb), c.q_d));
  return ((hi32(db) >= 0x43300000u) ? db : rb) & kMask52;
}

// (x * g) mod q as a canonical word, for a signed Arith52S word |x| < 4q (a
// forward transform's output before canonicalisation) and a canonical g < q:
// x reduced to |x| < 2q (csubS), the fine rounded-reciprocal product
// (mul_recip_fine, |T| < 0.875q), then one fix-up to [0, q)
// (Arith52S::canon_small): 10 FP64 operations per word instead of canon +
// mulmod_canon (15): the fused poly_mult_mod forward multiplies before
// canonicalising.
__device__ __forceinline__ uint64_t mulmod_signed_canon(uint64_t xbits, uint64_t g, const LimbConstDev& c) {
  const double x = csubS(as_d(xbits), c.twoq_d);
  const double gd = __dsub_rn(as_d(g | kDBias), kC52);
  return Arith52S::canon_small(mul_recip_fine(x, gd, c.qinv, c.q_d), c);
}

// Final word of a forward transform (small_mod(x, q, 4) when fout == 1,
// ntt.hpp:282-284) and of an inverse (n^-1 Shoup pass, ntt.hpp:429-432, then
// small_mod(x, q, 2) when fout == 1, ntt.hpp:303-305), as stored integers.
template <class A>
__device__ __forceinline__ uint64_t fwd_out(uint64_t x, const LimbConstDev& c, int fout) {
  if constexpr (A::kLoose) {
    return A::red16(x, c);  // canonical-only policy
  } else if constexpr (A::kSigned) {
    return A::canon(as_d(x), c);
  } else {
    return A::store(fout == 1 ? A::red4(x, c) : x);
  }
}
template <class A>
__device__ __forceinline__ uint64_t inv_out(uint64_t x, const LimbConstDev& c, int fout) {
  const uint64_t y = A::scale_ninv(x, c);
  if constexpr (A::kLoose) {
    return A::red4(y, c);  // canonical-only policy
  } else if constexpr (A::kSigned) {
    return A::canon(as_d(y), c);
  } else {
    return A::store(fout == 1 ? A::red2(y, c) : y);
  }
}

}  // namespace nk
