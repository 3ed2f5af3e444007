// Host-side precomputation for the device tables (product code, C++17).
//
// Reproduces the reference's table construction bit for bit so that lazy
// (non-canonical) outputs match:
//   is_prime               modarith.hpp:75-98   (deterministic Miller-Rabin, 12 witnesses)
//   Modulus                modarith.hpp:106-129 (bits, Barrett factor floor(2^(63+bits)/q))
//   minimal_primitive_root ntt.hpp:172-197      (smallest primitive 2n-th root)
//   NttTables ctor         ntt.hpp:217-247      (validation order and messages)
//   build_tables<B>        ntt.hpp:343-361      (psi^i at bit_reverse(i), floor(W*2^B/q))
// Plain 128-bit % arithmetic is used: every quantity above is canonical, so the
// arithmetic route does not matter, only the definitions do.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace nk {
namespace host {

using u128 = unsigned __int128;

inline uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q) {
  return static_cast<uint64_t>(static_cast<u128>(a) * b % q);
}
inline uint64_t powmod(uint64_t b, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  b %= q;
  while (e) {
    if (e & 1) r = mulmod(r, b, q);
    b = mulmod(b, b, q);
    e >>= 1;
  }
  return r;
}

inline bool is_prime(uint64_t n) {
  static const uint64_t wit[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return false;
  for (uint64_t p : wit)
    if (n % p == 0) return n == p;
  uint64_t d = n - 1;
  const int s = __builtin_ctzll(d);
  d >>= s;
  for (uint64_t a : wit) {
    uint64_t x = powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool composite = true;
    for (int i = 1; i < s; ++i) {
      x = mulmod(x, x, n);
      if (x == n - 1) { composite = false; break; }
    }
    if (composite) return false;
  }
  return true;
}

inline unsigned bit_width(uint64_t x) { return x ? 64u - static_cast<unsigned>(__builtin_clzll(x)) : 0u; }

struct Modulus {
  uint64_t q = 0;
  unsigned bits = 0;
  uint64_t barrett = 0;
};

// Returns false for an invalid modulus (modarith.hpp:109-111).
inline bool make_modulus(uint64_t q, Modulus* m) {
  if (q < 3 || q >= (uint64_t{1} << 62) || !is_prime(q)) return false;
  m->q = q;
  m->bits = bit_width(q);
  m->barrett = static_cast<uint64_t>((u128{1} << (63 + m->bits)) / q);
  return true;
}

inline uint64_t bit_reverse(uint64_t i, unsigned logn) {
  uint64_t r = 0;
  for (unsigned b = 0; b < logn; ++b) { r = (r << 1) | (i & 1); i >>= 1; }
  return r;
}

// 0 if order is not a power of two dividing q-1.
inline uint64_t minimal_primitive_root(uint64_t order, uint64_t q) {
  if (order == 0 || (order & (order - 1)) || (q - 1) % order) return 0;
  if (order == 1) return 1;
  const uint64_t half = order / 2, e = (q - 1) / order;
  uint64_t w0 = 0;
  for (uint64_t g = 2; g < q; ++g) {
    const uint64_t w = powmod(g, e, q);
    if (powmod(w, half, q) == q - 1) { w0 = w; break; }
  }
  if (!w0) return 0;
  const uint64_t sq = mulmod(w0, w0, q);
  uint64_t cur = w0, best = w0;
  for (uint64_t i = 1; i < half; ++i) {
    cur = mulmod(cur, sq, q);
    if (cur < best) best = cur;
  }
  return best;
}

struct Tables {
  uint64_t n = 0, q = 0, psi = 0, psi_inv = 0, ninv = 0, ninvp = 0;
  unsigned logn = 0;
  int bs = 0;
  std::vector<uint64_t> w, wp, wi, wip;  // bit-reversed root powers and precons
};

// Error codes follow include/nttkit_b200.h; *msg receives the reference's text.
inline int build_tables(uint64_t n, uint64_t q, const uint64_t* root, int bit_shift, Tables* t,
                        std::string* msg) {
  Modulus m;
  if (!make_modulus(q, &m)) { *msg = "Modulus: value must be a prime in [3, 2^62)"; return -1; }
  if (n < 2 || n > (uint64_t{1} << 20) || (n & (n - 1))) {
    *msg = "NttTables: n must be a power of two in [2, 2^20]"; return -2;
  }
  if (q % (2 * n) != 1) { *msg = "NttTables: q must satisfy q == 1 (mod 2n)"; return -3; }
  if (bit_shift == 0) bit_shift = (u128{4} * q < (u128{1} << 52)) ? 52 : 64;
  if (bit_shift != 52 && bit_shift != 64) {
    *msg = "NttTables: accumulator width must be 52 or 64"; return -4;
  }
  if (bit_shift == 52 && u128{4} * q >= (u128{1} << 52)) {
    *msg = "NttTables: 52-bit accumulator requires 4q < 2^52"; return -5;
  }
  uint64_t psi;
  if (root != nullptr) {  // an explicit root, as std::optional<uint64_t> (ntt.hpp:232-237)
    if (*root == 0 || *root >= q || powmod(*root, n, q) != q - 1) {
      *msg = "NttTables: root is not a primitive 2n'th root of unity"; return -6;
    }
    psi = *root;
  } else {
    psi = minimal_primitive_root(2 * n, q);
  }
  t->n = n; t->q = q; t->bs = bit_shift; t->psi = psi;
  t->psi_inv = powmod(psi, q - 2, q);
  t->logn = bit_width(n) - 1;
  t->w.assign(n, 0); t->wp.assign(n, 0); t->wi.assign(n, 0); t->wip.assign(n, 0);
  uint64_t f = 1, iv = 1;
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t r = bit_reverse(i, t->logn);
    t->w[r] = f;
    t->wi[r] = iv;
    t->wp[r] = static_cast<uint64_t>((static_cast<u128>(f) << bit_shift) / q);
    t->wip[r] = static_cast<uint64_t>((static_cast<u128>(iv) << bit_shift) / q);
    f = mulmod(f, psi, q);
    iv = mulmod(iv, t->psi_inv, q);
  }
  t->ninv = powmod(n % q, q - 2, q);
  t->ninvp = static_cast<uint64_t>((static_cast<u128>(t->ninv) << bit_shift) / q);
  return 0;
}

}  // namespace host
}  // namespace nk
