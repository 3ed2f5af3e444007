/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the B200 NTT / element-wise path.
 * See nttkit_oracle.h for the contract. Every function restates the reference
 * algorithm at the cited /root/reference/proj/ file:line; nothing here is
 * shipped or called by the product library.
 */
#include "nttkit_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

#define MIN64(a, b) ((a) < (b) ? (a) : (b))

/* ------------------------------------------------------------------------ */
/* modarith.hpp                                                              */
/* ------------------------------------------------------------------------ */

/* detail::mul_mod_u64 / pow_mod_u64, modarith.hpp:56-69 */
static uint64_t mulmod_full(uint64_t a, uint64_t b, uint64_t m) {
  return (uint64_t)(((u128)a * b) % m);
}
static uint64_t powmod_full(uint64_t base, uint64_t exp, uint64_t m) {
  uint64_t result = 1 % m;
  base %= m;
  while (exp) {
    if (exp & 1) result = mulmod_full(result, base, m);
    base = mulmod_full(base, base, m);
    exp >>= 1;
  }
  return result;
}

/* Deterministic Miller-Rabin with the first twelve primes, modarith.hpp:75-98 */
int oc_is_prime(uint64_t n) {
  static const uint64_t w[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return 0;
  for (int i = 0; i < 12; ++i)
    if (n % w[i] == 0) return n == w[i];
  uint64_t d = n - 1;
  int s = __builtin_ctzll(d);
  d >>= s;
  for (int i = 0; i < 12; ++i) {
    uint64_t x = powmod_full(w[i], d, n);
    if (x == 1 || x == n - 1) continue;
    int composite = 1;
    for (int k = 1; k < s; ++k) {
      x = mulmod_full(x, x, n);
      if (x == n - 1) { composite = 0; break; }
    }
    if (composite) return 0;
  }
  return 1;
}

static unsigned bit_width(uint64_t x) { return x ? 64u - (unsigned)__builtin_clzll(x) : 0u; }

/* Modulus ctor, modarith.hpp:108-115: prime q in [3, 2^62); k = floor(2^(63+bits)/q) */
int oc_modulus(uint64_t q, uint32_t* bits, uint64_t* barrett_factor) {
  if (q < 3 || q >= ((uint64_t)1 << 62) || !oc_is_prime(q)) return -1;
  unsigned b = bit_width(q);
  if (bits) *bits = b;
  if (barrett_factor) *barrett_factor = (uint64_t)(((u128)1 << (63 + b)) / q);
  return 0;
}

/* barrett_reduce, modarith.hpp:191-200 (d < 2^(63+bits)) */
static uint64_t barrett(u128 d, uint64_t q, unsigned bits, uint64_t k) {
  uint64_t c1 = (uint64_t)(d >> (bits - 1));
  uint64_t c3 = (uint64_t)(((u128)c1 * k) >> 64);
  uint64_t r = (uint64_t)d - c3 * q;
  r = MIN64(r, r - 2 * q);
  r = MIN64(r, r - q);
  return r;
}
uint64_t oc_barrett_reduce(uint64_t d_hi, uint64_t d_lo, uint64_t q) {
  uint32_t bits; uint64_t k;
  if (oc_modulus(q, &bits, &k)) return ~(uint64_t)0;
  return barrett(((u128)d_hi << 64) | d_lo, q, bits, k);
}

/* mul_mod, modarith.hpp:203-206 */
uint64_t oc_mul_mod(uint64_t a, uint64_t b, uint64_t q) {
  uint32_t bits; uint64_t k;
  oc_modulus(q, &bits, &k);
  return barrett((u128)a * b, q, bits, k);
}

/* pow_mod, modarith.hpp:228-237 (square-and-multiply over Barrett products) */
static uint64_t pow_mod_b(uint64_t base, uint64_t exp, uint64_t q, unsigned bits, uint64_t k) {
  uint64_t result = 1;
  base %= q;
  while (exp) {
    if (exp & 1) result = barrett((u128)result * base, q, bits, k);
    base = barrett((u128)base * base, q, bits, k);
    exp >>= 1;
  }
  return result;
}
uint64_t oc_pow_mod(uint64_t base, uint64_t exp, uint64_t q) {
  uint32_t bits; uint64_t k;
  oc_modulus(q, &bits, &k);
  return pow_mod_b(base, exp, q, bits, k);
}

/* inv_mod via Fermat, modarith.hpp:240-246; returns 0 for a zero input */
uint64_t oc_inv_mod(uint64_t x, uint64_t q) {
  x %= q;
  if (x == 0) return 0;
  return oc_pow_mod(x, q - 2, q);
}

/* small_mod, modarith.hpp:217-225 */
uint64_t oc_small_mod(uint64_t x, uint64_t q, uint64_t factor) {
  if (factor == 8) x = MIN64(x, x - 4 * q);
  if (factor >= 4) x = MIN64(x, x - 2 * q);
  if (factor >= 2) x = MIN64(x, x - q);
  return x;
}

/* precompute_factor<B>, modarith.hpp:176-183: floor(w * 2^B / q) */
uint64_t oc_precompute_factor(uint64_t w, uint64_t q, int bit_shift) {
  return (uint64_t)(((u128)w << bit_shift) / q);
}

/* bit_reverse, ntt.hpp:37-46 */
uint64_t oc_bit_reverse(uint64_t i, unsigned log2n) {
  uint64_t r = 0;
  for (unsigned b = 0; b < log2n; ++b) { r = (r << 1) | (i & 1); i >>= 1; }
  return r;
}

/* ------------------------------------------------------------------------ */
/* ntt.hpp                                                                    */
/* ------------------------------------------------------------------------ */

/* minimal_primitive_root, ntt.hpp:172-197 */
uint64_t oc_minimal_primitive_root(uint64_t order, uint64_t q) {
  uint32_t bits; uint64_t k;
  if (oc_modulus(q, &bits, &k)) return 0;
  if (order == 0 || (order & (order - 1)) || (q - 1) % order) return 0;
  if (order == 1) return 1;
  const uint64_t half = order / 2, e = (q - 1) / order;
  uint64_t w0 = 0;
  for (uint64_t g = 2; g < q; ++g) {
    uint64_t w = pow_mod_b(g, e, q, bits, k);
    if (pow_mod_b(w, half, q, bits, k) == q - 1) { w0 = w; break; }
  }
  if (!w0) return 0;
  const uint64_t w0sq = barrett((u128)w0 * w0, q, bits, k);
  uint64_t cur = w0, best = w0;
  for (uint64_t i = 1; i < half; ++i) {
    cur = barrett((u128)cur * w0sq, q, bits, k);
    if (cur < best) best = cur;
  }
  return best;
}

/* A table set for one (n, q), as NttTables holds it (ntt.hpp:206-247, 343-361). */
typedef struct {
  uint64_t n, q, twice_q, neg_q;
  unsigned log2n;
  int bs; /* 52 or 64 */
  uint64_t *w, *wp, *wi, *wip;
  uint64_t ninv, ninvp;
} tables_t;

static void tables_free(tables_t* t) {
  free(t->w); free(t->wp); free(t->wi); free(t->wip);
  memset(t, 0, sizeof(*t));
}

/* NttTables ctor validation ntt.hpp:219-241, select_bit_shift ntt.hpp:323-325,
 * build_tables ntt.hpp:343-361 */
static int tables_build(tables_t* t, uint64_t n, uint64_t q, uint64_t root, int bit_shift) {
  uint32_t bits; uint64_t k;
  memset(t, 0, sizeof(*t));
  if (oc_modulus(q, &bits, &k)) return -1;
  if (n < 2 || n > ((uint64_t)1 << 20) || (n & (n - 1))) return -2;
  if (q % (2 * n) != 1) return -3;
  if (bit_shift == 0) bit_shift = ((u128)4 * q < ((u128)1 << 52)) ? 52 : 64;
  if (bit_shift != 52 && bit_shift != 64) return -4;
  if (bit_shift == 52 && (u128)4 * q >= ((u128)1 << 52)) return -5;
  uint64_t psi;
  if (root) {
    if (root >= q || pow_mod_b(root, n, q, bits, k) != q - 1) return -6;
    psi = root;
  } else {
    psi = oc_minimal_primitive_root(2 * n, q);
  }
  const uint64_t psi_inv = pow_mod_b(psi, q - 2, q, bits, k);
  t->n = n; t->q = q; t->twice_q = 2 * q; t->bs = bit_shift;
  t->log2n = bit_width(n) - 1;
  /* negated_modulus<B>, ntt.hpp:85-92 */
  t->neg_q = bit_shift == 52 ? (((uint64_t)1 << 52) - q) : (~q + 1);
  t->w = malloc(n * 8); t->wp = malloc(n * 8); t->wi = malloc(n * 8); t->wip = malloc(n * 8);
  uint64_t fwd = 1, inv = 1;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t r = oc_bit_reverse(i, t->log2n);
    t->w[r] = fwd; t->wi[r] = inv;
    t->wp[r] = oc_precompute_factor(fwd, q, bit_shift);
    t->wip[r] = oc_precompute_factor(inv, q, bit_shift);
    fwd = barrett((u128)fwd * psi, q, bits, k);
    inv = barrett((u128)inv * psi_inv, q, bits, k);
  }
  t->ninv = pow_mod_b(n % q, q - 2, q, bits, k);
  t->ninvp = oc_precompute_factor(t->ninv, q, bit_shift);
  return 0;
}

int oc_ntt_tables(uint64_t n, uint64_t q, uint64_t root, int bit_shift,
                  uint64_t* psi_out, uint64_t* psi_inv_out,
                  uint64_t* psi_rev, uint64_t* psi_precon_rev,
                  uint64_t* psi_inv_rev, uint64_t* psi_inv_precon_rev,
                  uint64_t* n_inv, uint64_t* n_inv_precon) {
  tables_t t;
  int rc = tables_build(&t, n, q, root, bit_shift);
  if (rc) return rc;
  /* psi_rev[bit_reverse(1)] = psi^1 (ntt.hpp:257-258) */
  if (psi_out) *psi_out = t.w[n >> 1];
  if (psi_inv_out) *psi_inv_out = t.wi[n >> 1];
  if (psi_rev) memcpy(psi_rev, t.w, n * 8);
  if (psi_precon_rev) memcpy(psi_precon_rev, t.wp, n * 8);
  if (psi_inv_rev) memcpy(psi_inv_rev, t.wi, n * 8);
  if (psi_inv_precon_rev) memcpy(psi_inv_precon_rev, t.wip, n * 8);
  if (n_inv) *n_inv = t.ninv;
  if (n_inv_precon) *n_inv_precon = t.ninvp;
  int bs = t.bs;
  tables_free(&t);
  return bs;
}

/* mul_hi/mul_lo/mul_lo_add<B> (modarith.hpp:131-165) composed as
 * mul_factor_lazy<B> (ntt.hpp:97-101) */
static inline uint64_t mul_factor_lazy(uint64_t x, uint64_t w, uint64_t wp, uint64_t neg_q, int bs) {
  if (bs == 52) {
    const uint64_t mask = ((uint64_t)1 << 52) - 1;
    uint64_t qhat = (uint64_t)(((u128)wp * x) >> 52);
    return ((w * x & mask) + qhat * neg_q) & mask;
  }
  uint64_t qhat = (uint64_t)(((u128)wp * x) >> 64);
  return w * x + qhat * neg_q;
}

/* fwd_butterfly<B, ILTM>, ntt.hpp:103-113 */
static inline void fwd_bfly(uint64_t* x0, uint64_t* x1, uint64_t w, uint64_t wp,
                            const tables_t* t, int iltm) {
  uint64_t u = *x0;
  if (!iltm) u = MIN64(u, u - t->twice_q);
  uint64_t v = mul_factor_lazy(*x1, w, wp, t->neg_q, t->bs);
  *x0 = u + v;
  *x1 = u + t->twice_q - v;
}

/* inv_butterfly<B, ILTM>, ntt.hpp:115-130 */
static inline void inv_bfly(uint64_t* x0, uint64_t* x1, uint64_t w, uint64_t wp,
                            const tables_t* t, int iltm) {
  uint64_t x1m = *x1 - t->twice_q;
  uint64_t v = *x0 - x1m;
  if (t->bs == 52) v &= ((uint64_t)1 << 52) - 1;
  uint64_t sum = *x0 + *x1;
  if (!iltm) sum = MIN64(sum, sum - t->twice_q);
  *x0 = sum;
  *x1 = mul_factor_lazy(v, w, wp, t->neg_q, t->bs);
}

/* the scalar butterflies of the public API, harvey_forward_butterfly /
 * harvey_inverse_butterfly (ntt.hpp:137-166): one butterfly per element pair,
 * twiddle w with its precon for width bs, ILTM off */
int oc_butterflies(int fwd, uint64_t q, int bs, uint64_t w, const uint64_t* x0, const uint64_t* x1,
                   uint64_t n, uint64_t* y0, uint64_t* y1) {
  if (bs != 52 && bs != 64) return -1;
  tables_t t;
  memset(&t, 0, sizeof t);
  t.q = q;
  t.twice_q = 2 * q;
  t.bs = bs;
  t.neg_q = bs == 52 ? (((uint64_t)1 << 52) - q) : (~q + 1);
  const uint64_t wp = (uint64_t)(((u128)w << bs) / q);
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t a = x0[i], b = x1[i];
    if (fwd) fwd_bfly(&a, &b, w, wp, &t, 0);
    else inv_bfly(&a, &b, w, wp, &t, 0);
    y0[i] = a;
    y1[i] = b;
  }
  return 0;
}

/* forward_impl<B>, ntt.hpp:363-394, then the fout==1 pass ntt.hpp:282-284 */
static void forward_row(const tables_t* t, uint64_t* a, uint64_t fin, uint64_t fout) {
  const uint64_t n = t->n;
  uint64_t tt = n >> 1, m = 1;
  if (fin == 1) {
    uint64_t* y = a + tt;
    for (uint64_t j = 0; j < tt; ++j) fwd_bfly(&a[j], &y[j], t->w[1], t->wp[1], t, 1);
    m = 2; tt >>= 1;
  }
  for (; m < n; m <<= 1, tt >>= 1) {
    for (uint64_t i = 0; i < m; ++i) {
      const uint64_t w = t->w[m + i], wp = t->wp[m + i];
      uint64_t* x = a + 2 * i * tt;
      uint64_t* y = x + tt;
      for (uint64_t j = 0; j < tt; ++j) fwd_bfly(&x[j], &y[j], w, wp, t, 0);
    }
  }
  if (fout == 1)
    for (uint64_t j = 0; j < n; ++j) a[j] = oc_small_mod(a[j], t->q, 4);
}

/* inverse_impl<B>, ntt.hpp:396-433, then the fout==1 pass ntt.hpp:303-305 */
static void inverse_row(const tables_t* t, uint64_t* a, uint64_t fin, uint64_t fout) {
  const uint64_t n = t->n;
  uint64_t tt = 1, m = n;
  if (fin == 1) {
    const uint64_t h = m >> 1;
    for (uint64_t i = 0; i < h; ++i)
      inv_bfly(&a[2 * i], &a[2 * i + 1], t->wi[h + i], t->wip[h + i], t, 1);
    m = h; tt = 2;
  }
  for (; m > 1; m >>= 1, tt <<= 1) {
    const uint64_t h = m >> 1;
    uint64_t j1 = 0;
    for (uint64_t i = 0; i < h; ++i) {
      const uint64_t w = t->wi[h + i], wp = t->wip[h + i];
      uint64_t* x = a + j1;
      uint64_t* y = x + tt;
      for (uint64_t j = 0; j < tt; ++j) inv_bfly(&x[j], &y[j], w, wp, t, 0);
      j1 += 2 * tt;
    }
  }
  for (uint64_t j = 0; j < n; ++j) a[j] = mul_factor_lazy(a[j], t->ninv, t->ninvp, t->neg_q, t->bs);
  if (fout == 1)
    for (uint64_t j = 0; j < n; ++j) a[j] = oc_small_mod(a[j], t->q, 2);
}

/* ---- batch driver with optional pthreads over independent rows ---- */
typedef struct {
  const tables_t* tabs; uint32_t nmod; uint64_t n;
  uint64_t* res; const uint64_t* op; uint64_t r0, r1, fin, fout; int dir;
  const uint64_t* g; /* poly mult second operand */
} job_t;

static void poly_mult_row(const tables_t* t, uint64_t* res, const uint64_t* f, const uint64_t* g);

static void* run_job(void* p) {
  job_t* j = (job_t*)p;
  for (uint64_t r = j->r0; r < j->r1; ++r) {
    const tables_t* t = &j->tabs[r % j->nmod];
    uint64_t* dst = j->res + r * j->n;
    if (j->dir == 2) { poly_mult_row(t, dst, j->op + r * j->n, j->g + r * j->n); continue; }
    if (dst != j->op + r * j->n) memcpy(dst, j->op + r * j->n, j->n * 8);
    if (j->dir == 0) forward_row(t, dst, j->fin, j->fout);
    else inverse_row(t, dst, j->fin, j->fout);
  }
  return NULL;
}

static int run_batch(uint64_t n, const uint64_t* moduli, uint32_t nmod, int bit_shift,
                     uint64_t* res, const uint64_t* op, const uint64_t* g, uint64_t rows,
                     uint64_t fin, uint64_t fout, int dir, int threads) {
  if (nmod == 0) return -10;
  tables_t* tabs = calloc(nmod, sizeof(tables_t));
  int rc = 0;
  for (uint32_t i = 0; i < nmod && !rc; ++i) rc = tables_build(&tabs[i], n, moduli[i], 0, bit_shift);
  if (!rc) {
    if (threads < 1) threads = 1;
    if ((uint64_t)threads > rows) threads = rows ? (int)rows : 1;
    pthread_t* th = calloc(threads, sizeof(pthread_t));
    job_t* jobs = calloc(threads, sizeof(job_t));
    for (int i = 0; i < threads; ++i) {
      jobs[i] = (job_t){tabs, nmod, n, res, op, rows * i / threads, rows * (i + 1) / threads,
                        fin, fout, dir, g};
      if (threads == 1) run_job(&jobs[i]);
      else pthread_create(&th[i], NULL, run_job, &jobs[i]);
    }
    if (threads > 1)
      for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
    free(th); free(jobs);
  }
  for (uint32_t i = 0; i < nmod; ++i) tables_free(&tabs[i]);
  free(tabs);
  return rc;
}

/* NttTables::forward factor checks, ntt.hpp:270-275 */
int oc_ntt_forward(uint64_t n, const uint64_t* moduli, uint32_t nmod, int bit_shift,
                   uint64_t* result, const uint64_t* operand, uint64_t rows,
                   uint64_t fin, uint64_t fout, int threads) {
  if (fin != 1 && fin != 2 && fin != 4) return -20;
  if (fout != 1 && fout != 4) return -21;
  return run_batch(n, moduli, nmod, bit_shift, result, operand, NULL, rows, fin, fout, 0, threads);
}

/* NttTables::inverse factor checks, ntt.hpp:291-296 */
int oc_ntt_inverse(uint64_t n, const uint64_t* moduli, uint32_t nmod, int bit_shift,
                   uint64_t* result, const uint64_t* operand, uint64_t rows,
                   uint64_t fin, uint64_t fout, int threads) {
  if (fin != 1 && fin != 2) return -22;
  if (fout != 1 && fout != 2) return -23;
  return run_batch(n, moduli, nmod, bit_shift, result, operand, NULL, rows, fin, fout, 1, threads);
}

/* One row with an explicit root (NttTables(n, m, root), ntt.hpp:212-213); dir 0 fwd, 1 inv */
int oc_ntt_root(uint64_t n, uint64_t q, uint64_t root, int bit_shift, int dir, uint64_t* result,
                const uint64_t* operand, uint64_t fin, uint64_t fout) {
  tables_t t;
  int rc = tables_build(&t, n, q, root, bit_shift);
  if (rc) return rc;
  if (result != operand) memcpy(result, operand, n * 8);
  if (dir == 0) forward_row(&t, result, fin, fout);
  else inverse_row(&t, result, fin, fout);
  tables_free(&t);
  return 0;
}

/* First `nstages` stages of forward_impl / inverse_impl (debug aid for kernel bring-up) */
int oc_ntt_stages(uint64_t n, uint64_t q, int dir, uint64_t* a, uint64_t fin, int nstages) {
  tables_t t;
  int rc = tables_build(&t, n, q, 0, 0);
  if (rc) return rc;
  if (dir == 0) {
    uint64_t tt = n >> 1, m = 1;
    for (int s = 0; m < n && s < nstages; m <<= 1, tt >>= 1, ++s)
      for (uint64_t i = 0; i < m; ++i)
        for (uint64_t j = 0; j < tt; ++j)
          fwd_bfly(&a[2 * i * tt + j], &a[2 * i * tt + j + tt], t.w[m + i], t.wp[m + i], &t,
                   s == 0 && fin == 1);
  } else {
    uint64_t tt = 1, m = n;
    for (int s = 0; m > 1 && s < nstages; m >>= 1, tt <<= 1, ++s) {
      const uint64_t h = m >> 1;
      for (uint64_t i = 0; i < h; ++i)
        for (uint64_t j = 0; j < tt; ++j)
          inv_bfly(&a[2 * i * tt + j], &a[2 * i * tt + j + tt], t.wi[h + i], t.wip[h + i], &t,
                   s == 0 && fin == 1);
    }
  }
  tables_free(&t);
  return 0;
}

/* reference_ntt, ntt.hpp:457-508 (independent: only full-width % arithmetic) */
int oc_reference_ntt(uint64_t n, uint64_t q, uint64_t psi, int dir, const uint64_t* a, uint64_t* out) {
  if (n < 2 || (n & (n - 1))) return -1;
  unsigned lg = bit_width(n) - 1;
  if (dir == 0) {
    const uint64_t omega = mulmod_full(psi, psi, q);
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t wi = powmod_full(omega, i, q);
      uint64_t acc = 0, coeff = 1;
      const uint64_t step = mulmod_full(psi, wi, q);
      for (uint64_t j = 0; j < n; ++j) {
        acc = (acc + mulmod_full(a[j], coeff, q)) % q;
        coeff = mulmod_full(coeff, step, q);
      }
      out[oc_bit_reverse(i, lg)] = acc;
    }
  } else {
    uint64_t* std_ = malloc(n * 8);
    for (uint64_t i = 0; i < n; ++i) std_[oc_bit_reverse(i, lg)] = a[i];
    const uint64_t psi_inv = powmod_full(psi, 2 * n - 1, q);
    const uint64_t omega_inv = mulmod_full(psi_inv, psi_inv, q);
    const uint64_t n_inv = powmod_full(n % q, q - 2, q);
    for (uint64_t i = 0; i < n; ++i) {
      uint64_t acc = 0, coeff = 1;
      const uint64_t step = powmod_full(omega_inv, i, q);
      for (uint64_t j = 0; j < n; ++j) {
        acc = (acc + mulmod_full(std_[j], coeff, q)) % q;
        coeff = mulmod_full(coeff, step, q);
      }
      acc = mulmod_full(acc, powmod_full(psi_inv, i, q), q);
      out[i] = mulmod_full(acc, n_inv, q);
    }
    free(std_);
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* eltwise.hpp                                                                */
/* ------------------------------------------------------------------------ */

/* eltwise_add_mod, eltwise.hpp:47-57 */
int oc_eltwise_add_mod(uint64_t* r, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t q) {
  for (uint64_t i = 0; i < n; ++i) { uint64_t s = a[i] + b[i]; r[i] = MIN64(s, s - q); }
  return 0;
}

/* eltwise_neg_mod, eltwise.hpp:60-70 */
int oc_eltwise_neg_mod(uint64_t* r, const uint64_t* a, uint64_t n, uint64_t q) {
  for (uint64_t i = 0; i < n; ++i) r[i] = a[i] == 0 ? 0 : q - a[i];
  return 0;
}

/* inv_modulus_round_up, eltwise.hpp:95-104 */
static double inv_modulus_round_up(uint64_t q) {
  const double qd = (double)q;
  double u = 1.0 / qd;
  const double p = u * qd;
  const double e = fma(u, qd, -p);
  if (p < 1.0 || (p == 1.0 && e < 0.0)) u = nextafter(u, INFINITY);
  return u;
}

/* eltwise_mult_mod dispatch eltwise.hpp:180-188; int path eltwise.hpp:137-154 + loop 74-92;
 * float path eltwise.hpp:158-175 + loop 106-125 */
int oc_eltwise_mult_mod(uint64_t* r, const uint64_t* a, const uint64_t* b, uint64_t n,
                        uint64_t q, uint64_t fin, int path) {
  uint32_t bits; uint64_t k;
  if (oc_modulus(q, &bits, &k)) return -1;
  if (fin != 1 && fin != 2 && fin != 4) return -30;
  if (path == 0) path = q < ((uint64_t)1 << 50) ? 2 : 1;
  if (path == 1) {
    if ((u128)fin * q >= ((u128)1 << 63)) return -31;
    const unsigned shift = bits - 1;
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t x = oc_small_mod(a[i], q, fin), y = oc_small_mod(b[i], q, fin);
      const u128 prod = (u128)x * y;
      const uint64_t c1 = (uint64_t)(prod >> shift);
      const uint64_t c3 = (uint64_t)(((u128)c1 * k) >> 64);
      uint64_t c4 = (uint64_t)prod - c3 * q;
      c4 = MIN64(c4, c4 - 2 * q);
      c4 = MIN64(c4, c4 - q);
      r[i] = c4;
    }
  } else {
    if (q >= ((uint64_t)1 << 50)) return -32;
    const double qd = (double)q, u = inv_modulus_round_up(q);
    for (uint64_t i = 0; i < n; ++i) {
      const double x = (double)oc_small_mod(a[i], q, fin), y = (double)oc_small_mod(b[i], q, fin);
      const double h = x * y;
      const double l = fma(x, y, -h);
      const double c = floor(h * u);
      const double d = fma(-c, qd, h);
      double g = d + l;
      if (g < 0.0) g += qd;
      if (g >= qd) g -= qd;
      r[i] = (uint64_t)g;
    }
  }
  return 0;
}

/* eltwise_fma_mod: auto width eltwise.hpp:263-271, checks 236-251, loop 192-209 */
int oc_eltwise_fma_mod(uint64_t* r, const uint64_t* a, uint64_t y, const uint64_t* z,
                       uint64_t n, uint64_t q, uint64_t fin, int bit_shift) {
  if (oc_modulus(q, NULL, NULL)) return -1;
  if (bit_shift == 0) bit_shift = ((u128)fin * q < ((u128)1 << 52)) ? 52 : 64;
  if (fin != 1 && fin != 2 && fin != 4 && fin != 8) return -40;
  if (q >= ((uint64_t)1 << 61)) return -41;
  if (y >= q) return -42;
  if ((u128)fin * q >= ((u128)1 << bit_shift)) return -43;
  const uint64_t yb = (uint64_t)(((u128)y << bit_shift) / q);
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t x = oc_small_mod(a[i], q, fin);
    const uint64_t hi = (uint64_t)(((u128)x * yb) >> bit_shift);
    uint64_t v = x * y - hi * q;
    v = MIN64(v, v - q);
    if (z) { v += oc_small_mod(z[i], q, fin); v = MIN64(v, v - q); }
    r[i] = v;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* ring.hpp                                                                   */
/* ------------------------------------------------------------------------ */

/* poly_mult_mod, ring.hpp:28-43: fwd(1,4) x2, eltwise_mult_mod(.,4), inv(1,1) */
static void poly_mult_row(const tables_t* t, uint64_t* res, const uint64_t* f, const uint64_t* g) {
  const uint64_t n = t->n;
  uint64_t* fh = malloc(n * 8);
  uint64_t* gh = malloc(n * 8);
  memcpy(fh, f, n * 8); memcpy(gh, g, n * 8);
  forward_row(t, fh, 1, 4);
  forward_row(t, gh, 1, 4);
  oc_eltwise_mult_mod(res, fh, gh, n, t->q, 4, 0);
  inverse_row(t, res, 1, 1);
  free(fh); free(gh);
}

int oc_poly_mult_mod(uint64_t n, const uint64_t* moduli, uint32_t nmod, uint64_t* result,
                     const uint64_t* f, const uint64_t* g, uint64_t rows, int threads) {
  for (uint32_t i = 0; i < nmod; ++i)
    if (moduli[i] >= ((uint64_t)1 << 61)) return -50; /* ring.hpp:34-36 */
  return run_batch(n, moduli, nmod, 0, result, f, g, rows, 1, 1, 2, threads);
}

/* naive_negacyclic, ring.hpp:56-75 */
int oc_naive_negacyclic(uint64_t n, uint64_t q, const uint64_t* f, const uint64_t* g, uint64_t* c) {
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t plus = 0, minus = 0;
    for (uint64_t j = 0; j <= i; ++j) plus = (plus + mulmod_full(f[j], g[i - j], q)) % q;
    for (uint64_t j = i + 1; j < n; ++j) minus = (minus + mulmod_full(f[j], g[n + i - j], q)) % q;
    c[i] = (plus + q - minus) % q;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* std::mt19937_64 (the engine bench.hpp:126-131 and tests/test_util.hpp:38-53
 * seed inputs with), restated from its published definition (Matsumoto &
 * Nishimura 64-bit MT: n=312, m=156, r=31) so Python and C produce the same
 * streams as the reference.                                                  */
/* ------------------------------------------------------------------------ */
void oc_mt19937_64_fill(uint64_t seed, uint64_t* out, uint64_t count, uint64_t bound) {
  enum { NN = 312, MM = 156 };
  static const uint64_t MATRIX_A = 0xB5026F5AA96619E9ULL, UM = 0xFFFFFFFF80000000ULL,
                        LM = 0x7FFFFFFFULL;
  uint64_t mt[NN];
  int mti;
  mt[0] = seed;
  for (mti = 1; mti < NN; ++mti)
    mt[mti] = 6364136223846793005ULL * (mt[mti - 1] ^ (mt[mti - 1] >> 62)) + (uint64_t)mti;
  for (uint64_t c = 0; c < count; ++c) {
    if (mti >= NN) {
      int i;
      uint64_t x;
      for (i = 0; i < NN - MM; ++i) {
        x = (mt[i] & UM) | (mt[i + 1] & LM);
        mt[i] = mt[i + MM] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
      }
      for (; i < NN - 1; ++i) {
        x = (mt[i] & UM) | (mt[i + 1] & LM);
        mt[i] = mt[i + (MM - NN)] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
      }
      x = (mt[NN - 1] & UM) | (mt[0] & LM);
      mt[NN - 1] = mt[MM - 1] ^ (x >> 1) ^ ((x & 1ULL) ? MATRIX_A : 0ULL);
      mti = 0;
    }
    uint64_t x = mt[mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    out[c] = bound ? x % bound : x;
  }
}
