/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the B200 hot path.
 *
 * A plain-C restatement of the reference algorithms (nttkit, the portable
 * restatement of Intel HEXL, arXiv 2103.16400) for the negacyclic NTT and the
 * element-wise modular kernels. Every function cites the reference file:line
 * it follows (paths relative to /root/reference/proj/).
 *
 * Parity is PINNED: the oracle is checked against (1) the known answers of the
 * reference's own tests (tests/test_*.cpp), ported by value, and (2) the
 * reference itself compiled from its headers into oracle/_ref/ (see
 * oracle/Makefile, oracle/ref_shim.cpp) through golden fixtures under
 * tests/golden/ and live cross-checks in tests/test_oracle.py.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. The product path
 * (paper_2103_16400_b200/) never links or calls it.
 *
 * Return codes: 0 on success, negative on argument errors (the reference
 * throws std::invalid_argument at the cited lines).
 */
#ifndef NTTKIT_ORACLE_H
#define NTTKIT_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- scalar arithmetic (modarith.hpp) ---- */
int      oc_is_prime(uint64_t n);
/* bits/barrett factor; returns 0 or -1 for invalid modulus (modarith.hpp:108-115) */
int      oc_modulus(uint64_t q, uint32_t* bits, uint64_t* barrett_factor);
uint64_t oc_barrett_reduce(uint64_t d_hi, uint64_t d_lo, uint64_t q);
uint64_t oc_mul_mod(uint64_t a, uint64_t b, uint64_t q);
uint64_t oc_pow_mod(uint64_t base, uint64_t exp, uint64_t q);
uint64_t oc_inv_mod(uint64_t x, uint64_t q);
uint64_t oc_small_mod(uint64_t x, uint64_t q, uint64_t factor);
uint64_t oc_precompute_factor(uint64_t w, uint64_t q, int bit_shift);
uint64_t oc_bit_reverse(uint64_t i, unsigned log2n);
/* harvey_forward/inverse_butterfly (ntt.hpp:137-166) on n element pairs */
int oc_butterflies(int fwd, uint64_t q, int bs, uint64_t w, const uint64_t* x0, const uint64_t* x1,
                   uint64_t n, uint64_t* y0, uint64_t* y1);

/* ---- tables (ntt.hpp) ---- */
/* minimal primitive `order`-th root; 0 on error (ntt.hpp:172-197) */
uint64_t oc_minimal_primitive_root(uint64_t order, uint64_t q);
/* bit_shift: 0 = auto (ntt.hpp:323-325). root: 0 = minimal root.
 * out arrays (n each) may be NULL. Returns chosen bit shift (52/64) or <0 error. */
int oc_ntt_tables(uint64_t n, uint64_t q, uint64_t root, int bit_shift,
                  uint64_t* psi_out, uint64_t* psi_inv_out,
                  uint64_t* psi_rev, uint64_t* psi_precon_rev,
                  uint64_t* psi_inv_rev, uint64_t* psi_inv_precon_rev,
                  uint64_t* n_inv, uint64_t* n_inv_precon);

/* ---- transforms: batch of `rows` contiguous rows of n, row r uses moduli[r % nmod] ----
 * result may equal operand (in place). threads: 0/1 = single thread. */
int oc_ntt_forward(uint64_t n, const uint64_t* moduli, uint32_t nmod, int bit_shift,
                   uint64_t* result, const uint64_t* operand, uint64_t rows,
                   uint64_t fin, uint64_t fout, int threads);
int oc_ntt_inverse(uint64_t n, const uint64_t* moduli, uint32_t nmod, int bit_shift,
                   uint64_t* result, const uint64_t* operand, uint64_t rows,
                   uint64_t fin, uint64_t fout, int threads);
int oc_ntt_root(uint64_t n, uint64_t q, uint64_t root, int bit_shift, int dir, uint64_t* result,
                const uint64_t* operand, uint64_t fin, uint64_t fout);
int oc_ntt_stages(uint64_t n, uint64_t q, int dir, uint64_t* a, uint64_t fin, int nstages);
/* O(n^2) definitional transform (ntt.hpp:457-508); dir 0 = forward, 1 = inverse */
int oc_reference_ntt(uint64_t n, uint64_t q, uint64_t psi, int dir,
                     const uint64_t* a, uint64_t* out);

/* ---- element-wise (eltwise.hpp) ---- */
int oc_eltwise_add_mod(uint64_t* r, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t q);
int oc_eltwise_neg_mod(uint64_t* r, const uint64_t* a, uint64_t n, uint64_t q);
/* path: 0 = dispatch as the reference (float iff q<2^50), 1 = int, 2 = float */
int oc_eltwise_mult_mod(uint64_t* r, const uint64_t* a, const uint64_t* b, uint64_t n,
                        uint64_t q, uint64_t fin, int path);
/* z may be NULL; bit_shift 0 = auto (eltwise.hpp:263-271) */
int oc_eltwise_fma_mod(uint64_t* r, const uint64_t* a, uint64_t y, const uint64_t* z,
                       uint64_t n, uint64_t q, uint64_t fin, int bit_shift);

/* ---- ring (ring.hpp) ---- */
int oc_poly_mult_mod(uint64_t n, const uint64_t* moduli, uint32_t nmod, uint64_t* result,
                     const uint64_t* f, const uint64_t* g, uint64_t rows, int threads);
int oc_naive_negacyclic(uint64_t n, uint64_t q, const uint64_t* f, const uint64_t* g,
                        uint64_t* out);

/* ---- seeded inputs: std::mt19937_64(seed), eng() % bound (bench.hpp:126-131) ---- */
void oc_mt19937_64_fill(uint64_t seed, uint64_t* out, uint64_t count, uint64_t bound);

#ifdef __cplusplus
}
#endif
#endif
