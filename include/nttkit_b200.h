/*
 * nttkit_b200 — C-ABI drop-in for the polynomial-arithmetic hot path of Intel
 * HEXL (arXiv 2103.16400) as restated by nttkit (/root/reference/proj/), run on
 * B200 (sm_100a) kernels.
 *
 * Plain C types only: pointers, sizes, a CUDA stream as `void*` (a
 * cudaStream_t; NULL = the legacy default stream). Every entry point returns 0
 * on success and a negative NK_ERR_* code otherwise; nk_last_error() gives the
 * message (thread-local), which is the reference's std::invalid_argument text
 * for argument errors.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj/):
 *   nk_plan_create          NttTables(n, Modulus)                 include/nttkit/ntt.hpp:210
 *                           NttTables(n, Modulus, root)           include/nttkit/ntt.hpp:212-213
 *                           NttTables(n, m, optional root, bs)    include/nttkit/ntt.hpp:217-247
 *                           (HEXL: NTT(degree, q[, root])         PAPER.md:468,476)
 *                           — one plan holds the tables of `nlimbs` RNS moduli.
 *   nk_ntt_forward[_host]   NttTables::forward(result, operand, in, out)  ntt.hpp:268-285
 *                           (HEXL: NTT::ComputeForward            PAPER.md:485-486)
 *   nk_ntt_inverse[_host]   NttTables::inverse(result, operand, in, out)  ntt.hpp:289-306
 *                           (HEXL: NTT::ComputeInverse            PAPER.md:495-496)
 *   nk_eltwise_mult_mod[_host]  eltwise_mult_mod(r, a, b, Modulus, f)     eltwise.hpp:180-188
 *   nk_eltwise_mult_mod_int[_host]    eltwise_mult_mod_int            eltwise.hpp:137-154
 *   nk_eltwise_mult_mod_float[_host]  eltwise_mult_mod_float          eltwise.hpp:158-175
 *                           (HEXL: EltwiseMultMod                 PAPER.md:542-544)
 *   nk_eltwise_fma_mod[_host]   eltwise_fma_mod(r, a, y, z?, Modulus, f)  eltwise.hpp:263-271
 *                           and eltwise_fma_mod<B>                eltwise.hpp:231-259
 *                           (HEXL: EltwiseFMAMod, z == NULL is the vector-scalar
 *                            multiply                             PAPER.md:521,527-529)
 *   nk_eltwise_add_mod[_host]  eltwise_add_mod                    eltwise.hpp:47-57
 *   nk_eltwise_neg_mod[_host]  eltwise_neg_mod                    eltwise.hpp:60-70
 *   nk_poly_mult_mod[_host] poly_mult_mod(result, f, g, tables)   ring.hpp:28-43
 *   nk_modulus              Modulus(q)                            modarith.hpp:106-129
 *   nk_minimal_primitive_root  minimal_primitive_root             ntt.hpp:172-197
 *   nk_precompute_factor    precompute_factor<B>                  modarith.hpp:176-183
 *   nk_harvey_butterflies   harvey_forward/inverse_butterfly<B>   ntt.hpp:137-166
 *   nk_tables_host          NttTables table accessors             ntt.hpp:249-261
 *
 * Batched layout (device entry points): `npolys * nlimbs` contiguous rows of n
 * uint64 words, polynomial-major: row r = poly * nlimbs + l holds limb
 * (limb0 + l) of the plan. A single-polynomial reference call is
 * npolys = nlimbs = 1. result and operand must be identical (in place) or
 * disjoint (ntt.hpp:267-268); partial overlap is NK_ERR_OVERLAP.
 *
 * Device entry points are asynchronous on `stream`. *_host entry points take
 * host buffers and block until the result is back in host memory, like the
 * reference calls.
 */
#ifndef NTTKIT_B200_H
#define NTTKIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  NK_OK = 0,
  NK_ERR_MODULUS = -1,          /* "Modulus: value must be a prime in [3, 2^62)"            modarith.hpp:109-111 */
  NK_ERR_N = -2,                /* "NttTables: n must be a power of two in [2, 2^20]"         ntt.hpp:219-221 */
  NK_ERR_Q_MOD_2N = -3,         /* "NttTables: q must satisfy q == 1 (mod 2n)"                ntt.hpp:223-225 */
  NK_ERR_BIT_SHIFT = -4,        /* "NttTables: accumulator width must be 52 or 64"            ntt.hpp:226-228 */
  NK_ERR_BIT_SHIFT_52 = -5,     /* "NttTables: 52-bit accumulator requires 4q < 2^52"         ntt.hpp:229-231 */
  NK_ERR_ROOT = -6,             /* "NttTables: root is not a primitive 2n'th root of unity"   ntt.hpp:232-236 */
  NK_ERR_FWD_IN_FACTOR = -7,    /* "forward: input_mod_factor must be 1, 2 or 4"              ntt.hpp:270-272 */
  NK_ERR_FWD_OUT_FACTOR = -8,   /* "forward: output_mod_factor must be 1 or 4"                ntt.hpp:273-275 */
  NK_ERR_INV_IN_FACTOR = -9,    /* "inverse: input_mod_factor must be 1 or 2"                 ntt.hpp:291-293 */
  NK_ERR_INV_OUT_FACTOR = -10,  /* "inverse: output_mod_factor must be 1 or 2"                ntt.hpp:294-296 */
  NK_ERR_LENGTH = -11,          /* "transform: buffer length must equal n" / "eltwise: operand lengths must match"
                                   ntt.hpp:329-331, eltwise.hpp:26-30, ring.hpp:31-33 */
  NK_ERR_MULT_FACTOR = -12,     /* "eltwise_mult_mod: input_mod_factor must be 1, 2 or 4"     eltwise.hpp:141-143,162-164 */
  NK_ERR_MULT_INT_RANGE = -13,  /* "eltwise_mult_mod_int: requires input_mod_factor*q < 2^63" eltwise.hpp:144-146 */
  NK_ERR_MULT_FLOAT_RANGE = -14,/* "eltwise_mult_mod_float: requires q < 2^50"                eltwise.hpp:165-167 */
  NK_ERR_FMA_FACTOR = -15,      /* "eltwise_fma_mod: input_mod_factor must be 1, 2, 4 or 8"   eltwise.hpp:239-242 */
  NK_ERR_FMA_MODULUS = -16,     /* "eltwise_fma_mod: requires q < 2^61"                       eltwise.hpp:243-245 */
  NK_ERR_FMA_SCALAR = -17,      /* "eltwise_fma_mod: scalar must be < q"                      eltwise.hpp:246-248 */
  NK_ERR_FMA_WIDTH = -18,       /* "eltwise_fma_mod: requires input_mod_factor*q < 2^BitShift" eltwise.hpp:249-251 */
  NK_ERR_POLY_MODULUS = -19,    /* "poly_mult_mod: requires q < 2^61"                         ring.hpp:34-36 */
  NK_ERR_OVERLAP = -20,         /* result/operand partially overlap (ntt.hpp:267-268 contract) */
  NK_ERR_LIMB = -21,            /* limb range outside the plan */
  NK_ERR_NULL = -22,            /* NULL pointer where a buffer is required */
  NK_ERR_FACTOR_OPERAND = -23,  /* "precompute_factor: operand must be < q"                   modarith.hpp:179 */
  NK_ERR_BETA = -24,            /* "precompute_factor: requires q < beta/4"                   modarith.hpp:180-181 */
  NK_ERR_RANGE = -25,           /* "harvey_*_butterfly: inputs must be < 4q / < 2q"           ntt.hpp:144,161 */
  NK_ERR_CUDA = -100            /* CUDA runtime error; message has the CUDA error string */
};

typedef struct nk_plan nk_plan;

/* ---------------- host-only (no GPU needed) ---------------- */
const char* nk_last_error(void);
const char* nk_version(void);
/* Modulus(q): bits = bit_width(q), barrett = floor(2^(63+bits)/q). */
int nk_modulus(uint64_t q, uint32_t* bits, uint64_t* barrett_factor);
/* Smallest primitive `order`-th root of unity mod q (order a power of two dividing q-1). */
int nk_minimal_primitive_root(uint64_t order, uint64_t q, uint64_t* root);
/* precompute_factor<bit_shift>(w, Modulus(q)).precon = floor(w 2^bit_shift / q)
 * (modarith.hpp:176-183). Host-only. */
int nk_precompute_factor(uint64_t w, uint64_t q, int bit_shift, uint64_t* precon);
/* harvey_forward_butterfly / harvey_inverse_butterfly (ntt.hpp:137-166) on n
 * host element pairs, run on the GPU in the reference's integer arithmetic:
 * (x0, x1) -> (y0, y1) with the factor (w, precon) of width bit_shift. Inputs
 * must be < 4q (forward) / < 2q (inverse), checked (the reference's checked
 * build aborts, ntt.hpp:144,161). Blocking. */
int nk_harvey_butterflies(int fwd, uint64_t q, int bit_shift, uint64_t w, uint64_t precon,
                          const uint64_t* x0, const uint64_t* x1, uint64_t n, uint64_t* y0,
                          uint64_t* y1, int device);
/* Host precompute exactly as NttTables: root = NULL selects the minimal root (an explicit
 * *root is validated like std::optional<uint64_t> root, ntt.hpp:232-237), bit_shift = 0 selects
 * 52 iff 4q < 2^52. Any output pointer may be NULL; arrays hold n words. */
int nk_tables_host(uint64_t n, uint64_t q, const uint64_t* root, int bit_shift, uint64_t* psi,
                   uint64_t* root_powers_rev, uint64_t* root_precons_rev,
                   uint64_t* inv_root_powers_rev, uint64_t* inv_root_precons_rev,
                   uint64_t* inv_n, uint64_t* inv_n_precon, int* bit_shift_out);

/* ---------------- plans (device tables) ---------------- */
/* roots: NULL selects each limb's minimal root; otherwise nlimbs explicit roots, each
 * validated as NttTables(n, m, root) does (0 is rejected, ntt.hpp:234).
 * bit_shift: 0 = automatic per limb, else 52 or 64 for every limb. */
int nk_plan_create(nk_plan** plan, int device, uint64_t n, const uint64_t* moduli,
                   const uint64_t* roots, uint32_t nlimbs, int bit_shift);
void nk_plan_destroy(nk_plan* plan);
int nk_plan_info(const nk_plan* plan, uint32_t limb, uint64_t* n, uint64_t* q, uint64_t* psi,
                 int* bit_shift, uint32_t* nlimbs);

/* ---------------- device-pointer entry points (async on stream) ---------------- */
int nk_ntt_forward(const nk_plan* plan, uint64_t* d_result, const uint64_t* d_operand,
                   uint32_t limb0, uint32_t nlimbs, uint32_t npolys,
                   uint64_t input_mod_factor, uint64_t output_mod_factor, void* stream);
int nk_ntt_inverse(const nk_plan* plan, uint64_t* d_result, const uint64_t* d_operand,
                   uint32_t limb0, uint32_t nlimbs, uint32_t npolys,
                   uint64_t input_mod_factor, uint64_t output_mod_factor, void* stream);
/* Dyadic product of rows under each row's limb modulus (eltwise_mult_mod per row). */
int nk_plan_eltwise_mult_mod(const nk_plan* plan, uint64_t* d_result, const uint64_t* d_a,
                             const uint64_t* d_b, uint32_t limb0, uint32_t nlimbs,
                             uint32_t npolys, uint64_t input_mod_factor, void* stream);
/* poly_mult_mod over npolys*nlimbs row pairs: the canonical result of fwd(1,4) x2, mult(4),
 * inv(1,1) (ring.hpp:39-43). One kernel for N = 2^10 .. 2^14 when the limbs share one
 * accumulator width and q < 2^60 (2^50 at N = 2^14), else that sequence of launches. */
int nk_poly_mult_mod(const nk_plan* plan, uint64_t* d_result, const uint64_t* d_f,
                     const uint64_t* d_g, uint32_t limb0, uint32_t nlimbs, uint32_t npolys,
                     void* stream);

/* eltwise_mult_mod picks the path like the reference (eltwise.hpp:180-188): FP64
 * (DFMA) for q < 2^50, integer Barrett otherwise; _int / _float force one path
 * with that path's checks (eltwise.hpp:137-154 / 158-175). Results are identical. */
int nk_eltwise_mult_mod(uint64_t* d_result, const uint64_t* d_a, const uint64_t* d_b,
                        uint64_t n, uint64_t q, uint64_t input_mod_factor, void* stream);
int nk_eltwise_mult_mod_int(uint64_t* d_result, const uint64_t* d_a, const uint64_t* d_b,
                            uint64_t n, uint64_t q, uint64_t input_mod_factor, void* stream);
int nk_eltwise_mult_mod_float(uint64_t* d_result, const uint64_t* d_a, const uint64_t* d_b,
                              uint64_t n, uint64_t q, uint64_t input_mod_factor, void* stream);
/* d_z may be NULL (vector-scalar multiply). bit_shift: 0 = automatic, 52 or 64. */
int nk_eltwise_fma_mod(uint64_t* d_result, const uint64_t* d_a, uint64_t y, const uint64_t* d_z,
                       uint64_t n, uint64_t q, uint64_t input_mod_factor, int bit_shift,
                       void* stream);
int nk_eltwise_add_mod(uint64_t* d_result, const uint64_t* d_a, const uint64_t* d_b, uint64_t n,
                       uint64_t q, void* stream);
int nk_eltwise_neg_mod(uint64_t* d_result, const uint64_t* d_a, uint64_t n, uint64_t q,
                       void* stream);

/* ---------------- host-buffer entry points (blocking, reference semantics) ----------------
 * Copy host -> device, run, copy device -> host on the plan's device. Pinned host
 * memory gives full PCIe bandwidth; pageable memory works too. `length` is the
 * number of words in each buffer and must equal npolys*nlimbs*n (NK_ERR_LENGTH). */
int nk_ntt_forward_host(const nk_plan* plan, uint64_t* result, const uint64_t* operand,
                        uint64_t length, uint32_t limb0, uint32_t nlimbs, uint32_t npolys,
                        uint64_t input_mod_factor, uint64_t output_mod_factor, void* stream);
int nk_ntt_inverse_host(const nk_plan* plan, uint64_t* result, const uint64_t* operand,
                        uint64_t length, uint32_t limb0, uint32_t nlimbs, uint32_t npolys,
                        uint64_t input_mod_factor, uint64_t output_mod_factor, void* stream);
int nk_poly_mult_mod_host(const nk_plan* plan, uint64_t* result, const uint64_t* f,
                          const uint64_t* g, uint64_t length, uint32_t limb0, uint32_t nlimbs,
                          uint32_t npolys, void* stream);
int nk_eltwise_add_mod_host(uint64_t* result, const uint64_t* a, const uint64_t* b, uint64_t n,
                            uint64_t q, int device, void* stream);
int nk_eltwise_neg_mod_host(uint64_t* result, const uint64_t* a, uint64_t n, uint64_t q, int device,
                            void* stream);
int nk_eltwise_mult_mod_host(uint64_t* result, const uint64_t* a, const uint64_t* b, uint64_t n,
                             uint64_t q, uint64_t input_mod_factor, int device, void* stream);
int nk_eltwise_mult_mod_int_host(uint64_t* result, const uint64_t* a, const uint64_t* b, uint64_t n,
                                 uint64_t q, uint64_t input_mod_factor, int device, void* stream);
int nk_eltwise_mult_mod_float_host(uint64_t* result, const uint64_t* a, const uint64_t* b, uint64_t n,
                                   uint64_t q, uint64_t input_mod_factor, int device, void* stream);
int nk_eltwise_fma_mod_host(uint64_t* result, const uint64_t* a, uint64_t y, const uint64_t* z,
                            uint64_t n, uint64_t q, uint64_t input_mod_factor, int bit_shift,
                            int device, void* stream);

/* Number of kernels the library has launched in this process (for the bench's
 * gpu_launches claim). */
uint64_t nk_launch_count(void);
/* Debug aid: device buffer that a library built with -DNK_DBG_TIMELINE fills
 * with per-warp phase timestamps of the CTA-pair forward kernel
 * (tools/timeline.py; 296 x 8 x 32 x 16 words). NULL (the default) disables it;
 * the normal build ignores it. Per calling thread. */
void nk_debug_dump_to(uint64_t* d_buf);
/* Testing aid: when on, every beta = 2^52 transform uses the exact lazy
 * arithmetic (the reference's representatives) even where only the canonical
 * result is observable, so the tests can cover both arithmetic paths. Off by
 * default; applies to calls made by the calling thread only. */
void nk_debug_exact_only(int on);
/* Testing aid: which kernel transforms 16384-word blocks. -1 (default) = 2,
 * 0 = the CTA-pair kernel, 1 = the group-exchange kernel, 2 = two streams per
 * thread (ntt_str14 / ntt_stri14); 3 = defaults, but the single-kernel
 * poly_mult_mod by the group-exchange poly_mul14 instead of poly_str14;
 * 6 = defaults, but batches of 2^11..2^13-word rows smaller than the SM count
 * take the plain block kernel instead of the latency kernel (ntt_block_lat).
 * Applies to calls made by the calling thread only. */
void nk_debug_block_kernel(int which);
/* Testing aid: one butterfly per element pair (x0[i], x1[i]) -> (y0[i], y1[i])
 * in an arithmetic policy of the kernels (0 = ArithInt<64>, 1 = ArithInt<52>,
 * 2 = Arith52P, 3 = Arith52S with int64 words in and out, 4 = ArithIntL,
 * 5 / 6 = Arith52S (int64 words) / ArithIntL stage without its conditional
 * subtraction),
 * twiddle w with its Shoup quotient for the policy's width;
 * fwd != 0: the forward (CT) butterfly, else the inverse (GS). Device buffers. */
int nk_debug_butterflies(int policy, int fwd, uint64_t q, uint64_t w, const uint64_t* d_x0,
                         const uint64_t* d_x1, uint64_t n, uint64_t* d_y0, uint64_t* d_y1);

#ifdef __cplusplus
}
#endif
#endif
