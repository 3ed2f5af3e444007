// Host-side state and helpers shared by the library's translation units
// (capi.cu: the C-ABI; ntt_inst.cu: one transform policy x direction each;
// eltwise.cu: the element-wise launchers). Nothing here computes: every
// transform and product runs in the sm_100a kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "ntt_kernels.cuh"

namespace nk {
struct MultConst;
struct FmaConst;
struct PolyArgs;
struct PolyBlkArgs;
}  // namespace nk

namespace nk::rt {

// error reporting (nk_last_error is thread-local, like errno)
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define NK_CUDA(call)                                            \
  do {                                                           \
    cudaError_t e_ = (call);                                     \
    if (e_ != cudaSuccess) return ::nk::rt::cuda_fail(e_, #call); \
  } while (0)

// kernels launched by this process (nk_launch_count)
extern std::atomic<uint64_t> launches;

// Testing aids, per calling thread (nk_debug_block_kernel / nk_debug_exact_only /
// nk_debug_dump_to): they change dispatch only for calls made by the thread
// that set them.
extern thread_local int block_kernel;  // -1 auto, 0 CTA pair, 1 group exchange (16384-word blocks; poly_mult_mod: see capi.cu)
extern thread_local bool no_lat;       // small batches take ntt_block instead of ntt_block_lat
extern thread_local bool exact_only;   // beta = 2^52 transforms always take the lazy-exact policy
extern thread_local uint64_t* dbg;     // NK_DBG_TIMELINE builds: per-warp phase stamps

int sm_count();  // of the current device

// Full transform of a.rows rows with arithmetic policy A (dispatch.cuh,
// instantiated per policy and direction in ntt_inst.cu). buf_words: words in
// the input buffer (for the TMA tensor maps).
template <class A, bool FWD>
int run_ntt(NttArgs a, uint64_t buf_words, cudaStream_t st);

// poly_mult_mod of N = 16384 rows in one kernel (poly.cu, ntt_poly.cuh):
// signed FP64 policy, canonical f and g with 16-byte aligned rows.
int run_poly_mul14(const PolyArgs& pa, const uint64_t* f, const uint64_t* g, cudaStream_t st);

// poly_mult_mod of whole rows of N = 2^10 .. 2^13 in one kernel (polyblk.cu,
// ntt_polyblk.cuh): fp64 = the signed FP64 policy (every limb beta = 2^52),
// else the loose integer policy (every limb beta = 2^64, q < 2^60).
int run_poly_block(const PolyBlkArgs& pa, uint64_t rows, bool fp64, cudaStream_t st);

// element-wise launchers (eltwise.cu)
int launch_mult(uint64_t* r, const uint64_t* a, const uint64_t* b, uint64_t total, uint32_t logn,
                const MultConst& c0, const MultConst* consts, uint32_t nlimbs, int fin, bool loose,
                cudaStream_t st);
int launch_mult_float(uint64_t* r, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t q, int fin,
                      cudaStream_t st);
int launch_fma(uint64_t* r, const uint64_t* a, const uint64_t* z, uint64_t n, const FmaConst& c,
               cudaStream_t st);
int launch_add(uint64_t* r, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t q, cudaStream_t st);
int launch_neg(uint64_t* r, const uint64_t* a, uint64_t n, uint64_t q, cudaStream_t st);

}  // namespace nk::rt
