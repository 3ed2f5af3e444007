// Element-wise launchers (eltwise_kernels.cuh): vector width from the
// pointers' alignment, grid from the kernel's resident CTAs per SM,
// programmatic stream serialisation. Argument checks live in capi.cu.
#include <cuda_runtime.h>

#include <initializer_list>
#include <mutex>
#include <unordered_map>

#include "eltwise_kernels.cuh"
#include "runtime.hpp"

namespace nk::rt {
namespace {

// Resident CTAs per SM of an element-wise kernel (occupancy API, cached per
// kernel and device).
int resident_ctas(const void* kern, int block) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto& c = cache[dev & 63];
  auto it = c.find(kern);
  if (it != c.end()) return it->second;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, block, 0) != cudaSuccess || n < 1) n = 1;
  c[kern] = n;
  return n;
}

unsigned eltwise_grid(uint64_t work, const void* kern, int ku = kU) {
  // work = vector chunks; each thread takes ku chunks per sweep; up to two
  // waves of resident CTAs, grid-stride beyond
  const uint64_t per = 256ull * ku;
  uint64_t g = (work + per - 1) / per;
  const uint64_t cap = 2ull * sm_count() * resident_ctas(kern, 256);
  return static_cast<unsigned>(g < 1 ? 1 : (g > cap ? cap : g));
}

// widest vector access all pointers allow (32 / 16 / 8 bytes)
int vec_of(std::initializer_list<const void*> ptrs) {
  uintptr_t x = 0;
  for (const void* p : ptrs) x |= reinterpret_cast<uintptr_t>(p);
  return (x & 31) == 0 ? 4 : ((x & 15) == 0 ? 2 : 1);
}

// launch with programmatic stream serialisation (the kernels call
// griddepcontrol.wait before touching memory, nk::pdl_enter); grid sized for
// `work` vector chunks at ku chunks per thread
template <class... KArgs, class... Args>
int launch_pdl(const char* what, void (*kern)(KArgs...), uint64_t work, int ku, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(eltwise_grid(work, reinterpret_cast<const void*>(kern), ku));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  launches++;
  if (e != cudaSuccess) return cuda_fail(e, what);
  return 0;
}

template <int FIN, bool LOOSE, bool BATCHED>
int launch_mult_t(uint64_t* r, const uint64_t* a, const uint64_t* b, uint64_t total, uint32_t logn,
                  const MultConst& c0, const MultConst* consts, uint32_t nlimbs, cudaStream_t st) {
  const int vec = vec_of({r, a, b});
#define NK_MV(V)                                                                                              \
  return launch_pdl("eltwise_mult_kernel launch", eltwise_mult_kernel<FIN, LOOSE, BATCHED, V>, total / V + 1, \
                    kU, st, r, a, b, total, logn, c0, consts, nlimbs)
  if (vec == 4) NK_MV(4);
  if (vec == 2) NK_MV(2);
  NK_MV(1);
#undef NK_MV
}

}  // namespace

int launch_mult(uint64_t* r, const uint64_t* a, const uint64_t* b, uint64_t total, uint32_t logn,
                const MultConst& c0, const MultConst* consts, uint32_t nlimbs, int fin, bool loose,
                cudaStream_t st) {
  const bool batched = consts != nullptr;
#define NK_M(F, S, B) return launch_mult_t<F, S, B>(r, a, b, total, logn, c0, consts, nlimbs, st)
#define NK_M2(F)                                     \
  if (loose) {                                       \
    if (batched) NK_M(F, true, true);                \
    NK_M(F, true, false);                            \
  }                                                  \
  if (batched) NK_M(F, false, true);                 \
  NK_M(F, false, false)
  switch (fin) {
    case 1: NK_M2(1);
    case 2: NK_M2(2);
    default: NK_M2(4);
  }
#undef NK_M2
#undef NK_M
}

int launch_mult_float(uint64_t* r, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t q, int fin,
                      cudaStream_t st) {
  LimbConstDev c{};
  c.q = q;
  c.q_d = static_cast<double>(q);
  c.qinv = 1.0 / static_cast<double>(q);
  c.q_bias = static_cast<double>(q) + 4503599627370496.0;
  const int vec = vec_of({r, a, b});
#define NK_MFV(F, V) \
  return launch_pdl("eltwise_mult_float_kernel launch", eltwise_mult_float_kernel<F, V>, n / V + 1, 1, st, r, a, b, n, c)
#define NK_MF(F)                 \
  if (vec == 4) NK_MFV(F, 4);    \
  if (vec == 2) NK_MFV(F, 2);    \
  NK_MFV(F, 1)
  switch (fin) {
    case 1: NK_MF(1);
    case 2: NK_MF(2);
    default: NK_MF(4);
  }
#undef NK_MF
#undef NK_MFV
}

int launch_fma(uint64_t* r, const uint64_t* a, const uint64_t* z, uint64_t n, const FmaConst& c, cudaStream_t st) {
  const int vec = z ? vec_of({r, a, z}) : vec_of({r, a});
#define NK_FMAV(BS, Z, F, V)                                                                                  \
  return launch_pdl("eltwise_fma_kernel launch", eltwise_fma_kernel<BS, Z, F, V>, n / V + 1, fma_ku(Z), st, r, \
                    a, z, n, c)
#define NK_FMA(BS, Z, F)             \
  if (vec == 4) NK_FMAV(BS, Z, F, 4); \
  if (vec == 2) NK_FMAV(BS, Z, F, 2); \
  NK_FMAV(BS, Z, F, 1)
#define NK_FMA_F(BS, Z)      \
  switch (c.fin) {           \
    case 1: NK_FMA(BS, Z, 1); \
    case 2: NK_FMA(BS, Z, 2); \
    case 4: NK_FMA(BS, Z, 4); \
    default: NK_FMA(BS, Z, 8); \
  }
  if (c.bs == 52) {
    if (z) { NK_FMA_F(52, true) }
    NK_FMA_F(52, false)
  }
  if (z) { NK_FMA_F(64, true) }
  NK_FMA_F(64, false)
#undef NK_FMA_F
#undef NK_FMA
#undef NK_FMAV
}

int launch_add(uint64_t* r, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t q, cudaStream_t st) {
  const int vec = vec_of({r, a, b});
  if (vec == 4) return launch_pdl("eltwise_add_kernel launch", eltwise_add_kernel<4>, n / 4 + 1, 1, st, r, a, b, n, q);
  if (vec == 2) return launch_pdl("eltwise_add_kernel launch", eltwise_add_kernel<2>, n / 2 + 1, 1, st, r, a, b, n, q);
  return launch_pdl("eltwise_add_kernel launch", eltwise_add_kernel<1>, n, 1, st, r, a, b, n, q);
}

int launch_neg(uint64_t* r, const uint64_t* a, uint64_t n, uint64_t q, cudaStream_t st) {
  const int vec = vec_of({r, a});
  if (vec == 4) return launch_pdl("eltwise_neg_kernel launch", eltwise_neg_kernel<4>, n / 4 + 1, 1, st, r, a, n, q);
  if (vec == 2) return launch_pdl("eltwise_neg_kernel launch", eltwise_neg_kernel<2>, n / 2 + 1, 1, st, r, a, n, q);
  return launch_pdl("eltwise_neg_kernel launch", eltwise_neg_kernel<1>, n, 1, st, r, a, n, q);
}

}  // namespace nk::rt
