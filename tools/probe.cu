// Live pipe probes for bench.py's rooflines (measurement tooling, not part of
// the product library): the FP64 pipe rate (independent DFMA chains) and the
// in-register butterfly rate of the transforms' arithmetic policies
// (modmath.cuh) on the box the bench runs on. Built by tools/Makefile into
// tools/libnkprobe.so; bench.py calls it through ctypes.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <type_traits>

#include "modmath.cuh"

using namespace nk;

namespace {

constexpr int kChains = 8;
constexpr int kProbeStages = 4;

__global__ void __launch_bounds__(256) dfma_loop(double* out, int iters) {
  double a[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) a[k] = 1.0 + 1e-3 * (threadIdx.x + k);
  const double m = 0.9999999, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) a[k] = __fma_rn(a[k], m, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += a[k];
  if (s == 12345.0) out[threadIdx.x] = s;
}

// butterflies over V register words, four stages per iteration (spans 1, 2,
// 4, 8), two twiddles: the transforms' inner loop without memory or exchanges.
// The forward reduces x0 on every other stage only, as in the 16384-word
// kernels (modmath.cuh, Arith52S::fwd_skip / ArithIntL::fwd_skip).
template <class Tw>
__device__ __forceinline__ Tw as_tw(ulonglong2 w) {
  if constexpr (std::is_same_v<Tw, uint64_t>) return w.x;  // w only (Arith52S's 8-byte tables)
  else return w;
}

template <class A, int V, bool INV>
__global__ void __launch_bounds__(512, 1) bfly_loop(uint64_t* out, LimbConstDev c, ulonglong2 w0, ulonglong2 w1,
                                                    int iters) {
  uint64_t v[V];
#pragma unroll
  for (int i = 0; i < V; ++i) v[i] = A::load((threadIdx.x * 977u + i * 131u) % 1000003u);
  const typename A::Tw w[2] = {as_tw<typename A::Tw>(w0), as_tw<typename A::Tw>(w1)};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < kProbeStages; ++s) {
      const int h = 1 << s;
#pragma unroll
      for (int i = 0; i < V; ++i) {
        if ((i & h) || h >= V) continue;
        if (INV) A::template inv<false>(v[i], v[i + h], w[(i >> 1) & 1], c);
        else if (A::fwd_skip(false, s)) A::template fwd<true>(v[i], v[i + h], w[(i >> 1) & 1], c);
        else A::template fwd<false>(v[i], v[i + h], w[(i >> 1) & 1], c);
      }
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < V; ++i) s ^= v[i];
  if (s == 0x12345) out[threadIdx.x] = s;
}

uint64_t dbits(double d) {
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
}

int sms(int* n) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  return cudaDeviceGetAttribute(n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess ? 0 : -1;
}

template <class K>
int time_ms(K&& launch, float* ms) {
  launch();  // warm-up (clock ramp, module load)
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

template <class A, bool INV>
int bfly_rate(const LimbConstDev& c, ulonglong2 w0, ulonglong2 w1, double* per_s) {
  int nsm = 0;
  if (sms(&nsm)) return -1;
  uint64_t* out = nullptr;
  if (cudaMalloc(&out, 1 << 16) != cudaSuccess) return -1;
  constexpr int V = 32, kIters = 2048;
  float ms = 0;
  const int rc = time_ms([&] { bfly_loop<A, V, INV><<<nsm, 512>>>(out, c, w0, w1, kIters); }, &ms);
  cudaFree(out);
  if (rc) return rc;
  *per_s = double(nsm) * 512 * kIters * kProbeStages * (V / 2) / (ms * 1e-3);
  return 0;
}

}  // namespace

extern "C" {

// FP64 pipe: DFMA lane-operations per second over the whole GPU
int probe_fp64_rate(double* ops_per_s) {
  int nsm = 0;
  if (sms(&nsm)) return -1;
  double* out = nullptr;
  if (cudaMalloc(&out, 1 << 16) != cudaSuccess) return -1;
  constexpr int kIters = 1 << 15;
  const int grid = nsm * 4;
  float ms = 0;
  const int rc = time_ms([&] { dfma_loop<<<grid, 256>>>(out, kIters); }, &ms);
  cudaFree(out);
  if (rc) return rc;
  *ops_per_s = double(grid) * 256 * kIters * kChains / (ms * 1e-3);
  return 0;
}

// In-register butterflies per second (32 words per thread, one 512-thread CTA
// per SM): policy 0 = Arith52S (q = cfg3's first 50-bit limb), 1 = ArithIntL
// (q = cfg4's first 60-bit limb); inv != 0 for the inverse butterfly.
int probe_bfly_rate(int policy, int inv, double* bfly_per_s) {
  LimbConstDev c{};
  if (policy == 0) {
    const uint64_t q = 1125899904679937ull, w = 184459094098ull;
    const uint64_t wp = static_cast<uint64_t>((static_cast<unsigned __int128>(w) << 52) / q);
    c.q = q;
    c.twoq = 2 * q;
    c.negq = 0 - q;
    c.qq = double(q) / 4503599627370496.0;
    c.twoq_d = double(2 * q);
    c.bs = 52;
    c.q_d = double(q);
    c.qinv = 1.0 / double(q);
    c.q_bias = double(q) + 4503599627370496.0;
    const ulonglong2 w0{dbits(double(w)), dbits(double(wp))}, w1{dbits(double(w + 1)), dbits(double(wp))};
    return inv ? bfly_rate<Arith52S, true>(c, w0, w1, bfly_per_s) : bfly_rate<Arith52S, false>(c, w0, w1, bfly_per_s);
  }
  const uint64_t q = 1152921504606584833ull, w = 18043022392882ull;
  const uint64_t wp = static_cast<uint64_t>((static_cast<unsigned __int128>(w) << 64) / q);
  c.q = q;
  c.twoq = 2 * q;
  c.negq = 0 - q;
  c.fourq = 4 * q;
  c.bs = 64;
  const ulonglong2 w0{w, wp}, w1{w + 1, wp};
  return inv ? bfly_rate<ArithIntL, true>(c, w0, w1, bfly_per_s) : bfly_rate<ArithIntL, false>(c, w0, w1, bfly_per_s);
}

}  // extern "C"
