// Microbenchmark: butterflies/clk/SM of the forward Harvey butterfly in the
// arithmetic policies of modmath.cuh, at several words-per-thread (ILP) and
// warps-per-SM (TLP) points. Pure register work: isolates the arithmetic
// ceiling of the NTT kernels from their exchanges and memory traffic.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2103_16400_b200/csrc \
//        -o tools/bfly_bench tools/bfly_bench.cu
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "modmath.cuh"

using namespace nk;

template <class A, int V, int ITERS, bool INV>
__global__ void kern(uint64_t* out, LimbConstDev c, ulonglong2 w0, ulonglong2 w1) {
  uint64_t v[V];
#pragma unroll
  for (int i = 0; i < V; ++i) v[i] = A::load((threadIdx.x * 977u + i * 131u) % 1000003u);
  ulonglong2 w[2] = {w0, w1};
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      const int h = 1 << (s % 3);
#pragma unroll
      for (int i = 0; i < V; ++i) {
        if (i & h) continue;
        if (h >= V) continue;
        if (INV) A::template inv<false>(v[i], v[i + h], w[(i >> 1) & 1], c);
        else A::template fwd<false>(v[i], v[i + h], w[(i >> 1) & 1], c);
      }
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < V; ++i) s ^= v[i];
  if (s == 0x12345) out[threadIdx.x] = s;
}

template <class A, int V, bool INV = false>
void run(const char* name, int threads, int ctas_per_sm, const LimbConstDev& c, ulonglong2 w0, ulonglong2 w1) {
  constexpr int ITERS = 2048;
  uint64_t* out;
  cudaMalloc(&out, 1 << 16);
  const int grid = 148 * ctas_per_sm;
  kern<A, V, ITERS, INV><<<grid, threads>>>(out, c, w0, w1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<A, V, ITERS, INV><<<grid, threads>>>(out, c, w0, w1);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaError_t err = cudaGetLastError();
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bf = double(grid) * threads * ITERS * 3 * (V / 2);
  const double per_s = bf / (ms * 1e-3);
  printf("%-22s %s V=%2d thr=%4d ctas/SM=%d: %8.3f ms  %7.1f Gbfly/s  %5.2f bfly/clk/SM (1965 MHz)%s\n", name, INV ? "inv" : "fwd", V,
         threads, ctas_per_sm, ms, per_s / 1e9, per_s / 148 / 1.965e9, err ? cudaGetErrorString(err) : "");
  cudaFree(out);
}

static uint64_t dbits(double d) {
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
}

int main() {
  const uint64_t q = 1125899904679937ull;  // 50-bit
  LimbConstDev c{};
  c.q = q;
  c.twoq = 2 * q;
  c.negq = 0 - q;
  c.qq = double(q) / 4503599627370496.0;
  c.twoq_d = double(2 * q);
  c.bs = 52;
  const uint64_t w = 184459094098ull;
  const uint64_t wp = (uint64_t)(((unsigned __int128)w << 52) / q);
  ulonglong2 wi{w, wp};
  ulonglong2 wd{dbits(double(w)), dbits(double(wp))};
  ulonglong2 wi2{w + 1, wp}, wd2{dbits(double(w + 1)), wd.y};
  c.q_d = double(q);
  c.qinv = 1.0 / double(q);
  c.q_bias = double(q) + 4503599627370496.0;
  run<Arith52P, 32>("Arith52P", 512, 1, c, wd, wd2);
  run<Arith52P, 32, true>("Arith52P", 512, 1, c, wd, wd2);
  run<Arith52S, 32>("Arith52S", 512, 1, c, wd, wd2);
  run<Arith52S, 32, true>("Arith52S", 512, 1, c, wd, wd2);
  run<Arith52P, 16>("Arith52P", 512, 2, c, wd, wd2);
  run<Arith52S, 16>("Arith52S", 512, 2, c, wd, wd2);
  run<Arith52S, 16, true>("Arith52S", 512, 2, c, wd, wd2);
  return 0;
}
