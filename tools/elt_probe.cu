// Microbenchmark: EltwiseMultMod (cfg2: 2^20 x 60-bit) launch shapes. 16
// back-to-back calls on rotating buffer sets (384 MiB > L2) captured in one
// CUDA graph, with programmatic dependent launch, for several (CTAs per SM,
// chunks per thread) shapes of the same kernel body as eltwise_kernels.cuh.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2103_16400_b200/csrc -o tools/elt_probe tools/elt_probe.cu
#include <cstdio>
#include <vector>

#include "eltwise_kernels.cuh"

using namespace nk;

template <int KU, int MINB, bool EARLY>
__global__ void __launch_bounds__(256, MINB) kern(uint64_t* __restrict__ r, const uint64_t* __restrict__ a,
                                                  const uint64_t* __restrict__ b, uint64_t total, MultConst c) {
  if (!EARLY) pdl_enter();
  const uint64_t chunks = total / 4;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < chunks;
       i0 += KU * stride) {
    WordVec<4> x[KU], y[KU];
    if (EARLY) asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < chunks) {
        x[u] = ld_stream<4>(a + i * 4);
        y[u] = ld_stream<4>(b + i * 4);
      }
    }
    if (EARLY) asm volatile("griddepcontrol.launch_dependents;" :::);
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < chunks) {
        WordVec<4> o;
#pragma unroll
        for (int k = 0; k < 4; ++k) o.w[k] = mult_barrett<1, true>(x[u].w[k], y[u].w[k], c);
        st_stream<4>(r + i * 4, o);
      }
    }
  }
}


// vector-scalar multiply (eltwise_fma_mod without addend), 60-bit q: one input stream
template <int KU, int MINB>
__global__ void __launch_bounds__(256, MINB) vs_kern(uint64_t* __restrict__ r, const uint64_t* __restrict__ a,
                                                     uint64_t total, FmaConst c) {
  pdl_enter();
  const uint64_t chunks = total / 4;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < chunks;
       i0 += KU * stride) {
    WordVec<4> x[KU];
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < chunks) x[u] = ld_stream<4>(a + i * 4);
    }
#pragma unroll
    for (int u = 0; u < KU; ++u) {
      const uint64_t i = i0 + u * stride;
      if (i < chunks) {
        WordVec<4> o;
#pragma unroll
        for (int k = 0; k < 4; ++k) o.w[k] = fma_one<64, false, 1>(x[u].w[k], 0, c);
        st_stream<4>(r + i * 4, o);
      }
    }
  }
}

template <int KU, int MINB>
void run_vs(const char* name, unsigned grid, std::vector<uint64_t*>& R, std::vector<uint64_t*>& A, uint64_t n,
            FmaConst c) {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  auto k = vs_kern<KU, MINB>;
  const int sets = static_cast<int>(R.size());
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < sets; ++i) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, R[i], (const uint64_t*)A[i], n, c);
  }
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 20;
  cudaEventRecord(e0, st);
  for (int w = 0; w < reps; ++w) cudaGraphLaunch(ge, st);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms * 1e3 / (reps * sets);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0);
  printf("%-34s grid %4u occ %d: %6.2f us/call  %6.0f GB/s\n", name, grid, occ, us, 16.0 * n / us / 1e3);
}

template <class K>
void launch(K kern, unsigned grid, cudaStream_t st, bool pdl, uint64_t* r, const uint64_t* a, const uint64_t* b,
            uint64_t n, MultConst c) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, r, a, b, n, c);
}

template <int KU, int MINB, bool EARLY = false>
void run(const char* name, unsigned grid, bool pdl, std::vector<uint64_t*>& R, std::vector<uint64_t*>& A,
         std::vector<uint64_t*>& B, uint64_t n, MultConst c) {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  auto k = kern<KU, MINB, EARLY>;
  const int sets = static_cast<int>(R.size());
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < sets; ++i) launch(k, grid, st, pdl, R[i], A[i], B[i], n, c);
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 20;
  cudaEventRecord(e0, st);
  for (int w = 0; w < reps; ++w) cudaGraphLaunch(ge, st);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double us = ms * 1e3 / (reps * sets);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0);
  printf("%-34s grid %4u occ %d pdl %d: %6.2f us/call  %6.0f GB/s  %s\n", name, grid, occ, pdl, us, 24.0 * n / us / 1e3,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const uint64_t n = 1 << 20, q = 1152921504606846883ull;
  const int sets = 16;
  std::vector<uint64_t*> R(sets), A(sets), B(sets);
  std::vector<uint64_t> h(n);
  for (uint64_t i = 0; i < n; ++i) h[i] = (i * 0x9E3779B97F4A7C15ull) % q;
  for (int i = 0; i < sets; ++i) {
    cudaMalloc(&R[i], n * 8);
    cudaMalloc(&A[i], n * 8);
    cudaMalloc(&B[i], n * 8);
    cudaMemcpy(A[i], h.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(B[i], h.data(), n * 8, cudaMemcpyHostToDevice);
  }
  // barrett for q = 2^60 - 93: floor(2^(63+61)/q) (bits = 60 -> L = 63 + 60)
  const unsigned __int128 num = (unsigned __int128)1 << 123;
  MultConst c{q, 2 * q, (uint64_t)(num / q), 59, 1};
  const unsigned __int128 yb = ((unsigned __int128)123456789 << 64) / q;
  FmaConst fc{q, 123456789, (uint64_t)yb, 1, 64};
  run_vs<2, 1>("vs KU2 (library shape) grid 512", 512, R, A, n, fc);
  run_vs<1, 6>("vs KU1 minb6 grid 1024", 1024, R, A, n, fc);
  run_vs<1, 8>("vs KU1 minb8 grid 1024", 1024, R, A, n, fc);
  run_vs<2, 4>("vs KU2 minb4 grid 512", 512, R, A, n, fc);
  run_vs<2, 6>("vs KU2 minb6 grid 512", 512, R, A, n, fc);
  run_vs<4, 2>("vs KU4 minb2 grid 256", 256, R, A, n, fc);
  run_vs<4, 4>("vs KU4 minb4 grid 256", 256, R, A, n, fc);
  run_vs<2, 1>("vs KU2 grid 592", 592, R, A, n, fc);
  run_vs<1, 4>("vs KU1 minb4 grid 1024", 1024, R, A, n, fc);
  return 0;
}
