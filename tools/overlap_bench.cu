// Microbenchmark: do the FP64 pipe and the shared-memory (LSU) path overlap
// on one SM, (a) from different warps, (b) inside one warp's instruction
// stream? One 512-thread CTA per SM (the transform kernels' shape).
//   mode 0: all 16 warps DFMA            mode 1: all 16 warps LDS/STS
//   mode 2: warps 0-7 DFMA, 8-15 idle    mode 3: warps 0-7 DFMA, 8-15 LDS/STS
//   mode 4: every warp: K DFMA per LDS+STS pair, interleaved in program order
//   mode 5: every warp: a burst of 32 STS + 32 LDS, then the same DFMA count (phases)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/overlap_bench tools/overlap_bench.cu
#include <cstdint>
#include <cstdio>

#define CH 8

__device__ __forceinline__ void dfma8(double (&d)[CH], double e) {
#pragma unroll
  for (int i = 0; i < CH; ++i) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(e));
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) kern(uint64_t* out, long long* clk, int iters) {
  extern __shared__ uint64_t sm[];
  const uint32_t t = threadIdx.x, w = t >> 5;
  double d[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) d[i] = 1.0 + t * 1e-3 + i;
  const double e = 1.0000001;
  uint64_t x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = t + i;
  uint64_t* mine = sm + t;  // conflict-free 8-byte accesses, stride 512 words between slots
  __syncthreads();
  const long long c0 = clock64();
  const bool fp = (MODE == 0) || ((MODE == 2 || MODE == 3) && w < 8);
  const bool mem = (MODE == 1) || (MODE == 3 && w >= 8);
  if (MODE <= 3) {
    if (fp)
      for (int it = 0; it < iters; ++it) {
        dfma8(d, e);
        dfma8(d, e);
        dfma8(d, e);
        dfma8(d, e);
      }
    if (mem)
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("st.shared.u64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(mine + 512 * i)), "l"(x[i]) : "memory");
#pragma unroll
        for (int i = 0; i < 8; ++i) asm volatile("ld.shared.u64 %0, [%1];" : "=l"(x[i]) : "r"((uint32_t)__cvta_generic_to_shared(mine + 512 * ((i + 1) & 7))) : "memory");
      }
  } else if (MODE == 4) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        asm volatile("st.shared.u64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(mine + 512 * i)), "l"(x[i]) : "memory");
        dfma8(d, e);
        dfma8(d, e);
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(x[i]) : "r"((uint32_t)__cvta_generic_to_shared(mine + 512 * ((i + 1) & 7))) : "memory");
        dfma8(d, e);
        dfma8(d, e);
      }
    }
  } else {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("st.shared.u64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(mine + 512 * i)), "l"(x[i]) : "memory");
      __syncthreads();
#pragma unroll
      for (int i = 0; i < 8; ++i) asm volatile("ld.shared.u64 %0, [%1];" : "=l"(x[i]) : "r"((uint32_t)__cvta_generic_to_shared(mine + 512 * ((i + 1) & 7))) : "memory");
#pragma unroll
      for (int r = 0; r < 32; ++r) dfma8(d, e);
      __syncthreads();
    }
  }
  const long long c1 = clock64();
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += (uint64_t)d[i];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 0x12345) out[t] = s;
  if ((t & 31) == 0 && blockIdx.x == 0) clk[w] = c1 - c0;
}

template <int MODE>
void run(const char* name, int iters, double dfma_per_thread_iter, double smem_ops_per_thread_iter) {
  uint64_t* out;
  long long* clk;
  cudaMalloc(&out, 4096);
  cudaMalloc(&clk, 16 * 8);
  cudaMemset(clk, 0, 128);
  cudaFuncSetAttribute(kern<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  kern<MODE><<<148, 512, 64 * 1024>>>(out, clk, iters);
  kern<MODE><<<148, 512, 64 * 1024>>>(out, clk, iters);
  cudaDeviceSynchronize();
  long long h[16];
  cudaMemcpy(h, clk, 128, cudaMemcpyDeviceToHost);
  long long fpc = h[0], memc = h[15];
  printf("%-44s warp0 %9lld clk  warp15 %9lld clk", name, fpc, memc);
  if (dfma_per_thread_iter > 0) printf("  | DFMA %.1f lanes/clk/SM", dfma_per_thread_iter * iters * ((MODE == 2 || MODE == 3) ? 256 : 512) / fpc);
  if (smem_ops_per_thread_iter > 0)
    printf("  | smem %.1f B/clk/SM", smem_ops_per_thread_iter * iters * 8.0 * ((MODE == 3) ? 256 : 512) / (MODE == 3 ? memc : fpc));
  printf("\n");
  cudaFree(out);
  cudaFree(clk);
}

int main() {
  const int it = 2000;
  run<0>("0: 16 warps DFMA", it, 32, 0);
  run<1>("1: 16 warps STS+LDS", it, 0, 16);
  run<2>("2: 8 warps DFMA, 8 idle", it, 32, 0);
  run<3>("3: 8 warps DFMA + 8 warps STS+LDS", it, 32, 16);
  run<4>("4: each warp 16 DFMA per STS/LDS, interleaved", it / 4, 8 * 32, 16);
  run<5>("5: each warp 8 STS | 8 LDS | 256 DFMA | (phases)", it / 4, 256, 16);
  return 0;
}
