// Probe: on which SMs do the CTAs of 2- and 4-CTA clusters land (2 CTAs of
// 106 KiB per SM, as ntt_pair14)? Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/place_probe tools/place_probe.cu
#include <cstdio>
#include <cstdint>
template <int C>
__global__ void __launch_bounds__(256, 2) k(int* out, int iters) {
  extern __shared__ char sm[];
  uint32_t smid, rank, cid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(cid));
  if (threadIdx.x == 0) out[blockIdx.x] = smid;
  // keep busy a bit
  volatile double x = threadIdx.x;
  for (int i = 0; i < iters; ++i) x = x * 1.0000001 + 1e-9;
  sm[threadIdx.x] = (char)x;
}
template <int C>
void run() {
  int* d; cudaMalloc(&d, 4096 * 4);
  cudaFuncSetAttribute(k<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 106 * 1024);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(296); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = 106 * 1024;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  int ncl = 0; cudaOccupancyMaxActiveClusters(&ncl, (void*)k<C>, &cfg);
  cudaError_t e = cudaLaunchKernelEx(&cfg, k<C>, d, 100000);
  cudaDeviceSynchronize();
  int h[296]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("cluster %d: maxActiveClusters=%d err=%s\n", C, ncl, cudaGetErrorString(e));
  int same = 0, distinct_sets = 0;
  for (int c = 0; c < 296 / C && c < 12; ++c) {
    printf("  cl%2d:", c);
    for (int r = 0; r < C; ++r) printf(" %3d", h[c * C + r]);
    printf("\n");
  }
  // how many SMs does each cluster span, and do clusters share SM sets
  int span_hist[9] = {};
  for (int c = 0; c < 296 / C; ++c) {
    int u[8], nu = 0;
    for (int r = 0; r < C; ++r) { int s = h[c*C+r], f = 0; for (int i = 0; i < nu; ++i) f |= u[i]==s; if (!f) u[nu++] = s; }
    span_hist[nu]++;
  }
  printf("  span histogram:"); for (int i = 1; i <= C; ++i) printf(" %d:%d", i, span_hist[i]); printf("\n");
  // pairs (cluster 2): partner-set symmetry: for each SM, list the SMs of its CTAs' partners
  if (C == 2) {
    int sym = 0, tot = 0;
    for (int c = 0; c < 148; ++c) {
      int a = h[2*c], b = h[2*c+1];
      // find another cluster spanning the same {a,b}
      for (int d = 0; d < 148; ++d) if (d != c) { int x = h[2*d], y = h[2*d+1]; if ((x==a&&y==b)||(x==b&&y==a)) { sym++; break; } }
      tot++;
    }
    printf("  pairs whose SM set is shared by another pair: %d / %d\n", sym, tot);
  }
}
int main() { run<2>(); run<4>(); return 0; }
