// Microbenchmark: the register passes of the block kernels (pass14, real
// twiddle tables and index patterns), without exchanges or HBM traffic.
// Separates the compute-phase efficiency from the data movement.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2103_16400_b200/csrc \
//        -o tools/pass_bench tools/pass_bench.cu
#include <cstdio>
#include <cstring>
#include <vector>

#include "ntt_kernels.cuh"

using namespace nk;


// pass14 with twiddles read from a 4096-entry shared-memory table (indices
// masked): what the compute phases would reach if twiddle loads had shared
// memory latency (the access pattern differs, the latency question does not)
template <class A, bool FWD, class PD>
__device__ __forceinline__ void pass14_smem(uint64_t (&v)[32], const ulonglong2* tws, uint64_t xt,
                                            const LimbConstDev& c) {
  constexpr int K = PD::K, R = PD::R, G = PD::G;
  constexpr bool kLow = (PD::LO == 0 && PD::K == 5);
  constexpr bool kShared = (G == 2) && (PD::X >= 0) && (PD::X < PD::LO);
  constexpr int GL = kShared ? 1 : G;
  const uint32_t jhi = static_cast<uint32_t>(xt >> 5) & 511u;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    const int i = FWD ? (K - 1 - s) : s;
    const int b = PD::LO + i;
#pragma unroll
    for (int gl = 0; gl < GL; ++gl) {
      const uint64_t base = (xt + PD::jc(gl, 0)) >> (b + 1);
#pragma unroll
      for (int hi = 0; hi < (R >> (i + 1)); ++hi) {
        const uint32_t idx = kLow ? (low_index(b, hi, 0) + jhi) : static_cast<uint32_t>(base + hi);
        const ulonglong2 w = tws[idx & 4095u];
#pragma unroll
        for (int gg = 0; gg < G / GL; ++gg) {
#pragma unroll
          for (int l = 0; l < (1 << i); ++l) {
            const int g = kShared ? gg : gl;
            const int r0 = (hi << (i + 1)) | l;
            const int r1 = r0 | (1 << i);
            if (FWD) A::template fwd<false>(v[g * R + r0], v[g * R + r1], w, c);
            else A::template inv<false>(v[g * R + r0], v[g * R + r1], w, c);
          }
        }
      }
    }
  }
}

template <class A, bool FWD, int WHICH>
__global__ void __launch_bounds__(256, 2) kern(const ulonglong2* tw, const ulonglong2* twl, LimbConstDev c,
                                               uint32_t nlimbs, uint32_t iters, uint64_t* out) {
  using P1 = typename std::conditional<FWD, PassD<9, 5, -1>, PassD<0, 5, -1>>::type;
  using P2 = PassD<5, 4, 4>;
  using P3 = typename std::conditional<FWD, PassD<0, 5, -1>, PassD<9, 5, -1>>::type;
  const uint32_t t = threadIdx.x, l = t & 31, w = t >> 5, cta = blockIdx.x & 1;
  const uint32_t jt_p2 = (l & 15u) | ((l >> 4) << 9) | (w << 10) | (cta << 13);
  const uint32_t jt_low = (l << 5) | (w << 10) | (cta << 13);
  const uint32_t jt_hi = t | (cta << 8);
  const uint64_t n = 16384;
  uint64_t v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = A::load((t * 977u + i * 131u) % 1000003u);
  for (uint32_t it = 0; it < iters; ++it) {
    const uint32_t limb = (blockIdx.x / 2 + it * 148) % nlimbs;
    const ulonglong2* tl = tw + limb * n;
    const ulonglong2* tll = twl + limb * n + (jt_low >> 5);
    if (WHICH & 1) pass14<A, FWD, P1, false>(v, tl, tll, n, n + (FWD ? jt_hi : jt_low), c);
    if (WHICH & 2) pass14<A, FWD, P2, false>(v, tl, tll, n, n + jt_p2, c);
    if (WHICH & 4) pass14<A, FWD, P3, false>(v, tl, tll, n, n + (FWD ? jt_low : jt_hi), c);
    if (WHICH & 8) {
      extern __shared__ __align__(16) ulonglong2 tws[];
      if (it == 0) {
        for (uint32_t k = t; k < 4096; k += 256) tws[k] = tl[k];
        __syncthreads();
      }
      pass14_smem<A, FWD, P1>(v, tws, n + (FWD ? jt_hi : jt_low), c);
      pass14_smem<A, FWD, P2>(v, tws, n + jt_p2, c);
      pass14_smem<A, FWD, P3>(v, tws, n + (FWD ? jt_low : jt_hi), c);
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s ^= v[i];
  if (s == 0x12345) out[t] = s;
}

static uint64_t dbits(double d) {
  uint64_t u;
  memcpy(&u, &d, 8);
  return u;
}

template <class A, bool FWD, int WHICH>
void run(const char* name, const ulonglong2* tw, const ulonglong2* twl, const LimbConstDev& c, int bfly_per_iter,
         int grid = 296, int smem = 0) {
  // smem > 0: that much dynamic shared memory per CTA, so L1 shrinks to what
  // the real kernels leave it (~44 KiB per SM at two 106 KiB CTAs)
  cudaFuncSetAttribute(kern<A, FWD, WHICH>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  uint64_t* out;
  cudaMalloc(&out, 1 << 16);
  const uint32_t iters = 200;
  kern<A, FWD, WHICH><<<grid, 256, smem>>>(tw, twl, c, 32, 10, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<A, FWD, WHICH><<<grid, 256, smem>>>(tw, twl, c, 32, iters, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bf = double(grid) * 256 * iters * bfly_per_iter;
  printf("%-26s grid %3d %s: %8.3f ms  %5.2f bfly/clk/SM (1965 MHz)  %s\n", name, grid, FWD ? "fwd" : "inv", ms,
         bf / (ms * 1e-3) / 148 / 1.965e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  const uint64_t q = 1125899904679937ull, n = 16384;
  LimbConstDev c{};
  c.q = q;
  c.twoq = 2 * q;
  c.negq = 0 - q;
  c.qq = double(q) / 4503599627370496.0;
  c.twoq_d = double(2 * q);
  c.q_d = double(q);
  c.qinv = 1.0 / double(q);
  c.q_bias = double(q) + 4503599627370496.0;
  c.bs = 52;
  std::vector<ulonglong2> h(n * 32);
  for (size_t i = 0; i < h.size(); ++i) {
    const uint64_t w = (i * 0x9E3779B97F4A7C15ull) % q;
    const uint64_t wp = (uint64_t)(((unsigned __int128)w << 52) / q);
    h[i] = make_ulonglong2(dbits(double(w)), dbits(double(wp)));
  }
  ulonglong2 *tw, *twl;
  cudaMalloc(&tw, h.size() * 16);
  cudaMalloc(&twl, h.size() * 16);
  cudaMemcpy(tw, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(twl, h.data(), h.size() * 16, cudaMemcpyHostToDevice);
  const int sm = 106 * 1024;
  run<Arith52S, true, 7>("S all passes, small L1", tw, twl, c, 224, 296, sm);
  run<Arith52S, true, 8>("S all passes, smem twiddles", tw, twl, c, 224, 296, sm);
  run<Arith52S, false, 7>("S all inv, small L1", tw, twl, c, 224, 296, sm);
  run<Arith52S, false, 8>("S all inv, smem twiddles", tw, twl, c, 224, 296, sm);
  run<Arith52S, true, 7>("S all passes", tw, twl, c, 224);
  run<Arith52S, true, 7>("S all passes, 1 CTA/SM", tw, twl, c, 224, 148);
  run<Arith52S, true, 4>("S P3, 1 CTA/SM", tw, twl, c, 80, 148);
  run<Arith52S, true, 1>("S P1 (13..9)", tw, twl, c, 80);
  run<Arith52S, true, 2>("S P2 (8..5)", tw, twl, c, 64);
  run<Arith52S, true, 4>("S P3 (4..0, low table)", tw, twl, c, 80);
  run<Arith52S, false, 7>("S all passes", tw, twl, c, 224);
  run<Arith52S, false, 1>("S P1 (0..4, low table)", tw, twl, c, 80);
  run<Arith52S, false, 2>("S P2", tw, twl, c, 64);
  run<Arith52S, false, 4>("S P3 (9..13)", tw, twl, c, 80);
  return 0;
}
