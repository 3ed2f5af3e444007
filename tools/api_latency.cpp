// Per-call cost of the C-ABI entry points for small inputs (host issue rate
// and device completion), without Python in the loop.
// Build: g++ -std=c++17 -O2 -I include -I /usr/local/cuda/include tools/api_latency.cpp \
//        -L paper_2103_16400_b200 -lnttkit_b200 -L /usr/local/cuda/lib64 -lcudart \
//        -Wl,-rpath,$PWD/paper_2103_16400_b200 -o tools/api_latency
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdint>
#include <functional>
#include <vector>

#include "nttkit_b200.h"

static double per_call_us(const std::function<void()>& fn, int iters) {
  fn();
  cudaDeviceSynchronize();
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < iters; ++i) fn();
  const auto t1 = std::chrono::steady_clock::now();
  cudaDeviceSynchronize();
  const auto t2 = std::chrono::steady_clock::now();
  const double issue = std::chrono::duration<double, std::micro>(t1 - t0).count() / iters;
  const double total = std::chrono::duration<double, std::micro>(t2 - t0).count() / iters;
  std::printf("    issue %.2f us/call, completion %.2f us/call\n", issue, total);
  return total;
}

int main() {
  const uint64_t q60 = 1152921504606846883ull;
  const uint64_t n = 4096;
  const uint64_t q50 = 1125899906826241ull;  // cfg1
  uint64_t *a, *b, *r;
  cudaMalloc(&a, 1 << 20);
  cudaMalloc(&b, 1 << 20);
  cudaMalloc(&r, 1 << 20);
  cudaMemset(a, 0, 1 << 20);
  cudaMemset(b, 0, 1 << 20);
  cudaStream_t st;
  cudaStreamCreate(&st);
  nk_plan* p = nullptr;
  if (nk_plan_create(&p, 0, n, &q50, nullptr, 1, 0)) {
    std::printf("plan: %s\n", nk_last_error());
    return 1;
  }
  std::printf("nk_version x1: ");
  per_call_us([] { nk_version(); }, 100000);
  for (uint64_t len : {1024ull, 16384ull}) {
    std::printf("nk_eltwise_mult_mod n=%llu:\n", (unsigned long long)len);
    per_call_us([&] { nk_eltwise_mult_mod(r, a, b, len, q60, 1, st); }, 20000);
  }
  std::printf("nk_ntt_forward N=4096 (cfg1):\n");
  per_call_us([&] { nk_ntt_forward(p, r, a, 0, 1, 1, 1, 1, st); }, 20000);
  std::printf("nk_ntt_forward + nk_ntt_inverse N=4096 (cfg1 round trip):\n");
  per_call_us([&] {
    nk_ntt_forward(p, r, a, 0, 1, 1, 1, 1, st);
    nk_ntt_inverse(p, b, r, 0, 1, 1, 1, 1, st);
  }, 10000);
  nk_plan_destroy(p);
  return 0;
}
