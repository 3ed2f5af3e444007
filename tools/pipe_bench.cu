// Microbenchmark: per-SM throughput of the instructions the NTT butterfly is
// built from (IMAD, IMAD.WIDE, IMAD.HI, IADD3, DFMA, DADD, mixes) on B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pipe_bench tools/pipe_bench.cu
#include <cstdint>
#include <cstdio>

#define ITERS 4096
#define CH 8  // independent chains per thread

template <int OP>
__global__ void __launch_bounds__(512) kern(uint64_t* out, uint32_t seed) {
  uint32_t a[CH], b[CH];
  uint64_t w[CH];
  double d[CH], e[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    a[i] = seed * (threadIdx.x + 1) + i;
    b[i] = a[i] ^ 0x9e3779b9u;
    w[i] = (uint64_t(a[i]) << 20) | b[i];
    d[i] = (double)a[i];
    e[i] = (double)b[i] * 1e-9;
  }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (OP == 0) {  // IMAD (32-bit)
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b[i]), "r"(a[i]));
      } else if (OP == 1) {  // IMAD.WIDE.U32 with 64-bit accumulate
        asm volatile("{.reg .b32 t; cvt.u32.u64 t, %0; mad.wide.u32 %0, t, %1, %0;}" : "+l"(w[i]) : "r"(b[i]));
      } else if (OP == 2) {  // IMAD.HI.U32
        asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i]));
      } else if (OP == 3) {  // IADD3
        asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i]));
        asm volatile("xor.b32 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i]));
      } else if (OP == 4) {  // DFMA
        asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(e[i]));
      } else if (OP == 5) {  // DADD
        asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(d[i]) : "d"(e[i]));
      } else if (OP == 6) {  // IMAD + DFMA interleaved
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b[i]), "r"(a[i]));
        asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(e[i]));
      } else if (OP == 7) {  // IMAD.WIDE + IADD3 + DFMA
        asm volatile("{.reg .b32 t; cvt.u32.u64 t, %0; mad.wide.u32 %0, t, %1, %0;}" : "+l"(w[i]) : "r"(b[i]));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i]));
        asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(e[i]));
      } else if (OP == 8) {  // 64-bit add (IADD3 + IADD3.X)
        asm volatile("add.u64 %0, %0, %1;" : "+l"(w[i]) : "l"(w[(i + 1) % CH]));
      } else if (OP == 9) {  // IMAD + IADD3 (fma vs alu pipes)
        asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[i]) : "r"(b[i]), "r"(a[i]));
        asm volatile("add.u32 %0, %0, %1;" : "+r"(b[i]) : "r"(a[i]));
      } else if (OP == 10) {  // mul.lo.u64 (3 IMADs)
        asm volatile("mul.lo.u64 %0, %0, %1;" : "+l"(w[i]) : "l"(w[(i + 3) % CH]));
      } else if (OP == 11) {  // DFMA.RM
        asm volatile("fma.rm.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(e[i]));
      } else if (OP == 12) {  // FRND.F64 alone
        asm volatile("cvt.rni.f64.f64 %0, %0;" : "+d"(e[i]));
      } else if (OP == 13) {  // 8 DFMA (kernel's FP64 : FRND ratio), no FRND
#pragma unroll
        for (int r = 0; r < 8; ++r) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(e[i]));
      } else if (OP == 14) {  // 8 DFMA + 1 FRND.F64 on an independent chain
#pragma unroll
        for (int r = 0; r < 8; ++r) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(e[i]));
        asm volatile("cvt.rni.f64.f64 %0, %0;" : "+d"(e[(i + 1) % CH]));
      } else if (OP == 15) {  // 8 DFMA + 2 FRND.F64
#pragma unroll
        for (int r = 0; r < 8; ++r) asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(e[i]));
        asm volatile("cvt.rni.f64.f64 %0, %0;" : "+d"(e[(i + 1) % CH]));
        asm volatile("cvt.rni.f64.f64 %0, %0;" : "+d"(e[(i + 2) % CH]));
      } else if (OP == 16) {  // 8 DFMA + 8 LOP3/IADD (issue-slot sharing)
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(e[i]));
          asm volatile("xor.b32 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i]));
        }
      } else if (OP == 17) {  // 8 DFMA + 1 FRND + 8 LOP3
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          asm volatile("fma.rn.f64 %0, %0, %1, %1;" : "+d"(d[i]) : "d"(e[i]));
          asm volatile("xor.b32 %0, %0, %1;" : "+r"(a[i]) : "r"(b[i]));
        }
        asm volatile("cvt.rni.f64.f64 %0, %0;" : "+d"(e[(i + 1) % CH]));
      }
    }
  }
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += a[i] + b[i] + w[i] + (uint64_t)d[i];
  if (s == 0x12345) out[threadIdx.x] = s;
}

template <int OP>
void run(const char* name, int ops_per_iter) {
  uint64_t* out;
  cudaMalloc(&out, 4096);
  const int grid = 148 * 4, block = 512;
  kern<OP><<<grid, block>>>(out, 1);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<OP><<<grid, block>>>(out, 2);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double ops = double(grid) * block * ITERS * CH * ops_per_iter;
  const double per_s = ops / (ms * 1e-3);
  printf("%-28s %8.3f ms  %8.1f Gop/s  %6.1f thread-ops/clk/SM (at %d MHz)\n", name, ms,
         per_s / 1e9, per_s / 148 / (clk * 1e3), clk / 1000);
  cudaFree(out);
}

int main() {
  run<0>("IMAD (mad.lo.u32)", 1);
  run<1>("IMAD.WIDE.U32 acc", 1);
  run<2>("IMAD.HI.U32", 1);
  run<3>("IADD3+LOP3", 2);
  run<4>("DFMA", 1);
  run<11>("DFMA.RM", 1);
  run<5>("DADD", 1);
  run<6>("IMAD+DFMA (pairs)", 2);
  run<7>("WIDE+IADD3+DFMA (triples)", 3);
  run<8>("add.u64", 1);
  run<9>("IMAD+IADD3 (pairs)", 2);
  run<10>("mul.lo.u64", 1);
  run<12>("FRND.F64", 1);
  run<13>("8 DFMA", 8);
  run<14>("8 DFMA + FRND (count 8)", 8);
  run<15>("8 DFMA + 2 FRND (count 8)", 8);
  run<16>("8 DFMA + 8 LOP3 (count 8)", 8);
  run<17>("8 DFMA + 8 LOP3 + FRND (c8)", 8);
  return 0;
}
