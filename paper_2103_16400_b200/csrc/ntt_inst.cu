// One arithmetic policy x direction of the transform dispatch per object
// file: the Makefile compiles this source eight times with NK_INST = 0..7
// (bit 0 = forward, bits 1-2 = policy), in parallel.
#include "dispatch.cuh"

#ifndef NK_INST
#error "compile with -DNK_INST=0..7"
#endif

namespace nk::rt {
#if (NK_INST >> 1) == 0
using InstPolicy = Arith52S;
#elif (NK_INST >> 1) == 1
using InstPolicy = Arith52P;
#elif (NK_INST >> 1) == 2
using InstPolicy = ArithIntL;
#else
using InstPolicy = ArithInt<64>;
#endif
template int run_ntt<InstPolicy, (NK_INST & 1) != 0>(NttArgs, uint64_t, cudaStream_t);
}  // namespace nk::rt
