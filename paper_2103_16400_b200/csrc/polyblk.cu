// Launcher of the single-kernel poly_mult_mod for whole rows of N = 2^10 ..
// 2^13 words (ntt_polyblk.cuh). The C-ABI (capi.cu) chooses it when every
// limb of the call shares one canonical-only arithmetic policy.
#include "dispatch.cuh"
#include "ntt_polyblk.cuh"

namespace nk::rt {
namespace {

template <int LOGB, int LOGV, class A>
int launch_polyblk_t(const PolyBlkArgs& pa, uint64_t rows, cudaStream_t st) {
  constexpr size_t smem = polyblk_smem_bytes<LOGB, LOGV>();
  constexpr auto kern = poly_block<LOGB, LOGV, A>;
  if (smem > 48 * 1024)
    if (int rc = set_smem_once<kern>(smem)) return rc;
  kern<<<static_cast<unsigned>(rows), 1 << (LOGB - LOGV), smem, st>>>(pa);
  launches++;
  NK_CUDA(cudaGetLastError());
  return 0;
}

// 32 words per thread for batches that fill the GPU, 8 for small ones (like launch_block)
template <class A>
int launch_polyblk(const PolyBlkArgs& pa, uint64_t rows, cudaStream_t st) {
  const bool small = rows < static_cast<uint64_t>(sm_count());
#define NK_PB(L) \
  if (small) return launch_polyblk_t<L, 3, A>(pa, rows, st); \
  return launch_polyblk_t<L, 5, A>(pa, rows, st)
  switch (pa.fw.logn) {
    case 10: NK_PB(10);
    case 11: NK_PB(11);
    case 12: NK_PB(12);
    case 13: NK_PB(13);
    default: return fail(NK_ERR_CUDA, "internal: poly_block row length");
  }
#undef NK_PB
}

}  // namespace

int run_poly_block(const PolyBlkArgs& pa, uint64_t rows, bool fp64, cudaStream_t st) {
  return fp64 ? launch_polyblk<Arith52S>(pa, rows, st) : launch_polyblk<ArithIntL>(pa, rows, st);
}

}  // namespace nk::rt
