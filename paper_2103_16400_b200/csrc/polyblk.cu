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

// Words per thread (tools/polyblk_bench.py, 2^25 coefficients, us per call for 8 / 16 / 32
// words per thread):
//   50-bit limbs: N = 1024 489 / 395 / 557, 2048 543 / 425 / 458, 4096 660 / 510 / 502, 8192 772 / 684 / 663
//   60-bit limbs:          829 / 900 / 1230,     948 / 973 / 1010,    1105 / 948 / 1168,    1189 / 1108 / 1561
// 8 for batches smaller than the SM count (more threads per row).
template <class A>
int launch_polyblk(const PolyBlkArgs& pa, uint64_t rows, cudaStream_t st) {
  const bool small = rows < static_cast<uint64_t>(sm_count());
#define NK_PB(L, V) \
  if (small) return launch_polyblk_t<L, 3, A>(pa, rows, st); \
  return launch_polyblk_t<L, V, A>(pa, rows, st)
  switch (pa.fw.logn) {
    case 10: NK_PB(10, (A::kSigned ? 4 : 3));
    case 11: NK_PB(11, (A::kSigned ? 4 : 3));
    case 12: NK_PB(12, 4);
    case 13: NK_PB(13, (A::kSigned ? 5 : 4));
    default: return fail(NK_ERR_CUDA, "internal: poly_block row length");
  }
#undef NK_PB
}

}  // namespace

int run_poly_block(const PolyBlkArgs& pa, uint64_t rows, bool fp64, cudaStream_t st) {
  return fp64 ? launch_polyblk<Arith52S>(pa, rows, st) : launch_polyblk<ArithIntL>(pa, rows, st);
}

}  // namespace nk::rt
