// Launcher of the single-kernel poly_mult_mod (ntt_poly.cuh) for N = 16384
// rows under the signed FP64 policy. The C-ABI (capi.cu) chooses it, or the
// multi-launch sequences, per plan and limb range.
#include "dispatch.cuh"
#include "ntt_poly.cuh"

namespace nk::rt {

int run_poly_mul14(const PolyArgs& pa, const uint64_t* f, const uint64_t* g, cudaStream_t st) {
  const uint64_t words = pa.a.rows * pa.a.n;
  CUtensorMap mf, mg;
  if (int rc = make_map(&mf, kRowMap, f, words)) return rc;
  if (int rc = make_map(&mg, kRowMap, g, words)) return rc;
  const uint64_t grid = pa.a.rows < static_cast<uint64_t>(sm_count()) ? pa.a.rows : sm_count();
  if (block_kernel == 3) {  // nk_debug_block_kernel(3): the group-exchange version
    if (int rc = set_smem_once<poly_mul14<Arith52S>>(kPolySmemBytes)) return rc;
    poly_mul14<Arith52S><<<static_cast<unsigned>(grid), 512, kPolySmemBytes, st>>>(mf, mg, pa,
                                                                                    static_cast<uint32_t>(pa.a.rows));
  } else {  // two streams per thread (ntt_str.cuh cores)
    CUtensorMap mo;  // the result leaves by bulk tensor stores
    if (int rc = make_map(&mo, kStriOutMap, pa.a.out, words)) return rc;
    if (int rc = set_smem_once<poly_str14<Arith52S>>(kPolyStrSmemBytes)) return rc;
    poly_str14<Arith52S><<<static_cast<unsigned>(grid), 512, kPolyStrSmemBytes, st>>>(
        mf, mg, mo, pa, static_cast<uint32_t>(pa.a.rows));
  }
  launches++;
  NK_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace nk::rt
