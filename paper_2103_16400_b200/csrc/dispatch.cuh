// Transform launchers: kernel choice per row length and batch, TMA tensor
// maps, launch shapes. Included only by ntt_inst.cu, which instantiates
// run_ntt<A, FWD> once per arithmetic policy and direction (one translation
// unit each, compiled in parallel).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>

#include "../../include/nttkit_b200.h"
#include "ntt_kernels.cuh"
#include "ntt_grp.cuh"
#include "ntt_pair.cuh"
#include "ntt_str.cuh"
#include "runtime.hpp"

namespace nk::rt {
namespace {

// ---- TMA tensor maps (driver entry point fetched through the runtime) ----
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int encode_fn(EncodeTiledFn* out) {
  static EncodeTiledFn fn = nullptr;
  static cudaError_t err = cudaSuccess;
  static std::once_flag once;
  std::call_once(once, [&] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (err == cudaSuccess && q != cudaDriverEntryPointSuccess) err = cudaErrorNotSupported;
    fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (err != cudaSuccess) return cuda_fail(err, "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
  *out = fn;
  return 0;
}

enum MapKind { kRowMap = 0, kSuperlineMap = 1, kOutMap = 2, kGrpOutMap = 3, kStrOutMap = 4, kStriOutMap = 5 };

// A tensor map is a pure function of (kind, base, words): the last few are
// cached per thread, so repeated calls on the same buffers (a serving loop,
// the host pipeline's chunk buffers) skip the encode.
int make_map(CUtensorMap* map, MapKind kind, const uint64_t* base, uint64_t words) {
  struct Entry {
    const uint64_t* base;
    uint64_t words;
    int kind;
    CUtensorMap map;
  };
  constexpr int kEntries = 8;
  thread_local Entry cache[kEntries] = {};
  thread_local int next = 0;
  for (const Entry& e : cache)
    if (e.base == base && e.words == words && e.kind == kind && base) {
      *map = e.map;
      return 0;
    }
  EncodeTiledFn fn;
  if (int rc = encode_fn(&fn)) return rc;
  CUresult r;
  void* p = const_cast<uint64_t*>(base);
  if (kind == kRowMap) {
    // 2D view [words/16][16] of a row buffer, 128B swizzle, boxes of 256 x 128 B
    const cuuint64_t dims[2] = {16, words / 16};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {16, 256};
    const cuuint32_t estr[2] = {1, 1};
    r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (kind == kSuperlineMap) {
    // 3D view [words/512][32 lines][16 words] (no swizzle), boxes 16 x 16 x 32:
    // one box = the 8192 words of a 16384-word block with index bit 8 fixed
    const cuuint64_t dims[3] = {16, 32, words / 512};
    const cuuint64_t strides[2] = {128, 4096};
    const cuuint32_t box[3] = {16, 16, 32};
    const cuuint32_t estr[3] = {1, 1, 1};
    r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (kind == kStrOutMap) {
    // 2D view [words/16][16] (128B swizzle), boxes of 32 x 128 B: the 512 consecutive
    // words of one warp's stream output in ntt_str14
    const cuuint64_t dims[2] = {16, words / 16};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {16, 32};
    const cuuint32_t estr[2] = {1, 1};
    r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (kind == kStriOutMap) {
    // 2D view [words/512][512] (no swizzle), boxes of 8 rows x 32 words: one warp's words
    // l | w << 5 | r << 9 for 8 values of r (ntt_stri14's output, str::out_half_tma)
    const cuuint64_t dims[2] = {512, words / 512};
    const cuuint64_t strides[1] = {4096};
    const cuuint32_t box[2] = {32, 8};
    const cuuint32_t estr[2] = {1, 1};
    r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (kind == kGrpOutMap) {
    // 5D view [words/512][4 (j7, j8)][4 (j5, j6)][2 halves][16 words] (128B swizzle),
    // boxes 16 x 1 x 1 x 1 x 8: one half of the runs j5j6 of 8 consecutive
    // 512-word pieces = 8 rows of a warp's output image in ntt_grp14
    const cuuint64_t dims[5] = {16, 2, 4, 4, words / 512};
    const cuuint64_t strides[4] = {128, 256, 1024, 4096};
    const cuuint32_t box[5] = {16, 1, 1, 1, 8};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    // 3D view [words/32][2][16] (128B swizzle), boxes 16 x 1 x 32: one half of
    // 32 consecutive 32-word runs = one warp's output round of ntt_pair14
    const cuuint64_t dims[3] = {16, 2, words / 32};
    const cuuint64_t strides[2] = {128, 256};
    const cuuint32_t box[3] = {16, 1, 32};
    const cuuint32_t estr[3] = {1, 1, 1};
    r = fn(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS)
    return fail(NK_ERR_CUDA, "cuTensorMapEncodeTiled(kind " + std::to_string(kind) + ") failed (" +
                                 std::to_string(r) + ")");
  cache[next] = Entry{base, words, kind, *map};
  next = (next + 1) % kEntries;
  return 0;
}

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev & 63;
}

// cudaFuncSetAttribute once per kernel and device (the attribute is per
// device; KERN identifies the instantiation)
template <auto KERN>
int set_smem_once(size_t bytes) {
  static std::atomic<uint64_t> done{0};
  const uint64_t bit = uint64_t{1} << current_device();
  if (done.load(std::memory_order_acquire) & bit) return 0;
  NK_CUDA(cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
  done.fetch_or(bit, std::memory_order_acq_rel);
  return 0;
}

// group-exchange kernel (ntt_grp.cuh): persistent, one 512-thread CTA per SM
template <auto KERN, bool FWD>
int launch_grp_k(const NttArgs& a, uint64_t nitems, uint64_t buf_words, cudaStream_t st) {
  CUtensorMap map, omap;
  if (int rc = make_map(&map, kRowMap, a.in, buf_words)) return rc;
  // the forward stores its result by TMA (the inverse with plain stores: omap unused)
  if (int rc = FWD ? make_map(&omap, kGrpOutMap, a.out, buf_words) : (omap = map, 0)) return rc;
  if (int rc = set_smem_once<KERN>(kGrpSmemBytes)) return rc;
  const uint64_t g = nitems < static_cast<uint64_t>(sm_count()) ? nitems : sm_count();
  KERN<<<static_cast<unsigned>(g), 512, kGrpSmemBytes, st>>>(map, omap, a, static_cast<uint32_t>(nitems));
  launches++;
  NK_CUDA(cudaGetLastError());
  return 0;
}

template <class A, bool FWD, bool IL>
int launch_grp_t(const NttArgs& a, uint64_t nitems, uint64_t buf_words, cudaStream_t st) {
  if constexpr (!FWD)
    if (a.logn > 14) return launch_grp_k<ntt_grp14<A, FWD, IL, true>, FWD>(a, nitems, buf_words, st);
  return launch_grp_k<ntt_grp14<A, FWD, IL>, FWD>(a, nitems, buf_words, st);
}

// two-stream forward (ntt_str.cuh): persistent, one 512-thread CTA per SM
template <class A, bool IL>
int launch_str_t(const NttArgs& a, uint64_t nitems, uint64_t buf_words, cudaStream_t st) {
  constexpr auto kern = ntt_str14<A, IL>;
  CUtensorMap map, omap;
  if (int rc = make_map(&map, kRowMap, a.in, buf_words)) return rc;
  if (int rc = make_map(&omap, kStrOutMap, a.out, buf_words)) return rc;
  if (int rc = set_smem_once<kern>(kStrSmemBytes)) return rc;
  const uint64_t g = nitems < static_cast<uint64_t>(sm_count()) ? nitems : sm_count();
  kern<<<static_cast<unsigned>(g), 512, kStrSmemBytes, st>>>(map, omap, a, static_cast<uint32_t>(nitems));
  launches++;
  NK_CUDA(cudaGetLastError());
  return 0;
}

template <auto KERN>
int launch_stri_k(const NttArgs& a, uint64_t nitems, uint64_t buf_words, cudaStream_t st) {
  CUtensorMap map, omap;
  if (int rc = make_map(&map, kRowMap, a.in, buf_words)) return rc;
  if (int rc = make_map(&omap, kStriOutMap, a.out, buf_words)) return rc;
  if (int rc = set_smem_once<KERN>(kStrSmemBytes)) return rc;
  const uint64_t g = nitems < static_cast<uint64_t>(sm_count()) ? nitems : sm_count();
  KERN<<<static_cast<unsigned>(g), 512, kStrSmemBytes, st>>>(map, omap, a, static_cast<uint32_t>(nitems));
  launches++;
  NK_CUDA(cudaGetLastError());
  return 0;
}
template <class A, bool IL>
int launch_stri_t(const NttArgs& a, uint64_t nitems, uint64_t buf_words, cudaStream_t st) {
  if (a.logn > 14) return launch_stri_k<ntt_stri14<A, IL, true>>(a, nitems, buf_words, st);
  return launch_stri_k<ntt_stri14<A, IL>>(a, nitems, buf_words, st);
}

// CTA-pair kernel (ntt_pair.cuh): persistent, one cluster of 2 per block in
// flight, as many clusters as fit (2 CTAs per SM).
template <auto KERN, bool FWD>
int launch_pair_k(const NttArgs& a, uint64_t nitems, uint64_t buf_words, cudaStream_t st) {
  CUtensorMap map, omap;
  if (int rc = make_map(&map, FWD ? kSuperlineMap : kRowMap, a.in, buf_words)) return rc;
  if (int rc = make_map(&omap, kOutMap, a.out, buf_words)) return rc;
  if (int rc = set_smem_once<KERN>(kPairSmemBytes)) return rc;
  static int max_clusters[64] = {};
  const int dev = current_device();
  if (!max_clusters[dev]) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * sm_count());
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = kPairSmemBytes;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 2;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    NK_CUDA(cudaOccupancyMaxActiveClusters(&n, KERN, &cfg));
    max_clusters[dev] = n > 0 ? n : sm_count();
  }
  const uint64_t mc = static_cast<uint64_t>(max_clusters[dev]);
  const uint64_t g = nitems < mc ? nitems : mc;
  KERN<<<static_cast<unsigned>(2 * g), 256, kPairSmemBytes, st>>>(map, omap, a, static_cast<uint32_t>(nitems));
  launches++;
  NK_CUDA(cudaGetLastError());
  return 0;
}

template <class A, bool FWD, bool IL>
int launch_pair_t(const NttArgs& a, uint64_t nitems, uint64_t buf_words, cudaStream_t st) {
  if constexpr (FWD && A::kSigned)
    if (a.mulb) return launch_pair_k<ntt_pair14<A, FWD, IL, true>, FWD>(a, nitems, buf_words, st);
  // the fused product exists only in the signed FP64 forward instance above:
  // any other policy reaching here with a multiplier is a dispatch bug
  if (a.mulb) return fail(NK_ERR_CUDA, "internal: fused product requested for a policy without it");
  return launch_pair_k<ntt_pair14<A, FWD, IL>, FWD>(a, nitems, buf_words, st);
}

template <class A, bool FWD>
int launch_tma(const NttArgs& a, uint64_t nitems, uint64_t buf_words, bool iltm, cudaStream_t st) {
  // measured on B200 (cfg3 / cfg4, forward / inverse): with the low tables in
  // thread order the group-exchange kernel is the faster one in both
  // directions (220 / 217 us against the CTA-pair kernel's 228 / 229 us on
  // cfg3; 363 / 348 us against 363 / 384 us on cfg4); the three-launch
  // poly_mult_mod's fused product lives in the pair forward only
  const bool pair = a.mulb || block_kernel == 0;
  if constexpr (FWD)
    if (!a.mulb && (block_kernel == 2 || block_kernel < 0 || block_kernel == 3))  // the default forward: two streams per thread
      return iltm ? launch_str_t<A, true>(a, nitems, buf_words, st) : launch_str_t<A, false>(a, nitems, buf_words, st);
  if constexpr (!FWD)
    if (block_kernel == 2 || block_kernel < 0 || block_kernel == 3)  // the default inverse: two streams per thread
      return iltm ? launch_stri_t<A, true>(a, nitems, buf_words, st) : launch_stri_t<A, false>(a, nitems, buf_words, st);
  if (pair)
    return iltm ? launch_pair_t<A, FWD, true>(a, nitems, buf_words, st)
                : launch_pair_t<A, FWD, false>(a, nitems, buf_words, st);
  return iltm ? launch_grp_t<A, FWD, true>(a, nitems, buf_words, st)
              : launch_grp_t<A, FWD, false>(a, nitems, buf_words, st);
}

// LOGV = log2(words per thread): 8 for small batches (cfg1: one row), where
// the row's latency is the metric and more threads per row cut it; for batches
// that fill the GPU 16, or 32 where that measured faster (block_logv).
// 2^25 coefficients, us per call with 32 / 16 / 8 words per thread
// (tools/prof_ntt.py, 16 limbs):
//   50-bit, forward: N = 1024 177 / 150 / 162, 2048 164 / 161 / 168, 4096 199 / 189 / 207, 8192 222 / 215 / 326
//   50-bit, inverse:          172 / 143 / 173,      164 / 151 / 180,      195 / 206 / 227,      231 / 219 / 309
//   60-bit, forward:          279 / 231 / 247,      290 / 245 / 274,      327 / 286 / 322,      404 / 331 / 409
//   60-bit, inverse:          308 / 237 / 254,      345 / 256 / 281,      340 / 321 / 331,      354 / 329 / 411
template <class A, bool FWD>
constexpr int block_logv(int logb) {
  if (!FWD && A::kFP && logb == 12) return 5;
  return 4;
}

template <int LOGB, int LOGV, class A, bool FWD, bool IL>
int launch_block_t(const NttArgs& a, uint64_t grid, cudaStream_t st) {
  constexpr size_t smem = block_smem_bytes<LOGB, LOGV>();
  constexpr auto kern = ntt_block<LOGB, LOGV, A, FWD, IL>;
  if (smem > 48 * 1024)
    if (int rc = set_smem_once<kern>(smem)) return rc;
  kern<<<static_cast<unsigned>(grid), 1 << (LOGB - LOGV), smem, st>>>(a);
  launches++;
  NK_CUDA(cudaGetLastError());
  return 0;
}

// latency path (ntt_block_lat): programmatic dependent launch, twiddle row
// staged into shared memory before griddepcontrol.wait
template <int LOGB, int LOGV, class A, bool FWD, bool IL>
int launch_block_lat_t(const NttArgs& a, uint64_t grid, cudaStream_t st) {
  constexpr size_t smem = lat_smem_bytes<LOGB, LOGV>();
  constexpr auto kern = ntt_block_lat<LOGB, LOGV, A, FWD, IL>;
  if (int rc = set_smem_once<kern>(smem)) return rc;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(1u << (LOGB - LOGV));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  launches++;
  if (e != cudaSuccess) return cuda_fail(e, "ntt_block_lat launch");
  return 0;
}

template <class A, bool FWD>
int launch_block(uint32_t logb, const NttArgs& a, uint64_t grid, bool iltm, cudaStream_t st) {
  const bool small = a.rows < static_cast<uint64_t>(sm_count());
  if (small && a.logn == logb && !no_lat) {  // whole rows, few of them: the latency path
    switch (logb) {
      case 10: return iltm ? launch_block_lat_t<10, 3, A, FWD, true>(a, grid, st) : launch_block_lat_t<10, 3, A, FWD, false>(a, grid, st);
      case 11: return iltm ? launch_block_lat_t<11, 3, A, FWD, true>(a, grid, st) : launch_block_lat_t<11, 3, A, FWD, false>(a, grid, st);
      case 12: return iltm ? launch_block_lat_t<12, 3, A, FWD, true>(a, grid, st) : launch_block_lat_t<12, 3, A, FWD, false>(a, grid, st);
      default: return iltm ? launch_block_lat_t<13, 3, A, FWD, true>(a, grid, st) : launch_block_lat_t<13, 3, A, FWD, false>(a, grid, st);
    }
  }
#define NK_LB2(L, V) \
  return iltm ? launch_block_t<L, V, A, FWD, true>(a, grid, st) : launch_block_t<L, V, A, FWD, false>(a, grid, st)
#define NK_LB(L) \
  if (small) NK_LB2(L, 3); \
  NK_LB2(L, (block_logv<A, FWD>(L)))
  switch (logb) {
    case 10: NK_LB(10);
    case 11: NK_LB(11);
    case 12: NK_LB(12);
    default: NK_LB(13);
  }
#undef NK_LB
#undef NK_LB2
}

template <class A, bool FWD>
int launch_global(uint32_t k, uint32_t lo, bool first_iltm, bool last, const NttArgs& a, cudaStream_t st) {
  const uint64_t threads = a.rows << (a.logn - k);
  const unsigned grid = static_cast<unsigned>((threads + 255) / 256);
  switch (k) {
    case 1: ntt_global_pass<1, A, FWD><<<grid, 256, 0, st>>>(a, lo, first_iltm, last); break;
    case 2: ntt_global_pass<2, A, FWD><<<grid, 256, 0, st>>>(a, lo, first_iltm, last); break;
    default: ntt_global_pass<3, A, FWD><<<grid, 256, 0, st>>>(a, lo, first_iltm, last); break;
  }
  launches++;
  NK_CUDA(cudaGetLastError());
  return 0;
}

template <class A, bool FWD>
int launch_small(const NttArgs& a, cudaStream_t st) {
  const size_t smem = a.n * sizeof(uint64_t);
  const unsigned threads = static_cast<unsigned>(a.n / 2 < 256 ? a.n / 2 : 256);
  ntt_small<A, FWD><<<static_cast<unsigned>(a.rows), threads, smem, st>>>(a);
  launches++;
  NK_CUDA(cudaGetLastError());
  return 0;
}

}  // namespace

constexpr uint32_t kLogBlock = 14;

template <class A, bool FWD>
int run_ntt(NttArgs a, uint64_t buf_words, cudaStream_t st) {
  a.dbg = dbg;
  const uint32_t logn = a.logn;
  if (logn < 10) return launch_small<A, FWD>(a, st);
  if (logn < kLogBlock) return launch_block<A, FWD>(logn, a, a.rows, a.fin == 1, st);
  if (logn == kLogBlock) return launch_tma<A, FWD>(a, a.rows, buf_words, a.fin == 1, st);
  // long rows: high bits in global passes of <= 3 stages, low 14 bits per block
  const uint32_t gbits = logn - kLogBlock;
  uint32_t ks[2] = {gbits, 0};
  if (gbits > 3) {
    ks[0] = (gbits + 1) / 2;
    ks[1] = gbits - ks[0];
  }
  const int np = ks[1] ? 2 : 1;
  const uint64_t nitems = a.rows << gbits;
  if constexpr (FWD) {
    uint32_t top = logn;
    for (int p = 0; p < np; ++p) {
      const uint32_t lo = top - ks[p];
      if (int rc = launch_global<A, true>(ks[p], lo, p == 0 && a.fin == 1, false, a, st)) return rc;
      a.in = a.out;  // later passes run in place on the result
      top = lo;
    }
    return launch_tma<A, true>(a, nitems, buf_words, false, st);
  } else {
    if (int rc = launch_tma<A, false>(a, nitems, buf_words, a.fin == 1, st)) return rc;
    a.in = a.out;
    uint32_t lo = kLogBlock;
    for (int p = 0; p < np; ++p) {
      if (int rc = launch_global<A, false>(ks[p], lo, false, p == np - 1, a, st)) return rc;
      lo += ks[p];
    }
    return 0;
  }
}

}  // namespace nk::rt
