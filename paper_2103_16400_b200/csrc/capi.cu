// C-ABI of nttkit_b200 (include/nttkit_b200.h): argument validation that
// mirrors the reference's std::invalid_argument checks, plan (device table)
// management, and kernel launches. No CPU compute fallback exists: every
// transform and element-wise product runs in the sm_100a kernels below, and a
// missing/failed CUDA device is reported as NK_ERR_CUDA.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <condition_variable>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/nttkit_b200.h"
#include "eltwise_kernels.cuh"
#include "host_math.hpp"
#include "ntt_poly.cuh"
#include "ntt_polyblk.cuh"
#include "ntt_str.cuh"
#include "runtime.hpp"

using nk::host::u128;

// ---------------------------------------------------------------------------
// shared runtime state (runtime.hpp)
// ---------------------------------------------------------------------------
namespace nk::rt {
thread_local std::string g_err;
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  return fail(NK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
std::atomic<uint64_t> launches{0};
thread_local int block_kernel = -1;
thread_local bool no_lat = false;
thread_local bool exact_only = false;
thread_local uint64_t* dbg = nullptr;

int sm_count() {
  static int n[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!n[dev & 63]) cudaDeviceGetAttribute(&n[dev & 63], cudaDevAttrMultiProcessorCount, dev);
  return n[dev & 63] ? n[dev & 63] : 148;
}
}  // namespace nk::rt

using nk::rt::cuda_fail;
using nk::rt::fail;

namespace {

// Small per-thread cache of validated moduli: Modulus(q) runs Miller-Rabin
// (modarith.hpp:108-115); element-wise calls re-validate the same q repeatedly.
bool valid_modulus(uint64_t q, nk::host::Modulus* m) {
  thread_local nk::host::Modulus cache[4];
  thread_local int next = 0;
  for (auto& c : cache)
    if (c.q == q && q != 0) { *m = c; return true; }
  if (!nk::host::make_modulus(q, m)) return false;
  cache[next] = *m;
  next = (next + 1) & 3;
  return true;
}

bool overlap_bad(const void* a, const void* b, uint64_t bytes) {
  if (a == b) return false;
  const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  return x < y + bytes && y < x + bytes;
}

cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }

uint64_t dbits(double d) {
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
}
// a beta = 2^52 table word (the bit pattern of the double w, 0 <= w < q) as the balanced
// representative of the same residue: w - q when 2w > q (exact: both are integers below 2^52)
uint64_t balanced8(uint64_t wbits, uint64_t q) {
  double w;
  std::memcpy(&w, &wbits, 8);
  const uint64_t wi = static_cast<uint64_t>(w);
  return 2 * wi > q ? dbits(w - static_cast<double>(q)) : wbits;
}

// the balanced representative of w mod q as a double (q < 2^50)
double bal_d(uint64_t w, uint64_t q) {
  return 2 * w > q ? -static_cast<double>(q - w) : static_cast<double>(w);
}

// Makes `dev` current for the duration of one entry-point call and restores
// the caller's device on return (a call on a plan of another GPU must not
// move the caller's torch/CUDA current device).
class DeviceScope {
 public:
  DeviceScope() = default;
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;
  ~DeviceScope() {
    if (prev_ >= 0) cudaSetDevice(prev_);
  }
  int enter(int dev) {
    int cur = -1;
    NK_CUDA(cudaGetDevice(&cur));
    if (cur != dev) {
      NK_CUDA(cudaSetDevice(dev));
      prev_ = cur;
    }
    // stream-ordered scratch (poly_mult_mod's g^, unaligned views, the host
    // pipeline's chunks) comes from the device's default pool; keep freed
    // blocks in the pool instead of returning them to the driver at every
    // synchronisation
    static std::once_flag pool_once[64];
    std::call_once(pool_once[dev & 63], [dev] {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
    });
    return 0;
  }

 private:
  int prev_ = -1;
};

}  // namespace

struct nk_plan {
  int device = 0;
  uint64_t n = 0;
  uint32_t logn = 0, nlimbs = 0;
  std::vector<uint64_t> q, psi;
  std::vector<int> bs;
  ulonglong2* tw_fwd = nullptr;  // [limb][n]
  ulonglong2* tw_inv = nullptr;  // [limb][n]
  ulonglong2* twl_fwd = nullptr;  // [limb][n] low-bit-stage tables, transposed (nk::low_index)
  ulonglong2* twl_inv = nullptr;
  uint64_t* tw8_fwd = nullptr;   // [limb][n] w only (double bits) for the Arith52S kernels
  uint64_t* tw8_inv = nullptr;
  uint64_t* twl8_fwd = nullptr;  // [limb][n] low-table order
  uint64_t* twl8_inv = nullptr;
  // the low tables in the group-exchange kernels' thread order (NttArgs::twg)
  ulonglong2* twg_fwd = nullptr;
  ulonglong2* twg_inv = nullptr;
  uint64_t* twg8_fwd = nullptr;
  uint64_t* twg8_inv = nullptr;
  // forward low-stage twiddles of the two-stream kernel (NttArgs::twq), [limb][block][stream][entry][thread]
  ulonglong2* twq_fwd = nullptr;
  uint64_t* twq8_fwd = nullptr;
  ulonglong2* twq_inv = nullptr;
  uint64_t* twq8_inv = nullptr;
  void* slab = nullptr;          // the allocation the tables above live in
  nk::LimbConst* lc = nullptr;   // [limb]
  nk::MultConst* mc[3] = {nullptr, nullptr, nullptr};  // fin = 1, 2, 4
};

// ---------------------------------------------------------------------------
// transform dispatch (kernel choice: dispatch.cuh, compiled per policy in ntt_inst.cu)
// ---------------------------------------------------------------------------
namespace nk::rt {
extern template int run_ntt<Arith52S, true>(NttArgs, uint64_t, cudaStream_t);
extern template int run_ntt<Arith52S, false>(NttArgs, uint64_t, cudaStream_t);
extern template int run_ntt<Arith52P, true>(NttArgs, uint64_t, cudaStream_t);
extern template int run_ntt<Arith52P, false>(NttArgs, uint64_t, cudaStream_t);
extern template int run_ntt<ArithIntL, true>(NttArgs, uint64_t, cudaStream_t);
extern template int run_ntt<ArithIntL, false>(NttArgs, uint64_t, cudaStream_t);
extern template int run_ntt<ArithInt<64>, true>(NttArgs, uint64_t, cudaStream_t);
extern template int run_ntt<ArithInt<64>, false>(NttArgs, uint64_t, cudaStream_t);
}  // namespace nk::rt

namespace {
using nk::rt::run_ntt;
constexpr uint32_t kLogBlock = 14;

int check_limbs(const nk_plan* p, uint32_t limb0, uint32_t nlimbs) {
  if (!p) return fail(NK_ERR_NULL, "plan is NULL");
  if (nlimbs == 0 || static_cast<uint64_t>(limb0) + nlimbs > p->nlimbs)
    return fail(NK_ERR_LIMB, "limb range outside the plan");
  return 0;
}

// largest modulus of limbs [l0, l0 + cnt)
uint64_t max_q(const nk_plan* p, uint32_t l0, uint32_t cnt) {
  uint64_t m = 0;
  for (uint32_t l = l0; l < l0 + cnt; ++l) m = p->q[l] > m ? p->q[l] : m;
  return m;
}

int ntt_dispatch_aligned(const nk_plan* p, bool fwd, uint64_t* res, const uint64_t* op, uint32_t limb0,
                         uint32_t nlimbs, uint32_t npolys, uint64_t fin, uint64_t fout, cudaStream_t st,
                         const uint64_t* mulb);

// The transform kernels use 16/32-byte vector accesses and TMA on row
// starts: buffers that are not 32-byte aligned (e.g. a view starting at an odd
// word) run through an aligned stream-ordered copy instead of faulting.
int ntt_dispatch(const nk_plan* p, bool fwd, uint64_t* res, const uint64_t* op, uint32_t limb0,
                 uint32_t nlimbs, uint32_t npolys, uint64_t fin, uint64_t fout, cudaStream_t st,
                 const uint64_t* mulb = nullptr) {
  const uintptr_t mis = (reinterpret_cast<uintptr_t>(res) | reinterpret_cast<uintptr_t>(op) |
                         reinterpret_cast<uintptr_t>(mulb)) & 31;
  if (!mis || npolys == 0)
    return ntt_dispatch_aligned(p, fwd, res, op, limb0, nlimbs, npolys, fin, fout, st, mulb);
  const size_t bytes = static_cast<size_t>(npolys) * nlimbs * p->n * 8;
  uint64_t *t = nullptr, *tm = nullptr;
  int rc = 0;
  cudaError_t e = cudaMallocAsync(&t, bytes, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(t, op, bytes, cudaMemcpyDeviceToDevice, st);
  if (e == cudaSuccess && mulb) {
    e = cudaMallocAsync(&tm, bytes, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(tm, mulb, bytes, cudaMemcpyDeviceToDevice, st);
  }
  if (e != cudaSuccess) rc = cuda_fail(e, "unaligned view: aligned copy");
  if (!rc) rc = ntt_dispatch_aligned(p, fwd, t, t, limb0, nlimbs, npolys, fin, fout, st, mulb ? tm : nullptr);
  if (!rc) {
    e = cudaMemcpyAsync(res, t, bytes, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaMemcpyAsync(unaligned result)");
  }
  // the scratch goes back to the pool on every path
  if (t) cudaFreeAsync(t, st);
  if (tm) cudaFreeAsync(tm, st);
  return rc;
}

int ntt_dispatch_aligned(const nk_plan* p, bool fwd, uint64_t* res, const uint64_t* op, uint32_t limb0,
                         uint32_t nlimbs, uint32_t npolys, uint64_t fin, uint64_t fout, cudaStream_t st,
                         const uint64_t* mulb) {
  nk::NttArgs a{};
  a.mulb = mulb;
  a.out = res;
  a.in = op;
  a.tw = fwd ? p->tw_fwd : p->tw_inv;
  a.twl = fwd ? p->twl_fwd : p->twl_inv;
  a.tw8 = fwd ? p->tw8_fwd : p->tw8_inv;
  a.twl8 = fwd ? p->twl8_fwd : p->twl8_inv;
  a.twg = fwd ? p->twg_fwd : p->twg_inv;
  a.twg8 = fwd ? p->twg8_fwd : p->twg8_inv;
  a.twq = fwd ? p->twq_fwd : p->twq_inv;
  a.twq8 = fwd ? p->twq8_fwd : p->twq8_inv;
  a.lc = p->lc;
  a.n = p->n;
  a.logn = p->logn;
  a.limb0 = limb0;
  a.nlimbs = nlimbs;
  a.fin = static_cast<int>(fin);
  a.fout = static_cast<int>(fout);
  if (npolys == 0) return 0;
  // one launch when the limb range shares an accumulator width, else one per limb
  bool uniform = true;
  for (uint32_t l = 1; l < nlimbs; ++l) uniform &= p->bs[limb0 + l] == p->bs[limb0];
  const uint32_t runs = uniform ? 1 : nlimbs;
  for (uint32_t l = 0; l < runs; ++l) {
    nk::NttArgs b = a;
    if (uniform) {
      b.rows = static_cast<uint64_t>(npolys) * nlimbs;
      b.row_mul = 1;
      b.row_add = 0;
    } else {
      b.rows = npolys;
      b.row_mul = nlimbs;
      b.row_add = l;
    }
    const int bs = p->bs[limb0 + (uniform ? 0 : l)];
    const uint64_t words = static_cast<uint64_t>(npolys) * nlimbs * p->n;
    int rc;
    // beta = 2^52: signed FP64 arithmetic when only the canonical result is
    // observable (fout == 1 and one kernel holds the whole row), else the
    // reference's exact lazy representatives (nk::Arith52P)
    const bool canon = (b.fout == 1) && (b.logn <= kLogBlock) && !nk::rt::exact_only;
    if (bs == 52 && canon)
      rc = fwd ? run_ntt<nk::Arith52S, true>(b, words, st) : run_ntt<nk::Arith52S, false>(b, words, st);
    else if (bs == 52)
      rc = fwd ? run_ntt<nk::Arith52P, true>(b, words, st) : run_ntt<nk::Arith52P, false>(b, words, st);
    else if (b.fout == 1 && !nk::rt::exact_only && max_q(p, limb0 + (uniform ? 0 : l), uniform ? nlimbs : 1) < (uint64_t{1} << 60))
      // beta = 2^64, canonical result only: loose Shoup quotients (nk::ArithIntL)
      rc = fwd ? run_ntt<nk::ArithIntL, true>(b, words, st) : run_ntt<nk::ArithIntL, false>(b, words, st);
    else
      rc = fwd ? run_ntt<nk::ArithInt<64>, true>(b, words, st)
               : run_ntt<nk::ArithInt<64>, false>(b, words, st);
    if (rc) return rc;
  }
  return 0;
}

// loose Barrett quotients (eltwise_kernels.cuh) need 5q < 2^63
bool loose_barrett(uint64_t q) { return u128{5} * q < (u128{1} << 63); }

}  // namespace

// ---------------------------------------------------------------------------
// testing aid: single butterflies in each arithmetic policy (nk_debug_butterflies)
// ---------------------------------------------------------------------------
namespace nk {
template <class A, bool FWD, bool SIGNED_IO, bool SKIP = false>
__global__ void bfly_test_kernel(const uint64_t* x0, const uint64_t* x1, uint64_t n, ulonglong2 w,
                                 LimbConstDev c, uint64_t* y0, uint64_t* y1) {
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t a, b;
  if (SIGNED_IO) {  // Arith52S words are signed doubles: int64 in and out
    a = as_u(static_cast<double>(static_cast<int64_t>(x0[i])));
    b = as_u(static_cast<double>(static_cast<int64_t>(x1[i])));
  } else {
    a = A::load(x0[i]);
    b = A::load(x1[i]);
  }
  typename A::Tw wt;
  if constexpr (std::is_same_v<typename A::Tw, uint64_t>) wt = w.x;  // w only (Arith52S)
  else wt = w;
  if (FWD) A::template fwd<SKIP>(a, b, wt, c);  // SKIP: a stage without its conditional subtraction
  else A::template inv<SKIP>(a, b, wt, c);
  if (SIGNED_IO) {
    y0[i] = static_cast<uint64_t>(static_cast<int64_t>(as_d(a)));
    y1[i] = static_cast<uint64_t>(static_cast<int64_t>(as_d(b)));
  } else {
    y0[i] = A::store(a);
    y1[i] = A::store(b);
  }
}
}  // namespace nk

namespace {
template <class A, bool SIGNED_IO, bool SKIP = false>
int run_bfly_test(bool fwd, const uint64_t* x0, const uint64_t* x1, uint64_t n, ulonglong2 w,
                  const nk::LimbConstDev& c, uint64_t* y0, uint64_t* y1) {
  const unsigned grid = static_cast<unsigned>((n + 255) / 256);
  if (fwd) nk::bfly_test_kernel<A, true, SIGNED_IO, SKIP><<<grid, 256>>>(x0, x1, n, w, c, y0, y1);
  else nk::bfly_test_kernel<A, false, SIGNED_IO><<<grid, 256>>>(x0, x1, n, w, c, y0, y1);
  nk::rt::launches++;
  NK_CUDA(cudaGetLastError());
  return 0;
}
}  // namespace

// ---------------------------------------------------------------------------
// host-only entry points
// ---------------------------------------------------------------------------
extern "C" {

const char* nk_last_error(void) { return nk::rt::g_err.c_str(); }
const char* nk_version(void) { return "nttkit_b200 0.1 (sm_100a)"; }
uint64_t nk_launch_count(void) { return nk::rt::launches.load(); }
void nk_debug_dump_to(uint64_t* d_buf) { nk::rt::dbg = d_buf; }
void nk_debug_exact_only(int on) { nk::rt::exact_only = on != 0; }
int nk_debug_butterflies(int policy, int fwd, uint64_t q, uint64_t w, const uint64_t* d_x0, const uint64_t* d_x1,
                         uint64_t n, uint64_t* d_y0, uint64_t* d_y1) {
  nk::host::Modulus m;
  if (!valid_modulus(q, &m)) return fail(NK_ERR_MODULUS, "Modulus: value must be a prime in [3, 2^62)");
  if (w >= q) return fail(NK_ERR_ROOT, "debug_butterflies: twiddle must be < q");
  const bool b52 = policy == 1 || policy == 2 || policy == 3 || policy == 5;
  if (policy < 0 || policy > 6) return fail(NK_ERR_BIT_SHIFT, "debug_butterflies: policy must be 0..6");
  if (b52 && u128{4} * q >= (u128{1} << 52))
    return fail(NK_ERR_BIT_SHIFT_52, "NttTables: 52-bit accumulator requires 4q < 2^52");
  if ((policy == 4 || policy == 6) && q >= (uint64_t{1} << 60))
    return fail(NK_ERR_MODULUS, "debug_butterflies: the loose policy requires q < 2^60");
  if (n == 0) return 0;
  if (!d_x0 || !d_x1 || !d_y0 || !d_y1) return fail(NK_ERR_NULL, "debug_butterflies: NULL buffer");
  const int bs = b52 ? 52 : 64;
  const uint64_t wp = static_cast<uint64_t>((static_cast<u128>(w) << bs) / q);
  const bool fp = policy == 2 || policy == 3 || policy == 5;
  auto enc = [fp](uint64_t x) { return fp ? dbits(static_cast<double>(x)) : x; };
  nk::LimbConstDev c{};
  c.q = q;
  c.twoq = 2 * q;
  c.negq = ~q + 1;
  c.qq = std::ldexp(static_cast<double>(q), -52);
  c.twoq_d = static_cast<double>(2 * q);
  c.bs = bs;
  c.q_d = static_cast<double>(q);
  c.qinv = 1.0 / static_cast<double>(q);
  c.q_bias = static_cast<double>(q) + 4503599627370496.0;
  c.fourq = 4 * q;
  const ulonglong2 tw = make_ulonglong2(policy == 3 || policy == 5 ? balanced8(enc(w), q) : enc(w), enc(wp));
  const bool f = fwd != 0;
  switch (policy) {
    case 0: return run_bfly_test<nk::ArithInt<64>, false>(f, d_x0, d_x1, n, tw, c, d_y0, d_y1);
    case 1: return run_bfly_test<nk::ArithInt<52>, false>(f, d_x0, d_x1, n, tw, c, d_y0, d_y1);
    case 2: return run_bfly_test<nk::Arith52P, false>(f, d_x0, d_x1, n, tw, c, d_y0, d_y1);
    case 3: return run_bfly_test<nk::Arith52S, true>(f, d_x0, d_x1, n, tw, c, d_y0, d_y1);
    case 5: return run_bfly_test<nk::Arith52S, true, true>(f, d_x0, d_x1, n, tw, c, d_y0, d_y1);
    case 6: return run_bfly_test<nk::ArithIntL, false, true>(f, d_x0, d_x1, n, tw, c, d_y0, d_y1);
    default: return run_bfly_test<nk::ArithIntL, false>(f, d_x0, d_x1, n, tw, c, d_y0, d_y1);
  }
}

int nk_precompute_factor(uint64_t w, uint64_t q, int bit_shift, uint64_t* precon) {
  nk::host::Modulus m;
  if (!valid_modulus(q, &m)) return fail(NK_ERR_MODULUS, "Modulus: value must be a prime in [3, 2^62)");
  if (bit_shift != 52 && bit_shift != 64)
    return fail(NK_ERR_BIT_SHIFT, "NttTables: accumulator width must be 52 or 64");
  if (w >= q) return fail(NK_ERR_FACTOR_OPERAND, "precompute_factor: operand must be < q");
  if (u128{q} * 4 > (u128{1} << bit_shift))
    return fail(NK_ERR_BETA, "precompute_factor: requires q < beta/4");
  if (precon) *precon = static_cast<uint64_t>((static_cast<u128>(w) << bit_shift) / q);
  return 0;
}

int nk_harvey_butterflies(int fwd, uint64_t q, int bit_shift, uint64_t w, uint64_t precon, const uint64_t* x0,
                          const uint64_t* x1, uint64_t n, uint64_t* y0, uint64_t* y1, int device) {
  uint64_t wp = 0;
  if (int rc = nk_precompute_factor(w, q, bit_shift, &wp)) return rc;
  if (precon != wp) return fail(NK_ERR_FACTOR_OPERAND, "harvey butterfly: precon does not match the operand");
  if (n == 0) return 0;
  if (!x0 || !x1 || !y0 || !y1) return fail(NK_ERR_NULL, "harvey butterfly: NULL buffer");
  const uint64_t bound = (fwd ? 4 : 2) * q;  // ntt.hpp:144 / 161
  for (uint64_t i = 0; i < n; ++i)
    if (x0[i] >= bound || x1[i] >= bound)
      return fail(NK_ERR_RANGE, fwd ? "harvey_forward_butterfly: inputs must be < 4q"
                                    : "harvey_inverse_butterfly: inputs must be < 2q");
  DeviceScope ds;
  if (int rc = ds.enter(device)) return rc;
  uint64_t* d = nullptr;
  NK_CUDA(cudaMalloc(&d, 4 * n * sizeof(uint64_t)));
  int rc = 0;
  cudaError_t e = cudaMemcpy(d, x0, n * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(d + n, x1, n * 8, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) rc = cuda_fail(e, "cudaMemcpy(H2D)");
  // the reference's exact integer arithmetic for the width (ArithInt<52/64>)
  if (!rc) rc = nk_debug_butterflies(bit_shift == 52 ? 1 : 0, fwd, q, w, d, d + n, n, d + 2 * n, d + 3 * n);
  if (!rc) {
    e = cudaMemcpy(y0, d + 2 * n, n * 8, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(y1, d + 3 * n, n * 8, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaMemcpy(D2H)");
  }
  cudaFree(d);
  return rc;
}

void nk_debug_block_kernel(int which) {
  nk::rt::no_lat = (which == 6);
  nk::rt::block_kernel = (which >= 0 && which <= 3) ? which : -1;  // 3: defaults, but poly_mult_mod by poly_mul14
}

int nk_modulus(uint64_t q, uint32_t* bits, uint64_t* barrett_factor) {
  nk::host::Modulus m;
  if (!nk::host::make_modulus(q, &m))
    return fail(NK_ERR_MODULUS, "Modulus: value must be a prime in [3, 2^62)");
  if (bits) *bits = m.bits;
  if (barrett_factor) *barrett_factor = m.barrett;
  return 0;
}

int nk_minimal_primitive_root(uint64_t order, uint64_t q, uint64_t* root) {
  nk::host::Modulus m;
  if (!nk::host::make_modulus(q, &m))
    return fail(NK_ERR_MODULUS, "Modulus: value must be a prime in [3, 2^62)");
  const uint64_t r = nk::host::minimal_primitive_root(order, q);
  if (!r)
    return fail(NK_ERR_Q_MOD_2N,
                "minimal_primitive_root: order must be a power of two dividing q-1");
  if (root) *root = r;
  return 0;
}

int nk_tables_host(uint64_t n, uint64_t q, const uint64_t* root, int bit_shift, uint64_t* psi,
                   uint64_t* w, uint64_t* wp, uint64_t* wi, uint64_t* wip, uint64_t* ninv,
                   uint64_t* ninvp, int* bs_out) {
  nk::host::Tables t;
  std::string msg;
  if (int rc = nk::host::build_tables(n, q, root, bit_shift, &t, &msg)) return fail(rc, msg);
  if (psi) *psi = t.psi;
  if (w) std::memcpy(w, t.w.data(), n * 8);
  if (wp) std::memcpy(wp, t.wp.data(), n * 8);
  if (wi) std::memcpy(wi, t.wi.data(), n * 8);
  if (wip) std::memcpy(wip, t.wip.data(), n * 8);
  if (ninv) *ninv = t.ninv;
  if (ninvp) *ninvp = t.ninvp;
  if (bs_out) *bs_out = t.bs;
  return 0;
}

// ---------------------------------------------------------------------------
// plans
// ---------------------------------------------------------------------------
void nk_plan_destroy(nk_plan* p) {
  if (!p) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(p->device);
  cudaFree(p->slab);  // every twiddle table
  cudaFree(p->lc);
  for (auto* m : p->mc) cudaFree(m);
  cudaSetDevice(cur);
  delete p;
}

int nk_plan_create(nk_plan** out, int device, uint64_t n, const uint64_t* moduli,
                   const uint64_t* roots, uint32_t nlimbs, int bit_shift) {
  if (!out || !moduli) return fail(NK_ERR_NULL, "nk_plan_create: NULL argument");
  *out = nullptr;
  if (nlimbs == 0) return fail(NK_ERR_LIMB, "nk_plan_create: at least one modulus is required");
  // host tables first: argument errors are reported before any device work
  std::vector<nk::host::Tables> tabs(nlimbs);
  std::string msg;
  for (uint32_t l = 0; l < nlimbs; ++l)
    if (int rc = nk::host::build_tables(n, moduli[l], roots ? &roots[l] : nullptr, bit_shift,
                                        &tabs[l], &msg))
      return fail(rc, msg);
  DeviceScope ds;
  if (int rc = ds.enter(device)) return rc;
  nk_plan* p = new nk_plan();
  p->device = device;
  p->n = n;
  p->logn = tabs[0].logn;
  p->nlimbs = nlimbs;
  std::vector<ulonglong2> hf(n * nlimbs), hi(n * nlimbs), hlf(n * nlimbs), hli(n * nlimbs);
  const bool blocks = n >= (uint64_t{1} << 14);
  std::vector<ulonglong2> hgf(blocks ? n * nlimbs : 0), hgi(blocks ? n * nlimbs : 0);
  const uint64_t qper = (n >> 14) * nk::kStrTableWords;  // two-stream table entries per limb
  std::vector<ulonglong2> hqf(blocks ? qper * nlimbs : 0), hqi(blocks ? qper * nlimbs : 0);
  std::vector<nk::LimbConst> hl(nlimbs);
  std::vector<nk::MultConst> hm[3];
  for (auto& v : hm) v.resize(nlimbs);
  for (uint32_t l = 0; l < nlimbs; ++l) {
    const auto& t = tabs[l];
    p->q.push_back(t.q);
    p->psi.push_back(t.psi);
    p->bs.push_back(t.bs);
    // beta = 2^52 limbs run on the FP64 pipe (nk::Arith52P / Arith52S): table words hold the
    // doubles' bit patterns (exact: every value is below 2^52)
    const bool fp = (t.bs == 52);
    auto enc = [fp](uint64_t x) { return fp ? dbits(static_cast<double>(x)) : x; };
    for (uint64_t i = 0; i < n; ++i) {
      hf[l * n + i] = make_ulonglong2(enc(t.w[i]), enc(t.wp[i]));
      hi[l * n + i] = make_ulonglong2(enc(t.wi[i]), enc(t.wip[i]));
    }
    if (n >= (uint64_t{1} << 14)) {  // per 16384-word block (nk::low_index)
      for (uint64_t blk = 0; blk < (n >> 14); ++blk)
        for (int b = 0; b < 5; ++b)
          for (uint64_t d = 0; d < (uint64_t{1} << (4 - b)); ++d)
            for (uint64_t jhi = 0; jhi < 512; ++jhi) {
              const uint64_t src = (n >> (b + 1)) + (((blk << 9) + jhi) << (4 - b)) + d;
              const uint64_t dst = (blk << 14) + nk::low_index(b, static_cast<int>(d), static_cast<uint32_t>(jhi));
              hlf[l * n + dst] = hf[l * n + src];
              hli[l * n + dst] = hi[l * n + src];
            }
      // thread order of the group-exchange kernels' low pass (forward P3, inverse P1)
      for (uint64_t blk = 0; blk < (n >> 14); ++blk)
        for (int b = 0; b < 5; ++b)
          for (int d = 0; d < (1 << (4 - b)); ++d)
            for (uint32_t t = 0; t < 512; ++t) {
              const uint64_t dst = l * n + (blk << 14) + nk::low_index(b, d, t);
              const uint32_t jf = nk::GrpMap<true>::jt3(t >> 5, t & 31u) >> 5;
              const uint32_t ji = nk::GrpMap<false>::jt1(t >> 5, t & 31u) >> 5;
              hgf[dst] = hlf[l * n + (blk << 14) + nk::low_index(b, d, jf)];
              hgi[dst] = hli[l * n + (blk << 14) + nk::low_index(b, d, ji)];
            }
      for (uint64_t blk = 0; blk < (n >> 14); ++blk)
        for (uint32_t S = 0; S < 2; ++S)
          for (int e = 0; e < nk::kStrEntries; ++e)
            for (uint32_t t = 0; t < 512; ++t) {
              const uint64_t dst = l * qper + blk * nk::kStrTableWords + (S * nk::kStrEntries + e) * 512 + t;
              const uint64_t src = l * n + nk::str_tw_index(n, blk << 14, S, e, t);
              hqf[dst] = hf[src];
              hqi[dst] = hi[src];
            }
    }
    // -q modulo 2^64 (the 52-bit negated modulus of ntt.hpp:85-92 agrees modulo 2^52,
    // see modmath.cuh)
    // folded last inverse stage: n^-1 * w_1 (w_1 = inverse table entry 1)
    const uint64_t nw = static_cast<uint64_t>(static_cast<u128>(t.ninv) * t.wi[1] % t.q);
    const uint64_t nwp = static_cast<uint64_t>((static_cast<u128>(nw) << t.bs) / t.q);
    hl[l] = nk::LimbConst{t.q, 2 * t.q, ~t.q + 1, enc(t.ninv), enc(t.ninvp),
                          std::ldexp(static_cast<double>(t.q), -52), static_cast<double>(2 * t.q),
                          t.bs, 0, static_cast<double>(t.q), 1.0 / static_cast<double>(t.q),
                          static_cast<double>(t.q) + 4503599627370496.0, enc(nw), enc(nwp), 4 * t.q,
                          fp ? bal_d(t.ninv, t.q) : 0.0, fp ? bal_d(nw, t.q) : 0.0};
    nk::host::Modulus m;
    nk::host::make_modulus(t.q, &m);
    const int fins[3] = {1, 2, 4};
    for (int f = 0; f < 3; ++f) hm[f][l] = nk::MultConst{t.q, 2 * t.q, m.barrett, m.bits - 1, fins[f]};
  }
  auto cleanup = [&](int rc) { nk_plan_destroy(p); return rc; };
  cudaError_t e;
  // One slab for every twiddle table, packed back to back with a different
  // 256-byte-multiple skew in front of each (one allocation to manage, and the
  // tables' relative placement is the same for every plan of a shape). Measured:
  // poly_mult_mod's time still varies by ~5% between otherwise identical plans
  // (589..619 us on cfg5) with the physical pages the slab lands on.
  {
    struct Slot { void** p; size_t bytes; };
    const size_t b16 = hf.size() * sizeof(ulonglong2), b8 = hf.size() * 8;
    const size_t q16 = hqf.size() * sizeof(ulonglong2), q8 = hqf.size() * 8;
    const size_t g16 = hgf.size() * sizeof(ulonglong2), g8 = hgf.size() * 8;
    Slot slots[] = {{reinterpret_cast<void**>(&p->tw8_fwd), b8},   {reinterpret_cast<void**>(&p->tw8_inv), b8},
                    {reinterpret_cast<void**>(&p->twq8_fwd), q8},  {reinterpret_cast<void**>(&p->twq8_inv), q8},
                    {reinterpret_cast<void**>(&p->twg8_fwd), g8},  {reinterpret_cast<void**>(&p->twg8_inv), g8},
                    {reinterpret_cast<void**>(&p->twl8_fwd), b8},  {reinterpret_cast<void**>(&p->twl8_inv), b8},
                    {reinterpret_cast<void**>(&p->tw_fwd), b16},   {reinterpret_cast<void**>(&p->tw_inv), b16},
                    {reinterpret_cast<void**>(&p->twq_fwd), q16},  {reinterpret_cast<void**>(&p->twq_inv), q16},
                    {reinterpret_cast<void**>(&p->twg_fwd), g16},  {reinterpret_cast<void**>(&p->twg_inv), g16},
                    {reinterpret_cast<void**>(&p->twl_fwd), b16},  {reinterpret_cast<void**>(&p->twl_inv), b16}};
    size_t total = 0, idx = 0;
    for (const Slot& sl : slots) total += ((sl.bytes + 255) & ~size_t{255}) + 256 * (++idx);
    if ((e = cudaMalloc(&p->slab, total))) return cleanup(cuda_fail(e, "cudaMalloc(plan tables)"));
    size_t off = 0;
    idx = 0;
    for (const Slot& sl : slots) {
      off += 256 * (++idx);
      *sl.p = sl.bytes ? static_cast<char*>(p->slab) + off : nullptr;
      off += (sl.bytes + 255) & ~size_t{255};
    }
  }
  if ((e = cudaMalloc(&p->lc, hl.size() * sizeof(nk::LimbConst))))
    return cleanup(cuda_fail(e, "cudaMalloc(plan tables)"));
  for (int f = 0; f < 3; ++f)
    if ((e = cudaMalloc(&p->mc[f], nlimbs * sizeof(nk::MultConst))))
      return cleanup(cuda_fail(e, "cudaMalloc(plan consts)"));
  // uploads on a private stream, complete before the plan is returned: a first
  // call on any stream (blocking or not) reads finished tables
  cudaStream_t up = nullptr;
  if ((e = cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking))) return cleanup(cuda_fail(e, "cudaStreamCreate(plan upload)"));
  auto put = [&](void* dst, const void* src, size_t bytes) {
    return e == cudaSuccess ? (e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, up)) : e;
  };
  put(p->twl_fwd, hlf.data(), hlf.size() * sizeof(ulonglong2));
  put(p->twl_inv, hli.data(), hli.size() * sizeof(ulonglong2));
  put(p->tw_fwd, hf.data(), hf.size() * sizeof(ulonglong2));
  put(p->tw_inv, hi.data(), hi.size() * sizeof(ulonglong2));
  // the w halves of the beta = 2^52 entries (double bits; other limbs' words are unused)
  std::vector<uint64_t> h8[8];
  const std::vector<ulonglong2>* src8[8] = {&hf, &hi, &hlf, &hli, &hgf, &hgi, &hqf, &hqi};
  // ... stored BALANCED, w in (-q/2, q/2] (w - q for 2w > q, the same residue): |w v| < 2q^2 for
  // |v| < 4q, the range of the signed policy's integer-grid quotient (modmath.cuh, mul_recip_fine)
  for (int i = 0; i < 8; ++i) {
    h8[i].resize(src8[i]->size());
    const size_t per_limb = h8[i].size() / nlimbs;
    for (size_t k = 0; k < h8[i].size(); ++k) {
      const uint32_t l = static_cast<uint32_t>(k / per_limb);
      h8[i][k] = p->bs[l] == 52 ? balanced8((*src8[i])[k].x, p->q[l]) : (*src8[i])[k].x;
    }
  }
  put(p->tw8_fwd, h8[0].data(), h8[0].size() * 8);
  put(p->tw8_inv, h8[1].data(), h8[1].size() * 8);
  put(p->twl8_fwd, h8[2].data(), h8[2].size() * 8);
  put(p->twl8_inv, h8[3].data(), h8[3].size() * 8);
  if (blocks) {
    put(p->twg_fwd, hgf.data(), hgf.size() * sizeof(ulonglong2));
    put(p->twg_inv, hgi.data(), hgi.size() * sizeof(ulonglong2));
    put(p->twg8_fwd, h8[4].data(), h8[4].size() * 8);
    put(p->twg8_inv, h8[5].data(), h8[5].size() * 8);
    put(p->twq_fwd, hqf.data(), hqf.size() * sizeof(ulonglong2));
    put(p->twq8_fwd, h8[6].data(), h8[6].size() * 8);
    put(p->twq_inv, hqi.data(), hqi.size() * sizeof(ulonglong2));
    put(p->twq8_inv, h8[7].data(), h8[7].size() * 8);
  }
  put(p->lc, hl.data(), hl.size() * sizeof(nk::LimbConst));
  for (int f = 0; f < 3; ++f) put(p->mc[f], hm[f].data(), nlimbs * sizeof(nk::MultConst));
  const cudaError_t es = cudaStreamSynchronize(up);
  cudaStreamDestroy(up);
  if (e == cudaSuccess) e = es;
  if (e != cudaSuccess) return cleanup(cuda_fail(e, "cudaMemcpyAsync(plan tables)"));
  *out = p;
  return 0;
}

int nk_plan_info(const nk_plan* p, uint32_t limb, uint64_t* n, uint64_t* q, uint64_t* psi,
                 int* bit_shift, uint32_t* nlimbs) {
  if (!p) return fail(NK_ERR_NULL, "plan is NULL");
  if (limb >= p->nlimbs) return fail(NK_ERR_LIMB, "limb outside the plan");
  if (n) *n = p->n;
  if (q) *q = p->q[limb];
  if (psi) *psi = p->psi[limb];
  if (bit_shift) *bit_shift = p->bs[limb];
  if (nlimbs) *nlimbs = p->nlimbs;
  return 0;
}

// ---------------------------------------------------------------------------
// transforms
// ---------------------------------------------------------------------------
int nk_ntt_forward(const nk_plan* p, uint64_t* res, const uint64_t* op, uint32_t limb0,
                   uint32_t nlimbs, uint32_t npolys, uint64_t fin, uint64_t fout, void* stream) {
  if (fin != 1 && fin != 2 && fin != 4)
    return fail(NK_ERR_FWD_IN_FACTOR, "forward: input_mod_factor must be 1, 2 or 4");
  if (fout != 1 && fout != 4)
    return fail(NK_ERR_FWD_OUT_FACTOR, "forward: output_mod_factor must be 1 or 4");
  if (int rc = check_limbs(p, limb0, nlimbs)) return rc;
  if (!res || !op) return fail(NK_ERR_NULL, "forward: NULL buffer");
  if (overlap_bad(res, op, static_cast<uint64_t>(npolys) * nlimbs * p->n * 8))
    return fail(NK_ERR_OVERLAP, "forward: result and operand must alias fully or not overlap");
  DeviceScope ds;
  if (int rc = ds.enter(p->device)) return rc;
  return ntt_dispatch(p, true, res, op, limb0, nlimbs, npolys, fin, fout, S(stream));
}

int nk_ntt_inverse(const nk_plan* p, uint64_t* res, const uint64_t* op, uint32_t limb0,
                   uint32_t nlimbs, uint32_t npolys, uint64_t fin, uint64_t fout, void* stream) {
  if (fin != 1 && fin != 2)
    return fail(NK_ERR_INV_IN_FACTOR, "inverse: input_mod_factor must be 1 or 2");
  if (fout != 1 && fout != 2)
    return fail(NK_ERR_INV_OUT_FACTOR, "inverse: output_mod_factor must be 1 or 2");
  if (int rc = check_limbs(p, limb0, nlimbs)) return rc;
  if (!res || !op) return fail(NK_ERR_NULL, "inverse: NULL buffer");
  if (overlap_bad(res, op, static_cast<uint64_t>(npolys) * nlimbs * p->n * 8))
    return fail(NK_ERR_OVERLAP, "inverse: result and operand must alias fully or not overlap");
  DeviceScope ds;
  if (int rc = ds.enter(p->device)) return rc;
  return ntt_dispatch(p, false, res, op, limb0, nlimbs, npolys, fin, fout, S(stream));
}

int nk_plan_eltwise_mult_mod(const nk_plan* p, uint64_t* res, const uint64_t* a, const uint64_t* b,
                             uint32_t limb0, uint32_t nlimbs, uint32_t npolys, uint64_t fin,
                             void* stream) {
  if (int rc = check_limbs(p, limb0, nlimbs)) return rc;
  if (fin != 1 && fin != 2 && fin != 4)
    return fail(NK_ERR_MULT_FACTOR, "eltwise_mult_mod: input_mod_factor must be 1, 2 or 4");
  for (uint32_t l = 0; l < nlimbs; ++l)
    if (p->q[limb0 + l] >= (uint64_t{1} << 50) && u128{fin} * p->q[limb0 + l] >= (u128{1} << 63))
      return fail(NK_ERR_MULT_INT_RANGE, "eltwise_mult_mod_int: requires input_mod_factor*q < 2^63");
  if (!res || !a || !b) return fail(NK_ERR_NULL, "eltwise_mult_mod: NULL buffer");
  if (npolys == 0) return 0;
  DeviceScope ds;
  if (int rc = ds.enter(p->device)) return rc;
  const int fi = fin == 1 ? 0 : (fin == 2 ? 1 : 2);
  const uint64_t rows = static_cast<uint64_t>(npolys) * nlimbs;
  bool small = true;
  for (uint32_t l = 0; l < nlimbs; ++l) small &= loose_barrett(p->q[limb0 + l]);
  return nk::rt::launch_mult(res, a, b, rows * p->n, p->logn, nk::MultConst{}, p->mc[fi] + limb0, nlimbs,
                     static_cast<int>(fin), small, S(stream));
}

int nk_poly_mult_mod(const nk_plan* p, uint64_t* res, const uint64_t* f, const uint64_t* g,
                     uint32_t limb0, uint32_t nlimbs, uint32_t npolys, void* stream) {
  if (int rc = check_limbs(p, limb0, nlimbs)) return rc;
  for (uint32_t l = 0; l < nlimbs; ++l)
    if (p->q[limb0 + l] >= (uint64_t{1} << 61))
      return fail(NK_ERR_POLY_MODULUS, "poly_mult_mod: requires q < 2^61");
  if (!res || !f || !g) return fail(NK_ERR_NULL, "poly_mult_mod: NULL buffer");
  const uint64_t bytes = static_cast<uint64_t>(npolys) * nlimbs * p->n * 8;
  if (overlap_bad(res, f, bytes) || overlap_bad(res, g, bytes))
    return fail(NK_ERR_OVERLAP, "poly_mult_mod: result must alias an operand fully or not overlap");
  if (npolys == 0) return 0;
  DeviceScope ds;
  if (int rc = ds.enter(p->device)) return rc;
  cudaStream_t st = S(stream);
  // When every limb takes the signed FP64 arithmetic (N = 16384, q < 2^50)
  // the result is canonical and unique, so any schedule equals the
  // reference's fwd(1,4) x2 / mult(4) / inv(1,1) sequence (ring.hpp:28-43)
  // word for word:
  //  * one kernel (ntt_poly.cuh): both forwards, the product and the inverse
  //    on chip, 24 B of HBM traffic per coefficient (operands 16-byte aligned,
  //    for TMA);
  //  * nk_debug_block_kernel(0): three launches, canonical g^, then f^ with
  //    the product applied in the forward's store (CTA-pair kernel), then the
  //    inverse;
  //  * nk_debug_block_kernel(1) or exact_only: the reference's sequence.
  bool fused = p->logn == kLogBlock && !nk::rt::exact_only && (nk::rt::block_kernel <= 0 || nk::rt::block_kernel == 3);
  for (uint32_t l = 0; l < nlimbs; ++l) fused &= p->bs[limb0 + l] == 52;
  const bool aligned = ((reinterpret_cast<uintptr_t>(f) | reinterpret_cast<uintptr_t>(g)) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(res) & 7) == 0;
  if (fused && (nk::rt::block_kernel < 0 || nk::rt::block_kernel == 3) && aligned) {
    nk::PolyArgs pa{};
    pa.a.out = res;
    pa.a.in = f;
    pa.a.tw8 = p->tw8_fwd;
    pa.a.twg8 = p->twg8_fwd;
    pa.a.twq8 = p->twq8_fwd;
    pa.itwq8 = p->twq8_inv;
    pa.a.lc = p->lc;
    pa.a.n = p->n;
    pa.a.logn = p->logn;
    pa.a.rows = static_cast<uint64_t>(npolys) * nlimbs;
    pa.a.limb0 = limb0;
    pa.a.nlimbs = nlimbs;
    pa.a.row_mul = 1;
    pa.a.fin = 1;
    pa.a.fout = 1;
    pa.itw8 = p->tw8_inv;
    pa.itwg8 = p->twg8_inv;
    return nk::rt::run_poly_mul14(pa, f, g, st);
  }
  // Whole rows of N = 2^10 .. 2^13 whose limbs share one canonical-only
  // policy (all beta = 2^52: signed FP64; all beta = 2^64 with q < 2^60: loose
  // integer): one kernel, one CTA per row pair (ntt_polyblk.cuh), 24 B/coeff.
  // nk_debug_block_kernel(>= 0) / exact_only keep the reference's sequence.
  if (p->logn >= 10 && p->logn < kLogBlock && !nk::rt::exact_only && nk::rt::block_kernel < 0) {
    bool all52 = true, all64 = true;
    for (uint32_t l = 0; l < nlimbs; ++l) {
      all52 &= p->bs[limb0 + l] == 52;
      all64 &= p->bs[limb0 + l] == 64;
    }
    if (all52 || (all64 && max_q(p, limb0, nlimbs) < (uint64_t{1} << 60))) {
      nk::PolyBlkArgs pb{};
      pb.out = res;
      pb.f = f;
      pb.g = g;
      pb.mc = p->mc[0];
      for (nk::NttArgs* a : {&pb.fw, &pb.iv}) {
        a->lc = p->lc;
        a->n = p->n;
        a->logn = p->logn;
        a->limb0 = limb0;
        a->nlimbs = nlimbs;
        a->row_mul = 1;
        a->row_add = 0;
        a->fin = 1;
        a->fout = 1;
      }
      pb.fw.tw = p->tw_fwd;
      pb.fw.tw8 = p->tw8_fwd;
      pb.iv.tw = p->tw_inv;
      pb.iv.tw8 = p->tw8_inv;
      return nk::rt::run_poly_block(pb, static_cast<uint64_t>(npolys) * nlimbs, all52, st);
    }
  }
  uint64_t* gh = nullptr;
  NK_CUDA(cudaMallocAsync(&gh, bytes, st));
  if (fused) {
    int rc = ntt_dispatch(p, true, gh, g, limb0, nlimbs, npolys, 1, 1, st);
    if (!rc) rc = ntt_dispatch(p, true, res, f, limb0, nlimbs, npolys, 1, 1, st, gh);
    if (!rc) rc = ntt_dispatch(p, false, res, res, limb0, nlimbs, npolys, 1, 1, st);
    cudaError_t e = cudaFreeAsync(gh, st);
    if (rc) return rc;
    if (e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
    return 0;
  }
  // ring.hpp:39-42: g^ = fwd(g,1,4) first so that result may alias g. Only the canonical
  // result is observable, so unless exact_only asks for the reference's own sequence the
  // spectra are canonical too (fwd(1,1), mult(1)): the same words, and limbs below 2^60
  // then take the faster canonical-only transforms (ArithIntL).
  const uint64_t lazy = nk::rt::exact_only ? 4 : 1;
  int rc = ntt_dispatch(p, true, gh, g, limb0, nlimbs, npolys, 1, lazy, st);
  if (!rc) rc = ntt_dispatch(p, true, res, f, limb0, nlimbs, npolys, 1, lazy, st);
  if (!rc) rc = nk_plan_eltwise_mult_mod(p, res, res, gh, limb0, nlimbs, npolys, lazy, stream);
  if (!rc) rc = ntt_dispatch(p, false, res, res, limb0, nlimbs, npolys, 1, 1, st);
  cudaError_t e = cudaFreeAsync(gh, st);
  if (rc) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "cudaFreeAsync");
  return 0;
}

// ---------------------------------------------------------------------------
// element-wise (single modulus)
// ---------------------------------------------------------------------------
namespace {
// element-wise multiply paths: the dispatch of eltwise.hpp:180-188 (FP64 for
// q < 2^50, else integer Barrett) or one path forced, as the reference's
// eltwise_mult_mod_int / eltwise_mult_mod_float (eltwise.hpp:137-175)
enum MultPath { kMultAuto = 0, kMultInt = 1, kMultFloat = 2 };
constexpr uint64_t kFloatPathBound = uint64_t{1} << 50;  // eltwise.hpp:132

MultPath resolve_path(MultPath path, uint64_t q) {
  return path != kMultAuto ? path : (q < kFloatPathBound ? kMultFloat : kMultInt);
}

// Modulus(q) plus the checks of the path that runs (eltwise.hpp:141-146, 162-167)
int validate_mult(uint64_t q, uint64_t fin, nk::host::Modulus* m, MultPath path = kMultAuto) {
  if (!valid_modulus(q, m)) return fail(NK_ERR_MODULUS, "Modulus: value must be a prime in [3, 2^62)");
  if (fin != 1 && fin != 2 && fin != 4)
    return fail(NK_ERR_MULT_FACTOR, "eltwise_mult_mod: input_mod_factor must be 1, 2 or 4");
  path = resolve_path(path, q);
  if (path == kMultInt && u128{fin} * q >= (u128{1} << 63))
    return fail(NK_ERR_MULT_INT_RANGE, "eltwise_mult_mod_int: requires input_mod_factor*q < 2^63");
  if (path == kMultFloat && q >= kFloatPathBound)
    return fail(NK_ERR_MULT_FLOAT_RANGE, "eltwise_mult_mod_float: requires q < 2^50");
  return 0;
}

int eltwise_mult_path(uint64_t* res, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t q,
                      uint64_t fin, MultPath path, void* stream) {
  nk::host::Modulus m;
  if (int rc = validate_mult(q, fin, &m, path)) return rc;
  if (n == 0) return 0;
  if (!res || !a || !b) return fail(NK_ERR_NULL, "eltwise_mult_mod: NULL buffer");
  if (resolve_path(path, q) == kMultFloat)
    return nk::rt::launch_mult_float(res, a, b, n, q, static_cast<int>(fin), S(stream));
  const nk::MultConst c{q, 2 * q, m.barrett, m.bits - 1, static_cast<int>(fin)};
  return nk::rt::launch_mult(res, a, b, n, 0, c, nullptr, 1, static_cast<int>(fin), loose_barrett(q), S(stream));
}

// eltwise.hpp:236-251 (+ the automatic width of eltwise.hpp:263-271); *bs receives the width
int validate_fma(uint64_t q, uint64_t y, uint64_t fin, int bit_shift, int* bs) {
  nk::host::Modulus m;
  if (!valid_modulus(q, &m)) return fail(NK_ERR_MODULUS, "Modulus: value must be a prime in [3, 2^62)");
  *bs = bit_shift;
  if (*bs == 0) *bs = (u128{fin} * q < (u128{1} << 52)) ? 52 : 64;
  if (*bs != 52 && *bs != 64) return fail(NK_ERR_BIT_SHIFT, "eltwise_fma_mod: accumulator width must be 52 or 64");
  if (fin != 1 && fin != 2 && fin != 4 && fin != 8)
    return fail(NK_ERR_FMA_FACTOR, "eltwise_fma_mod: input_mod_factor must be 1, 2, 4 or 8");
  if (q >= (uint64_t{1} << 61)) return fail(NK_ERR_FMA_MODULUS, "eltwise_fma_mod: requires q < 2^61");
  if (y >= q) return fail(NK_ERR_FMA_SCALAR, "eltwise_fma_mod: scalar must be < q");
  if (u128{fin} * q >= (u128{1} << *bs))
    return fail(NK_ERR_FMA_WIDTH, "eltwise_fma_mod: requires input_mod_factor*q < 2^BitShift");
  return 0;
}
}  // namespace

int nk_eltwise_mult_mod(uint64_t* res, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t q,
                        uint64_t fin, void* stream) {
  return eltwise_mult_path(res, a, b, n, q, fin, kMultAuto, stream);
}

int nk_eltwise_mult_mod_int(uint64_t* res, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t q,
                            uint64_t fin, void* stream) {
  return eltwise_mult_path(res, a, b, n, q, fin, kMultInt, stream);
}

int nk_eltwise_mult_mod_float(uint64_t* res, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t q,
                              uint64_t fin, void* stream) {
  return eltwise_mult_path(res, a, b, n, q, fin, kMultFloat, stream);
}

int nk_eltwise_fma_mod(uint64_t* res, const uint64_t* a, uint64_t y, const uint64_t* z, uint64_t n,
                       uint64_t q, uint64_t fin, int bit_shift, void* stream) {
  int bs = 0;
  if (int rc = validate_fma(q, y, fin, bit_shift, &bs)) return rc;
  if (n == 0) return 0;
  if (!res || !a) return fail(NK_ERR_NULL, "eltwise_fma_mod: NULL buffer");
  const nk::FmaConst c{q, y, static_cast<uint64_t>((static_cast<u128>(y) << bs) / q),
                       static_cast<int>(fin), bs};
  return nk::rt::launch_fma(res, a, z, n, c, S(stream));
}

int nk_eltwise_add_mod(uint64_t* res, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t q,
                       void* stream) {
  nk::host::Modulus m;
  if (!valid_modulus(q, &m)) return fail(NK_ERR_MODULUS, "Modulus: value must be a prime in [3, 2^62)");
  if (n == 0) return 0;
  if (!res || !a || !b) return fail(NK_ERR_NULL, "eltwise_add_mod: NULL buffer");
  return nk::rt::launch_add(res, a, b, n, q, S(stream));
}

int nk_eltwise_neg_mod(uint64_t* res, const uint64_t* a, uint64_t n, uint64_t q, void* stream) {
  nk::host::Modulus m;
  if (!valid_modulus(q, &m)) return fail(NK_ERR_MODULUS, "Modulus: value must be a prime in [3, 2^62)");
  if (n == 0) return 0;
  if (!res || !a) return fail(NK_ERR_NULL, "eltwise_neg_mod: NULL buffer");
  return nk::rt::launch_neg(res, a, n, q, S(stream));
}

}  // extern "C"

// ---------------------------------------------------------------------------
// host-buffer wrappers: chunked H2D / kernels / D2H pipeline, then wait.
// ---------------------------------------------------------------------------
namespace {

// Pipelined host-buffer execution. The work is cut into chunks of whole
// units (polynomials for transforms, words for element-wise ops) of about
// kChunkBytes. Uploads, kernels and downloads run on three internal streams
// linked by per-slot events, with separate input and output buffers per slot:
// an upload waits only for the kernel that read its slot's inputs, a kernel
// for its upload and for the download that emptied its slot's output, so the
// two DMA directions stream back to back (PCIe is full duplex and the kernels
// are ~50x faster than the copies). Blocking: returns when the results are in
// host memory. Work previously queued on the caller's stream is ordered
// before the chunks.
constexpr uint64_t kChunkBytes = 16ull << 20;
constexpr int kMaxDepth = 4;

// chunk size and pipeline depth (buffers / internal streams); tunable through
// NK_HOST_CHUNK_MB / NK_HOST_DEPTH for measurements
uint64_t host_chunk_bytes() {
  static const uint64_t v = [] {
    const char* e = getenv("NK_HOST_CHUNK_MB");
    const long mb = e ? atol(e) : 0;
    return mb > 0 ? static_cast<uint64_t>(mb) << 20 : kChunkBytes;
  }();
  return v;
}
int host_depth() {
  static const int v = [] {
    const char* e = getenv("NK_HOST_DEPTH");
    const int d = e ? atoi(e) : 0;
    return d >= 2 && d <= kMaxDepth ? d : 3;
  }();
  return v;
}

// Parallel host memcpy for pageable buffers: a small persistent pool (the
// caller takes a share too). One copy at a time; each splits into equal parts.
class CopyPool {
 public:
  static CopyPool& get() {
    static CopyPool pool;
    return pool;
  }
  void copy(void* dst, const void* src, size_t bytes) {
    if (bytes < (size_t{1} << 20) || workers_.empty()) {
      std::memcpy(dst, src, bytes);
      return;
    }
    std::lock_guard<std::mutex> one(call_mu_);
    const int parts = static_cast<int>(workers_.size()) + 1;
    {
      std::lock_guard<std::mutex> lk(mu_);
      dst_ = static_cast<char*>(dst);
      src_ = static_cast<const char*>(src);
      bytes_ = bytes;
      parts_ = parts;
      next_ = 0;
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    run_parts();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return done_ == parts_; });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }

 private:
  CopyPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    const unsigned n = hw >= 4 ? std::min(8u, hw / 2) : 0;
    for (unsigned i = 1; i < n; ++i) workers_.emplace_back([this] { work(); });
  }
  void run_parts() {
    for (;;) {
      int part;
      char* d;
      const char* sp;
      size_t bytes;
      int parts;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (next_ >= parts_) return;
        part = next_++;
        d = dst_;
        sp = src_;
        bytes = bytes_;
        parts = parts_;
      }
      const size_t b0 = bytes * part / parts, b1 = bytes * (part + 1) / parts;
      std::memcpy(d + b0, sp + b0, b1 - b0);
      std::lock_guard<std::mutex> lk(mu_);
      if (++done_ == parts_) done_cv_.notify_all();
    }
  }
  void work() {
    uint64_t seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      run_parts();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_cv_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0;
  int parts_ = 0, next_ = 0, done_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// host memory the DMA engines can read directly (pinned / registered), as
// opposed to pageable memory the driver would stage through its own buffer
bool is_pinned(const void* p) {
  if (!p) return true;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type != cudaMemoryTypeUnregistered;
}

// One pipeline (streams, events, pinned staging buffers for pageable
// callers) per device. Host-buffer calls from several threads (the reference
// allows concurrent calls on shared tables, ntt.hpp:203-205,
// test_ntt.cpp:349-375) take turns on it: they are PCIe-bound, so
// serialising them costs no throughput, and the ordering event is never
// re-recorded by one call while another waits on it.
struct HostPipe {
  cudaStream_t s[3] = {};  // uploads, kernels, downloads
  cudaEvent_t start = nullptr;
  cudaEvent_t up[kMaxDepth] = {};    // slot's uploads done (its input staging may be refilled)
  cudaEvent_t kern[kMaxDepth] = {};  // slot's kernels done (its device inputs may be refilled)
  cudaEvent_t down[kMaxDepth] = {};  // slot's download done (its output buffer / staging may be reused)
  uint64_t* stage[kMaxDepth][3] = {};  // pinned staging: inputs 0..1, output 2
  uint64_t stage_bytes = 0;
  std::mutex mu;
};

int host_pipe(int dev, HostPipe** out) {
  static HostPipe pipes[64];
  static std::once_flag once[64];
  static cudaError_t err[64];
  std::call_once(once[dev & 63], [dev] {
    HostPipe& hp = pipes[dev & 63];
    cudaError_t e = cudaSuccess;
    for (auto& st : hp.s)
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&hp.start, cudaEventDisableTiming);
    for (int k = 0; k < kMaxDepth && e == cudaSuccess; ++k) {
      e = cudaEventCreateWithFlags(&hp.up[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&hp.kern[k], cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&hp.down[k], cudaEventDisableTiming);
    }
    err[dev & 63] = e;
  });
  if (err[dev & 63] != cudaSuccess) return cuda_fail(err[dev & 63], "host pipeline streams");
  *out = &pipes[dev & 63];
  return 0;
}

// pinned staging of at least `bytes` per slot and buffer (kept for later calls)
int stage_reserve(HostPipe* hp, uint64_t bytes) {
  if (hp->stage_bytes >= bytes) return 0;
  for (auto& slot : hp->stage)
    for (auto*& b : slot) {
      if (b) cudaFreeHost(b);
      b = nullptr;
    }
  hp->stage_bytes = 0;
  for (auto& slot : hp->stage)
    for (auto*& b : slot) NK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&b), bytes, cudaHostAllocDefault));
  hp->stage_bytes = bytes;
  return 0;
}

// fn(device input buffers of the chunk, device output buffer, first unit,
//    units in chunk, stream) -> int
// Pageable host buffers go through pinned staging: the host copies chunk c's
// inputs in (and chunk c - depth's result out) with CopyPool while the DMA
// engines move the pinned chunks, instead of the driver's serial staging.
template <class Fn>
int run_pipelined(int dev, cudaStream_t user, uint64_t units, uint64_t unit_words,
                  std::initializer_list<const uint64_t*> hin, uint64_t* hout, Fn&& fn) {
  HostPipe* hp = nullptr;
  if (int rc = host_pipe(dev, &hp)) return rc;
  std::lock_guard<std::mutex> lock(hp->mu);
  const int nin = static_cast<int>(hin.size());
  const uint64_t* in[2] = {nullptr, nullptr};
  bool in_staged[2] = {false, false};
  {
    int j = 0;
    for (const uint64_t* h : hin) {
      in[j] = h;
      in_staged[j] = !is_pinned(h);
      ++j;
    }
  }
  const bool out_staged = !is_pinned(hout);
  const uint64_t unit_bytes = unit_words * 8;
  uint64_t per = host_chunk_bytes() / unit_bytes;
  if (per < 1) per = 1;
  if (per > units) per = units;
  // Chunk schedule: full chunks, except that long runs start and end with a
  // quarter and a half chunk. The first upload and the last download are not
  // overlapped with anything, so they should be short; every chunk also costs
  // a fixed ~20-30 us (copy / kernel hand-offs), so the middle stays large.
  std::vector<uint64_t> first;  // first unit of chunk c, plus a final entry = units
  {
    std::vector<uint64_t> sizes;
    if (per >= 4 && units >= 4 * per) {
      const uint64_t q4 = per / 4, q2 = per / 2;
      sizes = {q4, q2};
      for (uint64_t mid = units - 2 * (q4 + q2); mid;) {
        const uint64_t c = mid < per ? mid : per;
        sizes.push_back(c);
        mid -= c;
      }
      sizes.push_back(q2);
      sizes.push_back(q4);
    } else {
      for (uint64_t u = 0; u < units; u += per) sizes.push_back(units - u < per ? units - u : per);
    }
    first.push_back(0);
    for (uint64_t c : sizes) first.push_back(first.back() + c);
  }
  const uint64_t nchunks = first.size() - 1;
  const bool any_staged = out_staged || in_staged[0] || in_staged[1];
  if (any_staged)
    if (int rc = stage_reserve(hp, per * unit_bytes)) return rc;
  NK_CUDA(cudaEventRecord(hp->start, user));
  cudaStream_t su = hp->s[0], sk = hp->s[1], sd = hp->s[2];
  uint64_t* buf[kMaxDepth][2] = {};
  uint64_t* obuf[kMaxDepth] = {};
  int rc = 0;
  const int nst = static_cast<int>(nchunks < static_cast<uint64_t>(host_depth()) ? nchunks : host_depth());
  {
    cudaError_t e = cudaSuccess;
    for (cudaStream_t st : {su, sk, sd})
      if (e == cudaSuccess) e = cudaStreamWaitEvent(st, hp->start, 0);
    for (int k = 0; k < nst && e == cudaSuccess; ++k) {
      for (int j = 0; j < nin && e == cudaSuccess; ++j) e = cudaMallocAsync(&buf[k][j], per * unit_bytes, su);
      if (e == cudaSuccess) e = cudaMallocAsync(&obuf[k], per * unit_bytes, su);
    }
    // the kernel and download streams use the buffers after su allocated them
    if (e == cudaSuccess) e = cudaEventRecord(hp->up[0], su);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sk, hp->up[0], 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sd, hp->up[0], 0);
    if (e != cudaSuccess) rc = cuda_fail(e, "host pipeline buffers");
  }
  auto chunk_of = [&](uint64_t c, uint64_t& off, uint64_t& bytes, uint64_t& u0, uint64_t& nu) {
    u0 = first[c];
    nu = first[c + 1] - u0;
    off = u0 * unit_words;
    bytes = nu * unit_bytes;
  };
  // copy chunk c's result from its slot's output staging to the caller's buffer
  auto drain = [&](uint64_t c) -> int {
    if (!out_staged) return 0;
    const int k = static_cast<int>(c % nst);
    uint64_t off, bytes, u0, nu;
    chunk_of(c, off, bytes, u0, nu);
    NK_CUDA(cudaEventSynchronize(hp->down[k]));
    CopyPool::get().copy(hout + off, hp->stage[k][2], bytes);
    return 0;
  };
  for (uint64_t c = 0; c < nchunks && !rc; ++c) {
    const int k = static_cast<int>(c % nst);
    const bool reuse = c >= static_cast<uint64_t>(nst);  // slot k held chunk c - nst
    uint64_t off, bytes, u0, nu;
    chunk_of(c, off, bytes, u0, nu);
    if (reuse) {
      if ((rc = drain(c - nst))) break;  // the slot's previous result is out of its staging
      if (in_staged[0] || in_staged[1]) {
        const cudaError_t e = cudaEventSynchronize(hp->up[k]);  // its previous uploads are done
        if (e != cudaSuccess) { rc = cuda_fail(e, "cudaEventSynchronize(host pipeline)"); break; }
      }
    }
    // uploads: after the kernels that read the slot's previous inputs
    cudaError_t e = reuse ? cudaStreamWaitEvent(su, hp->kern[k], 0) : cudaSuccess;
    for (int j = 0; j < nin && e == cudaSuccess; ++j) {
      if (!in[j]) continue;
      const uint64_t* src = in[j] + off;
      if (in_staged[j]) {
        CopyPool::get().copy(hp->stage[k][j], src, bytes);
        src = hp->stage[k][j];
      }
      e = cudaMemcpyAsync(buf[k][j], src, bytes, cudaMemcpyHostToDevice, su);
    }
    if (e == cudaSuccess) e = cudaEventRecord(hp->up[k], su);
    if (e != cudaSuccess) { rc = cuda_fail(e, "cudaMemcpyAsync(H2D)"); break; }
    // kernels: after the uploads, and after the download that emptied the slot's output
    e = cudaStreamWaitEvent(sk, hp->up[k], 0);
    if (e == cudaSuccess && reuse) e = cudaStreamWaitEvent(sk, hp->down[k], 0);
    if (e != cudaSuccess) { rc = cuda_fail(e, "cudaStreamWaitEvent(host pipeline)"); break; }
    if ((rc = fn(buf[k], obuf[k], u0, nu, sk))) break;
    e = cudaEventRecord(hp->kern[k], sk);
    // download: after the kernels
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sd, hp->kern[k], 0);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(out_staged ? hp->stage[k][2] : hout + off, obuf[k], bytes, cudaMemcpyDeviceToHost, sd);
    if (e == cudaSuccess) e = cudaEventRecord(hp->down[k], sd);
    if (e != cudaSuccess) rc = cuda_fail(e, "cudaMemcpyAsync(D2H)");
  }
  if (!rc)
    for (uint64_t c = nchunks > static_cast<uint64_t>(nst) ? nchunks - nst : 0; c < nchunks && !rc; ++c)
      rc = drain(c);
  // every use of the buffers precedes the last download in sd's order only
  // through events; join the other streams into sd before freeing
  {
    cudaError_t e = cudaEventRecord(hp->up[0], su);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sd, hp->up[0], 0);
    if (e == cudaSuccess) e = cudaEventRecord(hp->kern[0], sk);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(sd, hp->kern[0], 0);
    for (int k = 0; k < nst; ++k) {
      for (int j = 0; j < nin; ++j)
        if (buf[k][j]) cudaFreeAsync(buf[k][j], sd);
      if (obuf[k]) cudaFreeAsync(obuf[k], sd);
    }
    for (cudaStream_t st : {su, sk, sd}) {
      const cudaError_t e2 = cudaStreamSynchronize(st);
      if (e == cudaSuccess) e = e2;
    }
    if (!rc && e != cudaSuccess) rc = cuda_fail(e, "cudaStreamSynchronize(host pipeline)");
  }
  return rc;
}

int ntt_host(bool fwd, const nk_plan* p, uint64_t* res, const uint64_t* op, uint64_t length,
             uint32_t limb0, uint32_t nlimbs, uint32_t npolys, uint64_t fin, uint64_t fout,
             void* stream) {
  if (!p) return fail(NK_ERR_NULL, "plan is NULL");
  const uint64_t words = static_cast<uint64_t>(npolys) * nlimbs * p->n;
  if (length != words) return fail(NK_ERR_LENGTH, "transform: buffer length must equal n");
  if (!res || !op) return fail(NK_ERR_NULL, "transform: NULL buffer");
  if (npolys == 0) return 0;
  DeviceScope ds;
  if (int rc = ds.enter(p->device)) return rc;
  return run_pipelined(p->device, S(stream), npolys, static_cast<uint64_t>(nlimbs) * p->n, {op}, res,
                       [&](uint64_t* const* d, uint64_t* o, uint64_t, uint64_t nu, cudaStream_t st) {
                         const uint32_t np = static_cast<uint32_t>(nu);
                         return fwd ? nk_ntt_forward(p, o, d[0], limb0, nlimbs, np, fin, fout, st)
                                    : nk_ntt_inverse(p, o, d[0], limb0, nlimbs, np, fin, fout, st);
                       });
}

}  // namespace

extern "C" {

int nk_ntt_forward_host(const nk_plan* p, uint64_t* res, const uint64_t* op, uint64_t length,
                        uint32_t limb0, uint32_t nlimbs, uint32_t npolys, uint64_t fin,
                        uint64_t fout, void* stream) {
  if (fin != 1 && fin != 2 && fin != 4)
    return fail(NK_ERR_FWD_IN_FACTOR, "forward: input_mod_factor must be 1, 2 or 4");
  if (fout != 1 && fout != 4)
    return fail(NK_ERR_FWD_OUT_FACTOR, "forward: output_mod_factor must be 1 or 4");
  return ntt_host(true, p, res, op, length, limb0, nlimbs, npolys, fin, fout, stream);
}

int nk_ntt_inverse_host(const nk_plan* p, uint64_t* res, const uint64_t* op, uint64_t length,
                        uint32_t limb0, uint32_t nlimbs, uint32_t npolys, uint64_t fin,
                        uint64_t fout, void* stream) {
  if (fin != 1 && fin != 2)
    return fail(NK_ERR_INV_IN_FACTOR, "inverse: input_mod_factor must be 1 or 2");
  if (fout != 1 && fout != 2)
    return fail(NK_ERR_INV_OUT_FACTOR, "inverse: output_mod_factor must be 1 or 2");
  return ntt_host(false, p, res, op, length, limb0, nlimbs, npolys, fin, fout, stream);
}

int nk_poly_mult_mod_host(const nk_plan* p, uint64_t* res, const uint64_t* f, const uint64_t* g,
                          uint64_t length, uint32_t limb0, uint32_t nlimbs, uint32_t npolys,
                          void* stream) {
  if (!p) return fail(NK_ERR_NULL, "plan is NULL");
  const uint64_t words = static_cast<uint64_t>(npolys) * nlimbs * p->n;
  if (length != words) return fail(NK_ERR_LENGTH, "poly_mult_mod: operand lengths must equal n");
  if (!res || !f || !g) return fail(NK_ERR_NULL, "poly_mult_mod: NULL buffer");
  for (uint32_t l = 0; l < nlimbs && limb0 + l < p->nlimbs; ++l)
    if (p->q[limb0 + l] >= (uint64_t{1} << 61))
      return fail(NK_ERR_POLY_MODULUS, "poly_mult_mod: requires q < 2^61");
  if (npolys == 0) return 0;
  DeviceScope ds;
  if (int rc = ds.enter(p->device)) return rc;
  return run_pipelined(p->device, S(stream), npolys, static_cast<uint64_t>(nlimbs) * p->n, {f, g}, res,
                       [&](uint64_t* const* d, uint64_t* o, uint64_t, uint64_t nu, cudaStream_t st) {
                         return nk_poly_mult_mod(p, o, d[0], d[1], limb0, nlimbs, static_cast<uint32_t>(nu),
                                                 st);
                       });
}

namespace {
int eltwise_mult_host(uint64_t* res, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t q,
                      uint64_t fin, MultPath path, int device, void* stream) {
  if (!res || !a || !b) return fail(NK_ERR_NULL, "eltwise_mult_mod: NULL buffer");
  nk::host::Modulus m;
  if (int rc = validate_mult(q, fin, &m, path)) return rc;
  if (n == 0) return 0;
  DeviceScope ds;
  if (int rc = ds.enter(device)) return rc;
  return run_pipelined(device, S(stream), n, 1, {a, b}, res,
                       [&](uint64_t* const* d, uint64_t* o, uint64_t, uint64_t nu, cudaStream_t st) {
                         return eltwise_mult_path(o, d[0], d[1], nu, q, fin, path, st);
                       });
}
}  // namespace

int nk_eltwise_add_mod_host(uint64_t* res, const uint64_t* a, const uint64_t* b, uint64_t n, uint64_t q,
                            int device, void* stream) {
  nk::host::Modulus m;
  if (!valid_modulus(q, &m)) return fail(NK_ERR_MODULUS, "Modulus: value must be a prime in [3, 2^62)");
  if (n == 0) return 0;
  if (!res || !a || !b) return fail(NK_ERR_NULL, "eltwise_add_mod: NULL buffer");
  DeviceScope ds;
  if (int rc = ds.enter(device)) return rc;
  return run_pipelined(device, S(stream), n, 1, {a, b}, res,
                       [&](uint64_t* const* d, uint64_t* o, uint64_t, uint64_t nu, cudaStream_t st) {
                         return nk_eltwise_add_mod(o, d[0], d[1], nu, q, st);
                       });
}

int nk_eltwise_neg_mod_host(uint64_t* res, const uint64_t* a, uint64_t n, uint64_t q, int device,
                            void* stream) {
  nk::host::Modulus m;
  if (!valid_modulus(q, &m)) return fail(NK_ERR_MODULUS, "Modulus: value must be a prime in [3, 2^62)");
  if (n == 0) return 0;
  if (!res || !a) return fail(NK_ERR_NULL, "eltwise_neg_mod: NULL buffer");
  DeviceScope ds;
  if (int rc = ds.enter(device)) return rc;
  return run_pipelined(device, S(stream), n, 1, {a}, res,
                       [&](uint64_t* const* d, uint64_t* o, uint64_t, uint64_t nu, cudaStream_t st) {
                         return nk_eltwise_neg_mod(o, d[0], nu, q, st);
                       });
}

int nk_eltwise_mult_mod_host(uint64_t* res, const uint64_t* a, const uint64_t* b, uint64_t n,
                             uint64_t q, uint64_t fin, int device, void* stream) {
  return eltwise_mult_host(res, a, b, n, q, fin, kMultAuto, device, stream);
}
int nk_eltwise_mult_mod_int_host(uint64_t* res, const uint64_t* a, const uint64_t* b, uint64_t n,
                                 uint64_t q, uint64_t fin, int device, void* stream) {
  return eltwise_mult_host(res, a, b, n, q, fin, kMultInt, device, stream);
}
int nk_eltwise_mult_mod_float_host(uint64_t* res, const uint64_t* a, const uint64_t* b, uint64_t n,
                                   uint64_t q, uint64_t fin, int device, void* stream) {
  return eltwise_mult_host(res, a, b, n, q, fin, kMultFloat, device, stream);
}

int nk_eltwise_fma_mod_host(uint64_t* res, const uint64_t* a, uint64_t y, const uint64_t* z,
                            uint64_t n, uint64_t q, uint64_t fin, int bit_shift, int device,
                            void* stream) {
  if (!res || !a) return fail(NK_ERR_NULL, "eltwise_fma_mod: NULL buffer");
  int bs = 0;
  if (int rc = validate_fma(q, y, fin, bit_shift, &bs)) return rc;
  if (n == 0) return 0;
  DeviceScope ds;
  if (int rc = ds.enter(device)) return rc;
  return run_pipelined(device, S(stream), n, 1, {a, z}, res,
                       [&](uint64_t* const* d, uint64_t* o, uint64_t, uint64_t nu, cudaStream_t st) {
                         return nk_eltwise_fma_mod(o, d[0], y, z ? d[1] : nullptr, nu, q, fin, bit_shift, st);
                       });
}

}  // extern "C"
