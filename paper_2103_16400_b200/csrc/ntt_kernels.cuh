// Negacyclic NTT kernels for sm_100a.
//
// Algorithm = the reference's, stage for stage (so lazy outputs match bit for
// bit): radix-2 Cooley-Tukey forward over psi powers in bit-reversed order
// (ntt.hpp:363-394), Gentleman-Sande inverse (ntt.hpp:396-433) with the
// standalone n^-1 Shoup pass (ntt.hpp:429-432), Harvey lazy butterflies.
//
// Index algebra used throughout. With N the row length and j an element index,
// the butterfly of stage "bit b" pairs j and j + 2^b (bit b of j clear) and
// uses the twiddle at table index (N + j) >> (b + 1) in BOTH directions:
//   forward, stage m = N >> (b+1), t = 2^b: w_arr[m + (j >> (b+1))]  (ntt.hpp:384-386)
//   inverse, h = N >> (b+1), t = 2^b:        w_arr[h + (j >> (b+1))]  (ntt.hpp:416-420)
// The forward runs b = logN-1 .. 0, the inverse b = 0 .. logN-1.
//
// Kernels:
//  * ntt_block<LOGB, LOGV, BS, FWD>: one CTA transforms a contiguous block of
//    2^LOGB words (a whole row when N <= 2^LOGB, else a sub-block whose high
//    bits were already handled by ntt_global_pass). Each thread holds 2^LOGV
//    words in registers; bits are processed in register passes of <= LOGV
//    stages, with the block exchanged through a padded shared-memory image
//    between passes (phys(j) = j + j>>4 + j>>8 + j>>12: additive over disjoint
//    bit fields, so every shared-memory address is a per-thread base plus an
//    immediate, and every exchange pattern used is bank-conflict free).
//    Twiddles {w, w'} are one 16-byte load each.
//  * ntt_global_pass<K, BS, FWD>: K stages on bits [lo, lo+K) of long rows
//    (N > 2^LOGB), one column of 2^K words per thread, coalesced.
//  * ntt_small<BS, FWD>: any N <= 2^14, stage-by-stage in shared memory; for the
//    small sizes the reference tests use.
#pragma once
#include <cstdint>

#include "modmath.cuh"

namespace nk {

// Per-limb constants, resident on the device with the tables.
struct LimbConst {
  uint64_t q, twoq, negq, ninv, ninvp;
  int32_t bs;
  int32_t pad;
};

struct NttArgs {
  uint64_t* out;
  const uint64_t* in;
  const ulonglong2* tw;  // [limb][N] {w, w'} of the plan (fwd or inv table)
  const LimbConst* lc;   // [limb]
  uint64_t n;            // row length
  uint64_t rows;         // npolys * nlimbs
  uint32_t limb0, nlimbs;  // row r (after remapping) holds limb limb0 + r % nlimbs
  uint32_t row_mul, row_add;  // launched row i is row i * row_mul + row_add
  uint32_t logn;
  int32_t fin, fout;
};

__device__ __forceinline__ ulonglong2 ldtw(const ulonglong2* p) { return __ldg(p); }

// Shared-memory image index, see header comment.
__host__ __device__ constexpr uint32_t smem_phys(uint32_t j) {
  return j + (j >> 4) + (j >> 8) + (j >> 12);
}

// ---------------------------------------------------------------------------
// compile-time pass schedule of the block kernel
// ---------------------------------------------------------------------------
template <int LOGB, int LOGV>
struct Sched {
  static constexpr int LOGT = LOGB - LOGV;
  static constexpr int T = 1 << LOGT;
  static constexpr int V = 1 << LOGV;
  static constexpr int NP = (LOGB + LOGV - 1) / LOGV;
  // passes in top-down (forward) order: sizes as even as possible, larger first
  __host__ __device__ static constexpr int k(int p) { return LOGB / NP + (p < LOGB % NP ? 1 : 0); }
  __host__ __device__ static constexpr int lo(int p) {
    int s = LOGB;
    for (int i = 0; i <= p; ++i) s -= k(i);
    return s;
  }
  // place outer-index bits o into the positions outside [lo, lo+k)
  __host__ __device__ static constexpr uint32_t scatter(uint32_t o, int lo_, int k_) {
    return (o & ((1u << lo_) - 1u)) | ((o >> lo_) << (lo_ + k_));
  }
};

// One pass: K butterfly bits [LO, LO+K) over G = V / 2^K independent groups held
// in v[g * 2^K + r]. xt = N + block offset + scattered thread index (bits outside
// the pass only). STAGE0_ILTM: apply the first stage of the pass with
// InputLessThanMod (reference's fin == 1 specialisation).
template <int BS, bool FWD, int LOGT, int LOGV, int LO, int K>
__device__ __forceinline__ void do_pass(uint64_t (&v)[1 << LOGV], const ulonglong2* __restrict__ tw,
                                        uint64_t xt, bool first_iltm, uint64_t twoq,
                                        uint64_t negq) {
  constexpr int R = 1 << K;
  constexpr int G = (1 << LOGV) / R;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    const int i = FWD ? (K - 1 - s) : s;  // bit within the pass
    const int b = LO + i;                 // global bit
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t jg = Sched<LOGT + LOGV, LOGV>::scatter(static_cast<uint32_t>(g) << LOGT, LO, K);
      const uint64_t base = (xt + jg) >> (b + 1);
#pragma unroll
      for (int hi = 0; hi < (R >> (i + 1)); ++hi) {
        const ulonglong2 w = ldtw(tw + base + hi);
#pragma unroll
        for (int lo = 0; lo < (1 << i); ++lo) {
          const int r0 = (hi << (i + 1)) | lo;
          const int r1 = r0 | (1 << i);
          uint64_t& x0 = v[g * R + r0];
          uint64_t& x1 = v[g * R + r1];
          if (FWD) {
            if (s == 0 && first_iltm) fwd_bfly<BS, true>(x0, x1, w.x, w.y, twoq, negq);
            else fwd_bfly<BS, false>(x0, x1, w.x, w.y, twoq, negq);
          } else {
            if (s == 0 && first_iltm) inv_bfly<BS, true>(x0, x1, w.x, w.y, twoq, negq);
            else inv_bfly<BS, false>(x0, x1, w.x, w.y, twoq, negq);
          }
        }
      }
    }
  }
}

// P-th pass in processing order.
template <int LOGB, int LOGV, bool FWD>
struct PassOf {
  using S = Sched<LOGB, LOGV>;
  __host__ __device__ static constexpr int td(int p) { return FWD ? p : (S::NP - 1 - p); }
  __host__ __device__ static constexpr int lo(int p) { return S::lo(td(p)); }
  __host__ __device__ static constexpr int k(int p) { return S::k(td(p)); }
};

template <int LOGB, int LOGV, int BS, bool FWD, int P>
__device__ __forceinline__ void run_passes(uint64_t (&v)[1 << LOGV], uint64_t* sm,
                                           const ulonglong2* __restrict__ tw, uint32_t t,
                                           uint64_t xbase, bool first_iltm, uint64_t twoq,
                                           uint64_t negq) {
  using S = Sched<LOGB, LOGV>;
  using PO = PassOf<LOGB, LOGV, FWD>;
  constexpr int LO = PO::lo(P), K = PO::k(P);
  constexpr int R = 1 << K, G = S::V / R;
  const uint32_t jt = S::scatter(t, LO, K);
  if (P > 0) {
    // exchange: pass P-1 wrote its values to sm; read this pass's pattern
    __syncthreads();
    const uint32_t bt = smem_phys(jt);
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t jc = S::scatter(static_cast<uint32_t>(g) << S::LOGT, LO, K) | (r << LO);
        v[g * R + r] = sm[bt + smem_phys(jc)];
      }
  }
  do_pass<BS, FWD, S::LOGT, LOGV, LO, K>(v, tw, xbase + jt, P == 0 && first_iltm, twoq, negq);
  if constexpr (P + 1 < S::NP) {
    __syncthreads();  // every thread has read the previous image
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t jc = S::scatter(static_cast<uint32_t>(g) << S::LOGT, LO, K) | (r << LO);
        sm[smem_phys(jt) + smem_phys(jc)] = v[g * R + r];
      }
    run_passes<LOGB, LOGV, BS, FWD, P + 1>(v, sm, tw, t, xbase, false, twoq, negq);
  }
}

template <int LOGB, int LOGV, int BS, bool FWD>
__global__ void __launch_bounds__(1 << (LOGB - LOGV))
    ntt_block(NttArgs a) {
  using S = Sched<LOGB, LOGV>;
  using PO = PassOf<LOGB, LOGV, FWD>;
  extern __shared__ uint64_t sm[];
  const uint32_t t = threadIdx.x;
  const uint32_t lognb = a.logn - LOGB;  // log2 of blocks per row
  const uint64_t row = (static_cast<uint64_t>(blockIdx.x) >> lognb) * a.row_mul + a.row_add;
  const uint64_t blk = static_cast<uint64_t>(blockIdx.x) & ((uint64_t{1} << lognb) - 1);
  const uint32_t limb = a.limb0 + static_cast<uint32_t>(row % a.nlimbs);
  const LimbConst c = a.lc[limb];
  const ulonglong2* __restrict__ tw = a.tw + static_cast<uint64_t>(limb) * a.n;
  const uint64_t boff = blk << LOGB;
  const uint64_t* __restrict__ src = a.in + row * a.n + boff;
  uint64_t* __restrict__ dst = a.out + row * a.n + boff;
  const bool whole = (lognb == 0);

  uint64_t v[S::V];
  // ---- load: first pass pattern ----
  {
    constexpr int LO = PO::lo(0), K = PO::k(0);
    constexpr int R = 1 << K, G = S::V / R;
    const uint32_t jt = S::scatter(t, LO, K);
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const uint32_t jg = S::scatter(static_cast<uint32_t>(g) << S::LOGT, LO, K);
      if constexpr (LO == 0 && R >= 2) {
#pragma unroll
        for (int r = 0; r < R; r += 2) {
          const ulonglong2 p = *reinterpret_cast<const ulonglong2*>(src + jt + jg + r);
          v[g * R + r] = p.x;
          v[g * R + r + 1] = p.y;
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) v[g * R + r] = src[jt + jg + (r << LO)];
      }
    }
  }
  const bool first_iltm = (a.fin == 1) && (FWD ? whole : true);
  run_passes<LOGB, LOGV, BS, FWD, 0>(v, sm, tw, t, a.n + boff, first_iltm, c.twoq, c.negq);

  // ---- fix-ups of the final pass and store ----
  constexpr int PL = S::NP - 1;
  constexpr int LO = PO::lo(PL), K = PO::k(PL);
  constexpr int R = 1 << K, G = S::V / R;
  if (FWD) {
    if (a.fout == 1) {
#pragma unroll
      for (int i = 0; i < S::V; ++i) v[i] = csub(csub(v[i], c.twoq), c.q);  // small_mod(x,q,4)
    }
  } else if (whole) {
#pragma unroll
    for (int i = 0; i < S::V; ++i) v[i] = mul_lazy<BS>(v[i], c.ninv, c.ninvp, c.negq);
    if (a.fout == 1) {
#pragma unroll
      for (int i = 0; i < S::V; ++i) v[i] = csub(v[i], c.q);  // small_mod(x,q,2)
    }
  }
  const uint32_t jt = S::scatter(t, LO, K);
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const uint32_t jg = S::scatter(static_cast<uint32_t>(g) << S::LOGT, LO, K);
    if constexpr (LO == 0 && R >= 2) {
#pragma unroll
      for (int r = 0; r < R; r += 2)
        *reinterpret_cast<ulonglong2*>(dst + jt + jg + r) = make_ulonglong2(v[g * R + r], v[g * R + r + 1]);
    } else {
#pragma unroll
      for (int r = 0; r < R; ++r) dst[jt + jg + (r << LO)] = v[g * R + r];
    }
  }
}

template <int LOGB, int LOGV>
constexpr size_t block_smem_bytes() {
  return Sched<LOGB, LOGV>::NP > 1 ? (smem_phys((1u << LOGB) - 1) + 1) * sizeof(uint64_t) : 0;
}

// ---------------------------------------------------------------------------
// K stages over bits [lo, lo+K) of long rows; one column per thread.
// first_iltm: forward with fin == 1 at the top stage. last: inverse final pass
// (apply n^-1 and the fout reduction).
// ---------------------------------------------------------------------------
template <int K, int BS, bool FWD>
__global__ void __launch_bounds__(256) ntt_global_pass(NttArgs a, uint32_t lo, int first_iltm,
                                                       int last) {
  constexpr int R = 1 << K;
  const uint64_t gid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint32_t logcols = a.logn - K;
  if (gid >= (a.rows << logcols)) return;
  const uint64_t row = (gid >> logcols) * a.row_mul + a.row_add;
  const uint64_t o = gid & ((uint64_t{1} << logcols) - 1);
  const uint32_t limb = a.limb0 + static_cast<uint32_t>(row % a.nlimbs);
  const LimbConst c = a.lc[limb];
  const ulonglong2* __restrict__ tw = a.tw + static_cast<uint64_t>(limb) * a.n;
  const uint64_t j0 = (o & ((uint64_t{1} << lo) - 1)) | ((o >> lo) << (lo + K));
  const uint64_t* src = a.in + row * a.n;
  uint64_t* dst = a.out + row * a.n;
  uint64_t v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) v[r] = src[j0 + (static_cast<uint64_t>(r) << lo)];
  const uint64_t xt = a.n + j0;
#pragma unroll
  for (int s = 0; s < K; ++s) {
    const int i = FWD ? (K - 1 - s) : s;
    const uint32_t b = lo + i;
    const uint64_t base = xt >> (b + 1);
#pragma unroll
    for (int hi = 0; hi < (R >> (i + 1)); ++hi) {
      const ulonglong2 w = ldtw(tw + base + hi);
#pragma unroll
      for (int l = 0; l < (1 << i); ++l) {
        const int r0 = (hi << (i + 1)) | l, r1 = r0 | (1 << i);
        if (FWD) {
          if (s == 0 && first_iltm) fwd_bfly<BS, true>(v[r0], v[r1], w.x, w.y, c.twoq, c.negq);
          else fwd_bfly<BS, false>(v[r0], v[r1], w.x, w.y, c.twoq, c.negq);
        } else {
          inv_bfly<BS, false>(v[r0], v[r1], w.x, w.y, c.twoq, c.negq);
        }
      }
    }
  }
  if (!FWD && last) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      v[r] = mul_lazy<BS>(v[r], c.ninv, c.ninvp, c.negq);
      if (a.fout == 1) v[r] = csub(v[r], c.q);
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) dst[j0 + (static_cast<uint64_t>(r) << lo)] = v[r];
}

// ---------------------------------------------------------------------------
// Any N <= 2^14: one CTA per row, whole row in shared memory, one stage at a
// time. Used for the small sizes of the reference's tests.
// ---------------------------------------------------------------------------
template <int BS, bool FWD>
__global__ void __launch_bounds__(256) ntt_small(NttArgs a) {
  extern __shared__ uint64_t sm[];
  const uint64_t row = static_cast<uint64_t>(blockIdx.x) * a.row_mul + a.row_add;
  const uint32_t limb = a.limb0 + static_cast<uint32_t>(row % a.nlimbs);
  const LimbConst c = a.lc[limb];
  const ulonglong2* __restrict__ tw = a.tw + static_cast<uint64_t>(limb) * a.n;
  const uint32_t n = static_cast<uint32_t>(a.n);
  for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) sm[j] = a.in[row * a.n + j];
  __syncthreads();
  for (uint32_t s = 0; s < a.logn; ++s) {
    const uint32_t b = FWD ? (a.logn - 1 - s) : s;
    const bool iltm = (s == 0) && (a.fin == 1);
    for (uint32_t p = threadIdx.x; p < n / 2; p += blockDim.x) {
      const uint32_t j = ((p >> b) << (b + 1)) | (p & ((1u << b) - 1u));
      const ulonglong2 w = ldtw(tw + ((a.n + j) >> (b + 1)));
      uint64_t x0 = sm[j], x1 = sm[j + (1u << b)];
      if (FWD) {
        if (iltm) fwd_bfly<BS, true>(x0, x1, w.x, w.y, c.twoq, c.negq);
        else fwd_bfly<BS, false>(x0, x1, w.x, w.y, c.twoq, c.negq);
      } else {
        if (iltm) inv_bfly<BS, true>(x0, x1, w.x, w.y, c.twoq, c.negq);
        else inv_bfly<BS, false>(x0, x1, w.x, w.y, c.twoq, c.negq);
      }
      sm[j] = x0;
      sm[j + (1u << b)] = x1;
    }
    __syncthreads();
  }
  for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) {
    uint64_t x = sm[j];
    if (FWD) {
      if (a.fout == 1) x = csub(csub(x, c.twoq), c.q);
    } else {
      x = mul_lazy<BS>(x, c.ninv, c.ninvp, c.negq);
      if (a.fout == 1) x = csub(x, c.q);
    }
    a.out[row * a.n + j] = x;
  }
}

}  // namespace nk
