// ntt_grp14: the 16384-word block transform on ONE 512-thread CTA per SM whose
// exchanges run inside groups of four warps (named barriers) instead of the
// whole CTA or a CTA pair.
//
// Why: the block is 14 stages in three register passes (5 + 4/5 + 5 stages,
// 32 words per thread). A pass's thread index bits and the next pass's share
// some index bits; the threads holding a fixed value of those common bits
// exchange only among themselves. With the thread numbering below, two of the
// common bits are warp-index bits on BOTH sides of an exchange, so each
// exchange is four independent 4-warp exchanges: a warp waits for its 3
// partners (one per SMSP), never for the slowest of 16 warps on two SMs, and
// no data crosses the SM (no DSMEM).
//
// Index bits of a block word j (regs = the register bits, w = warp bits
// (w>>2, w&3), the remaining thread bits are lane bits):
//
//   forward (stages 13..0)                  inverse (stages 0..13)
//   P1 regs 9..13   w: (2,3) (7,8)           P1 regs 0..4    w: (11,12) (7,8)
//      lanes 0 4 5 6 1                          lanes 5 6 13 9 10
//   -- ex1: groups w>>2 = j2,j3, in place     -- ex1: groups w>>2 = j11,j12, in place
//      in the TMA staging buffer --              in the TMA staging buffer --
//   P2 regs 5..8 + 4  w: (2,3) (12,13)       P2 regs 5..8 + 13  w: (11,12) (3,4)
//      lanes 0 9 10 11 1                        lanes 0 1 2 9 10
//   -- ex2: groups w&3 = j12,j13, two        -- ex2: groups w&3 = j3,j4, two
//      rounds on bit 4 through E --             rounds on bit 13 through E --
//   P3 regs 0..4    w: (7,8) (12,13)         P3 regs 9..13   w: (7,8) (3,4)
//      lanes 9 10 11 5 6                        lanes 0 1 2 5 6
//
// Exchange 1 rewrites each group's words into the group's own slots of the
// staging buffer (a permutation within the slots whose index bits w>>2 are
// fixed), after every warp of the group has read its P1 words (per-group
// mbarrier, arrived right after the reads, waited on just before the writes)
// and before the P2 reads (named barrier). The slot permutation XORs thread
// bits into the swizzled line bits so that both sides are conflict free.
// When the last of the 16 warps has read its P2 words (shared counter), that
// warp issues the next block's TMA into the staging buffer. Exchange 2 goes
// through a separate 64 KiB image E, 16 KiB per group, in two rounds split on
// a register bit common to both passes.
//
// Twiddles and butterflies are those of pass14 (ntt_kernels.cuh), including
// the transposed low table for the pass over bits 0..4.
#pragma once
#include "ntt_kernels.cuh"
#include "ntt_pair.cuh"

namespace nk {

constexpr uint32_t kGrpExBytes = 4u * 16384u;  // E: 4 groups x 2048 words
constexpr uint32_t kGrpOutBytes = 16u * 2048u;  // forward output images: 2 KiB per warp
// [1 KiB align][staging 128 KiB][E 64 KiB][O 32 KiB][limb constants x2]
// [mbarriers: full, ex1 reads x4, ex2 reads x4][counter][output images read x4]
constexpr size_t kGrpSmemBytes = 1024 + kStageBytes + kGrpExBytes + kGrpOutBytes + 2 * sizeof(LimbConst) + 16 * 8;

__device__ __forceinline__ void named_sync128(uint32_t id) {
  asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
}

__device__ __forceinline__ void st_v4_u64(uint64_t* p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}

// thread index bits (block-local j) of each pass; see the header table
template <bool FWD>
struct GrpMap;
template <>
struct GrpMap<true> {
  __host__ __device__ static constexpr uint32_t jt1(uint32_t w, uint32_t l) {
    return (l & 1u) | (((l >> 4) & 1u) << 1) | ((w >> 2) << 2) | (((l >> 1) & 7u) << 4) | ((w & 3u) << 7);
  }
  __host__ __device__ static constexpr uint32_t jt2(uint32_t w, uint32_t l) {
    return (l & 1u) | (((l >> 4) & 1u) << 1) | ((w >> 2) << 2) | (((l >> 1) & 7u) << 9) | ((w & 3u) << 12);
  }
  __host__ __device__ static constexpr uint32_t jt3(uint32_t w, uint32_t l) {
    return (((l >> 3) & 1u) << 5) | (((l >> 4) & 1u) << 6) | ((w >> 2) << 7) | ((l & 7u) << 9) | ((w & 3u) << 12);
  }
};
template <>
struct GrpMap<false> {
  __host__ __device__ static constexpr uint32_t jt1(uint32_t w, uint32_t l) {
    return ((l & 1u) << 5) | (((l >> 1) & 1u) << 6) | (((l >> 2) & 1u) << 13) | (((l >> 3) & 1u) << 9) |
           (((l >> 4) & 1u) << 10) | ((w & 3u) << 7) | ((w >> 2) << 11);
  }
  __host__ __device__ static constexpr uint32_t jt2(uint32_t w, uint32_t l) {
    return (l & 7u) | (((l >> 3) & 1u) << 9) | (((l >> 4) & 1u) << 10) | ((w & 3u) << 3) | ((w >> 2) << 11);
  }
  __host__ __device__ static constexpr uint32_t jt3(uint32_t w, uint32_t l) {
    return (l & 7u) | (((l >> 3) & 1u) << 5) | (((l >> 4) & 1u) << 6) | ((w & 3u) << 3) | ((w >> 2) << 7);
  }
};

// exchange-1 slot permutation (word j -> the staging slot of word ex1_perm(j)):
// XOR thread bits into the low line bits (swz_off's bank selector)
template <bool FWD>
__host__ __device__ __forceinline__ constexpr uint32_t ex1_perm(uint32_t j) {
  return FWD ? (j ^ (((j >> 9) & 7u) << 4)) : (j ^ (((j >> 13) & 1u) << 4) ^ (((j >> 9) & 1u) << 6));
}

// byte offset of word j in its group's 16 KiB slice of E (the slice index is
// added by the caller)
template <bool FWD>
__host__ __device__ __forceinline__ constexpr uint32_t ex2_off(uint32_t j) {
  if (FWD) {
    // row = j5..j11, 16-byte chunk (j1..j3) ^ (j9..j11), word j0
    const uint32_t row = (j >> 5) & 127u;
    const uint32_t chunk = ((j >> 1) & 7u) ^ ((j >> 9) & 7u);
    return (row << 7) | (chunk << 4) | ((j & 1u) << 3);
  } else {
    // row = (j6, j7, j8, j9, j10, j11, j12), bank word (j0, j1, j2, j5 ^ j9)
    const uint32_t row = ((j >> 6) & 7u) | (((j >> 9) & 15u) << 3);
    const uint32_t bank = (j & 7u) | ((((j >> 5) ^ (j >> 9)) & 1u) << 3);
    return (row << 7) | (bank << 3);
  }
}

namespace grp {

// P2-read base (both directions): swz_off(ex1_perm(jt2 | jc(g, r))) =
//   (q2 ^ (y * 0x90)) + (hi << 10), y = the 3 low line bits the registers
//   flip, hi = the register line bits above them (see ex1 below)
template <bool FWD>
__device__ __forceinline__ uint32_t q2_of(uint32_t jt2) {
  if (FWD) {
    // line = jt2 >> 4 (bits 5..9) | s, s = g + 2r; XOR m = j9..j11 into its low 3 bits
    const uint32_t m = (jt2 >> 9) & 7u, c1 = (jt2 >> 1) & 7u;
    return ((jt2 >> 4) << 7) | (m << 7) | ((m ^ c1) << 4) | ((jt2 & 1u) << 3);
  } else {
    // line bit0 = j4 ^ g, bit1 = r0, bit2 = r1 ^ j9, bits 3,4 = r2, r3, bits 5..8 = j9..j12, bit 9 = g
    const uint32_t rt = ((jt2 >> 4) & 1u) | (((jt2 >> 9) & 1u) << 2) | (((jt2 >> 9) & 15u) << 5);
    const uint32_t c1 = (jt2 >> 1) & 7u;
    return (rt << 7) | ((c1 ^ (rt & 7u)) << 4) | ((jt2 & 1u) << 3);
  }
}

// P1 words from the staging buffer. Forward: 32 words at stride 512, one
// 8-byte load each (base + immediate). Inverse: 32 contiguous words (two
// 16-word lines) as 16-byte chunks; `key` is XORed into the chunk swizzle
// (0 for the TMA layout; poly_mul14's product image uses j9..j11). RAW: the
// buffer already holds the policy's representation (no A::load).
template <class A, bool FWD, bool RAW = false>
__device__ __forceinline__ void p1_read(uint64_t (&v)[32], const uint8_t* St, uint32_t jt1, uint32_t key = 0) {
  if (FWD) {
    const uint32_t b1 = swz_off(jt1);
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const uint64_t x = *reinterpret_cast<const uint64_t*>(St + b1 + r * 4096);
      v[r] = RAW ? x : A::load(x);
    }
  } else {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t row16 = (jt1 >> 4) + h;
      const uint32_t rowoff = row16 << 7, sw = (row16 & 7) ^ key;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        const ulonglong2 p = *reinterpret_cast<const ulonglong2*>(St + rowoff + ((cc ^ sw) << 4));
        v[16 * h + 2 * cc] = RAW ? p.x : A::load(p.x);
        v[16 * h + 2 * cc + 1] = RAW ? p.y : A::load(p.y);
      }
    }
  }
}

// Exchange 1: in place, within the group's staging slots: wait (bar_r1g,
// `parity`) until every warp of the group has read its P1 words, write this
// thread's words to their exchange slots (ex1_write), sync the group, read the
// P2 words (ex1_read). The kernels interleave the pieces with arithmetic.
template <bool FWD>
__device__ __forceinline__ void ex1_write(const uint64_t (&v)[32], uint8_t* St, uint32_t jt1) {
  if (FWD) {
    // swz_off(ex1_perm(jt1 | r << 9)) = (swz_off(jt1) ^ ((r & 7) * 0x90)) + r * 4096
    const uint32_t b1 = swz_off(jt1);
#pragma unroll
    for (int r = 0; r < 32; ++r) *reinterpret_cast<uint64_t*>(St + ((b1 ^ ((r & 7) * 0x90u)) + r * 4096)) = v[r];
  } else {
    // swz_off(ex1_perm(jt1 | h << 4 | 2cc)) = wh ^ (cc << 4), wh from the
    // permuted line (jt1' >> 4) ^ h, jt1' = ex1_perm(jt1)
    const uint32_t rp = ex1_perm<false>(jt1) >> 4;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t rh = rp ^ static_cast<uint32_t>(h);
      const uint32_t wh = (rh << 7) | ((rh & 7u) << 4);
#pragma unroll
      for (int cc = 0; cc < 8; ++cc)
        *reinterpret_cast<ulonglong2*>(St + (wh ^ (cc << 4))) = make_ulonglong2(v[16 * h + 2 * cc], v[16 * h + 2 * cc + 1]);
    }
  }
}
template <bool FWD>
__device__ __forceinline__ void ex1_read(uint64_t (&v)[32], const uint8_t* St, uint32_t q2) {
#pragma unroll
  for (int g = 0; g < 2; ++g)
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      // forward: s = g + 2r (line bits 0..4); inverse: line bits (g, r0, r1) low, (r2, r3) << 3, g << 9
      const uint32_t y = FWD ? ((g + 2 * r) & 7) : (g | ((r & 3) << 1));
      const uint32_t hi = FWD ? (((g + 2 * r) >> 3) << 10) : (((r >> 2) << 10) | (g << 16));
      v[16 * g + r] = *reinterpret_cast<const uint64_t*>(St + ((q2 ^ (y * 0x90u)) + hi));
    }
}
template <bool FWD>
__device__ __forceinline__ void ex1(uint64_t (&v)[32], uint8_t* St, uint32_t jt1, uint32_t q2, uint64_t* bar_r1g,
                                    uint32_t parity, uint32_t g1) {
  mbar_wait(bar_r1g, parity);
  ex1_write<FWD>(v, St, jt1);
  named_sync128(1 + g1);
  ex1_read<FWD>(v, St, q2);
}

// This warp has consumed the staging buffer; the last of the 16 warps (shared
// counter) runs `refill` (e.g. issues the next TMA into the buffer).
template <class F>
__device__ __forceinline__ void staging_consumed(uint32_t* cnt, uint32_t l, F&& refill) {
  __syncwarp();
  if (l == 0) {
    __threadfence_block();
    const uint32_t old = atomicAdd(cnt, 1u);
    if ((old & 15u) == 15u) {
      __threadfence_block();
      refill();
    }
  }
}

// Exchange 2: through the group's slice Eg of E, two rounds on the register
// bit common to P2 and P3 (forward bit 4, inverse bit 13): round h moves
// registers 16h .. 16h + 15 (ex2_write, group sync, ex2_read; the round-0
// reads of every warp of the group precede the round-1 writes). Waits
// (bar_r2g, `parity`) for the previous exchange's last-round reads; arrives
// when this warp's last-round reads are done.
template <bool FWD>
__device__ __forceinline__ void ex2_write(const uint64_t (&v)[32], uint8_t* Eg, uint32_t e2w, int h) {
  // ex2_off(jt2 | r << 5): forward e2w + r * 128; inverse (e2w ^ ((r & 1) << 6)) + (r >> 1) * 128
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    const uint32_t off = FWD ? (e2w + r * 128) : ((e2w ^ ((r & 1) << 6)) + (r >> 1) * 128);
    *reinterpret_cast<uint64_t*>(Eg + off) = v[16 * h + r];
  }
}
template <bool FWD>
__device__ __forceinline__ void ex2_read(uint64_t (&v)[32], const uint8_t* Eg, uint32_t e2r, int h) {
  if (FWD) {
    // P3 round h: the 16 contiguous words j0..j3 (bit 4 = h) as 16-byte
    // chunks, ex2_off(jt3 | 2cc) = e2r ^ (cc << 4)
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const ulonglong2 p = *reinterpret_cast<const ulonglong2*>(Eg + (e2r ^ (cc << 4)));
      v[16 * h + 2 * cc] = p.x;
      v[16 * h + 2 * cc + 1] = p.y;
    }
  } else {
    // P3 round h: registers 16h + r hold j = jt3 | (16h + r) << 9 (bit 13 = h),
    // ex2_off(jt3 | r << 9) = (e2r ^ ((r & 1) << 6)) + r * 1024
#pragma unroll
    for (int r = 0; r < 16; ++r)
      v[16 * h + r] = *reinterpret_cast<const uint64_t*>(Eg + ((e2r ^ ((r & 1) << 6)) + r * 1024));
  }
}
template <bool FWD>
__device__ __forceinline__ void ex2(uint64_t (&v)[32], uint8_t* Eg, uint32_t e2w, uint32_t e2r, uint64_t* bar_r2g,
                                    uint32_t parity, uint32_t g2, uint32_t l) {
  mbar_wait(bar_r2g, parity);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (h == 1) named_sync128(5 + g2);  // round-0 reads done before round-1 writes
    ex2_write<FWD>(v, Eg, e2w, h);
    named_sync128(5 + g2);
    ex2_read<FWD>(v, Eg, e2r, h);
  }
  __syncwarp();
  if (l == 0) mbar_arrive_local(bar_r2g);
}

// Forward result words (32 contiguous per thread, a 256-byte run per lane) to
// global memory in four rounds through the warp's 2 KiB image Ow: each lane
// writes 64 bytes of its run as row l, then every STG.128 stores 8 rows x 64
// bytes (16-byte chunks XOR-swizzled by (row >> 1) & 3: both sides conflict
// free).
__device__ __forceinline__ void fwd_store(const uint64_t (&v)[32], uint8_t* Ow, uint32_t w, uint32_t l,
                                          uint64_t* __restrict__ dst) {
  const uint32_t wrow = ((l >> 1) << 7) | ((l & 1u) << 6), wsw = (l >> 1) & 3u;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (q) __syncwarp();  // the previous round's rows have been read
#pragma unroll
    for (int cc = 0; cc < 4; ++cc)
      *reinterpret_cast<ulonglong2*>(Ow + wrow + ((cc ^ wsw) << 4)) = make_ulonglong2(v[8 * q + 2 * cc], v[8 * q + 2 * cc + 1]);
    __syncwarp();
#pragma unroll
    for (int s2 = 0; s2 < 4; ++s2) {
      const uint32_t rw = (l >> 2) + 8 * s2, cc = l & 3u;
      const ulonglong2 p =
          *reinterpret_cast<const ulonglong2*>(Ow + ((rw >> 1) << 7) + ((rw & 1u) << 6) + ((cc ^ ((rw >> 1) & 3u)) << 4));
      *reinterpret_cast<ulonglong2*>(dst + GrpMap<true>::jt3(w, rw) + 8 * q + 2 * cc) = p;
    }
  }
}

}  // namespace grp

#ifndef NK_GRP_PIPE
#define NK_GRP_PIPE 1
#endif

#if defined(NK_DBG_TIMELINE)  // perf experiment: per-warp phase timestamps into a.dbg (tools/timeline.py --grp)
#define NK_GTS(id)                                                                             \
  do {                                                                                         \
    if (a.dbg && l == 0 && it_ < 16)                                                           \
      a.dbg[((static_cast<uint64_t>(blockIdx.x) * 16 + w) * 16 + it_) * 16 + (id)] = clock64(); \
  } while (0)
#else
#define NK_GTS(id) ((void)0)
#endif

template <class A, bool FWD, bool ILTM0, bool LONG = false>
__global__ void __launch_bounds__(512, 1)
    ntt_grp14(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, NttArgs a,
              uint32_t nitems) {
  using P1 = typename std::conditional<FWD, PassD<9, 5, -1>, PassD<0, 5, -1>>::type;
  using P2 = typename std::conditional<FWD, PassD<5, 4, 4>, PassD<5, 4, 13>>::type;
  using P3 = typename std::conditional<FWD, PassD<0, 5, -1>, PassD<9, 5, -1>>::type;
  using M = GrpMap<FWD>;
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* St = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);  // staging, 128B-swizzled lines
  uint8_t* E = St + kStageBytes;
  uint8_t* O = E + kGrpExBytes;
  // the block's limb constants arrive with its words (one more bulk copy on
  // bar_full), alternating between two slots: no global-load latency at the
  // start of a block, and the fields are read from shared memory where used
  const LimbConst* Cs = reinterpret_cast<const LimbConst*>(O + kGrpOutBytes);
  uint64_t* bar_full = reinterpret_cast<uint64_t*>(O + kGrpOutBytes + 2 * sizeof(LimbConst));
  uint64_t* bar_r1 = bar_full + 1;  // [4] ex1 groups: P1 reads done
  uint64_t* bar_r2 = bar_full + 5;  // [4] ex2 groups: last-round reads done
  uint32_t* cnt = reinterpret_cast<uint32_t*>(bar_full + 9);
  uint64_t* bar_o = bar_full + 10;  // [4] ex2 groups (forward): the output images in E have been read by their stores
  const uint32_t t = threadIdx.x, l = t & 31u, w = t >> 5;
  const uint32_t g1 = w >> 2, g2 = w & 3u;  // exchange-1 / exchange-2 group
  const uint32_t lognb = a.logn - kB14;
  const uint64_t rowwords16 = a.n >> 4;

  auto item_row = [&](uint32_t k, uint64_t& row, uint64_t& blk) {
    row = (static_cast<uint64_t>(k) >> lognb) * a.row_mul + a.row_add;
    blk = static_cast<uint64_t>(k) & ((uint64_t{1} << lognb) - 1);
  };
  // slot: parity of the block's position in this CTA's sequence
  auto issue = [&](uint32_t k, uint32_t slot) {
    uint64_t row, blk;
    item_row(k, row, blk);
    const int32_t y0 = static_cast<int32_t>(row * rowwords16 + (blk << (kB14 - 4)));
    const uint32_t limb = a.limb0 + static_cast<uint32_t>(row % a.nlimbs);
    mbar_expect_tx(bar_full, kStageBytes + static_cast<uint32_t>(sizeof(LimbConst)));
#pragma unroll
    for (int q = 0; q < 4; ++q) tma_load_2d(St + q * 32768, &tin, 0, y0 + q * 256, bar_full);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(Cs + slot)),
                 "l"(a.lc + limb), "r"(static_cast<uint32_t>(sizeof(LimbConst))), "r"(smem_u32(bar_full))
                 : "memory");
  };

  if (t == 0) {
    mbar_init(bar_full, 1);
    for (int i = 0; i < 4; ++i) {
      mbar_init(bar_r1 + i, 4);
      mbar_init(bar_r2 + i, 4);
      mbar_init(bar_o + i, 4);
    }
    *cnt = 0;
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tin)) : "memory");
    if (FWD) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tout)) : "memory");
  }
  __syncthreads();
  if (t == 0 && blockIdx.x < nitems) issue(blockIdx.x, 0);

  const uint32_t jt1 = M::jt1(w, l), jt2 = M::jt2(w, l), jt3 = M::jt3(w, l);
  uint8_t* Eg = E + (g2 << 14);           // this warp's exchange-2 group slice
  // Thread-constant byte bases: every shared access below is a base, at most
  // one XOR with an immediate, plus an immediate offset (derivations in the
  // helpers; swz_off is the 128B swizzle, ex1_perm / ex2_off the layouts).
  const uint32_t q2 = grp::q2_of<FWD>(jt2);
  const uint32_t e2w = ex2_off<FWD>(jt2), e2r = ex2_off<FWD>(jt3);
  uint32_t phase = 0;
  uint32_t it_ = 0;
  (void)it_;

  for (uint32_t k = blockIdx.x; k < nitems; k += gridDim.x) {
    uint64_t row, blk;
    item_row(k, row, blk);
    NK_GTS(0);
    const uint32_t limb = a.limb0 + static_cast<uint32_t>(row % a.nlimbs);
    const typename A::Tw* __restrict__ tw = tw_of<A>(a, limb);
    // low pass: the thread-order table (a warp's loads are 32 consecutive entries)
    const typename A::Tw* __restrict__ twl = twg_of<A>(a, limb) + (blk << kB14) + t;
    const uint64_t boff = blk << kB14;
    uint64_t* __restrict__ dst = a.out + row * a.n + boff;
    const uint64_t xbase = a.n + boff;
    uint64_t v[32];

    // ---- P1 words from the staging buffer (TMA layout) ----
    mbar_wait(bar_full, phase);
    // (register allocation: the inverse is spill-free with the fields copied to
    // registers here, the forward with the fields read where they are used)
    typename std::conditional<FWD, const LimbConst&, const LimbConst>::type c = Cs[phase];
    NK_GTS(1);
    grp::p1_read<A, FWD>(v, St, jt1);
    __syncwarp();
    if (l == 0) mbar_arrive_local(bar_r1 + g1);  // this warp's P1 slots may be rewritten
    NK_GTS(2);

    // Inverse, pipelined (kPipe): the exchanges' shared-memory traffic is
    // issued between arithmetic that does not depend on it. P1's last stage
    // (bit 4) runs after the wait for the group's P1 reads, so its results go
    // to their exchange slots as they are formed; P2 runs one half (bit 13)
    // at a time with the round-0 writes of exchange 2 between the halves;
    // P3's stages below bit 13 run per half, around the round-1 traffic.
    constexpr bool kPipe = !FWD && NK_GRP_PIPE;
    constexpr bool kFoldLast = !FWD && A::kSigned && !LONG;
    if constexpr (kPipe) {
      stages14<A, FWD, P1, ILTM0, 0, 4>(v, tw, twl, a.n, xbase + jt1, c);
      mbar_wait(bar_r1 + g1, phase);
      stages14<A, FWD, P1, ILTM0, 4, 5>(v, tw, twl, a.n, xbase + jt1, c);
      NK_GTS(3);
      grp::ex1_write<FWD>(v, St, jt1);
      named_sync128(1 + g1);
      grp::ex1_read<FWD>(v, St, q2);
      grp::staging_consumed(cnt, l, [&] {
        if (k + gridDim.x < nitems) {
          fence_proxy_async();
          issue(k + gridDim.x, phase ^ 1);
        }
      });
      NK_GTS(4);
      stages14<A, FWD, P2, false, 0, 4, 0>(v, tw, twl, a.n, xbase + jt2, c);
      mbar_wait(bar_r2 + g2, phase ^ 1);
      grp::ex2_write<FWD>(v, Eg, e2w, 0);
      stages14<A, FWD, P2, false, 0, 4, 1>(v, tw, twl, a.n, xbase + jt2, c);
      NK_GTS(5);
      named_sync128(5 + g2);
      grp::ex2_read<FWD>(v, Eg, e2r, 0);
      stages14<A, FWD, P3, false, 0, 1, 0>(v, tw, twl, a.n, xbase + jt3, c);
      named_sync128(5 + g2);  // round-0 reads done before round-1 writes
      grp::ex2_write<FWD>(v, Eg, e2w, 1);
      stages14<A, FWD, P3, false, 1, 3, 0>(v, tw, twl, a.n, xbase + jt3, c);
      named_sync128(5 + g2);
      grp::ex2_read<FWD>(v, Eg, e2r, 1);
      __syncwarp();
      if (l == 0) mbar_arrive_local(bar_r2 + g2);
      NK_GTS(6);
      stages14<A, FWD, P3, false, 3, 4, 0>(v, tw, twl, a.n, xbase + jt3, c);
      stages14<A, FWD, P3, false, 0, 4, 1>(v, tw, twl, a.n, xbase + jt3, c);
      if constexpr (kFoldLast) {
#pragma unroll
        for (int r = 0; r < 16; ++r) A::inv_fold(v[r], v[r + 16], c);
      } else {
        stages14<A, FWD, P3, false, 4, 5>(v, tw, twl, a.n, xbase + jt3, c);
      }
    } else {
    pass14<A, FWD, P1, ILTM0>(v, tw, twl, a.n, xbase + jt1, c);
    NK_GTS(3);
    if (FWD && l == 0) {  // the previous block's output stores have read this warp's images
      bulk_wait_read();
      mbar_arrive_local(bar_o + g2);
    }

    // ---- exchange 1: in place, within the group's staging slots ----
    grp::ex1<FWD>(v, St, jt1, q2, bar_r1 + g1, phase, g1);
    // staging consumed by this warp; the last of the 16 warps refills it
    grp::staging_consumed(cnt, l, [&] {
      if (k + gridDim.x < nitems) {
        fence_proxy_async();
        issue(k + gridDim.x, phase ^ 1);
      }
    });

    NK_GTS(4);
    pass14<A, FWD, P2, false>(v, tw, twl, a.n, xbase + jt2, c);
    NK_GTS(5);

    // ---- exchange 2: the previous block's last-round reads (first block: passes) ----
    if (FWD) mbar_wait(bar_o + g2, phase);  // ... and its output images have left the slice
    grp::ex2<FWD>(v, Eg, e2w, e2r, bar_r2 + g2, phase ^ 1, g2, l);
    NK_GTS(6);

    // canonical inverse (Arith52S, whole rows): n^-1 folded into the last
    // stage (bit 13, single twiddle), as in ntt_pair14 / ntt_grp14
    if constexpr (kFoldLast) {
      pass14<A, FWD, P3, false, 1>(v, tw, twl, a.n, xbase + jt3, c);
#pragma unroll
      for (int r = 0; r < 16; ++r) A::inv_fold(v[r], v[r + 16], c);
    } else {
      pass14<A, FWD, P3, false>(v, tw, twl, a.n, xbase + jt3, c);
    }
    }

    NK_GTS(7);
    // ---- final words and stores ----
    if (FWD) {
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = fwd_out<A>(v[i], c, a.fout);
      // Each thread holds a 256-byte run; a warp's 32 runs are 8 pieces (j9..j11)
      // of 4 consecutive runs (j5, j6). Two rounds (the run's halves): the warp
      // writes its 32 half-runs as the rows of a 4 KiB image (row = lane, 128B
      // swizzle: conflict free) in its quarter of the exchange-2 slice, then four
      // bulk tensor stores (one per j5j6: 8 rows, the box of the 5-D map) move it
      // out. The slice is free once the group's exchange-2 reads are done
      // (bar_r2), and taken again by the next block's exchange 2 after every
      // warp's stores have read their images (bar_o, arrived in the next block).
      uint8_t* Wb = Eg + ((w >> 2) << 12);
      mbar_wait(bar_r2 + g2, phase);
      const int32_t c4 = static_cast<int32_t>(((row * a.n + boff) >> 9) + 8u * (w & 3u));
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h == 1) {
          if (l == 0) bulk_wait_read();
          __syncwarp();
        }
#pragma unroll
        for (int cc = 0; cc < 8; ++cc)
          *reinterpret_cast<ulonglong2*>(Wb + (l << 7) + ((cc ^ (l & 7)) << 4)) =
              make_ulonglong2(v[16 * h + 2 * cc], v[16 * h + 2 * cc + 1]);
        fence_proxy_async();
        __syncwarp();
        if (l == 0) {
#pragma unroll
          for (int s2 = 0; s2 < 4; ++s2)
            asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                             reinterpret_cast<uint64_t>(&tout)),
                         "r"(0), "r"(h), "r"(s2), "r"(static_cast<int32_t>(w >> 2)), "r"(c4),
                         "r"(smem_u32(Wb + (s2 << 10)))
                         : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    } else {
      if constexpr (LONG) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = A::store(v[i]);  // intermediate of a long row
      } else if constexpr (!kFoldLast) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = inv_out<A>(v[i], c, a.fout);
      }
#pragma unroll
      for (int r = 0; r < 32; ++r) dst[jt3 | (static_cast<uint32_t>(r) << 9)] = v[r];
    }
    NK_GTS(8);
    phase ^= 1;
    ++it_;
  }
  if (FWD && l == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace nk
