"""CPU checks of the two-stream kernels' index algebra (csrc/ntt_str.cuh),
restated in Python: the thread numberings of every pass cover each 8192-word
stream, the closed-form byte offsets of the exchanges equal the layouts they
claim (word j' at j' ^ (((j' >> 4) & 7) << 1) for e1, word m at
m ^ (((m >> 5) & 7) << 1) for the warp-local e2, the plain layout for the
inverse's e1'), what one side writes is what the other side reads, every
8-byte access pattern is conflict free (the 16 lanes of a half-warp hit 16
distinct 8-byte slots of a 128-byte line), the 16-byte accesses to the
128B-swizzled output / input image are conflict free per quarter-warp, the
lane-pair shuffle delivers the words it claims, and the (stream, entry,
thread) twiddle table holds the reference's table index for every butterfly."""
import pytest

THREADS = [(w, l) for w in range(16) for l in range(32)]


def jt1(w, l):  # GrpMap<true>::jt1
    return (l & 1) | (((l >> 4) & 1) << 1) | ((w >> 2) << 2) | (((l >> 1) & 7) << 4) | ((w & 3) << 7)


def jt2(w, l):
    return l | (w << 9)


def jt3(w, l):
    return (l & 1) | ((l >> 1) << 5) | (w << 9)


def e1_phys(jp):
    return jp ^ (((jp >> 4) & 7) << 1)


def e2_phys(m):
    return m ^ (((m >> 5) & 7) << 1)


def conflict_free_8(byte_offsets_of_32_lanes):
    """8-byte accesses: each half-warp (16 lanes) must hit 16 distinct 8-byte slots modulo 128 bytes."""
    for h in range(2):
        slots = {(o >> 3) & 15 for o in byte_offsets_of_32_lanes[16 * h:16 * h + 16]}
        if len(slots) != 16:
            return False
    return True


def conflict_free_16(byte_offsets_of_32_lanes):
    """16-byte accesses: each quarter-warp (8 lanes) must hit 8 distinct 16-byte chunks modulo 128 bytes."""
    for q in range(4):
        chunks = {(o >> 4) & 7 for o in byte_offsets_of_32_lanes[8 * q:8 * q + 8]}
        if len(chunks) != 8:
            return False
    return True


def test_pass_maps_cover_a_stream():
    assert len({jt1(w, l) | (r << 9) for w, l in THREADS for r in range(16)}) == 8192  # P1 (per stream)
    assert len({jt2(w, l) | (r << 5) for w, l in THREADS for r in range(16)}) == 8192  # Q2
    assert len({jt3(w, l) | (r << 1) for w, l in THREADS for r in range(16)}) == 8192  # Q3
    # Q4: registers (j0; j2, j3, j4), lane bit 0 = j1
    assert len({(jt3(w, l) & ~1) | ((l & 1) << 1) | (hi << 2) | j0 for w, l in THREADS for hi in range(8)
                for j0 in range(2)}) == 8192
    # inverse P1': lanes j0..j4, warps j5..j8, registers j9..j12
    assert len({l | (w << 5) | (r << 9) for w, l in THREADS for r in range(16)}) == 8192


def test_forward_e1_offsets_and_conflicts():
    where = {}
    for w in range(16):
        for r in range(16):
            offs = []
            for l in range(32):
                j1 = jt1(w, l)
                e1w = (j1 ^ (((j1 >> 4) & 7) << 1)) << 3
                off = e1w + r * 4096
                assert off == e1_phys(j1 | (r << 9)) << 3
                where[j1 | (r << 9)] = off
                offs.append(off)
            assert conflict_free_8(offs)
    assert len(set(where.values())) == 8192 and max(where.values()) < 65536
    for w in range(16):
        for r in range(16):
            offs = []
            for l in range(32):
                e1r = ((l ^ ((l >> 4) << 1)) << 3) + (w << 12)
                off = (e1r ^ ((r & 3) << 5)) + r * 256
                assert off == where[jt2(w, l) | (r << 5)]  # reads what P1 wrote
                offs.append(off)
            assert conflict_free_8(offs)


def test_e2_offsets_and_conflicts():
    # forward: Q2 map writes, Q3 map reads; the inverse uses the same offsets with the roles swapped
    for r in range(16):
        wr, rd = [], []
        for l in range(32):
            off = ((l << 3) ^ ((r & 7) << 4)) + r * 256
            assert off == e2_phys(l | (r << 5)) << 3
            wr.append(off)
            e2r = ((l & 1) << 3) | (((l >> 1) & 7) << 4) | ((l >> 1) << 8)
            off = e2r ^ (r << 4)
            assert off == e2_phys((l & 1) | (r << 1) | ((l >> 1) << 5)) << 3
            rd.append(off)
        assert conflict_free_8(wr) and conflict_free_8(rd)
    assert len({e2_phys(m) for m in range(512)}) == 512


def test_inverse_e1_is_plain_and_conflict_free():
    where = {}
    for w in range(16):
        for r in range(16):
            offs = [(l << 3) + (w << 12) + r * 256 for l in range(32)]  # Q2' map writes
            for l in range(32):
                where[jt2(w, l) | (r << 5)] = offs[l]
                assert offs[l] == (jt2(w, l) | (r << 5)) << 3
            assert conflict_free_8(offs)
    for w in range(16):
        for r in range(16):
            offs = [(l << 3) + (w << 8) + r * 4096 for l in range(32)]  # P1' map reads
            for l in range(32):
                assert offs[l] == where[l | (w << 5) | (r << 9)]
            assert conflict_free_8(offs)


def test_image_offsets_and_conflicts():
    """Forward output image = inverse input: word m = j0 | j1 << 1 | hi << 2 | (l >> 1) << 5 of the warp's 512
    words in 128-byte rows with the 128B swizzle (16-byte chunk ^= row & 7), 16-byte accesses."""
    seen = set()
    for hi in range(8):
        offs = []
        for l in range(32):
            rowi = (hi >> 2) + 2 * (l >> 1)
            chunk = ((l & 1) | ((hi & 3) << 1)) ^ (rowi & 7)
            off = (rowi << 7) + (chunk << 4)
            m = ((l & 1) << 1) | (hi << 2) | ((l >> 1) << 5)  # j0 = 0 word of the pair
            assert rowi == m >> 4 and chunk == ((m >> 1) & 7) ^ (rowi & 7)
            offs.append(off)
            seen.add(off)
        assert conflict_free_16(offs)
    assert len(seen) == 256 and max(seen) < 4096


def test_lane_pair_shuffle():
    """Forward: a lane holds (j0 = its bit 0; j1 = 0, 1) and ends with (j0 = 0, 1; j1 = its bit 0)."""
    for hi in range(8):
        for b in range(2):  # this lane's bit 0
            own = {j1: ("w", b, j1) for j1 in range(2)}            # (j0 = b, j1)
            partner = {j1: ("w", 1 - b, j1) for j1 in range(2)}    # (j0 = 1 - b, j1)
            recv = partner[0] if (1 - b) else partner[1]          # the partner sends odd ? own0 : own1
            y0 = recv if b else own[0]
            y1 = own[1] if b else recv
            assert y0 == ("w", 0, b) and y1 == ("w", 1, b)


@pytest.mark.parametrize("n,boff", [(16384, 0), (65536, 16384), (65536, 49152)])
def test_twiddle_table_indices(n, boff):
    """str_tw_index: entry e of thread t in stream S is the table index (N + j) >> (b + 1) of the butterflies
    that thread computes with it."""
    def idx(S, e, t):
        w, l = t >> 5, t & 31
        jb = boff + (S << 13)
        if e < 15:
            b = 4 if e == 0 else (3 if e < 3 else (2 if e < 7 else 1))
            hi = 0 if e == 0 else (e - 1 if e < 3 else (e - 3 if e < 7 else e - 7))
            return (n + jb + jt3(w, l) + (hi << (b + 1))) >> (b + 1)
        hi = e - 15
        return (n + jb + (jt3(w, l) & ~1) + ((l & 1) << 1) + (hi << 2)) >> 1
    for S in range(2):
        for t in range(0, 512, 7):
            w, l = t >> 5, t & 31
            base = boff + (S << 13) + jt3(w, l)
            for r in range(16):      # Q3 registers r = (j1..j4)
                j = base | (r << 1)
                for i in range(4):   # stage bit b = 1 + i; the entry for the register bits above b
                    b = 1 + i
                    hi = r >> (i + 1)
                    e = [7, 3, 1, 0][i] + hi
                    assert idx(S, e, t) == (n + j) >> (b + 1)
            for hi in range(8):      # Q4: bit 0
                j = boff + (S << 13) + (jt3(w, l) & ~1) + ((l & 1) << 1) + (hi << 2)
                assert idx(S, 15 + hi, t) == (n + j) >> 1 == (n + j + 1) >> 1
