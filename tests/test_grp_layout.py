"""CPU checks of ntt_grp14's index algebra (csrc/ntt_grp.cuh), restated in
Python: each pass's thread numbering covers the block, the exchange-1 slot
permutation stays inside each 4-warp group's slots, the exchange-2 image is a
bijection per group and round, the closed-form byte offsets the kernel uses
equal the generic layout functions, and every shared-memory access pattern is
free of bank conflicts except the inverse's first read of the TMA staging
buffer (two-way, fixed by the TMA's 128B swizzle)."""
import pytest


def swz_off(j):
    row, col = j >> 4, j & 15
    return (row << 7) + ((((col >> 1) ^ (row & 7))) << 4) + ((col & 1) << 3)


def perm(fwd, j):
    return (j ^ (((j >> 9) & 7) << 4)) if fwd else (j ^ (((j >> 13) & 1) << 4) ^ (((j >> 9) & 1) << 6))


def ex2(fwd, j):
    if fwd:
        row = (j >> 5) & 127
        ch = ((j >> 1) & 7) ^ ((j >> 9) & 7)
        return (row << 7) | (ch << 4) | ((j & 1) << 3)
    row = ((j >> 6) & 7) | (((j >> 9) & 15) << 3)
    bank = (j & 7) | ((((j >> 5) ^ (j >> 9)) & 1) << 3)
    return (row << 7) | (bank << 3)


def jt(fwd, p, w, l):
    if fwd:
        return [(l & 1) | (((l >> 4) & 1) << 1) | ((w >> 2) << 2) | (((l >> 1) & 7) << 4) | ((w & 3) << 7),
                (l & 1) | (((l >> 4) & 1) << 1) | ((w >> 2) << 2) | (((l >> 1) & 7) << 9) | ((w & 3) << 12),
                (((l >> 3) & 1) << 5) | (((l >> 4) & 1) << 6) | ((w >> 2) << 7) | ((l & 7) << 9) | ((w & 3) << 12)][p]
    return [((l & 1) << 5) | (((l >> 1) & 1) << 6) | (((l >> 2) & 1) << 13) | (((l >> 3) & 1) << 9)
            | (((l >> 4) & 1) << 10) | ((w & 3) << 7) | ((w >> 2) << 11),
            (l & 7) | (((l >> 3) & 1) << 9) | (((l >> 4) & 1) << 10) | ((w & 3) << 3) | ((w >> 2) << 11),
            (l & 7) | (((l >> 3) & 1) << 5) | (((l >> 4) & 1) << 6) | ((w & 3) << 3) | ((w >> 2) << 7)][p]


THREADS = [(w, l) for w in range(16) for l in range(32)]


@pytest.mark.parametrize("fwd", [True, False], ids=["fwd", "inv"])
def test_pass_maps_cover_the_block(fwd):
    X = 4 if fwd else 13
    R1 = (lambda t, r: t | (r << 9)) if fwd else (lambda t, r: t | r)
    R3 = (lambda t, r: t | r) if fwd else (lambda t, r: t | (r << 9))
    assert len({R1(jt(fwd, 0, w, l), r) for w, l in THREADS for r in range(32)}) == 16384
    assert len({jt(fwd, 1, w, l) | (g << X) | (r << 5) for w, l in THREADS for g in range(2)
                for r in range(16)}) == 16384
    assert len({R3(jt(fwd, 2, w, l), r) for w, l in THREADS for r in range(32)}) == 16384


@pytest.mark.parametrize("fwd", [True, False], ids=["fwd", "inv"])
def test_exchange_groups_and_layouts(fwd):
    X = 4 if fwd else 13
    # exchange 1: the group key (w >> 2) is the same index bits on both sides
    g1 = (lambda j: (j >> 2) & 3) if fwd else (lambda j: (j >> 11) & 3)
    for w, l in THREADS:
        assert g1(jt(fwd, 0, w, l)) == w >> 2 == g1(jt(fwd, 1, w, l))
    assert sorted(perm(fwd, j) for j in range(16384)) == list(range(16384))
    assert all(g1(perm(fwd, j)) == g1(j) for j in range(16384))
    # exchange 2: the group key (w & 3) is the same index bits on both sides
    g2 = (lambda j: (j >> 12) & 3) if fwd else (lambda j: (j >> 3) & 3)
    for w, l in THREADS:
        assert g2(jt(fwd, 1, w, l)) == w & 3 == g2(jt(fwd, 2, w, l))
    for gg in range(4):
        for h in range(2):
            offs = {ex2(fwd, j) for j in range(16384) if g2(j) == gg and ((j >> X) & 1) == h}
            assert len(offs) == 2048 and max(offs) < 16384


@pytest.mark.parametrize("fwd", [True, False], ids=["fwd", "inv"])
def test_closed_form_offsets(fwd):
    for w, l in THREADS:
        j1, j2, j3 = (jt(fwd, p, w, l) for p in range(3))
        if fwd:
            b1 = swz_off(j1)
            for r in range(32):
                assert swz_off(perm(True, j1 | r << 9)) == (b1 ^ ((r & 7) * 0x90)) + r * 4096
            m, c1 = (j2 >> 9) & 7, (j2 >> 1) & 7
            q2 = ((j2 >> 4) << 7) | (m << 7) | ((m ^ c1) << 4) | ((j2 & 1) << 3)
        else:
            rp = perm(False, j1) >> 4
            for h in range(2):
                rh = rp ^ h
                wh = (rh << 7) | ((rh & 7) << 4)
                for cc in range(8):
                    assert swz_off(perm(False, j1 | h << 4 | cc << 1)) == wh ^ (cc << 4)
            rt = ((j2 >> 4) & 1) | (((j2 >> 9) & 1) << 2) | (((j2 >> 9) & 15) << 5)
            c1 = (j2 >> 1) & 7
            q2 = (rt << 7) | ((c1 ^ (rt & 7)) << 4) | ((j2 & 1) << 3)
        X = 4 if fwd else 13
        for g in range(2):
            for r in range(16):
                y = ((g + 2 * r) & 7) if fwd else (g | ((r & 3) << 1))
                hi = (((g + 2 * r) >> 3) << 10) if fwd else (((r >> 2) << 10) | (g << 16))
                assert swz_off(perm(fwd, j2 | (g << X) | (r << 5))) == (q2 ^ (y * 0x90)) + hi
        e2w, e2r = ex2(fwd, j2), ex2(fwd, j3)
        for r in range(16):
            off = (e2w + r * 128) if fwd else ((e2w ^ ((r & 1) << 6)) + (r >> 1) * 128)
            assert ex2(fwd, j2 | r << 5) == off
        if fwd:
            for cc in range(8):
                assert ex2(True, j3 | cc << 1) == e2r ^ (cc << 4)
        else:
            for r in range(16):
                assert ex2(False, j3 | r << 9) == (e2r ^ ((r & 1) << 6)) + r * 1024


def _ways(offsets, unit):
    """Shared-memory wavefronts needed beyond the minimum: 8-byte accesses are
    served per half-warp (16 distinct 8-byte bank words), 16-byte ones per
    quarter-warp (8 distinct 16-byte chunks)."""
    group = 16 if unit == 8 else 8
    worst = 1
    for g0 in range(0, 32, group):
        banks = [(o // unit) % (128 // unit) for o in offsets[g0:g0 + group]]
        worst = max(worst, max(banks.count(b) for b in set(banks)))
    return worst


@pytest.mark.parametrize("fwd", [True, False], ids=["fwd", "inv"])
def test_shared_accesses_conflict_free(fwd):
    X = 4 if fwd else 13
    worst = {}

    def note(k, offs, unit):
        worst[k] = max(worst.get(k, 1), _ways(offs, unit))

    for w in range(16):
        if fwd:
            for r in range(32):
                note("p1 read", [swz_off(jt(fwd, 0, w, l) | r << 9) for l in range(32)], 8)
                note("ex1 write", [swz_off(perm(fwd, jt(fwd, 0, w, l) | r << 9)) for l in range(32)], 8)
            for cc in range(8):
                note("p3 read", [ex2(fwd, jt(fwd, 2, w, l) | cc << 1) for l in range(32)], 16)
        else:
            for h in range(2):
                for cc in range(8):
                    note("p1 read", [swz_off(jt(fwd, 0, w, l) | h << 4 | cc << 1) for l in range(32)], 16)
                    note("ex1 write", [swz_off(perm(fwd, jt(fwd, 0, w, l) | h << 4 | cc << 1))
                                       for l in range(32)], 16)
            for r in range(16):
                note("p3 read", [ex2(fwd, jt(fwd, 2, w, l) | r << 9) for l in range(32)], 8)
        for g in range(2):
            for r in range(16):
                note("p2 read", [swz_off(perm(fwd, jt(fwd, 1, w, l) | (g << X) | (r << 5))) for l in range(32)], 8)
        for r in range(16):
            note("ex2 write", [ex2(fwd, jt(fwd, 1, w, l) | r << 5) for l in range(32)], 8)
    expected = {k: 1 for k in worst}
    if not fwd:
        expected["p1 read"] = 2  # the TMA swizzle varies only two chunk bits across a quarter-warp
    assert worst == expected
