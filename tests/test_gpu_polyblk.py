"""GPU parity of the single-kernel poly_mult_mod for whole rows of N = 2^10 ..
2^13 words (csrc/ntt_polyblk.cuh) against the unmodified reference
(oracle/_ref/libnttref.so running ring.hpp:28-43's forward / forward / product /
inverse sequence) and against this library's own multi-launch sequence.

Covered: both canonical-only policies (50-bit limbs on the FP64 pipe, 60-bit
limbs on the integer pipes, also small moduli and an explicit 64-bit
accumulator for a small modulus), both launch shapes (fewer rows than SMs: 8
words per thread; more: 16 or 32 words per thread), limb sub-ranges, aliasing of the
result with either operand, extreme rows (all q-1, all zero), one launch per
call, and the fall-back for plans that mix accumulator widths.
"""
import numpy as np
import pytest
import torch

from oracle_lib import Ref
from primes import largest_ntt_primes, smallest_ntt_primes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    assert Ref.available(), "oracle/_ref/libnttref.so missing (build it with make -C oracle)"
    return Ref()


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.uint64).view(np.int64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint64)


def rows_uniform(oracle, moduli, n, rows, seed):
    L = len(moduli)
    return np.concatenate([oracle.mt19937_64(seed + r, n, moduli[r % L]) for r in range(rows)])


def threads(ref):
    return max(1, int(ref.lib.ref_hw_threads()))


@pytest.mark.parametrize("logn", [10, 11, 12, 13])
@pytest.mark.parametrize("bits", [50, 60])
@pytest.mark.parametrize("npolys", [2, 80])
def test_polyblk_vs_reference(nk, oracle, ref, logn, bits, npolys):
    """3 limbs x npolys row pairs (6 rows: the 8-words-per-thread shape; 240 rows:
    16 or 32 words per thread): one launch, every word equal to the reference's,
    and the same words from 20 repeated launches (the exchange image and the
    parked spectrum are reused across the three transforms of a row)."""
    n = 1 << logn
    moduli = largest_ntt_primes(bits, n, 3)
    plan = nk.RnsNtt(n, moduli)
    rows = npolys * len(moduli)
    f = rows_uniform(oracle, moduli, n, rows, 1000 * logn + bits)
    g = rows_uniform(oracle, moduli, n, rows, 7000 * logn + bits)
    # extreme rows: all q-1 times all q-1, zero times anything, q-1 times uniform
    f[:n] = moduli[0] - 1
    g[:n] = moduli[0] - 1
    f[n:2 * n] = 0
    g[2 * n:3 * n] = moduli[2] - 1
    want = ref.poly_mult_mod(n, moduli, f, g, threads=threads(ref))
    df, dg = dev(f), dev(g)
    out = torch.empty_like(df)
    before = nk.launch_count()
    plan.poly_mult_mod(out, df, dg)
    torch.cuda.synchronize()
    assert nk.launch_count() - before == 1
    assert np.array_equal(host(out), want)
    for _ in range(20):
        again = torch.empty_like(df)
        plan.poly_mult_mod(again, df, dg)
        assert torch.equal(again, out)
    # the library's own multi-launch sequence (the reference's order of operations)
    nk.set_block_kernel(1)
    try:
        out2 = torch.empty_like(df)
        before = nk.launch_count()
        plan.poly_mult_mod(out2, df, dg)
        torch.cuda.synchronize()
        assert nk.launch_count() - before > 1
        assert np.array_equal(host(out2), want)
    finally:
        nk.set_block_kernel(-1)
    # host-buffer entry point
    assert np.array_equal(plan.poly_mult_mod(None, f, g), want)


@pytest.mark.parametrize("logn", [10, 13])
@pytest.mark.parametrize("bits", [50, 60])
def test_polyblk_aliasing_and_limb_ranges(nk, oracle, ref, logn, bits):
    n = 1 << logn
    moduli = largest_ntt_primes(bits, n, 4)
    plan = nk.RnsNtt(n, moduli)
    sub = moduli[1:3]
    rows = 5 * len(sub)
    f = rows_uniform(oracle, sub, n, rows, 31 + logn)
    g = rows_uniform(oracle, sub, n, rows, 77 + logn)
    want = ref.poly_mult_mod(n, sub, f, g)
    df, dg = dev(f), dev(g)
    plan.poly_mult_mod(df, df, dg, limb0=1, nlimbs=2)  # result aliases f
    assert np.array_equal(host(df), want)
    df = dev(f)
    plan.poly_mult_mod(dg, df, dg, limb0=1, nlimbs=2)  # result aliases g
    assert np.array_equal(host(dg), want)
    # 8-byte aligned views (an odd word offset) need no staging copy here
    base = torch.zeros(f.size + 1, dtype=torch.int64, device="cuda")
    base[1:] = dev(f)
    out = torch.empty(f.size, dtype=torch.int64, device="cuda")
    plan.poly_mult_mod(out, base[1:], dev(g), limb0=1, nlimbs=2)
    assert np.array_equal(host(out), want)


@pytest.mark.parametrize("bits", [20, 30, 40, 49])
def test_polyblk_small_moduli(nk, oracle, ref, bits):
    """The smallest NTT primes of a width (the other end of each policy's range)."""
    n = 2048
    moduli = smallest_ntt_primes(bits, n, 2)
    plan = nk.RnsNtt(n, moduli)
    rows = 3 * len(moduli)
    f = rows_uniform(oracle, moduli, n, rows, 5 + bits)
    g = rows_uniform(oracle, moduli, n, rows, 9 + bits)
    f[:n] = moduli[0] - 1
    g[:n] = moduli[0] - 1
    want = ref.poly_mult_mod(n, moduli, f, g)
    out = torch.empty(f.size, dtype=torch.int64, device="cuda")
    before = nk.launch_count()
    plan.poly_mult_mod(out, dev(f), dev(g))
    torch.cuda.synchronize()
    assert nk.launch_count() - before == 1
    assert np.array_equal(host(out), want)


def test_polyblk_explicit_64bit_accumulator(nk, oracle, ref):
    """A 45-bit modulus with bit_shift = 64: the integer policy's tables."""
    n = 4096
    moduli = largest_ntt_primes(45, n, 2)
    plan = nk.RnsNtt(n, moduli, bit_shift=64)
    rows = 4
    f = rows_uniform(oracle, moduli, n, rows, 411)
    g = rows_uniform(oracle, moduli, n, rows, 412)
    want = ref.poly_mult_mod(n, moduli, f, g)
    out = torch.empty(f.size, dtype=torch.int64, device="cuda")
    before = nk.launch_count()
    plan.poly_mult_mod(out, dev(f), dev(g))
    torch.cuda.synchronize()
    assert nk.launch_count() - before == 1
    assert np.array_equal(host(out), want)


def test_polyblk_mixed_widths_fall_back(nk, oracle, ref):
    """A 50-bit and a 60-bit limb in one call (beta = 2^52 and 2^64): no common
    policy, so the multi-launch sequence runs; a 61-bit limb likewise (outside
    the loose integer policy's q < 2^60)."""
    n = 4096
    for moduli in ([largest_ntt_primes(50, n, 1)[0], largest_ntt_primes(60, n, 1)[0]],
                   largest_ntt_primes(61, n, 2)):
        plan = nk.RnsNtt(n, moduli)
        rows = 2 * len(moduli)
        f = rows_uniform(oracle, moduli, n, rows, 511)
        g = rows_uniform(oracle, moduli, n, rows, 512)
        want = ref.poly_mult_mod(n, moduli, f, g)
        out = torch.empty(f.size, dtype=torch.int64, device="cuda")
        before = nk.launch_count()
        plan.poly_mult_mod(out, dev(f), dev(g))
        torch.cuda.synchronize()
        assert nk.launch_count() - before > 1
        assert np.array_equal(host(out), want)


@pytest.mark.parametrize("logn,bits,npolys", [(10, 50, 1), (11, 60, 70), (12, 50, 60), (13, 60, 1), (13, 50, 40)])
def test_polyblk_writes_stay_in_bounds(nk, oracle, ref, logn, bits, npolys):
    """Guard words around the result stay untouched and the operands are left
    as they were (the kernel writes its result rows only)."""
    n = 1 << logn
    moduli = largest_ntt_primes(bits, n, 3)
    plan = nk.RnsNtt(n, moduli)
    rows = npolys * len(moduli)
    f = rows_uniform(oracle, moduli, n, rows, 2000 + logn)
    g = rows_uniform(oracle, moduli, n, rows, 3000 + logn)
    want = ref.poly_mult_mod(n, moduli, f, g, threads=threads(ref))
    guard = 64
    sentinel = 0x5A5A5A5A5A5A5A5A
    buf = torch.full((f.size + 2 * guard,), sentinel, dtype=torch.int64, device="cuda")
    df, dg = dev(f), dev(g)
    plan.poly_mult_mod(buf[guard:guard + f.size], df, dg)
    got = host(buf)
    assert np.array_equal(got[guard:guard + f.size], want)
    assert np.all(got[:guard] == np.uint64(sentinel)) and np.all(got[guard + f.size:] == np.uint64(sentinel))
    assert np.array_equal(host(df), f) and np.array_equal(host(dg), g)


@pytest.mark.parametrize("logn,bits", [(14, 60), (15, 50), (15, 60), (16, 60), (9, 50), (9, 60)])
def test_poly_multi_launch_sizes_vs_reference(nk, oracle, ref, logn, bits):
    """Sizes and limb widths without a single-kernel version (N = 16384 with
    60-bit limbs, N >= 32768, N <= 512): forward / forward / product / inverse
    launches with canonical spectra; the reference's own lazy sequence under
    exact_only. Both equal the reference's words."""
    n = 1 << logn
    moduli = largest_ntt_primes(bits, n, 2)
    plan = nk.RnsNtt(n, moduli)
    rows = 3 * len(moduli)
    f = rows_uniform(oracle, moduli, n, rows, 9000 + logn)
    g = rows_uniform(oracle, moduli, n, rows, 9500 + logn)
    f[:n] = moduli[0] - 1
    g[:n] = moduli[0] - 1
    want = ref.poly_mult_mod(n, moduli, f, g, threads=threads(ref))
    for exact in (False, True):
        nk.set_exact_only(exact)
        try:
            out = torch.empty(f.size, dtype=torch.int64, device="cuda")
            before = nk.launch_count()
            plan.poly_mult_mod(out, dev(f), dev(g))
            torch.cuda.synchronize()
            assert nk.launch_count() - before > 1
            assert np.array_equal(host(out), want), exact
        finally:
            nk.set_exact_only(False)
