"""GPU parity of the kernels' single butterflies, per arithmetic policy.

Mirrors tests/test_ntt.cpp:264-333 of the reference (ForwardButterfly /
InverseButterfly: exhaustive q = 17 congruence and range) through
nk_debug_butterflies, plus random samples at 50- and 60-bit moduli:
  * the exact policies (ArithInt<64>, ArithInt<52>, Arith52P) must
    return the reference's lazy representatives bit for bit (oracle);
  * the canonical-only policies (Arith52S: signed words, ArithIntL: loose
    quotients) must stay congruent and within their documented ranges
    (modmath.cuh), which is what their transforms' exactness rests on.
"""
import numpy as np
import pytest
import torch

from primes import largest_ntt_primes

pytestmark = pytest.mark.gpu

EXACT = {0: 64, 1: 52, 2: 52}  # policy -> accumulator width
ARITH52S, ARITHINTL = 3, 4


def dev(x):
    x = np.ascontiguousarray(x)
    return torch.from_numpy(x.view(np.int64) if x.dtype == np.uint64 else x.astype(np.int64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def exhaustive_pairs(lo, hi):
    a, b = np.meshgrid(np.arange(lo, hi, dtype=np.int64), np.arange(lo, hi, dtype=np.int64))
    return a.reshape(-1), b.reshape(-1)


def sample_pairs(q, rng, n, lo_f, hi_f):
    """Uniform in [lo_f q, hi_f q) plus the range edges (uint64 when the range
    is non-negative: 8q exceeds int64 at 61-bit q)."""
    lo, hi = int(lo_f * q), hi_f * q
    dt = np.uint64 if lo >= 0 else np.int64
    edges = [e for e in (lo, lo + 1, hi - 1, 0, q - 1, q, min(hi - 1, 2 * q)) if lo <= e < hi]
    edges = np.array(edges, dt)
    a = np.concatenate([edges, rng.integers(lo, hi, n, dtype=dt)])
    b = np.concatenate([edges[::-1], rng.integers(lo, hi, n, dtype=dt)])
    return a, b


def qs(policy):
    if policy in (0, ARITHINTL):
        return [17, largest_ntt_primes(60, 1024, 1)[0], largest_ntt_primes(61, 1024, 1)[0]]
    return [17, largest_ntt_primes(50, 1024, 1)[0]]


def twiddles(q, rng):
    return list(range(q)) if q == 17 else [0, 1, q - 1] + [int(w) for w in rng.integers(2, q - 1, 5)]


@pytest.mark.parametrize("policy", sorted(EXACT))
@pytest.mark.parametrize("fwd", [True, False], ids=["fwd", "inv"])
def test_exact_policies_match_reference_butterflies(nk, oracle, policy, fwd):
    rng = np.random.default_rng(policy * 2 + fwd)
    bs = EXACT[policy]
    for q in qs(policy):
        hi_f = 4 if fwd else 2  # [0, 4q) forward, [0, 2q) inverse (ntt.hpp:103-130)
        if q == 17:
            a, b = exhaustive_pairs(0, hi_f * q)
        else:
            a, b = sample_pairs(q, rng, 4096, 0, hi_f)
        for w in twiddles(q, rng):
            y0, y1 = nk.debug_butterflies(policy, fwd, q, w, dev(a.astype(np.uint64)),
                                          dev(b.astype(np.uint64)))
            w0, w1 = oracle.butterflies(fwd, q, bs, w, a.astype(np.uint64), b.astype(np.uint64))
            assert np.array_equal(host(y0).view(np.uint64), w0), (policy, q, w)
            assert np.array_equal(host(y1).view(np.uint64), w1), (policy, q, w)
            assert int(w0.max()) < hi_f * q and int(w1.max()) < hi_f * q  # reference ranges


@pytest.mark.parametrize("fwd", [True, False], ids=["fwd", "inv"])
def test_signed_policy_ranges(nk, fwd):
    """Arith52S: forward |x| < 4q -> |y| < 4q, inverse |x| < 2q -> |y| < 2q,
    congruent to the butterfly's value."""
    rng = np.random.default_rng(5 + fwd)
    for q in qs(ARITH52S):
        r = 4 if fwd else 2
        if q == 17:
            a, b = exhaustive_pairs(-r * q + 1, r * q)
        else:
            a, b = sample_pairs(q, rng, 4096, -r + 1e-9, r)
        for w in twiddles(q, rng):
            y0, y1 = nk.debug_butterflies(ARITH52S, fwd, q, w, dev(a), dev(b))
            y0, y1 = host(y0), host(y1)
            assert np.abs(y0).max() < r * q and np.abs(y1).max() < r * q, (q, w)
            A, B = a.astype(object), b.astype(object)
            if fwd:
                e0, e1 = (A + w * B) % q, (A - w * B) % q
            else:
                e0, e1 = (A + B) % q, (w * (A - B)) % q
            assert all(int(u) % q == v for u, v in zip(y0, e0)), (q, w)
            assert all(int(u) % q == v for u, v in zip(y1, e1)), (q, w)


def test_signed_policy_product_bound(nk):
    """Arith52S's rounded-reciprocal product (modmath.cuh mul_recip_fine, w
    alone, stored balanced, no Shoup table): with x0 = 0 the forward butterfly
    returns (T, -T), and the documented bound |T| < q must hold for every
    multiplicand |v| < 4q and every twiddle."""
    rng = np.random.default_rng(11)
    for q in qs(ARITH52S):
        if q == 17:
            b = np.arange(-4 * q + 1, 4 * q, dtype=np.int64)
        else:
            b = np.concatenate([np.array([4 * q - 1, -(4 * q - 1), 2 * q, -2 * q, 0, 1], np.int64),
                                rng.integers(-4 * q + 1, 4 * q, 8192, dtype=np.int64)])
        a = np.zeros_like(b)
        tws = twiddles(q, rng) + ([q - 1, q - 2, q // 2, q // 2 + 1] if q > 17 else list(range(1, q)))
        for w in tws:
            y0, y1 = nk.debug_butterflies(ARITH52S, True, q, w, dev(a), dev(b))
            y0, y1 = host(y0), host(y1)
            assert np.abs(y0).max() < q, (q, w, int(np.abs(y0).max()))
            assert np.array_equal(y0, -y1)
            B = b.astype(object)
            assert all(int(u) % q == (w * v) % q for u, v in zip(y0, B)), (q, w)


def test_signed_policy_alternating_stages(nk):
    """The 16384-word kernels' forward schedule (Arith52S::fwd_skip): a reducing
    stage maps |x| < 4q into |y| < 3q, the non-reducing stage after it |x| < 3q
    into |y| < 4q (policy 5), both congruent to the butterfly's value."""
    rng = np.random.default_rng(12)
    for q in qs(ARITH52S):
        for policy, rin, rout in ((ARITH52S, 4, 3), (5, 3, 4)):
            if q == 17:
                a, b = exhaustive_pairs(-rin * q + 1, rin * q)
            else:
                a, b = sample_pairs(q, rng, 4096, -rin + 1e-9, rin)
                edge = np.array([rin * q - 1, -(rin * q - 1)], np.int64)
                a = np.concatenate([a, edge, edge, -edge])
                b = np.concatenate([b, edge, -edge, edge])
            for w in twiddles(q, rng) + [q // 2, q // 2 + 1, q - 1]:
                y0, y1 = nk.debug_butterflies(policy, True, q, w, dev(a), dev(b))
                y0, y1 = host(y0), host(y1)
                assert np.abs(y0).max() < rout * q and np.abs(y1).max() < rout * q, (policy, q, w)
                A, B = a.astype(object), b.astype(object)
                e0, e1 = (A + w * B) % q, (A - w * B) % q
                assert all(int(u) % q == v for u, v in zip(y0, e0)), (policy, q, w)
                assert all(int(u) % q == v for u, v in zip(y1, e1)), (policy, q, w)


@pytest.mark.parametrize("fwd", [True, False], ids=["fwd", "inv"])
@pytest.mark.parametrize("skip", [False, True], ids=["reducing", "skipping"])
def test_loose_policy_ranges(nk, fwd, skip):
    """ArithIntL (q < 2^60, 16q <= 2^64), modmath.cuh: a reducing forward stage
    maps words in [0, 16q) into [0, 12q), the non-reducing stage after it
    [0, 12q) into [0, 16q); inverse words stay in [0, 8q), without the
    reduction when both inputs are products (below 4q). Congruent to the
    butterfly's value."""
    rng = np.random.default_rng(9 + fwd + 2 * skip)
    for q in [17, largest_ntt_primes(60, 1024, 1)[0]]:
        if fwd:
            rin, rout = (12, 16) if skip else (16, 12)
        else:
            rin, rout = (4, 8) if skip else (8, 8)
        if q == 17:
            a, b = exhaustive_pairs(0, rin * q)
        else:
            a, b = sample_pairs(q, rng, 4096, 0, rin)
        a, b = a.astype(np.uint64), b.astype(np.uint64)
        for w in twiddles(q, rng):
            y0, y1 = nk.debug_butterflies(6 if skip else ARITHINTL, fwd, q, w, dev(a), dev(b))
            y0, y1 = host(y0).view(np.uint64), host(y1).view(np.uint64)
            assert int(y0.max()) < rout * q and int(y1.max()) < rout * q, (q, w)
            A, B = a.astype(object), b.astype(object)
            if fwd:
                e0, e1 = (A + w * B) % q, (A - w * B) % q
            else:
                e0, e1 = (A + B) % q, (w * (A - B)) % q
            assert all(int(u) % q == v for u, v in zip(y0, e0)), (q, w)
            assert all(int(u) % q == v for u, v in zip(y1, e1)), (q, w)


def test_public_harvey_butterflies(nk, oracle):
    """The public scalar API (ntt.hpp:137-166) through nk_harvey_butterflies:
    test_ntt.cpp's ZeroAndZeroMultiplier / SymmetryAndZero known answers and
    the exhaustive q = 17 table, both widths, against the oracle."""
    q = 17
    for bs in (52, 64):
        w5 = nk.precompute_factor(5, q, bs)
        assert nk.harvey_forward_butterfly(0, 0, w5, q) == (0, 2 * q)  # test_ntt.cpp:264-275
        w0 = nk.precompute_factor(0, q, bs)
        for x0 in (0, 5, 40, 67):
            z0, z1 = nk.harvey_forward_butterfly(x0, 9, w0, q)
            assert z0 % q == x0 % q and z1 % q == x0 % q
        w3 = nk.precompute_factor(3, q, bs)
        for x in (0, 7, 30):  # test_ntt.cpp:301-313
            y0, y1 = nk.harvey_inverse_butterfly(x, x, w3, q)
            assert y1 % q == 0 and y0 % q == (2 * x) % q
        for fwd, r in ((True, 4), (False, 2)):
            a, b = np.meshgrid(np.arange(r * q, dtype=np.uint64), np.arange(r * q, dtype=np.uint64))
            a, b = a.reshape(-1), b.reshape(-1)
            for w in range(q):
                f = nk.precompute_factor(w, q, bs)
                fn = nk.harvey_forward_butterfly if fwd else nk.harvey_inverse_butterfly
                y0, y1 = fn(a, b, f, q)
                w0_, w1_ = oracle.butterflies(fwd, q, bs, w, a, b)
                assert np.array_equal(y0, w0_) and np.array_equal(y1, w1_), (bs, fwd, w)


def test_cpp_facade_on_device():
    """tests/cpp/facade_test (the C++ drop-in facade: reference and HEXL names)
    end to end on the GPU."""
    import os
    import subprocess

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "tests", "cpp", "facade_test")
    if not os.path.exists(exe):
        import sys
        sys.path.insert(0, root)
        import __graft_entry__
        __graft_entry__.build_facade_test()
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "facade gpu checks ok" in out.stdout
