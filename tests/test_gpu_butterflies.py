"""GPU parity of the kernels' single butterflies, per arithmetic policy.

Mirrors tests/test_ntt.cpp:264-333 of the reference (ForwardButterfly /
InverseButterfly: exhaustive q = 17 congruence and range) through
nk_debug_butterflies, plus random samples at 50- and 60-bit moduli:
  * the exact policies (ArithInt<64>, ArithInt<52>, Arith52P, Arith52F) must
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

EXACT = {0: 64, 1: 52, 2: 52, 5: 52}  # policy -> accumulator width
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


@pytest.mark.parametrize("fwd", [True, False], ids=["fwd", "inv"])
def test_loose_policy_ranges(nk, fwd):
    """ArithIntL: forward words in [0, 8q) stay there, inverse words in
    [0, 4q) stay there, congruent to the butterfly's value."""
    rng = np.random.default_rng(9 + fwd)
    for q in qs(ARITHINTL):
        r = 8 if fwd else 4
        if q == 17:
            a, b = exhaustive_pairs(0, r * q)
        else:
            a, b = sample_pairs(q, rng, 4096, 0, r)
        a, b = a.astype(np.uint64), b.astype(np.uint64)
        for w in twiddles(q, rng):
            y0, y1 = nk.debug_butterflies(ARITHINTL, fwd, q, w, dev(a), dev(b))
            y0, y1 = host(y0).view(np.uint64), host(y1).view(np.uint64)
            assert int(y0.max()) < r * q and int(y1.max()) < r * q, (q, w)
            A, B = a.astype(object), b.astype(object)
            if fwd:
                e0, e1 = (A + w * B) % q, (A - w * B) % q
            else:
                e0, e1 = (A + B) % q, (w * (A - B)) % q
            assert all(int(u) % q == v for u, v in zip(y0, e0)), (q, w)
            assert all(int(u) % q == v for u, v in zip(y1, e1)), (q, w)
