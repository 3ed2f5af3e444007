#!/usr/bin/env python
"""Small invocations of every kernel family for compute-sanitizer: each case
runs once, checked against the oracle, so a sanitizer report can be tied to a
kernel and a result. (compute-sanitizer is closed on this round's GPU pool;
the guard-word tests in tests/ stand in for memcheck there.)

    python tools/sanitize_cases.py [case ...]     (no args: all cases)
    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} \
        python tools/sanitize_cases.py <case>
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2103_16400_b200 as nk  # noqa: E402
from oracle_lib import Oracle  # noqa: E402
from primes import largest_ntt_primes  # noqa: E402

o = Oracle()


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x).view(np.int64)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint64)


def transform(n, bits, nlimbs, npolys, kernel=-1, fin=1, fout=1, exact=False):
    moduli = largest_ntt_primes(bits, n, nlimbs)
    x = np.concatenate([o.mt19937_64(11 + r, n, moduli[r % nlimbs]) for r in range(npolys * nlimbs)])
    nk.set_block_kernel(kernel)
    nk.set_exact_only(exact)
    try:
        plan = nk.RnsNtt(n, moduli)
        d = dev(x)
        f = host(plan.forward(torch.empty_like(d), d, fin, fout))
        assert np.array_equal(f, o.forward(n, moduli, x, fin, fout, threads=8)), "forward"
        b = host(plan.inverse(torch.empty_like(d), d, 1, 1))
        assert np.array_equal(b, o.inverse(n, moduli, x, 1, 1, threads=8)), "inverse"
    finally:
        nk.set_block_kernel(-1)
        nk.set_exact_only(False)


def eltwise():
    q = largest_ntt_primes(60, 2, 1)[0]
    a, b = o.mt19937_64(1, 4099, q), o.mt19937_64(2, 4099, q)
    r = torch.empty(4099, dtype=torch.int64, device="cuda")
    nk.eltwise_mult_mod(r, dev(a), dev(b), q, 1)
    assert np.array_equal(host(r), o.eltwise_mult_mod(a, b, q, 1))
    nk.eltwise_fma_mod(r, dev(a), 12345, dev(b), q, 1)
    assert np.array_equal(host(r), o.eltwise_fma_mod(a, 12345, b, q, 1))
    q50 = largest_ntt_primes(50, 2, 1)[0]
    a5, b5 = o.mt19937_64(3, 4099, q50), o.mt19937_64(4, 4099, q50)
    nk.eltwise_mult_mod(r, dev(a5), dev(b5), q50, 1)
    assert np.array_equal(host(r), o.eltwise_mult_mod(a5, b5, q50, 1))


def poly(kernel=-1):
    n = 16384
    moduli = largest_ntt_primes(50, n, 2)
    f = np.concatenate([o.mt19937_64(21 + r, n, moduli[r % 2]) for r in range(4)])
    g = np.concatenate([o.mt19937_64(31 + r, n, moduli[r % 2]) for r in range(4)])
    plan = nk.RnsNtt(n, moduli)
    nk.set_block_kernel(kernel)
    try:
        got = host(plan.poly_mult_mod(torch.empty(f.size, dtype=torch.int64, device="cuda"), dev(f), dev(g)))
    finally:
        nk.set_block_kernel(-1)
    assert np.array_equal(got, o.poly_mult_mod(n, moduli, f, g))


CASES = {
    "pair14_and_grp14": lambda: transform(16384, 50, 1, 3),            # ntt_pair14 fwd, ntt_grp14 inv
    "pair14_int": lambda: transform(16384, 60, 1, 2, fin=4),           # integer (ArithIntL) pair / grp
    "pair14_exact": lambda: transform(16384, 50, 1, 2, fout=4, exact=True),
    "pair_inverse": lambda: transform(16384, 50, 1, 2, kernel=0),
    "grp_forward": lambda: transform(16384, 50, 1, 2, kernel=1),
    "block_lat_4096": lambda: transform(4096, 50, 1, 1),               # ntt_block_lat
    "block_8192_batch": lambda: transform(8192, 50, 2, 80),            # ntt_block, >= SM count rows
    "small_1024": lambda: transform(1024, 30, 2, 2),                   # ntt_small
    "global_pass_65536": lambda: transform(65536, 60, 1, 1, fin=4),    # ntt_global_pass + block
    "eltwise": eltwise,
    "poly_single": poly,                                               # poly_mul14 (TMEM)
    "poly_three_launch": lambda: poly(kernel=0),                       # pair14 with the fused product
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for name in names:
        CASES[name]()
        print("ok", name, flush=True)
