#!/usr/bin/env python
"""poly_mult_mod of whole rows of N = 2^10 .. 2^13: the single kernel
(csrc/ntt_polyblk.cuh) against the multi-launch sequence (nk_debug_block_kernel(1)),
2^25 coefficients per operand (256 MiB each: larger than L2), 16 limbs.

    python tools/polyblk_bench.py [--iters 20]
One JSON line per (N, limb width).
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2103_16400_b200 as nk  # noqa: E402
from bench import largest_ntt_primes  # noqa: E402


def time_us(fn, iters):
    for _ in range(3):
        fn()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(iters):
        fn()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) * 1e3 / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--limbs", type=int, default=16)
    ap.add_argument("--logwords", type=int, default=25)
    a = ap.parse_args()
    gen = torch.Generator(device="cuda").manual_seed(1)
    words = 1 << a.logwords
    x = torch.randint(0, 1 << 49, (words,), dtype=torch.int64, device="cuda", generator=gen)
    y = torch.randint(0, 1 << 49, (words,), dtype=torch.int64, device="cuda", generator=gen)
    out = torch.empty_like(x)
    for bits in (50, 60):
        for logn in (10, 11, 12, 13):
            n = 1 << logn
            plan = nk.RnsNtt(n, largest_ntt_primes(bits, n, a.limbs))
            res = {"n": n, "bits": bits, "rows": words // n}
            for name, k in (("single_us", -1), ("multi_us", 1)):
                nk.set_block_kernel(k)
                before = nk.launch_count()
                plan.poly_mult_mod(out, x, y)
                res[name.replace("_us", "_launches")] = nk.launch_count() - before
                res[name] = round(time_us(lambda: plan.poly_mult_mod(out, x, y), a.iters), 1)
            nk.set_block_kernel(-1)
            res["hbm_GBs_single"] = round(24 * words / res["single_us"] / 1e3, 1)
            print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
