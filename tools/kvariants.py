#!/usr/bin/env python
"""Device time of the forward / inverse at a config under each 16384-word
block kernel (nk_debug_block_kernel: 0 CTA pair, 1 group exchange, 2 two streams per thread), CUDA
events over back-to-back calls.

    python tools/kvariants.py [--n 16384 --limbs 32 --polys 64 --bits 50] [--kernels 0,1]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import paper_2103_16400_b200 as nk  # noqa: E402
from bench import largest_ntt_primes  # noqa: E402


def timed(fn, reps):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--limbs", type=int, default=32)
    ap.add_argument("--polys", type=int, default=64)
    ap.add_argument("--bits", type=int, default=50)
    ap.add_argument("--kernels", default="0,1,2")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--fin", type=int, default=1)
    ap.add_argument("--fout", type=int, default=1)
    a = ap.parse_args()
    moduli = largest_ntt_primes(a.bits, a.n, a.limbs)
    plan = nk.RnsNtt(a.n, moduli)
    words = a.n * a.limbs * a.polys
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randint(0, 1 << 49, (words,), dtype=torch.int64, device="cuda", generator=g)
    out = torch.empty_like(x)
    for k in [int(s) for s in a.kernels.split(",")]:
        nk.set_block_kernel(k)
        fwd = timed(lambda: plan.forward(out, x, a.fin, a.fout), a.reps)
        inv = timed(lambda: plan.inverse(out, x, 1, min(a.fout, 2)), a.reps)
        print(json.dumps({"kernel": k, "n": a.n, "limbs": a.limbs, "polys": a.polys, "bits": a.bits,
                          "fwd_us": fwd, "inv_us": inv}), flush=True)
    nk.set_block_kernel(-1)


if __name__ == "__main__":
    main()
