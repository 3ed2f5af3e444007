#!/usr/bin/env python
"""Small driver for ncu / timing of one transform configuration.

    python tools/prof_ntt.py --n 16384 --limbs 32 --polys 64 --bits 50 --iters 3
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2103_16400_b200 as nk  # noqa: E402
from bench import largest_ntt_primes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--limbs", type=int, default=32)
    ap.add_argument("--polys", type=int, default=64)
    ap.add_argument("--bits", type=int, default=50)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--fin", type=int, default=1)
    ap.add_argument("--kernel", type=int, default=-1, help="nk_debug_block_kernel (-1 auto)")
    ap.add_argument("--op", default="both", choices=["fwd", "inv", "both", "poly", "mult"])
    a = ap.parse_args()
    nk.set_block_kernel(a.kernel)
    moduli = largest_ntt_primes(a.bits, a.n, a.limbs)
    plan = nk.RnsNtt(a.n, moduli)
    words = a.n * a.limbs * a.polys
    g = torch.Generator(device="cuda").manual_seed(1)
    # values < 2^49 < q: valid reduced inputs for every 50/60-bit limb
    x = torch.randint(0, 1 << 49, (words,), dtype=torch.int64, device="cuda", generator=g)
    y = torch.randint(0, 1 << 49, (words,), dtype=torch.int64, device="cuda", generator=g)
    out = torch.empty_like(x)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for it in range(a.iters + 1):
        if it == 1:
            ev[0].record()
        if a.op in ("fwd", "both"):
            plan.forward(out, x, a.fin, 1)
        if a.op in ("inv", "both"):
            plan.inverse(out, x, 1, 1)
        if a.op == "poly":
            plan.poly_mult_mod(out, x, y)
        if a.op == "mult":
            plan.eltwise_mult_mod(out, x, y, 1)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / max(1, a.iters)
    print(f"n={a.n} limbs={a.limbs} polys={a.polys} op={a.op}: {ms:.4f} ms/iter, "
          f"{words / ms / 1e3:.1f} Mcoeff/s per direction-op")


if __name__ == "__main__":
    main()
