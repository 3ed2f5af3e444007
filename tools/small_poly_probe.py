#!/usr/bin/env python
"""poly_mult_mod of batches smaller than the SM count (1 .. 147 row pairs), N = 1024 / 4096 /
8192: the single poly_block launch (8 words per thread) against the multi-launch sequence
(nk_debug_block_kernel(1)), as stream launches through the Python mirror (call overhead
included on both sides). One JSON line per shape.

    python tools/small_poly_probe.py
"""
import os, sys, json, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_2103_16400_b200 as nk
from bench import largest_ntt_primes
def time_us(fn, iters=200):
    for _ in range(10): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters
gen = torch.Generator(device="cuda").manual_seed(1)
for bits in (50, 60):
    for n in (1024, 4096, 8192):
        plan = nk.RnsNtt(n, largest_ntt_primes(bits, n, 1))
        for rows in (1, 4, 16, 64, 147):
            x = torch.randint(0, 1 << 49, (rows * n,), dtype=torch.int64, device="cuda", generator=gen)
            y = torch.randint(0, 1 << 49, (rows * n,), dtype=torch.int64, device="cuda", generator=gen)
            out = torch.empty_like(x)
            r = {"bits": bits, "n": n, "rows": rows}
            for name, k in (("single", -1), ("multi", 1)):
                nk.set_block_kernel(k)
                r[name] = round(time_us(lambda: plan.poly_mult_mod(out, x, y)), 2)
            nk.set_block_kernel(-1)
            print(json.dumps(r), flush=True)
