#!/usr/bin/env python
"""Device times of every BASELINE config on one B200 (CUDA events, inputs
resident, warm-up first). Prints one JSON line per config.

  cfg1  N=4096, 1 limb: forward(1,1)+inverse(1,1) latency (CUDA graph)
  cfg2  2^20 x 60-bit: EltwiseMultMod vv / vs (FMA, no addend) / FMA, 16
        rotating buffer sets > L2, one CUDA graph per op
  cfg3  N=16384, 32 limbs x 64 polys: forward(1,1), inverse(1,1)
  cfg4  N=65536, 24 60-bit limbs x 16 polys: forward(4,1), inverse(2,1)
  cfg5  N=16384, 16 limbs x 128 pairs: poly_mult_mod
Synthetic inputs (torch.randint below the smallest modulus); the bench and
the parity tests use the mt19937_64 streams.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import paper_2103_16400_b200 as nk  # noqa: E402
from bench import cfg2_modulus, largest_ntt_primes  # noqa: E402


def timed(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def rnd(words, hi, gen):
    return torch.randint(0, hi, (words,), dtype=torch.int64, device="cuda", generator=gen)


def graphed(fn):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g.replay


def main():
    gen = torch.Generator(device="cuda").manual_seed(7)
    out = []
    # cfg1
    n = 4096
    q1 = largest_ntt_primes(50, n, 1)[0]  # cfg1: q == 1 mod 2N
    p1 = nk.RnsNtt(n, [q1])
    x = rnd(n, q1, gen)
    f, b = torch.empty_like(x), torch.empty_like(x)
    step = graphed(lambda: (p1.forward(f, x, 1, 1), p1.inverse(b, f, 1, 1)))
    out.append({"cfg": 1, "op": "fwd(1,1)+inv(1,1) latency, CUDA graph", "us": 1e3 * timed(step, 200, 10)})
    nk.set_block_kernel(6)  # plain block kernel for comparison
    step = graphed(lambda: (p1.forward(f, x, 1, 1), p1.inverse(b, f, 1, 1)))
    out.append({"cfg": 1, "op": "fwd+inv latency, plain block kernel (mode 6)", "us": 1e3 * timed(step, 200, 10)})
    nk.set_block_kernel(-1)
    out.append({"cfg": 1, "op": "fwd+inv latency, stream launches (no graph)",
                "us": 1e3 * timed(lambda: (p1.forward(f, x, 1, 1), p1.inverse(b, f, 1, 1)), 200, 10)})
    # cfg2
    q = cfg2_modulus()
    n2, sets = 1 << 20, 16
    a = torch.stack([rnd(n2, q, gen) for _ in range(sets)])
    c = torch.stack([rnd(n2, q, gen) for _ in range(sets)])
    r = torch.empty_like(a)
    y = int(torch.randint(0, 1 << 59, (1,)).item()) % q
    ops = {
        "EltwiseMultMod vv (24 B/word)": (lambda i: nk.eltwise_mult_mod(r[i], a[i], c[i], q, 1), 24),
        "EltwiseFMAMod vs, no addend (16 B/word)": (lambda i: nk.eltwise_fma_mod(r[i], a[i], y, None, q, 1), 16),
        "EltwiseFMAMod (24 B/word)": (lambda i: nk.eltwise_fma_mod(r[i], a[i], y, c[i], q, 1), 24),
    }
    for name, (op, bpw) in ops.items():
        step = graphed(lambda: [op(i) for i in range(sets)])
        us = 1e3 * timed(step, 20, 3) / sets
        out.append({"cfg": 2, "op": name, "us_per_call": us, "GB_s": bpw * n2 / us / 1e3})
    del a, c, r
    # f-3: the two multiply paths at q < 2^50 (the reference takes the FP64 one)
    q50 = largest_ntt_primes(50, 2, 1)[0]
    a = torch.stack([rnd(n2, q50, gen) for _ in range(sets)])
    c = torch.stack([rnd(n2, q50, gen) for _ in range(sets)])
    r = torch.empty_like(a)
    for name, fn in (("int", nk.eltwise_mult_mod_int), ("float", nk.eltwise_mult_mod_float)):
        step = graphed(lambda: [fn(r[i], a[i], c[i], q50, 1) for i in range(sets)])
        us = 1e3 * timed(step, 20, 3) / sets
        out.append({"cfg": "2b", "op": f"EltwiseMultMod 50-bit q, {name} path", "us_per_call": us,
                    "GB_s": 24 * n2 / us / 1e3})
    del a, c, r
    # cfg3
    n = 16384
    m3 = largest_ntt_primes(50, n, 32)
    p3 = nk.RnsNtt(n, m3)
    words = 64 * 32 * n
    x = rnd(words, min(m3), gen)
    o = torch.empty_like(x)
    fwd = timed(lambda: p3.forward(o, x, 1, 1))
    inv = timed(lambda: p3.inverse(o, x, 1, 1))
    out.append({"cfg": 3, "op": "forward(1,1)", "us": 1e3 * fwd, "Gcoeff_s": words / fwd / 1e6})
    out.append({"cfg": 3, "op": "inverse(1,1)", "us": 1e3 * inv, "Gcoeff_s": words / inv / 1e6})
    del x, o
    # cfg4
    n = 65536
    m4 = largest_ntt_primes(60, n, 24)
    p4 = nk.RnsNtt(n, m4)
    words = 16 * 24 * n
    x = rnd(words, 4 * min(m4), gen)
    x2 = rnd(words, 2 * min(m4), gen)
    o = torch.empty_like(x)
    fwd = timed(lambda: p4.forward(o, x, 4, 1))
    inv = timed(lambda: p4.inverse(o, x2, 2, 1))
    out.append({"cfg": 4, "op": "forward(4,1)", "us": 1e3 * fwd, "Gcoeff_s": words / fwd / 1e6})
    out.append({"cfg": 4, "op": "inverse(2,1)", "us": 1e3 * inv, "Gcoeff_s": words / inv / 1e6})
    del x, x2, o
    # cfg5
    n = 16384
    m5 = m3[:16]
    p5 = nk.RnsNtt(n, m5)
    words = 128 * 16 * n
    fx, gx = rnd(words, min(m5), gen), rnd(words, min(m5), gen)
    o = torch.empty_like(fx)
    t5 = timed(lambda: p5.poly_mult_mod(o, fx, gx), 10, 2)
    out.append({"cfg": 5, "op": "poly_mult_mod (2048 row pairs)", "us": 1e3 * t5,
                "Gcoeff_s": words / t5 / 1e6, "hbm_floor_us": 24 * words / 6455.6e3})
    nk.set_block_kernel(0)  # the three-launch sequence, for comparison
    t5b = timed(lambda: p5.poly_mult_mod(o, fx, gx), 10, 2)
    nk.set_block_kernel(-1)
    out.append({"cfg": 5, "op": "poly_mult_mod, three launches", "us": 1e3 * t5b,
                "Gcoeff_s": words / t5b / 1e6})
    for line in out:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
