#!/usr/bin/env python
"""Generate tests/golden/golden.npz from the REFERENCE ITSELF.

Runs the unmodified nttkit headers (compiled into oracle/_ref/libnttref.so by
oracle/Makefile from /root/reference/proj/include) on seeded inputs and stores
inputs + outputs. The fixtures pin both the C oracle (tests/test_oracle.py,
CPU) and the GPU kernels (tests/test_gpu_golden.py) to the reference on a
machine where /root/reference is absent (the GPU box).

Usage (in the build container, where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import Oracle, Ref  # noqa: E402
from primes import cfg2_modulus, config_seed, largest_ntt_primes, smallest_ntt_primes  # noqa: E402


def main():
    ref, o = Ref(), Oracle()
    g = {}
    cases = []
    # ---- tables: (n, q) incl. the reference tests' q=17/97 and the config primes ----
    table_cases = [(4, 17, 0), (8, 97, 0), (16, 97, 0), (64, smallest_ntt_primes(50, 64, 1)[0], 0),
                   (64, smallest_ntt_primes(49, 64, 1)[0], 64),
                   (256, smallest_ntt_primes(61, 256, 1)[0], 0),
                   (4096, largest_ntt_primes(50, 4096, 1)[0], 0)]
    for i, (n, q, bs) in enumerate(table_cases):
        t = ref.tables(n, q, 0, bs)
        g[f"tab{i}_meta"] = np.array([n, q, bs, t["psi"], t["ninv"], t["ninvp"], t["bit_shift"]],
                                     np.uint64)
        for k in ("w", "wp", "wi", "wip"):
            g[f"tab{i}_{k}"] = t[k]
    # ---- transforms across sizes, bit classes and (fin, fout) with lifted inputs ----
    k = 0
    for n in (2, 4, 8, 16, 32, 64, 128, 256):
        for bits in (20, 30, 50, 61):
            q = smallest_ntt_primes(bits, n, 1)[0]
            x = o.mt19937_64(7000 + k, n, q)
            for fin, fout in ((1, 1), (1, 4), (2, 1), (4, 4)):
                xi = x + np.uint64(q) * o.mt19937_64(8000 + k, n, fin)
                g[f"fwd{k}_meta"] = np.array([n, q, fin, fout], np.uint64)
                g[f"fwd{k}_in"] = xi
                g[f"fwd{k}_out"] = ref.forward(n, [q], xi, fin, fout)
                k += 1
    kf = k
    k = 0
    for n in (2, 8, 64, 256):
        for bits in (20, 50, 61):
            q = smallest_ntt_primes(bits, n, 1)[0]
            x = o.mt19937_64(9000 + k, n, q)
            for fin, fout in ((1, 1), (1, 2), (2, 1), (2, 2)):
                xi = x + np.uint64(q) * o.mt19937_64(9500 + k, n, fin)
                g[f"inv{k}_meta"] = np.array([n, q, fin, fout], np.uint64)
                g[f"inv{k}_in"] = xi
                g[f"inv{k}_out"] = ref.inverse(n, [q], xi, fin, fout)
                k += 1
    ki = k
    # ---- cfg1: N=4096, 50-bit q, seeded input; canonical and lazy ----
    n, q = 4096, largest_ntt_primes(50, 4096, 1)[0]
    x = o.mt19937_64(config_seed(1), n, q)
    g["cfg1_x"] = x
    g["cfg1_q"] = np.array([q], np.uint64)
    g["cfg1_fwd11"] = ref.forward(n, [q], x, 1, 1)
    g["cfg1_fwd14"] = ref.forward(n, [q], x, 1, 4)
    g["cfg1_inv11"] = ref.inverse(n, [q], g["cfg1_fwd11"], 1, 1)
    g["cfg1_inv12"] = ref.inverse(n, [q], g["cfg1_fwd11"], 1, 2)
    # ---- element-wise: cfg2 modulus, first 4096 words, plus small moduli ----
    q2 = cfg2_modulus()
    s = config_seed(2)
    a = o.mt19937_64(s, 4096, q2)
    b = o.mt19937_64(s + 1, 4096, q2)
    z = o.mt19937_64(s + 2, 4096, q2)
    y = int(o.mt19937_64(s + 3, 1, q2)[0])
    g["elt_q"] = np.array([q2, y], np.uint64)
    g["elt_a"], g["elt_b"], g["elt_z"] = a, b, z
    g["elt_mult"] = ref.eltwise_mult_mod(a, b, q2, 1)
    g["elt_vs"] = ref.eltwise_fma_mod(a, y, None, q2, 1)
    g["elt_fma"] = ref.eltwise_fma_mod(a, y, z, q2, 1)
    # factor-4 products on a 50-bit modulus (reference takes its FP64 path)
    q50 = largest_ntt_primes(50, 1, 1)[0]
    a4 = o.mt19937_64(61, 4096, 4 * q50)
    b4 = o.mt19937_64(62, 4096, 4 * q50)
    g["elt4_q"] = np.array([q50], np.uint64)
    g["elt4_a"], g["elt4_b"] = a4, b4
    g["elt4_mult"] = ref.eltwise_mult_mod(a4, b4, q50, 4)
    g["elt4_fma8"] = ref.eltwise_fma_mod(o.mt19937_64(63, 4096, 8 * q50), 12345, None, q50, 8)
    g["elt4_fma8_in"] = o.mt19937_64(63, 4096, 8 * q50)
    # ---- ring: poly_mult_mod vs the reference at small n and one cfg5-size row ----
    for i, (n, bits) in enumerate(((16, 30), (256, 50), (256, 61), (16384, 50))):
        q = (largest_ntt_primes(50, n, 1) if n == 16384 else smallest_ntt_primes(bits, n, 1))[0]
        f = o.mt19937_64(70 + i, n, q)
        gg = o.mt19937_64(80 + i, n, q)
        g[f"poly{i}_meta"] = np.array([n, q], np.uint64)
        g[f"poly{i}_f"], g[f"poly{i}_g"] = f, gg
        g[f"poly{i}_out"] = ref.poly_mult_mod(n, [q], f, gg)
    g["counts"] = np.array([len(table_cases), kf, ki, 4], np.uint64)
    out = os.path.join(HERE, "golden.npz")
    np.savez_compressed(out, **g)
    print(f"wrote {out}: {os.path.getsize(out)} bytes, {len(g)} arrays")


if __name__ == "__main__":
    main()
