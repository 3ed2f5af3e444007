#!/usr/bin/env python
"""Benchmark records in the reference CLI's format.

Runs the reference's own harness (oracle/_ref/refbench: bench.hpp run_bench +
emit, built from the unmodified headers) for its records, then appends one
`gpu_sm100` row per (kernel, n, q_bits) measured on cuda:0 through this
package, in the same `kernel,n,q_bits,variant,median_ns,speedup_vs_naive`
CSV (or JSON). Same primes (bench.hpp:134-143 bench_prime), same inputs
(bench.hpp:126-131 with the per-record seed of run_bench), and the same rule:
the GPU output is verified against the reference's optimized variant before
it is timed (bench.hpp:346-356).

GPU timing: inputs resident on the device; median over `reps` samples, each a
CUDA-event-timed batch of calls sized to >= 200 us divided by its length
(the reference's calibrated batches, bench.hpp:212-228).

    python tools/bench_records.py [--sizes 1024,4096,16384] [--q-bits 50] [--format csv|json]
"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import paper_2103_16400_b200 as nk  # noqa: E402
from oracle_lib import Oracle, Ref  # noqa: E402
from primes import smallest_ntt_primes  # noqa: E402

KERNELS = ["fwd_ntt", "inv_ntt", "eltwise_mult", "eltwise_fma", "eltwise_add", "poly_mult"]
SEED = 20260809  # Config::seed


def record_seed(kernel, n, q_bits):
    return SEED ^ (KERNELS.index(kernel) << 40) ^ (n << 8) ^ q_bits


def gpu_median_ns(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    once = max(e0.elapsed_time(e1) * 1e6, 1.0)
    iters = max(1, int(2e5 / once))
    samples = []
    for _ in range(reps):
        fn()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        samples.append(e0.elapsed_time(e1) * 1e6 / iters)
    samples.sort()
    m = len(samples) // 2
    return samples[m] if len(samples) % 2 else 0.5 * (samples[m - 1] + samples[m])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1024,4096,16384")
    ap.add_argument("--q-bits", default="50")
    ap.add_argument("--kernels", default=",".join(KERNELS))
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--format", default="csv", choices=["csv", "json"])
    a = ap.parse_args()
    exe = os.path.join(ROOT, "oracle", "_ref", "refbench")
    csv = subprocess.run([exe, "--sizes", a.sizes, "--q-bits", a.q_bits, "--kernels", a.kernels,
                          "--reps", str(a.reps), "--format", "csv"],
                         check=True, capture_output=True, text=True).stdout
    recs = []
    for line in csv.strip().splitlines()[1:]:
        k, n, qb, var, med, sp = line.split(",")
        recs.append(dict(kernel=k, n=int(n), q_bits=int(qb), variant=var, median_ns=float(med),
                         speedup_vs_naive=float(sp)))
    o, ref = Oracle(), Ref()
    out = []
    for kernel in a.kernels.split(","):
        for n in [int(s) for s in a.sizes.split(",")]:
            for qb in [int(s) for s in a.q_bits.split(",")]:
                rows = [r for r in recs if (r["kernel"], r["n"], r["q_bits"]) == (kernel, n, qb)]
                out.extend(rows)
                naive = next(r["median_ns"] for r in rows if r["variant"] == "naive")
                q = smallest_ntt_primes(qb, n, 1)[0]  # bench_prime
                s = record_seed(kernel, n, qb)
                av = o.mt19937_64(s, n, q)
                bv = o.mt19937_64(s + 1, n, q)
                y = int(o.mt19937_64(s + 2, 1, q)[0])
                da = torch.from_numpy(av.view(np.int64)).cuda()
                db = torch.from_numpy(bv.view(np.int64)).cuda()
                dr = torch.empty_like(da)
                plan = nk.RnsNtt(n, [q]) if kernel in ("fwd_ntt", "inv_ntt", "poly_mult") else None
                if kernel == "fwd_ntt":
                    fn = lambda: plan.forward(dr, da, 1, 1)  # noqa: E731
                    want = ref.forward(n, [q], av, 1, 1, bit_shift=64)
                elif kernel == "inv_ntt":
                    fn = lambda: plan.inverse(dr, da, 1, 1)  # noqa: E731
                    want = ref.inverse(n, [q], av, 1, 1, bit_shift=64)
                elif kernel == "eltwise_mult":
                    fn = lambda: nk.eltwise_mult_mod(dr, da, db, q, 1)  # noqa: E731
                    want = ref.eltwise_mult_mod(av, bv, q, 1)
                elif kernel == "eltwise_fma":
                    fn = lambda: nk.eltwise_fma_mod(dr, da, y, db, q, 1)  # noqa: E731
                    want = ref.eltwise_fma_mod(av, y, bv, q, 1, bit_shift=64)
                elif kernel == "eltwise_add":
                    fn = lambda: nk.eltwise_add_mod(dr, da, db, q)  # noqa: E731
                    want = ref.eltwise_add_mod(av, bv, q)
                else:
                    fn = lambda: plan.poly_mult_mod(dr, da, db)  # noqa: E731
                    want = ref.poly_mult_mod(n, [q], av, bv)
                fn()
                torch.cuda.synchronize()
                got = dr.cpu().numpy().view(np.uint64)
                if not np.array_equal(got, want):
                    raise SystemExit(f"bench verification failed: {kernel} n={n} variant gpu_sm100")
                med = gpu_median_ns(fn, a.reps)
                out.append(dict(kernel=kernel, n=n, q_bits=qb, variant="gpu_sm100", median_ns=med,
                                speedup_vs_naive=naive / med))
    if a.format == "json":
        print(json.dumps(out, indent=2))
    else:
        print("kernel,n,q_bits,variant,median_ns,speedup_vs_naive")
        for r in out:
            print(f"{r['kernel']},{r['n']},{r['q_bits']},{r['variant']},{r['median_ns']:.1f},"
                  f"{r['speedup_vs_naive']:.4f}")


if __name__ == "__main__":
    main()
