#!/usr/bin/env python
"""Benchmark of the B200 NTT hot path (driver contract: one JSON line on rank 0).

Workload (BASELINE.json metric "fwd/inv NTT Mcoeff/s (N=16384, batched
limbs)", config 3): N = 16384, 32 RNS limbs of distinct 50-bit NTT primes
(largest < 2^50, == 1 mod 32768), 64 polynomials -> 2048 rows = 33,554,432
coefficients, uniform in [0, q) from std::mt19937_64 (bench.hpp:126-131).
A step = forward NTT (fin 1, fout 1) + inverse NTT (fin 1, fout 1) over the
whole batch; `value` = coefficient transforms per second (2 x 33.5 M per step)
across all ranks, in Mcoeff/s. Inputs (256 MiB) exceed the 126 MB L2.

Multi-GPU: one process per GPU, each rank transforms its own cfg3 batch
(independent ciphertext polynomials; no collective): weak scaling.

--impl reference: the reference's own CPU code (oracle/_ref/libnttref.so, built
from the unmodified nttkit headers) on all host threads, same config/metric, on
the full cfg3 batch per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "fwd/inv NTT Mcoeff/s (N=16384, batched limbs)"
FWD_KERNEL = "ntt_pair14<Arith52S,fwd>"  # the forward's only launch at cfg3
# FP64 operations per butterfly of the signed canonical arithmetic
# (modmath.cuh Arith52S: 6 for the Shoup product, 2 output adds, 1 for the
# conditional subtraction), the floor the transform kernels are bound by
DP_PER_BFLY = 9
N = 16384
NLIMBS = 32
NPOLYS = 64
SEED = 3 ^ 20260809


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


def _is_prime(n):
    """Deterministic Miller-Rabin for n < 2^64 (the first 12 primes as bases)."""
    if n < 2:
        return False
    small = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)
    for p in small:
        if n % p == 0:
            return n == p
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def largest_ntt_primes(bits, n, count):
    """Descending from 2^bits in steps of 2n: the primes q == 1 (mod 2n) below
    2^bits (the BASELINE configs' moduli)."""
    out, two_n = [], 2 * n
    c = ((1 << bits) - 1) // two_n * two_n + 1
    while len(out) < count and c > 2:
        if c < (1 << bits) and _is_prime(c):
            out.append(c)
        c -= two_n
    return out


def cfg3_moduli():
    """The 32 largest primes < 2^50 that are 1 mod 2N, descending
    (tests/test_bench_inputs.py pins the list)."""
    return largest_ntt_primes(50, N, NLIMBS)


def cfg2_modulus():
    """The largest prime below 2^60 (2^60 - 93)."""
    c = (1 << 60) - 1
    while not _is_prime(c):
        c -= 2
    return c


_MT_NN, _MT_MM = 312, 156
_MT_A, _MT_UM, _MT_LM = np.uint64(0xB5026F5AA96619E9), np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)


def mt19937_64_rows(seeds, count):
    """std::mt19937_64 streams, one per seed, vectorised over the seeds with
    numpy: returns [len(seeds)][count] raw outputs (C++ [rand.eng.mers],
    tests/test_bench_inputs.py checks it against the C generator)."""
    u = np.uint64
    rows = len(seeds)
    mt = np.empty((rows, _MT_NN), np.uint64)
    mt[:, 0] = np.asarray(seeds, np.uint64)
    with np.errstate(over="ignore"):
        for i in range(1, _MT_NN):
            prev = mt[:, i - 1]
            mt[:, i] = u(6364136223846793005) * (prev ^ (prev >> u(62))) + u(i)
    out = np.empty((rows, count), np.uint64)
    done = 0

    def mix(a, b):
        x = (a & _MT_UM) | (b & _MT_LM)
        return (x >> u(1)) ^ np.where((x & u(1)) != 0, _MT_A, u(0))

    while done < count:
        # twist in three vectorised blocks (each block reads only finished words)
        k = _MT_NN - _MT_MM
        mt[:, :k] = mt[:, _MT_MM:] ^ mix(mt[:, :k], mt[:, 1:k + 1])
        mt[:, k:_MT_NN - 1] = mt[:, :_MT_NN - 1 - k] ^ mix(mt[:, k:_MT_NN - 1], mt[:, k + 1:])
        mt[:, _MT_NN - 1] = mt[:, _MT_MM - 1] ^ mix(mt[:, _MT_NN - 1], mt[:, 0])
        y = mt.copy()
        y ^= (y >> u(29)) & u(0x5555555555555555)
        y ^= (y << u(17)) & u(0x71D67FFFEDA60000)
        y ^= (y << u(37)) & u(0xFFF7EEE000000000)
        y ^= y >> u(43)
        take = min(_MT_NN, count - done)
        out[:, done:done + take] = y[:, :take]
        done += take
    return out


def make_inputs(moduli, npolys, seed):
    """[npolys][nlimbs][N] uniform in [0, q_l): row r is std::mt19937_64(seed + r)
    reduced mod its limb's q, the reference bench's eng() % q
    (bench.hpp:126-131)."""
    L = len(moduli)
    rows = npolys * L
    raw = mt19937_64_rows([seed + r for r in range(rows)], N)
    q = np.asarray([moduli[r % L] for r in range(rows)], np.uint64)[:, None]
    return (raw % q).reshape(-1)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run_nvml():
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
                    ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4)]
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                self.samples.append([str(sm), str(mx), f"{pw:.1f}", hex(r)] +
                                    ["Active" if r & b else "Not Active" for _, b in bits])
                self._stop.wait(0.02)

        def run():
            try:
                return run_nvml()
            except Exception:
                pass
            q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                          f"--query-gpu={q}", "--format=csv,noheader,nounits"],
                                         capture_output=True, text=True, timeout=5).stdout
                    self.samples.append([s.strip() for s in out.strip().split(",")])
                except Exception:
                    pass
                self._stop.wait(0.1)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = [float(s[0]) for s in self.samples if len(s) >= 8 and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) >= 8 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            if len(s) >= 8:
                for k, name in enumerate(names):
                    if s[4 + k].lower().startswith("active"):
                        reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def cpu_reference(moduli, rows, reps, threads, min_seconds=0.0, warm_seconds=1.0, check_forward=None):
    """The reference's NttTables::forward/inverse (oracle/_ref, the unmodified
    nttkit headers) on `rows` rows with `threads` host threads; returns the
    per-step times (at least `reps` steps and at least `min_seconds` total)."""
    import ctypes as C

    from oracle_lib import Ref

    ref = Ref()
    npolys = max(1, rows // len(moduli))
    x = make_inputs(moduli, npolys, SEED)[: rows * N]
    out = np.empty_like(x)
    out.fill(0)  # pre-fault: first-touch page faults are not the reference's cost
    mods = np.asarray(moduli, np.uint64)
    p = ref.lib.ref_plan_create(N, mods.ctypes.data_as(C.POINTER(C.c_uint64)), mods.size)
    ptr = lambda a: a.ctypes.data_as(C.POINTER(C.c_uint64))  # noqa: E731
    # steady state: the first steps on a fresh box run up to 2x slower (thread
    # start-up, clock ramp), so at least warm_seconds of untimed steps first
    if check_forward is not None:  # the GPU forward's words against the reference's
        ref.lib.ref_plan_ntt(p, 0, ptr(out), ptr(x), rows, 1, 1, threads)
        assert np.array_equal(out, check_forward[: out.size]), "GPU forward differs from the reference"
    t_w = time.perf_counter()
    while time.perf_counter() - t_w < warm_seconds:
        ref.lib.ref_plan_ntt(p, 0, ptr(out), ptr(x), rows, 1, 1, threads)
        ref.lib.ref_plan_ntt(p, 1, ptr(out), ptr(out), rows, 1, 1, threads)
    times = []
    t_start = time.perf_counter()
    while len(times) < reps or time.perf_counter() - t_start < min_seconds:
        t0 = time.perf_counter()
        ref.lib.ref_plan_ntt(p, 0, ptr(out), ptr(x), rows, 1, 1, threads)
        ref.lib.ref_plan_ntt(p, 1, ptr(out), ptr(out), rows, 1, 1, threads)
        times.append(time.perf_counter() - t0)
    ref.lib.ref_plan_destroy(p)
    assert np.array_equal(out, x), "reference round trip failed"
    return times


def run_reference(args):
    """--impl reference: the reference's own CPU implementation of the path
    (nttkit NttTables::forward + inverse, compiled -O3 -DNDEBUG into
    oracle/_ref/libnttref.so) on all host threads, the full cfg3 batch per step.
    Under torchrun only rank 0 runs it."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    moduli = cfg3_moduli()
    threads = os.cpu_count() or 1
    rows = NPOLYS * NLIMBS
    # warm-up: W steps and at least 1 s of steady state (inside cpu_reference)
    times = cpu_reference(moduli, rows, args.steps, threads,
                          warm_seconds=max(1.0, args.warmup * 0.1))
    t = statistics.median(times)
    v = 2 * rows * N / t / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "Mcoeff/s",
        "n_gpus": args.gpus, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (mt19937_64, uniform [0,q))",
        "config": {"workload": "cfg3: N=16384, 32 limbs x 64 polys, fwd(1,1)+inv(1,1)",
                   "rows_per_step": rows},
        "cpu_baseline": {"value": v, "unit": "Mcoeff/s", "cores": threads, "kind": "reference",
                         "sample": f"full cfg3 batch ({rows} rows of N=16384) fwd+inv per step"},
        "e2e": {"value": v, "unit": "Mcoeff/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def ncu_traffic():
    """dram read+write bytes per forward launch from the committed ncu capture
    (profiles/ncu_summary.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        k = d["kernels"][FWD_KERNEL]
        return float(k["dram_bytes_read"]) + float(k["dram_bytes_write"])
    except Exception:
        return None


def modmul_bench(stream, reps=20):
    """cfg2 vector-vector EltwiseMultMod, 2^20 words, 60-bit q, on 16 rotating
    buffer sets (16 x 24 MiB > 126 MB L2): GB/s at 24 B/word."""
    import torch

    import paper_2103_16400_b200 as nk

    q = cfg2_modulus()
    n = 1 << 20
    sets = 16
    g = torch.Generator(device="cuda").manual_seed(2)
    a = torch.randint(0, 1 << 59, (sets, n), dtype=torch.int64, device="cuda", generator=g)
    b = torch.randint(0, 1 << 59, (sets, n), dtype=torch.int64, device="cuda", generator=g)
    r = torch.empty_like(a)
    for i in range(sets):
        nk.eltwise_mult_mod(r[i], a[i], b[i], q, 1)
    # one CUDA graph of `sets` launches: device time without host launch overhead
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for i in range(sets):
            nk.eltwise_mult_mod(r[i], a[i], b[i], q, 1)
    graph.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(reps):
        graph.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * sets)
    gbs = 24 * n / (us * 1e-6) / 1e9
    hbm = peaks()[0]
    return {"metric": "EltwiseMultMod GB/s (cfg2: 2^20 x 60-bit, 24 B/word)",
            "value": gbs, "us_per_call": us, "roofline_frac": gbs / hbm, "peak_gbs": hbm,
            "l2": "16 rotating buffer sets of 24 MiB (384 MiB > 126 MB L2)",
            "timing": "one CUDA graph of 16 back-to-back calls (programmatic dependent launch)"}


def pcie_probe(reps=4, nbytes=256 << 20):
    """Pinned-memory PCIe bandwidth on this box: H2D, D2H and both at once
    (GB/s per direction) -- the ceiling of the e2e number."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def rate(fn):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return reps * nbytes / (time.perf_counter() - t0) / 1e9

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    out = {"h2d_gbs": rate(lambda: d.copy_(h, non_blocking=True)),
           "d2h_gbs": rate(lambda: h2.copy_(d2, non_blocking=True)),
           "duplex_gbs_per_direction": rate(both)}
    del h, h2, d, d2
    return out


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2103_16400_b200 as nk

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    moduli = cfg3_moduli()
    plan = nk.RnsNtt(N, moduli, device=local)
    words = NPOLYS * NLIMBS * N
    x = make_inputs(moduli, NPOLYS, SEED + rank * 100003)
    d_in = torch.from_numpy(x.view(np.int64)).cuda()
    d_f = torch.empty_like(d_in)
    d_b = torch.empty_like(d_in)
    stream = torch.cuda.current_stream()

    def step():
        plan.forward(d_f, d_in, 1, 1)
        plan.inverse(d_b, d_f, 1, 1)

    # correctness gate before timing (bench.hpp:346-356 convention): the round
    # trip here; rank 0's cpu_baseline leg also checks the forward words
    # against the reference's own (the only use of oracle/ in this arm)
    step()
    torch.cuda.synchronize()
    assert torch.equal(d_b, d_in), "round trip mismatch"
    fwd_words = d_f.cpu().numpy().view(np.uint64) if (rank == 0 and not args.no_cpu_baseline) else None

    for _ in range(args.warmup):
        step()
    # per-kernel events on the launching stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    l0 = nk.launch_count()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    for i in range(args.steps):
        ev[i][0].record(stream)
        plan.forward(d_f, d_in, 1, 1)
        ev[i][1].record(stream)
        plan.inverse(d_b, d_f, 1, 1)
        ev[i][2].record(stream)
    t_end.record(stream)
    torch.cuda.synchronize()
    launches = nk.launch_count() - l0
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    total_ms = t_start.elapsed_time(t_end)
    fwd_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in ev)
    inv_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in ev)
    if world > 1:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_step = total_ms / args.steps
    coeffs_step = 2 * words * world
    value = coeffs_step / (ms_step * 1e-3) / 1e6

    # ---- end to end through the C-ABI host-buffer calls (pinned memory) ----
    hx = torch.from_numpy(x.view(np.int64)).pin_memory().numpy().view(np.uint64)
    hf = torch.empty(words, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
    hb = torch.empty(words, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
    e2e_steps = max(2, min(args.steps, 5))
    plan.forward(hf, hx, 1, 1)
    plan.inverse(hb, hf, 1, 1)
    assert np.array_equal(hb, x)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        plan.forward(hf, hx, 1, 1)
        plan.inverse(hb, hf, 1, 1)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = coeffs_step / e2e_s / 1e6

    pcie = pcie_probe() if rank == 0 else None
    if pcie:
        # each step moves 2 x 8 B/coeff each way per direction-op: the duplex ceiling
        pcie["e2e_ceiling_mcoeff_s"] = coeffs_step / (2 * 8 * words / (pcie["duplex_gbs_per_direction"] * 1e9)) / 1e6

    hbm, smmax, peak_kind = peaks()
    # dominant kernel: the forward block kernel (one launch per forward)
    fwd_bytes = 16 * words  # read + write each coefficient once
    achieved = fwd_bytes / (fwd_ms * 1e-3) / 1e9
    butterflies = (N // 2) * 14 * NPOLYS * NLIMBS
    sm_clock = clocks.get("sm_mhz") or smmax
    dp_floor_us = butterflies * DP_PER_BFLY / (64 * 148 * sm_clock * 1e6) * 1e6
    survey_int_us = butterflies * 30 / (128 * 148 * smmax * 1e6) * 1e6
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            rows = NPOLYS * NLIMBS
            times = cpu_reference(moduli, rows, 2, threads, min_seconds=10.0, check_forward=fwd_words)
            tt = statistics.median(times)
            cpu = {"value": 2 * rows * N / tt / 1e6, "unit": "Mcoeff/s", "cores": threads,
                   "kind": "reference",
                   "sample": f"full cfg3 batch fwd+inv, {len(times)} steps (~10 s), reference "
                             f"NttTables (-O3 -DNDEBUG) on {threads} threads"}
        modmul = modmul_bench(stream)
        line = {
            "metric": METRIC, "value": value, "unit": "Mcoeff/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (mt19937_64, uniform [0,q))",
            "config": {"workload": "cfg3: N=16384, 32 limbs x 64 polys per GPU, fwd(1,1)+inv(1,1)",
                       "rows_per_gpu": NPOLYS * NLIMBS, "l2": "inputs 256 MiB > 126 MB L2",
                       "parallelism": f"limb/poly sharding x{world}, no collective"},
            "fwd_ms": fwd_ms, "inv_ms": inv_ms,
            "fwd_mcoeff_s": words / fwd_ms / 1e3, "inv_mcoeff_s": words / inv_ms / 1e3,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": ncu_traffic(), "kernel": FWD_KERNEL,
                         "peak_kind": peak_kind, "algorithmic_bytes_per_launch": fwd_bytes,
                         "note": "traffic: dram read+write of one ncu --set full capture "
                                 "(profiles/ncu_summary.json); the kernel is FP64-pipe bound, "
                                 "see compute"},
            # the binding roofline of the transform: FP64 issue (64 DP ops/clk/SM,
            # tools/pipe_bench.cu) at the run's SM clock
            "compute": {"pipe": "fp64", "dp_ops_per_butterfly": DP_PER_BFLY,
                        "butterflies_per_launch": butterflies,
                        "t_floor_us": dp_floor_us, "t_measured_us": fwd_ms * 1e3,
                        "frac": dp_floor_us / (fwd_ms * 1e3),
                        "sm_mhz": sm_clock},
            "int_pipe": {"butterflies_per_launch": butterflies,
                         "gbfly_s": butterflies / (fwd_ms * 1e-3) / 1e9,
                         "survey_int_model_frac": survey_int_us / (fwd_ms * 1e3),
                         "survey_int_model": "30 integer instr/butterfly at 128 lanes/clk/SM "
                                             "(SURVEY.md 8(d))"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "Mcoeff/s", "h2d_bytes_per_step": 2 * 8 * words,
                    "d2h_bytes_per_step": 2 * 8 * words,
                    "path": "nk_ntt_forward_host + nk_ntt_inverse_host (pinned host buffers; chunked upload / compute / download pipeline, 4 PCIe transfers of 256 MiB per step)",
                    "pcie": pcie},
            "gpu_launches": launches, "clocks": clocks,
            "modmul": modmul,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
