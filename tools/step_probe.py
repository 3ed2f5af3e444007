#!/usr/bin/env python
"""What do the per-kernel CUDA events inside bench.py's timed region cost?
cfg3 forward + inverse steps timed (a) with two events around all steps,
(b) with three events per step as bench.py records them, (c) forwards only and
inverses only, back to back.
    python tools/step_probe.py"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2103_16400_b200 as nk  # noqa: E402
from bench import N, cfg3_moduli  # noqa: E402

plan = nk.RnsNtt(N, cfg3_moduli())
words = N * 32 * 64
g = torch.Generator(device="cuda").manual_seed(1)
x = torch.randint(0, 1 << 49, (words,), dtype=torch.int64, device="cuda", generator=g)
f, b = torch.empty_like(x), torch.empty_like(x)
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def run(steps, mode):
    for _ in range(5):
        plan.forward(f, x, 1, 1)
        plan.inverse(b, f, 1, 1)
    evs = [(E(), E(), E()) for _ in range(steps)]
    t0, t1 = E(), E()
    torch.cuda.synchronize()
    t0.record()
    for i in range(steps):
        if mode == "events":
            evs[i][0].record()
        if mode != "inv":
            plan.forward(f, x, 1, 1)
        if mode == "events":
            evs[i][1].record()
        if mode != "fwd":
            plan.inverse(b, f, 1, 1)
        if mode == "events":
            evs[i][2].record()
    t1.record()
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / steps * 1e3


for mode in ("plain", "events", "plain", "events", "fwd", "inv"):
    print(f"{mode:7s} {run(50, mode):8.1f} us per step", flush=True)
