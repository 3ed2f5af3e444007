#!/usr/bin/env python
"""Why does bench.py's cfg5 leg time poly_mult_mod slower than tools/prof_ntt.py?
Times the same call under the suspects: operand values (uniform mod q vs
< 2^49), buffers / plan created before or after other allocations, number of
warm-up calls and repetitions.
    python tools/cfg5_probe.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2103_16400_b200 as nk  # noqa: E402
from bench import N, BASE_SEED, cfg3_moduli, make_inputs, dev_time_ms  # noqa: E402

m5 = cfg3_moduli()[:16]
P5 = 128
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()  # noqa: E731


def t(plan, r, f, g, warm, reps):
    return 1e3 * dev_time_ms(lambda: plan.poly_mult_mod(r, f, g), reps, warm)


f5 = make_inputs(m5, P5, 5 ^ BASE_SEED)
g5 = make_inputs(m5, P5, (5 ^ BASE_SEED) + 7919)
words = f5.size
gen = torch.Generator(device="cuda").manual_seed(1)

p_a = nk.RnsNtt(N, m5)
xr = torch.randint(0, 1 << 49, (words,), dtype=torch.int64, device="cuda", generator=gen)
yr = torch.randint(0, 1 << 49, (words,), dtype=torch.int64, device="cuda", generator=gen)
out = torch.empty_like(xr)
for warm, reps in ((3, 10), (3, 10), (20, 50), (3, 10)):
    print(f"fresh plan, randint<2^49 operands, warm {warm} reps {reps}: {t(p_a, out, xr, yr, warm, reps):.1f} us", flush=True)
df, dg = dev(f5), dev(g5)
for warm, reps in ((3, 10), (20, 50)):
    print(f"fresh plan, uniform mod q operands, warm {warm} reps {reps}: {t(p_a, out, df, dg, warm, reps):.1f} us", flush=True)
print(f"fresh plan, randint operands again: {t(p_a, out, xr, yr, 3, 10):.1f} us", flush=True)
# canonical small operands (values < 2^20): does the operand magnitude matter?
xs = torch.randint(0, 1 << 20, (words,), dtype=torch.int64, device="cuda", generator=gen)
print(f"fresh plan, operands < 2^20: {t(p_a, out, xs, xs, 3, 10):.1f} us", flush=True)
# allocations in between (as bench.py's earlier legs leave the caching allocator), then a new plan
junk = [torch.empty(1 << 27, dtype=torch.int64, device="cuda") for _ in range(6)]  # 6 GiB
del junk
p_b = nk.RnsNtt(N, m5)
r2 = torch.empty_like(df)
print(f"second plan after 6 GiB of allocator churn, uniform operands, new result buffer: {t(p_b, r2, df, dg, 3, 10):.1f} us", flush=True)
print(f"second plan, randint operands: {t(p_b, out, xr, yr, 3, 10):.1f} us", flush=True)
print(f"first plan, uniform operands, new result buffer: {t(p_a, r2, df, dg, 3, 10):.1f} us", flush=True)
torch.cuda.empty_cache()
p_c = nk.RnsNtt(N, m5)
print(f"third plan after empty_cache, uniform operands: {t(p_c, r2, df, dg, 3, 10):.1f} us", flush=True)
# idle gap (the bench leg follows seconds of CPU work)
import time
time.sleep(3.0)
print(f"after 3 s idle, warm 3 reps 10: {t(p_a, r2, df, dg, 3, 10):.1f} us", flush=True)
print(f"right after: {t(p_a, r2, df, dg, 3, 10):.1f} us", flush=True)
