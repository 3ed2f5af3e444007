#!/usr/bin/env python
"""Per-phase durations and cross-warp skew of the group-exchange kernel (NK_DBG_TIMELINE build):
   make -C paper_2103_16400_b200 variant V=tl F=-DNK_DBG_TIMELINE
   NK_LIB_PATH=paper_2103_16400_b200/libnttkit_b200_tl.so python tools/timeline_grp.py [fwd|inv]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2103_16400_b200 as nk  # noqa: E402
from bench import largest_ntt_primes  # noqa: E402

op = sys.argv[1] if len(sys.argv) > 1 else "inv"
n = 16384
moduli = largest_ntt_primes(50, n, 32)
plan = nk.RnsNtt(n, moduli)
nk.set_block_kernel(1)
x = torch.randint(0, 1 << 49, (64 * 32 * n,), dtype=torch.int64, device="cuda")
o = torch.empty_like(x)
run = (lambda: plan.forward(o, x, 1, 1)) if op == "fwd" else (lambda: plan.inverse(o, x, 1, 1))
run()
dbg = torch.zeros(148 * 16 * 16 * 16, dtype=torch.int64, device="cuda")
nk.lib().nk_debug_dump_to(C.c_void_p(dbg.data_ptr()))
run()
torch.cuda.synchronize()
nk.lib().nk_debug_dump_to(None)
t = dbg.cpu().numpy().reshape(148, 16, 16, 16)[:, :, :, :9].astype(np.float64)  # [cta][warp][item][stamp]
valid = (t[..., 0] > 0) & (t[..., 8] > 0)
names = ["wait TMA", "P1 reads", "P1 compute", "ex1 + refill", "P2 compute", "ex2", "P3 compute", "output"]
d = np.diff(t, axis=-1)[valid]
tot = d.sum(axis=1)
print(f"{op}: items {valid.sum()}, mean item {tot.mean():.0f} clk, median {np.median(tot):.0f}")
for i, nm in enumerate(names):
    print(f"  {nm:14s} mean {d[:, i].mean():8.0f}  p50 {np.median(d[:, i]):8.0f}  p90 {np.percentile(d[:, i], 90):8.0f}"
          f"  share {100 * d[:, i].mean() / tot.mean():5.1f}%")
# skew across the 16 warps of a CTA at each stamp (items 2..12: steady state)
ts = t[:, :, 2:12, :]
ok = valid[:, :, 2:12].all(axis=1)
sk = (ts.max(axis=1) - ts.min(axis=1))[ok]
print("  skew across the CTA's 16 warps at each stamp (mean clk):", " ".join(f"{v:.0f}" for v in sk.mean(axis=0)))
# one CTA, one item: offsets of every warp's stamps relative to the first warp's start
c0 = t[5, :, 5, :] - t[5, :, 5, 0].min()
for w in range(16):
    print(f"  w{w:2d}", " ".join(f"{v:6.0f}" for v in c0[w]))
