#!/usr/bin/env python
"""Per-phase durations of the two-stream inverse ntt_stri14 (NK_DBG_TIMELINE build):
   NK_LIB_PATH=paper_2103_16400_b200/libnttkit_b200_tl.so python tools/timeline_stri.py"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2103_16400_b200 as nk  # noqa: E402
from bench import largest_ntt_primes  # noqa: E402

n = 16384
plan = nk.RnsNtt(n, largest_ntt_primes(50, n, 32))
nk.set_block_kernel(2)
x = torch.randint(0, 1 << 49, (64 * 32 * n,), dtype=torch.int64, device="cuda")
o = torch.empty_like(x)
plan.inverse(o, x, 1, 1)
dbg = torch.zeros(148 * 16 * 16 * 16, dtype=torch.int64, device="cuda")
nk.lib().nk_debug_dump_to(C.c_void_p(dbg.data_ptr()))
plan.inverse(o, x, 1, 1)
torch.cuda.synchronize()
nk.lib().nk_debug_dump_to(None)
t = dbg.cpu().numpy().reshape(148, 16, 16, 16)[:, :, :, :12].astype(np.float64)
valid = (t[..., 0] > 0) & (t[..., 11] > 0)
names = ["wait for the block", "input reads", "A: Q4', shuffle, Q3', e2' write", "B: Q4', shuffle, Q3'", "e2' read A, write B",
         "Q2' A, read B", "wait inputs read, e1' write A, Q2' B, e1' write B", "wait A written", "read A, P1' A",
         "wait B, read B, P1' B", "bit 13 (+ n^-1), stores"]
d = np.diff(t, axis=-1)[valid]
tot = d.sum(axis=1)
print(f"items {valid.sum()}, mean item {tot.mean():.0f} clk, median {np.median(tot):.0f}")
for i, nm in enumerate(names):
    print(f"  {nm:28s} mean {d[:, i].mean():8.0f}  p50 {np.median(d[:, i]):8.0f}  p90 {np.percentile(d[:, i], 90):8.0f}"
          f"  share {100 * d[:, i].mean() / tot.mean():5.1f}%")
ts = t[:, :, 2:12, :]
ok = valid[:, :, 2:12].all(axis=1)
sk = (ts.max(axis=1) - ts.min(axis=1))[ok]
print("  skew across the CTA's 16 warps at each stamp (mean clk):", " ".join(f"{v:.0f}" for v in sk.mean(axis=0)))
