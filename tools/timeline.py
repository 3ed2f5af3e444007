#!/usr/bin/env python
"""Per-phase durations of the CTA-pair forward kernel (NK_DBG_TIMELINE build):
   NK_LIB_PATH=paper_2103_16400_b200/libnttkit_b200_tl.so python tools/timeline.py"""
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
moduli = largest_ntt_primes(50, n, 32)
plan = nk.RnsNtt(n, moduli)
nk.set_block_kernel(0)  # the CTA-pair kernel
x = torch.randint(0, 1 << 49, (64 * 32 * n,), dtype=torch.int64, device="cuda")
o = torch.empty_like(x)
plan.forward(o, x, 1, 1)
dbg = torch.zeros(296 * 8 * 32 * 16, dtype=torch.int64, device="cuda")
nk.lib().nk_debug_dump_to(C.c_void_p(dbg.data_ptr()))
plan.forward(o, x, 1, 1)
torch.cuda.synchronize()
nk.lib().nk_debug_dump_to(None)
t = dbg.cpu().numpy().reshape(296, 8, 32, 16)[:, :, :, :10].astype(np.float64)
valid = (t[..., 0] > 0) & (t[..., 9] > 0)
names = ["wait TMA", "P1 loads", "P1 compute", "ex1 (DSMEM, rendezvous)", "P2 reads + TMA issue",
         "P2 compute", "ex2 (warp-local)", "P3 compute", "output"]
d = np.diff(t, axis=-1)[valid]
tot = d.sum(axis=1)
print(f"items {valid.sum()}, mean item {tot.mean():.0f} clk, median {np.median(tot):.0f}")
for i, nm in enumerate(names):
    print(f"  {nm:26s} mean {d[:, i].mean():8.0f}  p50 {np.median(d[:, i]):8.0f}  p90 {np.percentile(d[:, i], 90):8.0f}"
          f"  share {100 * d[:, i].mean() / tot.mean():5.1f}%")
# gap between items (end of item k to start of item k+1 on the same warp)
t0 = t[..., 0]
t9 = t[..., 9]
gaps = (t0[:, :, 1:] - t9[:, :, :-1])[valid[:, :, 1:] & valid[:, :, :-1]]
print(f"  gap between items mean {gaps.mean():.0f}")
