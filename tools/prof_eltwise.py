#!/usr/bin/env python
"""cfg2 element-wise kernels for ncu: EltwiseMultMod vv, FMA and vs-mult on
2^20 x 60-bit words (each launched a few times)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2103_16400_b200 as nk  # noqa: E402
from bench import cfg2_modulus  # noqa: E402

q = cfg2_modulus()
n = 1 << 20
g = torch.Generator(device="cuda").manual_seed(3)
a = torch.randint(0, q, (n,), dtype=torch.int64, device="cuda", generator=g)
b = torch.randint(0, q, (n,), dtype=torch.int64, device="cuda", generator=g)
r = torch.empty_like(a)
for _ in range(3):
    nk.eltwise_mult_mod(r, a, b, q, 1)
    nk.eltwise_fma_mod(r, a, 12345, b, q, 1)
    nk.eltwise_fma_mod(r, a, 12345, None, q, 1)
torch.cuda.synchronize()
print("ok")
