#!/usr/bin/env python
"""cfg2 element-wise kernels for ncu: EltwiseMultMod vv, FMA and vs-mult with
a 60-bit modulus (each launched a few times).

    python tools/prof_eltwise.py            2^20 words (cfg2's size; L2-resident)
    python tools/prof_eltwise.py --big      2^26 words per operand (512 MiB, far
                                            larger than L2): one launch streams
                                            from HBM in steady state, so ncu's
                                            dram__bytes and duration measure the
                                            kernel's sustained bandwidth
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2103_16400_b200 as nk  # noqa: E402
from bench import cfg2_modulus  # noqa: E402

q = cfg2_modulus()
n = 1 << (26 if "--big" in sys.argv else 20)
g = torch.Generator(device="cuda").manual_seed(3)
a = torch.randint(0, q, (n,), dtype=torch.int64, device="cuda", generator=g)
b = torch.randint(0, q, (n,), dtype=torch.int64, device="cuda", generator=g)
r = torch.empty_like(a)
for _ in range(3):
    nk.eltwise_mult_mod(r, a, b, q, 1)
    nk.eltwise_fma_mod(r, a, 12345, b, q, 1)
    nk.eltwise_fma_mod(r, a, 12345, None, q, 1)
torch.cuda.synchronize()
print("ok", n)
