import sys, os
import numpy as np, torch
sys.path[:0] = [".", "tests"]
import paper_2103_16400_b200 as nk
from oracle_lib import Oracle
from primes import largest_ntt_primes
o = Oracle()
n = 16384
for L, P in ((3, 3), (32, 64), (3, 100)):
    moduli = largest_ntt_primes(50, n, L)
    plan = nk.RnsNtt(n, moduli)
    x = np.concatenate([o.mt19937_64(7 + r, n, moduli[r % L]) for r in range(L * P)])
    d = torch.from_numpy(x.view(np.int64)).cuda()
    nk.set_block_kernel(4)
    out = torch.full_like(d, 7)
    plan.forward(out, d, 1, 1)
    torch.cuda.synchronize()
    got = out.cpu().numpy().view(np.uint64)
    nk.set_block_kernel(0)
    ref = torch.empty_like(d)
    plan.forward(ref, d, 1, 1)
    want = ref.cpu().numpy().view(np.uint64)
    bad = np.nonzero(got != want)[0]
    print(f"L={L} P={P}: mism {bad.size}/{got.size}", "" if not bad.size else
          f"first {bad[:6]} got {got[bad[:3]]} want {want[bad[:3]]} sevens {np.sum(got == 7)}")
