"""Debug: which words of a 16384-word transform differ from the oracle."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2103_16400_b200 as nk
from oracle_lib import Oracle
from primes import largest_ntt_primes
o = Oracle()
n = 16384
for bits in (30, 50):
    moduli = largest_ntt_primes(bits, n, 1)
    plan = nk.RnsNtt(n, moduli)
    for exact in (0, 1):
        nk.set_exact_only(exact)
        for kern in (0, 1):
            nk.set_block_kernel(kern)
            x = o.mt19937_64(5, n * 2, moduli[0])
            d = torch.from_numpy(x.view(np.int64)).cuda()
            for fwd in (True, False):
                out = torch.zeros_like(d)
                (plan.forward if fwd else plan.inverse)(out, d, 1, 1)
                torch.cuda.synchronize()
                got = out.cpu().numpy().view(np.uint64)
                want = (o.forward if fwd else o.inverse)(n, moduli, x, 1, 1)
                bad = np.nonzero(got != want)[0]
                print(f"bits={bits} exact={exact} kern={kern} fwd={fwd}: mism={bad.size}",
                      "" if bad.size == 0 else f"first={bad[:8]} last={bad[-4:]} zeros={np.sum(got[bad]==0)}")
