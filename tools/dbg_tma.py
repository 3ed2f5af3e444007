import sys, os, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2103_16400_b200 as nk
from oracle_lib import Oracle
from primes import largest_ntt_primes
o = Oracle()
n = 16384
for bits, nl, npolys in [(30, 3, 2), (50, 3, 2), (50, 1, 1), (50, 1, 300), (60, 3, 2)]:
    moduli = largest_ntt_primes(bits, n, nl)
    plan = nk.RnsNtt(n, moduli)
    rows = nl * npolys
    x = np.concatenate([o.mt19937_64(r + 1, n, moduli[r % nl]) for r in range(rows)])
    d = torch.from_numpy(x.view(np.int64)).cuda()
    for fwd in (True, False):
        out = torch.zeros_like(d)
        (plan.forward if fwd else plan.inverse)(out, d, 1, 1)
        torch.cuda.synchronize()
        got = out.cpu().numpy().view(np.uint64).reshape(rows, n)
        want = (o.forward if fwd else o.inverse)(n, moduli, x, 1, 1, threads=8).reshape(rows, n)
        bad = [r for r in range(rows) if not np.array_equal(got[r], want[r])]
        print(bits, nl, npolys, 'fwd' if fwd else 'inv', 'bad rows', bad[:10], len(bad))
        if bad:
            r = bad[0]
            m = np.nonzero(got[r] != want[r])[0]
            print('  first bad idx', m[:10], len(m), got[r][m[:3]], want[r][m[:3]])
