import sys, numpy as np, torch, ctypes as C
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2103_16400_b200 as nk
from oracle_lib import Oracle, _ptr
from primes import largest_ntt_primes
o = Oracle(); n = 16384
moduli = largest_ntt_primes(50, n, 1); q = moduli[0]
plan = nk.RnsNtt(n, moduli)
x = o.mt19937_64(1, n, q)
d = torch.from_numpy(x.view(np.int64)).cuda()
for fwd in (True, False):
    dbg = torch.zeros(4 * n + 18000, dtype=torch.int64, device='cuda')
    nk.lib().nk_debug_dump_to(C.c_void_p(dbg.data_ptr()))
    out = torch.zeros_like(d)
    (plan.forward if fwd else plan.inverse)(out, d, 1, 1)
    torch.cuda.synchronize()
    nk.lib().nk_debug_dump_to(None)
    dall = dbg.cpu().numpy().view(np.uint64); dd = dall[:4*n].reshape(4, n); Bd = dall[4*n:]
    for P, st in enumerate((5, 10, 14) if fwd else (4, 9, 14)):
        ref = x.copy()
        o.lib.oc_ntt_stages(n, q, 0 if fwd else 1, _ptr(ref), 1, st)
        bad = np.nonzero(dd[P] != ref)[0]
        print('fwd' if fwd else 'inv', 'pass', P, 'stages', st, 'bad', len(bad), bad[:8], bad[-4:] if len(bad) else '')
    ref = x.copy(); o.lib.oc_ntt_stages(n, q, 0 if fwd else 1, _ptr(ref), 1, 5 if fwd else 4)
    bad = np.nonzero(dd[3] != ref)[0]
    print('after exchange-1: bad', len(bad), bad[:8])
    print(dd[3][8192:8200], ref[8192:8200])
    print('stale?', np.array_equal(dd[3][8192:8200], ref[0:8]), np.array_equal(dd[3][8192:8200], ref[4096:4104]))
    pos = {int(v): i for i, v in enumerate(ref)}
    src = [pos.get(int(dd[3][j]), -1) for j in bad[:12]]
    print('bad j', list(bad[:12]), 'value found at ref index', src)
    # also check against raw input and against pass-0 dump
    pos0 = {int(v): i for i, v in enumerate(dd[0])}
    print('in pass0 dump at', [pos0.get(int(dd[3][j]), -1) for j in bad[:12]])
    # B image check: round h holds P1-state words j with bit13 == h at phys(j & 0x1FFF)
    phys = lambda j: j + (j >> 4) + (j >> 8) + (j >> 12)
    ref5 = x.copy(); o.lib.oc_ntt_stages(n, q, 0 if fwd else 1, _ptr(ref5), 1, 5 if fwd else 4)
    for h in range(2):
        badB = [j for j in range(8192) if (int(Bd[h * 9000 + phys(j)]) & ((1 << 52) - 1)) != int(ref5[j + 8192 * h])]
        print('B round', h, 'bad', len(badB), badB[:6])
