import sys, os, json
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2103_16400_b200 as nk
from bench import largest_ntt_primes
def timed(fn, reps=30):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps
for n, bits, limbs, polys, fin in ((16384, 50, 32, 64, 1), (16384, 50, 3, 5, 2), (16384, 60, 4, 8, 1), (16384, 60, 2, 3, 2), (65536, 60, 24, 16, 2)):
    moduli = largest_ntt_primes(bits, n, limbs)
    plan = nk.RnsNtt(n, moduli)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randint(0, 1 << (bits - 1), (limbs * polys * n,), dtype=torch.int64, device="cuda", generator=g)
    nk.set_block_kernel(1)
    ref = plan.inverse(torch.empty_like(x), x, fin, 1)
    ref2 = plan.inverse(torch.empty_like(x), x, fin, 2)
    nk.set_block_kernel(2)
    got = plan.inverse(torch.empty_like(x), x, fin, 1)
    got2 = plan.inverse(torch.empty_like(x), x, fin, 2)
    torch.cuda.synchronize()
    bad = (ref != got).nonzero()
    print(n, bits, limbs, polys, fin, "fout1 equal:", bool((ref == got).all()), "fout2 equal:", bool((ref2 == got2).all()),
          "mismatches:", int(bad.numel()), bad[:5].flatten().tolist())
    if limbs >= 24:
        out = torch.empty_like(x)
        for kk in (1, 2):
            nk.set_block_kernel(kk)
            print("  kernel", kk, "inv us", timed(lambda: plan.inverse(out, x, fin, 1)))
nk.set_block_kernel(-1)
