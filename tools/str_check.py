import sys, os, json
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2103_16400_b200 as nk
from bench import largest_ntt_primes
n = 16384
for bits, limbs, polys, fin in ((50, 32, 64, 1), (50, 3, 5, 1), (60, 4, 8, 4), (50, 2, 3, 2)):
    moduli = largest_ntt_primes(bits, n, limbs)
    plan = nk.RnsNtt(n, moduli)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randint(0, 1 << (bits - 1), (limbs * polys * n,), dtype=torch.int64, device="cuda", generator=g)
    nk.set_block_kernel(1)
    ref = plan.forward(torch.empty_like(x), x, fin, 1)
    ref4 = plan.forward(torch.empty_like(x), x, fin, 4)
    nk.set_block_kernel(2)
    got = plan.forward(torch.empty_like(x), x, fin, 1)
    got4 = plan.forward(torch.empty_like(x), x, fin, 4)
    torch.cuda.synchronize()
    bad = (ref != got).nonzero()
    print(bits, limbs, polys, fin, "fout1 equal:", bool((ref == got).all()), "fout4 equal:", bool((ref4 == got4).all()),
          "mismatches:", int(bad.numel()), bad[:5].flatten().tolist())
    if bits == 50 and limbs == 32:
        def timed(fn, reps=30):
            for _ in range(3): fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); e0.record()
            for _ in range(reps): fn()
            e1.record(); torch.cuda.synchronize()
            return e0.elapsed_time(e1) * 1e3 / reps
        out = torch.empty_like(x)
        for kk in (1, 2):
            nk.set_block_kernel(kk)
            print("kernel", kk, "fwd us", timed(lambda: plan.forward(out, x, 1, 1)))
nk.set_block_kernel(-1)
