import sys, os, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2103_16400_b200 as nk
from bench import largest_ntt_primes
def timed(fn, reps=20, warm=3):
    for _ in range(warm): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps
n = 16384
gen = torch.Generator(device="cuda").manual_seed(1)
m = largest_ntt_primes(50, n, 32)
words = 128 * 16 * n
bufs = [torch.randint(0, min(m), (words,), dtype=torch.int64, device="cuda", generator=gen) for _ in range(3)]
x = torch.randint(0, 1 << 49, (64 * 32 * n,), dtype=torch.int64, device="cuda", generator=gen)
o3 = torch.empty_like(x)
plans = []
for i in range(8):
    p = nk.RnsNtt(n, m[:16]); plans.append(p)
    t5 = timed(lambda: p.poly_mult_mod(bufs[2], bufs[0], bufs[1]), 20, 3)
    for kk in (3,):
        nk.set_block_kernel(kk); t5o = timed(lambda: p.poly_mult_mod(bufs[2], bufs[0], bufs[1]), 20, 3); nk.set_block_kernel(-1)
    p32 = nk.RnsNtt(n, m); plans.append(p32)
    f = timed(lambda: p32.forward(o3, x, 1, 1)); iv = timed(lambda: p32.inverse(o3, x, 1, 1))
    nk.set_block_kernel(1); f1 = timed(lambda: p32.forward(o3, x, 1, 1)); i1 = timed(lambda: p32.inverse(o3, x, 1, 1)); nk.set_block_kernel(-1)
    print(f"plan pair {i}: poly_str {t5:.1f}  poly_mul14 {t5o:.1f} | cfg3 str fwd {f:.1f} inv {iv:.1f} | grp fwd {f1:.1f} inv {i1:.1f}")
