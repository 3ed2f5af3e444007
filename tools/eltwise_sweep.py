import sys, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2103_16400_b200 as nk
from bench import cfg2_modulus
q = cfg2_modulus()
for logn in (18, 20, 22, 24, 26):
    n = 1 << logn; sets = max(2, (1 << 28) // (24 * n) + 1); reps = 10
    a = torch.randint(0, 1 << 59, (sets, n), dtype=torch.int64, device="cuda")
    b = torch.randint(0, 1 << 59, (sets, n), dtype=torch.int64, device="cuda")
    r = torch.empty_like(a)
    for i in range(sets): nk.eltwise_mult_mod(r[i], a[i], b[i], q, 1)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for i in range(sets): nk.eltwise_mult_mod(r[i], a[i], b[i], q, 1)
    graph.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): graph.replay()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * sets)
    # plain copy for reference
    c = torch.empty(3 * n // 2 * 2, dtype=torch.int64, device='cuda'); d = torch.empty_like(c)
    e0.record()
    for _ in range(reps): d.copy_(c)
    e1.record(); torch.cuda.synchronize()
    cu = e0.elapsed_time(e1) * 1e3 / reps
    print(f"n=2^{logn}: mult {us:8.2f} us {24*n/us/1e3:7.1f} GB/s | copy of same bytes {cu:8.2f} us {24*n/cu/1e3:7.1f} GB/s")
