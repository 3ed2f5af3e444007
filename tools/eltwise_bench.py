"""Device-time bench of the element-wise kernels (cfg2 shapes) via CUDA graphs."""
import sys, os
import torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2103_16400_b200 as nk
from bench import cfg2_modulus
q = cfg2_modulus(); n = 1 << 20; sets = 16; reps = 20
g = torch.Generator(device="cuda").manual_seed(2)
a = torch.randint(0, 1 << 59, (sets, n), dtype=torch.int64, device="cuda", generator=g)
b = torch.randint(0, 1 << 59, (sets, n), dtype=torch.int64, device="cuda", generator=g)
r = torch.empty_like(a)
y = 123456789
for name, fn, bytes_per in [
    ("mult", lambda i: nk.eltwise_mult_mod(r[i], a[i], b[i], q, 1), 24),
    ("vs-mult", lambda i: nk.eltwise_fma_mod(r[i], a[i], y, None, q, 1), 16),
    ("fma", lambda i: nk.eltwise_fma_mod(r[i], a[i], y, b[i], q, 1), 24)]:
    for i in range(sets): fn(i)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for i in range(sets): fn(i)
    graph.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): graph.replay()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * sets)
    print(f"{name:8s} {us:7.2f} us/call  {bytes_per * n / us / 1e3:8.1f} GB/s")
