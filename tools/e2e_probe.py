#!/usr/bin/env python
"""PCIe probe and host-buffer pipeline timing (cfg3 fwd_host + inv_host).

  python tools/e2e_probe.py pcie        # pinned H2D, D2H, both at once
  python tools/e2e_probe.py e2e         # NK_HOST_CHUNK_MB / NK_HOST_DEPTH from the env
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def pcie():
    n = 256 << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h2.copy_(d2, non_blocking=True))]:
        fn(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        print(f"{name}: {5 * n / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    print(f"both: {5 * n / (time.perf_counter() - t0) / 1e9:.1f} GB/s per direction")


def e2e():
    import paper_2103_16400_b200 as nk
    from bench import largest_ntt_primes
    n, limbs, polys = 16384, 32, 64
    m = largest_ntt_primes(50, n, limbs)
    plan = nk.RnsNtt(n, m)
    words = n * limbs * polys
    rng = np.random.default_rng(1)
    x = (rng.integers(0, min(m), words, dtype=np.int64)).astype(np.int64)
    hx = torch.from_numpy(x).pin_memory().numpy().view(np.uint64)
    hf = torch.empty(words, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
    hb = torch.empty(words, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
    plan.forward(hf, hx, 1, 1)
    plan.inverse(hb, hf, 1, 1)
    assert np.array_equal(hb, x.view(np.uint64))
    steps = 5
    t0 = time.perf_counter()
    for _ in range(steps):
        plan.forward(hf, hx, 1, 1)
        plan.inverse(hb, hf, 1, 1)
    s = (time.perf_counter() - t0) / steps
    print(f"chunk={os.environ.get('NK_HOST_CHUNK_MB', 'default')} depth={os.environ.get('NK_HOST_DEPTH', 'default')}: "
          f"{s * 1e3:.2f} ms/step, {2 * words / s / 1e6:.0f} Mcoeff/s")


if __name__ == "__main__":
    {"pcie": pcie, "e2e": e2e}[sys.argv[1]]()
