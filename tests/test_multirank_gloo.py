"""The N>1 path on CPU: world_size 2 over gloo (127.0.0.1).

Each rank takes its limb shard (sharding.limb_shard) of a cfg3-shaped batch
(smaller N), transforms it with the CPU oracle (standing in for its GPU, which
this container does not have), and the shards are all-gathered and compared
with the whole-batch transform: the partition covers every (poly, limb) row
exactly once and needs no exchange. Also checks the max-over-ranks timing
reduction the bench uses.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle_lib import Oracle
        from paper_2103_16400_b200.sharding import limb_shard, shard_rows
        from primes import largest_ntt_primes

        o = Oracle()
        n, nlimbs, npolys = 1024, 6, 4
        moduli = largest_ntt_primes(50, n, nlimbs)
        x = np.concatenate([o.mt19937_64(7 + r, n, moduli[r % nlimbs]) for r in range(npolys * nlimbs)])
        full = o.forward(n, moduli, x, 1, 1)
        l0, cnt = limb_shard(nlimbs, world, rank)
        mine = o.forward(n, moduli[l0:l0 + cnt], shard_rows(x, n, nlimbs, l0, cnt), 1, 1)
        sizes = [None] * world
        dist.all_gather_object(sizes, (l0, cnt))
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        rebuilt = np.empty((npolys, nlimbs, n), np.uint64)
        for (a, c), part in zip(sizes, gathered):
            rebuilt[:, a:a + c, :] = part.reshape(npolys, c, n)
        ok = np.array_equal(rebuilt.reshape(-1), full)
        covered = sorted(l for a, c in sizes for l in range(a, a + c)) == list(range(nlimbs))
        t = torch.tensor([1.0 + rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, ok, covered, float(t.item())))
    finally:
        dist.destroy_process_group()


def test_limb_sharding_two_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    results = sorted(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(ok and cov for _, ok, cov, _ in results), results
    assert all(m == 2.0 for *_, m in results)


@pytest.mark.parametrize("nlimbs,world", [(32, 1), (32, 2), (32, 8), (24, 8), (16, 8), (5, 2), (7, 4)])
def test_limb_shard_balanced(nlimbs, world):
    from paper_2103_16400_b200.sharding import limb_shard

    parts = [limb_shard(nlimbs, world, r) for r in range(world)]
    assert sum(c for _, c in parts) == nlimbs
    assert max(c for _, c in parts) - min(c for _, c in parts) <= 1
    pos = 0
    for a, c in parts:
        assert a == pos
        pos += c


def _bench_worker(rank, world, port, q):
    """bench.py's own multi-GPU helpers on CPU: each rank's share of the cfg3
    batch (rank_inputs, reduced N) and the max/sum-over-ranks reductions."""
    import sys

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import bench

        n, npolys = 64, 3
        limb0, nl, x = bench.rank_inputs(world, rank, n=n, npolys=npolys)
        parts = [None] * world
        dist.all_gather_object(parts, (limb0, nl, x))
        full = bench.make_inputs(bench.cfg3_moduli(), npolys, bench.SEED, n=n).reshape(npolys, bench.NLIMBS, n)
        rebuilt = np.empty_like(full)
        for a, c, part in parts:
            rebuilt[:, a:a + c, :] = part.reshape(npolys, c, n)
        ok = np.array_equal(rebuilt, full)
        mx = bench.reduce_over_ranks(10.0 * (rank + 1), "max", world, "gloo")
        sm = bench.reduce_over_ranks(1.0 + rank, "sum", world, "gloo")
        cfgs = [None] * world
        dist.all_gather_object(cfgs, bench.workload_config(world))
        q.put((rank, ok, mx, sm, all(c == cfgs[0] for c in cfgs)))
    finally:
        dist.destroy_process_group()


def test_bench_multirank_helpers_two_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    results = sorted(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(ok and same for _, ok, _, _, same in results), results
    assert all(mx == 20.0 and sm == 3.0 for _, _, mx, sm, _ in results), results
