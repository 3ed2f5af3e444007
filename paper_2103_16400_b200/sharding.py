"""Multi-GPU partition of the NTT work (one process per GPU, no collective on
the data path).

RNS limbs and ciphertext polynomials are independent: rank r
of a world of W transforms a contiguous range of limbs (strong scaling: the
limb set is fixed, e.g. BASELINE cfg3's 32 limbs over 1/2/4/8 GPUs) or its own
batch of polynomials (weak scaling). Collectives are used only by the bench
harness for the barrier and the max-over-ranks timing.
"""
from __future__ import annotations


def limb_shard(nlimbs: int, world: int, rank: int) -> tuple[int, int]:
    """(first limb, count) of rank's contiguous limb range; remainders go to the
    lowest ranks so counts differ by at most one."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("invalid world/rank")
    base, rem = divmod(nlimbs, world)
    count = base + (1 if rank < rem else 0)
    first = rank * base + min(rank, rem)
    return first, count


def poly_shard(npolys: int, world: int, rank: int) -> tuple[int, int]:
    """(first poly, count) — the same balanced split over polynomials."""
    return limb_shard(npolys, world, rank)


def shard_rows(x, n: int, nlimbs: int, limb0: int, count: int):
    """Rows of limbs [limb0, limb0+count) from a [npolys][nlimbs][n] batch, as a
    contiguous [npolys][count][n] array (numpy or torch)."""
    npolys = x.reshape(-1).shape[0] // (nlimbs * n)
    v = x.reshape(npolys, nlimbs, n)[:, limb0:limb0 + count, :]
    return v.reshape(-1).copy() if hasattr(v, "copy") else v.contiguous().reshape(-1)
