"""DeviceMesh(d1, d2) — PAPER.md §3.1 "Device Mesh" and §3.3.

rank = i1*d2 + i2: pinned by the §3.1 worked example: with
[Shard(1), Shard(0)] the column blocks belong to "rank-[0,1] and rank-[2,3]"
(i.e. ranks sharing i1), and with [Replicate, Shard(0)] "rank-0 and rank-2"
hold the same row block (ranks sharing i2).
"""
from __future__ import annotations


def enumerate_meshes(n: int) -> list[tuple[int, int]]:
    """All 2-D meshes (d1, d2) with d1*d2 = n, by descending d1."""
    if n < 1:
        raise ValueError("n must be >= 1")
    return [(d1, n // d1) for d1 in range(n, 0, -1) if n % d1 == 0]


def coords(d1: int, d2: int, rank: int) -> tuple[int, int]:
    if not 0 <= rank < d1 * d2:
        raise ValueError("rank out of range")
    return rank // d2, rank % d2


def rank_of(d1: int, d2: int, i1: int, i2: int) -> int:
    if not (0 <= i1 < d1 and 0 <= i2 < d2):
        raise ValueError("coordinate out of range")
    return i1 * d2 + i2


def groups(d1: int, d2: int, dim: int) -> list[list[int]]:
    """Communication groups of one mesh dimension ("each communication
    requires only one row or column of workers").

    dim 1: d2 groups, group i2 = the d1 ranks sharing i2, ordered by i1.
    dim 2: d1 groups, group i1 = the d2 ranks sharing i1, ordered by i2.
    """
    if dim == 1:
        return [[rank_of(d1, d2, i1, i2) for i1 in range(d1)] for i2 in range(d2)]
    if dim == 2:
        return [[rank_of(d1, d2, i1, i2) for i2 in range(d2)] for i1 in range(d1)]
    raise ValueError("dim must be 1 or 2")


def group_of(d1: int, d2: int, dim: int, rank: int) -> list[int]:
    i1, i2 = coords(d1, d2, rank)
    return groups(d1, d2, dim)[i2 if dim == 1 else i1]
