"""Per-rank shard index map of the ATP layer (product side, no oracle import).

Rank (i1, i2) of DeviceMesh(d1, d2), rank = i1*d2 + i2, holds these
contiguous blocks of each global tensor (math orientation W[in, out]):

    X, Y1, Z, dZ, dY1, dX   [T, h]    cols block i2 of d2          [Replicate, Shard(1)]
    Wqkv [h, 3h]            rows blk(h,d2,i2) x cols blk(3h,d1,i1) [Shard(1), Shard(0)]
    Wo   [h, h]             rows blk(h,d1,i1) x cols blk(h,d2,i2)  [Shard(0), Shard(1)]
    W1   [h, F]             rows blk(h,d2,i2) x cols blk(F,d1,i1)  column-first
    W2   [F, h]             rows blk(F,d1,i1) x cols blk(h,d2,i2)  row-first
    bqkv, b1, QKV, U, H     cols blk(., d1, i1)
    bo, b2                  cols blk(h, d2, i2)
    ctx  [T, h]             cols blk(h, d1, i1)   (whole heads, head-interleaved QKV, G19)

Each entry is (row0, nrows, col0, ncols) in the global tensor; 1-D tensors use
rows (0, 1).
"""
from __future__ import annotations


def blk(n: int, parts: int, i: int) -> tuple[int, int]:
    if n % parts:
        raise ValueError(f"{n} not divisible by {parts}")
    b = n // parts
    return i * b, b


def coords(d1: int, d2: int, rank: int) -> tuple[int, int]:
    return rank // d2, rank % d2


def shard_boxes(d1: int, d2: int, rank: int, T: int, h: int, F: int) -> dict:
    i1, i2 = coords(d1, d2, rank)
    ac = blk(h, d2, i2)
    full_T = (0, T)
    one = (0, 1)
    return {
        "x": full_T + ac, "dz": full_T + ac,
        "wqkv": blk(h, d2, i2) + blk(3 * h, d1, i1), "bqkv": one + blk(3 * h, d1, i1),
        "wo": blk(h, d1, i1) + blk(h, d2, i2), "bo": one + ac,
        "w1": blk(h, d2, i2) + blk(F, d1, i1), "b1": one + blk(F, d1, i1),
        "w2": blk(F, d1, i1) + blk(h, d2, i2), "b2": one + ac,
        # derived activations (for comparing with a gathered reference)
        "qkv": full_T + blk(3 * h, d1, i1), "ctx": full_T + blk(h, d1, i1),
        "y1": full_T + ac, "z": full_T + ac, "u": full_T + blk(F, d1, i1), "h": full_T + blk(F, d1, i1),
        "dx": full_T + ac, "dy1": full_T + ac,
    }


def local_widths(d1: int, d2: int, h: int, F: int) -> dict:
    return {"hc": h // d2, "h1": h // d1, "q1": 3 * h // d1, "F1": F // d1}
