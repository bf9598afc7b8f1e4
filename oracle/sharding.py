"""Sharding specs on a 2-D mesh — PAPER.md §3.1 "Sharding Spec".

A spec is one placement per MESH dimension ("we have chosen to bind the
strategy to the dimensions of the device mesh"):
    ("S", d)  Shard(d): split tensor dim d into equal contiguous blocks
    ("R",)    Replicate
    ("P",)    Partial(SUM): every rank holds an addend; sum = global tensor

When both mesh dimensions shard the same tensor dimension, mesh dim 1 splits
first and mesh dim 2 splits each resulting block (the "level" reading of P:161:
"the devices in the current group being divided into d_i sub-groups at the
i-th level").
"""
from __future__ import annotations

import numpy as np

from . import mesh as _mesh

S0 = ("S", 0)
S1 = ("S", 1)
R = ("R",)
P = ("P",)


def _block(x: np.ndarray, axis: int, n: int, i: int) -> np.ndarray:
    ext = x.shape[axis]
    if ext % n:
        raise ValueError(f"extent {ext} not divisible by {n}")
    b = ext // n
    sl = [slice(None)] * x.ndim
    sl[axis] = slice(i * b, (i + 1) * b)
    return x[tuple(sl)]


def local(global_t: np.ndarray, spec, d1: int, d2: int, rank: int) -> np.ndarray:
    """The local tensor of ``rank`` for a Partial-free ``spec`` (copy)."""
    i1, i2 = _mesh.coords(d1, d2, rank)
    out = global_t
    for (pl, n, i) in ((spec[0], d1, i1), (spec[1], d2, i2)):
        if pl[0] == "S":
            out = _block(out, pl[1], n, i)
        elif pl[0] == "P":
            raise ValueError("Partial has no canonical local split; use partial_split")
    return np.array(out, copy=True)


def shard(global_t: np.ndarray, spec, d1: int, d2: int) -> list[np.ndarray]:
    return [local(global_t, spec, d1, d2, r) for r in range(d1 * d2)]


def unshard(locals_: list[np.ndarray], spec, d1: int, d2: int) -> np.ndarray:
    """Reassemble the global tensor from per-rank locals (Partial-free spec).

    Replicated copies must agree exactly; Shard blocks are concatenated.
    """
    def rebuild(i1_fixed):
        # Build the tensor seen at mesh level 1 coordinate i1 (combine dim 2).
        pl2 = spec[1]
        parts = [locals_[_mesh.rank_of(d1, d2, i1_fixed, i2)] for i2 in range(d2)]
        if pl2[0] == "S":
            return np.concatenate(parts, axis=pl2[1])
        for p in parts[1:]:
            if not np.array_equal(p, parts[0]):
                raise ValueError("replicas disagree")
        return parts[0]

    lvl = [rebuild(i1) for i1 in range(d1)]
    pl1 = spec[0]
    if pl1[0] == "S":
        return np.concatenate(lvl, axis=pl1[1])
    for p in lvl[1:]:
        if not np.array_equal(p, lvl[0]):
            raise ValueError("replicas disagree")
    return lvl[0]


def local_shape(global_shape, spec, d1: int, d2: int) -> tuple:
    shp = list(global_shape)
    for pl, n in ((spec[0], d1), (spec[1], d2)):
        if pl[0] == "S":
            if shp[pl[1]] % n:
                raise ValueError("not divisible")
            shp[pl[1]] //= n
    return tuple(shp)
