"""ATP transformer linear block: dense definition and the sharded SPMD simulation.

Everything is float64 NumPy.  Citations are PAPER.md lines (P:n) with the
section they fall in; readings of silent/garbled points are SURVEY.md §8(c)
G-numbers, restated in DESIGN.md "Readings of the paper".

Dense definition (what ATP computes exactly, up to summation order — sharding
only re-associates sums):
    attention projections:
        QKV = X Wqkv + bqkv                 (Wqkv columns head-interleaved, G19)
        ctx = core(QKV)                     zero-FLOP stand-in: Q+K+V per head (G20)
        Y1  = X + ctx Wo + bo               (residual, G17)
    feed-forward:
        U   = Y1 W1 + b1,  H = GeLU(U)      (exact erf GeLU, G15)
        Z   = Y1 + H W2 + b2
    backward for a given dZ (dX = dY W^T, dW = X^T dY).

Sharded simulation (§3.2 Fig. 5/6; chunking §4.1):
    column-first linear: X [Replicate, Shard(1)], W [Shard(1), Shard(0)]
        -> local Y partial over mesh dim 2 -> all-reduce dim 2 -> [Shard(1), Replicate]
    row-first linear:    X [Shard(1), Replicate], W [Shard(0), Shard(1)]
        -> local Y [Partial, Shard(1)] -> all-reduce dim 1 -> [Replicate, Shard(1)]
    (dims per Eq. 2 / §3.2, reading G1).  Backward: the dX partial sums reduce on
    the conjugate dimension (col-first: dim 1, row-first: dim 2).
"""
from __future__ import annotations

import numpy as np
from scipy.special import erf

from . import mesh as _mesh
from . import sharding as _sh
from .sharding import P, R, S0, S1

SQRT2 = np.sqrt(2.0)
INV_SQRT_2PI = 1.0 / np.sqrt(2.0 * np.pi)

# Placements
COL_W = (S1, S0)      # column-first weight  [Shard(1), Shard(0)]
ROW_W = (S0, S1)      # row-first weight     [Shard(0), Shard(1)]
ACT = (R, S1)         # block input/output   [Replicate, Shard(1)]
COL_OUT = (S1, R)     # column-first output after the dim-2 all-reduce
BIAS_COL = (S0, R)    # 1-D bias of a column-first output: split by i1
BIAS_ROW = (R, S0)    # 1-D bias of a row-first output:    split by i2


# ---------------------------------------------------------------- elementwise
def gelu(x):
    """GeLU(x) = x * Phi(x), exact erf form (reading G15)."""
    return x * 0.5 * (1.0 + erf(x / SQRT2))


def gelu_grad(x):
    """d/dx [x Phi(x)] = Phi(x) + x phi(x)."""
    return 0.5 * (1.0 + erf(x / SQRT2)) + x * INV_SQRT_2PI * np.exp(-0.5 * x * x)


def core_fwd(qkv, heads: int):
    """Stand-in attention core (G20): ctx[:, j*d:(j+1)*d] = Q_j + K_j + V_j.

    qkv columns are head-interleaved: column = head*3d + s*d + j, s in {q,k,v}.
    """
    T, w = qkv.shape
    d = w // (3 * heads)
    return qkv.reshape(T, heads, 3, d).sum(axis=2).reshape(T, heads * d)


def core_bwd(dctx, heads: int):
    T, w = dctx.shape
    d = w // heads
    return np.repeat(dctx.reshape(T, heads, 1, d), 3, axis=2).reshape(T, 3 * w)


# ---------------------------------------------------------------- dense layer
def dense_forward(g: dict, heads: int) -> dict:
    x = g["x"]
    qkv = x @ g["wqkv"] + g["bqkv"]
    ctx = core_fwd(qkv, heads)
    y1 = x + (ctx @ g["wo"] + g["bo"])
    u = y1 @ g["w1"] + g["b1"]
    hh = gelu(u)
    z = y1 + (hh @ g["w2"] + g["b2"])
    return {"qkv": qkv, "ctx": ctx, "y1": y1, "u": u, "h": hh, "z": z}


def dense_backward(g: dict, c: dict, dz, heads: int) -> dict:
    """Analytic backward through Z, H, U, Y1, ctx, QKV."""
    dh = dz @ g["w2"].T
    dw2 = c["h"].T @ dz
    db2 = dz.sum(axis=0)
    du = dh * gelu_grad(c["u"])
    dw1 = c["y1"].T @ du
    db1 = du.sum(axis=0)
    dy1 = dz + du @ g["w1"].T
    dctx = dy1 @ g["wo"].T
    dwo = c["ctx"].T @ dy1
    dbo = dy1.sum(axis=0)
    dqkv = core_bwd(dctx, heads)
    dwqkv = g["x"].T @ dqkv
    dbqkv = dqkv.sum(axis=0)
    dx = dy1 + dqkv @ g["wqkv"].T
    return {"dx": dx, "dy1": dy1, "du": du, "dh": dh, "dctx": dctx, "dqkv": dqkv,
            "dwqkv": dwqkv, "dbqkv": dbqkv, "dwo": dwo, "dbo": dbo,
            "dw1": dw1, "db1": db1, "dw2": dw2, "db2": db2}


# ---------------------------------------------------------------- collectives
class CommLog:
    """Executed collective list: one entry per collective call (every rank
    makes the same call); size-1 dimensions are skipped (G7)."""

    def __init__(self):
        self.calls = []

    def add(self, phase, name, dim, p, elems):
        self.calls.append((phase, name, dim, p, int(elems)))


def all_reduce(parts: list, d1: int, d2: int, dim: int, log: CommLog | None = None,
               phase: str = "", name: str = ""):
    """Explicit grouped all-reduce over mesh ``dim``.

    Each group's members are summed in ascending mesh coordinate and the sum is
    assigned to every member (a Partial(SUM) -> Replicate conversion).
    """
    p = d1 if dim == 1 else d2
    out = [None] * len(parts)
    for grp in _mesh.groups(d1, d2, dim):
        s = parts[grp[0]].copy()
        for r in grp[1:]:
            s = s + parts[r]
        for r in grp:
            out[r] = s.copy()
    if log is not None and p > 1:
        log.add(phase, name, dim, p, parts[0].size)
    return out


# ---------------------------------------------------------------- one linear
def colfirst_forward(x_loc, w_loc, d1, d2, log=None, tag="col"):
    """Column-first TP GEMM: local X W, all-reduce on dim 2."""
    part = [xl @ wl for xl, wl in zip(x_loc, w_loc)]
    return all_reduce(part, d1, d2, 2, log, "fwd", tag)


def rowfirst_forward(x_loc, w_loc, d1, d2, log=None, tag="row"):
    """Row-first TP GEMM: local X W is [Partial, Shard(1)], all-reduce dim 1."""
    part = [xl @ wl for xl, wl in zip(x_loc, w_loc)]
    return all_reduce(part, d1, d2, 1, log, "fwd", tag)


def linear_backward(kind, x_loc, w_loc, dy_loc, d1, d2, log=None, tag=""):
    """dX = dY W^T reduced on the conjugate dim; dW = X^T dY local."""
    part = [dy @ wl.T for dy, wl in zip(dy_loc, w_loc)]
    dim = 1 if kind == "col" else 2
    dx = all_reduce(part, d1, d2, dim, log, "bwd", tag)
    dw = [xl.T @ dy for xl, dy in zip(x_loc, dy_loc)]
    return dx, dw


# ---------------------------------------------------------------- layer shards
def shard_layer(g: dict, d1: int, d2: int) -> dict:
    """Per-rank shards of the layer's global tensors."""
    sh = {}
    sh["x"] = _sh.shard(g["x"], ACT, d1, d2)
    sh["wqkv"] = _sh.shard(g["wqkv"], COL_W, d1, d2)
    sh["wo"] = _sh.shard(g["wo"], ROW_W, d1, d2)
    sh["w1"] = _sh.shard(g["w1"], COL_W, d1, d2)
    sh["w2"] = _sh.shard(g["w2"], ROW_W, d1, d2)
    for b, spec in (("bqkv", BIAS_COL), ("b1", BIAS_COL), ("bo", BIAS_ROW), ("b2", BIAS_ROW)):
        sh[b] = _bias_shards(g[b], spec, d1, d2)
    if "dz" in g:
        sh["dz"] = _sh.shard(g["dz"], ACT, d1, d2)
    return sh


def _bias_shards(b, spec, d1, d2):
    # A 1-D bias is a row vector [1, n]; Shard(0) of the vector = Shard(1) of the row.
    spec2 = tuple(S1 if pl == S0 else pl for pl in spec)
    return [_sh.local(b[None, :], spec2, d1, d2, r)[0] for r in range(d1 * d2)]


def _rows(a, k, c):
    m = a.shape[0] // c
    return a[k * m:(k + 1) * m]


def spmd_forward(sh: dict, d1: int, d2: int, heads: int, chunks: int = 1,
                 log: CommLog | None = None) -> dict:
    """Sharded layer forward, block by block, chunk by chunk (§3.2.1, §4.1).

    Each block processes chunks k = 0..c-1 independently; the bias of a
    reduced output is added once after the reduction (G16).
    """
    n = d1 * d2
    T = sh["x"][0].shape[0]
    if T % chunks:
        raise ValueError("T % chunks != 0")
    heads_loc = heads // d1
    st = {k: [[None] * chunks for _ in range(n)] for k in ("qkv", "ctx", "y1", "u", "h", "z")}
    # attention: QKV column-first (f1 on dim 2), Out row-first (f2 on dim 1)
    for k in range(chunks):
        xk = [_rows(sh["x"][r], k, chunks) for r in range(n)]
        red = colfirst_forward(xk, sh["wqkv"], d1, d2, log, "qkv")
        for r in range(n):
            st["qkv"][r][k] = red[r] + sh["bqkv"][r]
            st["ctx"][r][k] = core_fwd(st["qkv"][r][k], heads_loc)
    for k in range(chunks):
        red = rowfirst_forward([st["ctx"][r][k] for r in range(n)], sh["wo"], d1, d2, log, "out")
        for r in range(n):
            st["y1"][r][k] = _rows(sh["x"][r], k, chunks) + (red[r] + sh["bo"][r])
    # feed-forward: FC1 column-first (f3 on dim 2), FC2 row-first (f4 on dim 1)
    for k in range(chunks):
        red = colfirst_forward([st["y1"][r][k] for r in range(n)], sh["w1"], d1, d2, log, "fc1")
        for r in range(n):
            st["u"][r][k] = red[r] + sh["b1"][r]
            st["h"][r][k] = gelu(st["u"][r][k])
    for k in range(chunks):
        red = rowfirst_forward([st["h"][r][k] for r in range(n)], sh["w2"], d1, d2, log, "fc2")
        for r in range(n):
            st["z"][r][k] = st["y1"][r][k] + (red[r] + sh["b2"][r])
    return {key: [np.concatenate(v[r], axis=0) for r in range(n)] for key, v in st.items()}


def spmd_backward(sh: dict, fw: dict, dz_loc: list, d1: int, d2: int, heads: int,
                  chunks: int = 1, log: CommLog | None = None) -> dict:
    """Sharded layer backward: per linear, the dX partials of each
    chunk are all-reduced on the conjugate dimension; dW = X^T dY accumulates
    over chunks in order 0..c-1 and needs no communication."""
    n = d1 * d2
    heads_loc = heads // d1
    g = {k: [[None] * chunks for _ in range(n)] for k in ("dh", "du", "dy1", "dctx", "dqkv", "dx")}
    acc = {k: [None] * n for k in ("dw2", "dw1", "dwo", "dwqkv")}
    R_ = lambda a, k: _rows(a, k, chunks)

    def accum(name, r, val):
        acc[name][r] = val if acc[name][r] is None else acc[name][r] + val

    # FC2 (row-first): dH partial over dim 2
    for k in range(chunks):
        dzk = [R_(dz_loc[r], k) for r in range(n)]
        dx, dw = linear_backward("row", [R_(fw["h"][r], k) for r in range(n)], sh["w2"], dzk,
                                 d1, d2, log, "fc2")
        for r in range(n):
            g["dh"][r][k] = dx[r]
            accum("dw2", r, dw[r])
            g["du"][r][k] = dx[r] * gelu_grad(R_(fw["u"][r], k))
    # FC1 (column-first): dY1 partial over dim 1, plus the residual path dZ
    for k in range(chunks):
        dx, dw = linear_backward("col", [R_(fw["y1"][r], k) for r in range(n)], sh["w1"],
                                 [g["du"][r][k] for r in range(n)], d1, d2, log, "fc1")
        for r in range(n):
            g["dy1"][r][k] = R_(dz_loc[r], k) + dx[r]
            accum("dw1", r, dw[r])
    # Out (row-first): dctx partial over dim 2
    for k in range(chunks):
        dx, dw = linear_backward("row", [R_(fw["ctx"][r], k) for r in range(n)], sh["wo"],
                                 [g["dy1"][r][k] for r in range(n)], d1, d2, log, "out")
        for r in range(n):
            g["dctx"][r][k] = dx[r]
            accum("dwo", r, dw[r])
            g["dqkv"][r][k] = core_bwd(dx[r], heads_loc)
    # QKV (column-first): dX partial over dim 1, plus the residual path dY1
    for k in range(chunks):
        dx, dw = linear_backward("col", [R_(sh["x"][r], k) for r in range(n)], sh["wqkv"],
                                 [g["dqkv"][r][k] for r in range(n)], d1, d2, log, "qkv")
        for r in range(n):
            g["dx"][r][k] = g["dy1"][r][k] + dx[r]
            accum("dwqkv", r, dw[r])
    out = {key: [np.concatenate(v[r], axis=0) for r in range(n)] for key, v in g.items()}
    out.update(acc)
    out["db2"] = [dz_loc[r].sum(axis=0) for r in range(n)]
    out["db1"] = [out["du"][r].sum(axis=0) for r in range(n)]
    out["dbo"] = [out["dy1"][r].sum(axis=0) for r in range(n)]
    out["dbqkv"] = [out["dqkv"][r].sum(axis=0) for r in range(n)]
    return out


# Placement of every layer tensor after its block (for unsharding results).
SPECS = {
    "x": ACT, "y1": ACT, "z": ACT, "dz": ACT, "dy1": ACT, "dx": ACT,
    "qkv": COL_OUT, "ctx": COL_OUT, "u": COL_OUT, "h": COL_OUT,
    "dh": COL_OUT, "du": COL_OUT, "dctx": COL_OUT, "dqkv": COL_OUT,
    "wqkv": COL_W, "w1": COL_W, "dwqkv": COL_W, "dw1": COL_W,
    "wo": ROW_W, "w2": ROW_W, "dwo": ROW_W, "dw2": ROW_W,
}
BIAS_SPECS = {"bqkv": BIAS_COL, "b1": BIAS_COL, "dbqkv": BIAS_COL, "db1": BIAS_COL,
              "bo": BIAS_ROW, "b2": BIAS_ROW, "dbo": BIAS_ROW, "db2": BIAS_ROW}


def unshard_named(name: str, locals_: list, d1: int, d2: int) -> np.ndarray:
    if name in BIAS_SPECS:
        spec2 = tuple(S1 if pl == S0 else pl for pl in BIAS_SPECS[name])
        return _sh.unshard([l[None, :] for l in locals_], spec2, d1, d2)[0]
    return _sh.unshard(locals_, SPECS[name], d1, d2)


def run_layer(g: dict, d1: int, d2: int, heads: int, chunks: int = 1):
    """Convenience: shard, forward, backward; returns (shards, fwd, bwd, log)."""
    g = {k: np.asarray(v, dtype=np.float64) for k, v in g.items()}
    sh = shard_layer(g, d1, d2)
    log = CommLog()
    fw = spmd_forward(sh, d1, d2, heads, chunks, log)
    bw = spmd_backward(sh, fw, sh["dz"], d1, d2, heads, chunks, log)
    return sh, fw, bw, log


# ---------------------------------------------------------------- single rows
def dense_forward_rows(g_rows_x, g: dict, heads: int) -> dict:
    """Dense forward of a subset of token rows (the layer is row-local: no
    cross-token op on the hot path, G13/G20) — for sampled full-size checks."""
    gg = dict(g)
    gg["x"] = g_rows_x
    return dense_forward(gg, heads)
