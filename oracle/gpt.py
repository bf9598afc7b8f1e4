"""Full GPT layer: dense definition and sharded SPMD simulation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): imported by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / reference legs, never by
the product path.

Everything is float64 NumPy.  P:n = PAPER.md line; G-numbers = readings in
DESIGN.md §2 (G1-G28 from SURVEY §8(c); G29-G35 added for the full layer).

Dense definition, one pre-LN GPT layer on T = b*s token rows (batch-major):
    A   = LN1(X)                              (G29: pre-LN; LN affine, eps 1e-5)
    QKV = A Wqkv + bqkv                       (head-interleaved columns, G19)
    ctx = Attn(QKV) per sequence and head:    softmax(Q K^T / sqrt(d)) V   (Eq. 1)
                                              with a causal mask (G30)
    Y1  = X + ctx Wo + bo
    B   = LN2(Y1)
    U   = B W1 + b1,  H = GeLU(U)
    Z   = Y1 + H W2 + b2
and its analytic backward for a given dZ.

Sharded simulation (Fig. 6(a)): as the linear block (oracle/layer.py),
except that the attention core is fully sharded: the QKV partial sums are
REDUCE-SCATTERED over mesh dim 2 (member i2 receives head block i2 of its d1
block: a/(d1*d2) heads), the core runs on the local heads, and ctx is
ALL-GATHERED over dim 2 before the Out linear (G32).  Backward mirrors it: the
dctx partials are reduce-scattered on dim 2, dQKV is all-gathered on dim 2.
LayerNorm with the hidden dimension sharded over d2 all-reduces the per-row
partial sums (sum x, sum x^2) forward and (sum g, sum g*xhat) backward over
dim 2 (G33).  Chunks are whole sequences (G34).
"""
from __future__ import annotations

import numpy as np

from . import mesh as _mesh
from .layer import (ACT, BIAS_COL, BIAS_ROW, COL_W, ROW_W, CommLog, _bias_shards, all_reduce, gelu, gelu_grad)
from . import sharding as _sh

LN_EPS = 1e-5


# ---------------------------------------------------------------- LayerNorm
def layernorm_fwd(x, gamma, beta, eps=LN_EPS):
    """y = (x - mean) / sqrt(var + eps) * gamma + beta over the last axis
    (biased variance).  Returns (y, mean, rstd)."""
    mean = x.mean(axis=1)
    var = ((x - mean[:, None]) ** 2).mean(axis=1)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = (x - mean[:, None]) * rstd[:, None]
    return xhat * gamma + beta, mean, rstd


def layernorm_bwd(dy, x, gamma, mean, rstd):
    """Analytic LayerNorm backward: with g = dy*gamma and n = row width,
    dx = rstd * (g - mean(g) - xhat * mean(g*xhat)); dgamma = sum_rows dy*xhat;
    dbeta = sum_rows dy."""
    xhat = (x - mean[:, None]) * rstd[:, None]
    g = dy * gamma
    dx = rstd[:, None] * (g - g.mean(axis=1, keepdims=True) - xhat * (g * xhat).mean(axis=1, keepdims=True))
    return dx, (dy * xhat).sum(axis=0), dy.sum(axis=0)


# ---------------------------------------------------------------- attention core
def attention_fwd(q, k, v, causal=True):
    """One head of one sequence, Eq. 1: O = softmax(q k^T / sqrt(d)) v.
    Returns (O, lse) with lse = log sum_j exp(s_ij) of the scaled, masked scores."""
    s_len, d = q.shape
    s = (q @ k.T) / np.sqrt(d)
    if causal:
        s = np.where(np.tril(np.ones((s_len, s_len), dtype=bool)), s, -np.inf)
    m = s.max(axis=1, keepdims=True)
    p = np.exp(s - m)
    l = p.sum(axis=1, keepdims=True)
    return (p / l) @ v, (m + np.log(l))[:, 0]


def attention_bwd(do, q, k, v, causal=True):
    """Backward of attention_fwd: with P = softmax(S), S = q k^T / sqrt(d):
    dV = P^T dO; dP = dO V^T; dS = P * (dP - rowsum(dP * P)); dQ = dS K / sqrt(d);
    dK = dS^T Q / sqrt(d)."""
    s_len, d = q.shape
    s = (q @ k.T) / np.sqrt(d)
    if causal:
        s = np.where(np.tril(np.ones((s_len, s_len), dtype=bool)), s, -np.inf)
    p = np.exp(s - s.max(axis=1, keepdims=True))
    p /= p.sum(axis=1, keepdims=True)
    dv = p.T @ do
    dp = do @ v.T
    ds = p * (dp - (dp * p).sum(axis=1, keepdims=True))
    return ds @ k / np.sqrt(d), ds.T @ q / np.sqrt(d), dv


def _head_cols(j, d):
    """Columns of head j's q, k, v in a head-interleaved QKV block (G19)."""
    b = 3 * j * d
    return slice(b, b + d), slice(b + d, b + 2 * d), slice(b + 2 * d, b + 3 * d)


def core_softmax_fwd(qkv, heads: int, seq: int, causal=True):
    """Attention core over every sequence (rows [n*seq, (n+1)*seq)) and head of a
    head-interleaved QKV block [T, 3*heads*d].  Returns (ctx [T, heads*d], lse [heads, T])."""
    T, w = qkv.shape
    d = w // (3 * heads)
    ctx = np.zeros((T, heads * d))
    lse = np.zeros((heads, T))
    for n in range(T // seq):
        rows = slice(n * seq, (n + 1) * seq)
        for j in range(heads):
            cq, ck, cv = _head_cols(j, d)
            o, ls = attention_fwd(qkv[rows, cq], qkv[rows, ck], qkv[rows, cv], causal)
            ctx[rows, j * d:(j + 1) * d] = o
            lse[j, rows] = ls
    return ctx, lse


def core_softmax_bwd(dctx, qkv, heads: int, seq: int, causal=True):
    """dQKV [T, 3*heads*d] (head-interleaved) for the upstream gradient dctx."""
    T, w = qkv.shape
    d = w // (3 * heads)
    dqkv = np.zeros_like(qkv)
    for n in range(T // seq):
        rows = slice(n * seq, (n + 1) * seq)
        for j in range(heads):
            cq, ck, cv = _head_cols(j, d)
            dq, dk, dv = attention_bwd(dctx[rows, j * d:(j + 1) * d], qkv[rows, cq], qkv[rows, ck],
                                       qkv[rows, cv], causal)
            dqkv[rows, cq], dqkv[rows, ck], dqkv[rows, cv] = dq, dk, dv
    return dqkv


# ---------------------------------------------------------------- dense layer
def dense_forward(g: dict, heads: int, seq: int, causal=True) -> dict:
    x = g["x"]
    a, mu1, rs1 = layernorm_fwd(x, g["g1"], g["be1"])
    qkv = a @ g["wqkv"] + g["bqkv"]
    ctx, lse = core_softmax_fwd(qkv, heads, seq, causal)
    y1 = x + (ctx @ g["wo"] + g["bo"])
    bn, mu2, rs2 = layernorm_fwd(y1, g["g2"], g["be2"])
    u = bn @ g["w1"] + g["b1"]
    hh = gelu(u)
    z = y1 + (hh @ g["w2"] + g["b2"])
    return {"a": a, "mu1": mu1, "rs1": rs1, "qkv": qkv, "ctx": ctx, "lse": lse, "y1": y1,
            "bn": bn, "mu2": mu2, "rs2": rs2, "u": u, "h": hh, "z": z}


def dense_backward(g: dict, c: dict, dz, heads: int, seq: int, causal=True) -> dict:
    dh = dz @ g["w2"].T
    dw2 = c["h"].T @ dz
    db2 = dz.sum(axis=0)
    du = dh * gelu_grad(c["u"])
    dw1 = c["bn"].T @ du
    db1 = du.sum(axis=0)
    dbn = du @ g["w1"].T
    dln2, dg2, dbe2 = layernorm_bwd(dbn, c["y1"], g["g2"], c["mu2"], c["rs2"])
    dy1 = dz + dln2
    dctx = dy1 @ g["wo"].T
    dwo = c["ctx"].T @ dy1
    dbo = dy1.sum(axis=0)
    dqkv = core_softmax_bwd(dctx, c["qkv"], heads, seq, causal)
    dwqkv = c["a"].T @ dqkv
    dbqkv = dqkv.sum(axis=0)
    da = dqkv @ g["wqkv"].T
    dln1, dg1, dbe1 = layernorm_bwd(da, g["x"], g["g1"], c["mu1"], c["rs1"])
    dx = dy1 + dln1
    return {"dx": dx, "dy1": dy1, "dbn": dbn, "du": du, "dh": dh, "dctx": dctx, "dqkv": dqkv, "da": da,
            "dwqkv": dwqkv, "dbqkv": dbqkv, "dwo": dwo, "dbo": dbo, "dw1": dw1, "db1": db1,
            "dw2": dw2, "db2": db2, "dg1": dg1, "dbe1": dbe1, "dg2": dg2, "dbe2": dbe2}


# ---------------------------------------------------------------- collectives
def reduce_scatter_cols(parts: list, d1: int, d2: int, dim: int, log: CommLog | None = None,
                        phase: str = "", name: str = ""):
    """Grouped reduce-scatter over mesh ``dim`` (Fig. 6(a) scatter): the
    members' partials are summed in ascending mesh coordinate and member j keeps
    column block j (of p equal blocks)."""
    p = d1 if dim == 1 else d2
    out = [None] * len(parts)
    for grp in _mesh.groups(d1, d2, dim):
        s = parts[grp[0]].copy()
        for r in grp[1:]:
            s = s + parts[r]
        wb = s.shape[1] // p
        for j, r in enumerate(grp):
            out[r] = s[:, j * wb:(j + 1) * wb].copy()
    if log is not None and p > 1:
        log.add(phase, name + ":rs", dim, p, parts[0].size)
    return out


def all_gather_cols(parts: list, d1: int, d2: int, dim: int, log: CommLog | None = None,
                    phase: str = "", name: str = ""):
    """Grouped all-gather over mesh ``dim`` (Fig. 6(a) gather): every
    member gets the column concatenation of the members' blocks in ascending
    mesh coordinate."""
    p = d1 if dim == 1 else d2
    out = [None] * len(parts)
    for grp in _mesh.groups(d1, d2, dim):
        cat = np.concatenate([parts[r] for r in grp], axis=1)
        for r in grp:
            out[r] = cat.copy()
    if log is not None and p > 1:
        log.add(phase, name + ":ag", dim, p, parts[0].size * p)
    return out


# ---------------------------------------------------------------- sharding
def head_block(a, d1: int, d2: int, r: int):
    """Columns of rank r's attention heads in a global [T, heads*w] tensor:
    block i1*d2 + i2 of d1*d2 equal column blocks (G32)."""
    n = d1 * d2
    wb = a.shape[-1] // n
    return a[..., r * wb:(r + 1) * wb] if a.ndim == 1 else a[:, r * wb:(r + 1) * wb]


def shard_gpt(g: dict, d1: int, d2: int) -> dict:
    """Per-rank shards.  The linear weights and biases as
    in oracle/layer.shard_layer; LayerNorm gamma/beta follow the hidden split
    (Shard(0) over dim 2, replicated over dim 1, like bo/b2); bqkv is split
    like the local heads (it is added once, after the reduce-scatter)."""
    sh = {"x": _sh.shard(g["x"], ACT, d1, d2),
          "wqkv": _sh.shard(g["wqkv"], COL_W, d1, d2), "wo": _sh.shard(g["wo"], ROW_W, d1, d2),
          "w1": _sh.shard(g["w1"], COL_W, d1, d2), "w2": _sh.shard(g["w2"], ROW_W, d1, d2)}
    sh["bqkv"] = [head_block(g["bqkv"], d1, d2, r) for r in range(d1 * d2)]
    for b in ("bo", "b2", "g1", "be1", "g2", "be2"):
        sh[b] = _bias_shards(g[b], BIAS_ROW, d1, d2)
    sh["b1"] = _bias_shards(g["b1"], BIAS_COL, d1, d2)
    if "dz" in g:
        sh["dz"] = _sh.shard(g["dz"], ACT, d1, d2)
    return sh


def _ln_sharded_fwd(x_loc, gam, bet, width, d1, d2, log, name):
    """LayerNorm of [T, width] rows whose columns are split over dim 2: the per-row
    partial sums (sum x, sum x^2) are all-reduced over dim 2 (G33)."""
    n = d1 * d2
    part = [np.stack([x_loc[r].sum(axis=1), (x_loc[r] ** 2).sum(axis=1)], axis=1) for r in range(n)]
    tot = all_reduce(part, d1, d2, 2, log, "fwd", name + ":stats")
    out, mean, rstd = [], [], []
    for r in range(n):
        mu = tot[r][:, 0] / width
        var = tot[r][:, 1] / width - mu * mu
        rs = 1.0 / np.sqrt(var + LN_EPS)
        out.append((x_loc[r] - mu[:, None]) * rs[:, None] * gam[r] + bet[r])
        mean.append(mu)
        rstd.append(rs)
    return out, mean, rstd


def _ln_sharded_bwd(dy_loc, x_loc, gam, mean, rstd, width, d1, d2, log, name):
    n = d1 * d2
    xh = [(x_loc[r] - mean[r][:, None]) * rstd[r][:, None] for r in range(n)]
    gg = [dy_loc[r] * gam[r] for r in range(n)]
    part = [np.stack([gg[r].sum(axis=1), (gg[r] * xh[r]).sum(axis=1)], axis=1) for r in range(n)]
    tot = all_reduce(part, d1, d2, 2, log, "bwd", name + ":stats")
    dx = [rstd[r][:, None] * (gg[r] - tot[r][:, 0:1] / width - xh[r] * tot[r][:, 1:2] / width) for r in range(n)]
    dgam = [(dy_loc[r] * xh[r]).sum(axis=0) for r in range(n)]
    dbet = [dy_loc[r].sum(axis=0) for r in range(n)]
    return dx, dgam, dbet


def _rows(a, k, c):
    m = a.shape[0] // c
    return a[k * m:(k + 1) * m]


def spmd_forward(sh: dict, d1: int, d2: int, heads: int, seq: int, chunks: int = 1, causal=True,
                 log: CommLog | None = None) -> dict:
    """Sharded full-layer forward, chunk by chunk (chunks = whole sequences, G34)."""
    n = d1 * d2
    T, hloc = sh["x"][0].shape
    h = hloc * d2
    if T % (seq * chunks):
        raise ValueError("chunks must be whole sequences: T % (seq * chunks) != 0")
    if heads % (d1 * d2):
        raise ValueError("heads % (d1*d2) != 0 (Fig. 6(a) shards heads over both dims)")
    hl = heads // (d1 * d2)
    keys = ("a", "mu1", "rs1", "qkv", "ctx_loc", "lse", "ctx", "y1", "bn", "mu2", "rs2", "u", "h", "z")
    st = {k: [[None] * chunks for _ in range(n)] for k in keys}
    for k in range(chunks):
        xk = [_rows(sh["x"][r], k, chunks) for r in range(n)]
        a, mu, rs = _ln_sharded_fwd(xk, sh["g1"], sh["be1"], h, d1, d2, log, "ln1")
        part = [a[r] @ sh["wqkv"][r] for r in range(n)]
        qkv = reduce_scatter_cols(part, d1, d2, 2, log, "fwd", "qkv")
        ctx_loc = []
        for r in range(n):
            q = qkv[r] + sh["bqkv"][r]
            c, ls = core_softmax_fwd(q, hl, seq, causal)
            for key, v in (("a", a[r]), ("mu1", mu[r]), ("rs1", rs[r]), ("qkv", q), ("ctx_loc", c), ("lse", ls)):
                st[key][r][k] = v
            ctx_loc.append(c)
        ctx = all_gather_cols(ctx_loc, d1, d2, 2, log, "fwd", "ctx")
        red = all_reduce([ctx[r] @ sh["wo"][r] for r in range(n)], d1, d2, 1, log, "fwd", "out")
        y1 = [xk[r] + (red[r] + sh["bo"][r]) for r in range(n)]
        bn, mu, rs = _ln_sharded_fwd(y1, sh["g2"], sh["be2"], h, d1, d2, log, "ln2")
        red = all_reduce([bn[r] @ sh["w1"][r] for r in range(n)], d1, d2, 2, log, "fwd", "fc1")
        for r in range(n):
            st["ctx"][r][k], st["y1"][r][k], st["bn"][r][k] = ctx[r], y1[r], bn[r]
            st["mu2"][r][k], st["rs2"][r][k] = mu[r], rs[r]
            st["u"][r][k] = red[r] + sh["b1"][r]
            st["h"][r][k] = gelu(st["u"][r][k])
        red = all_reduce([st["h"][r][k] @ sh["w2"][r] for r in range(n)], d1, d2, 1, log, "fwd", "fc2")
        for r in range(n):
            st["z"][r][k] = y1[r] + (red[r] + sh["b2"][r])
    out = {}
    for key, v in st.items():
        ax = 1 if key == "lse" else 0
        out[key] = [np.concatenate(v[r], axis=ax) for r in range(n)]
    return out


def spmd_backward(sh: dict, fw: dict, dz_loc: list, d1: int, d2: int, heads: int, seq: int,
                  chunks: int = 1, causal=True, log: CommLog | None = None) -> dict:
    """Sharded full-layer backward (P:341-345 per linear; Fig. 6(a) conjugates
    for the core: reduce-scatter dctx on dim 2, all-gather dQKV on dim 2)."""
    n = d1 * d2
    T, hloc = sh["x"][0].shape
    h = hloc * d2
    hl = heads // (d1 * d2)
    names = ("dh", "du", "dbn", "dy1", "dctx_loc", "dqkv_loc", "dqkv", "da", "dx")
    gr = {k: [[None] * chunks for _ in range(n)] for k in names}
    acc = {k: [None] * n for k in ("dw2", "dw1", "dwo", "dwqkv", "dg1", "dbe1", "dg2", "dbe2")}
    Rk = lambda a, k: _rows(a, k, chunks)

    def accum(name, r, val):
        acc[name][r] = val if acc[name][r] is None else acc[name][r] + val

    for k in range(chunks):
        dz = [Rk(dz_loc[r], k) for r in range(n)]
        dh = all_reduce([dz[r] @ sh["w2"][r].T for r in range(n)], d1, d2, 2, log, "bwd", "fc2")
        du = [dh[r] * gelu_grad(Rk(fw["u"][r], k)) for r in range(n)]
        dbn = all_reduce([du[r] @ sh["w1"][r].T for r in range(n)], d1, d2, 1, log, "bwd", "fc1")
        y1 = [Rk(fw["y1"][r], k) for r in range(n)]
        dl2, dg2, dbe2 = _ln_sharded_bwd(dbn, y1, sh["g2"], [Rk(fw["mu2"][r], k) for r in range(n)],
                                         [Rk(fw["rs2"][r], k) for r in range(n)], h, d1, d2, log, "ln2")
        dy1 = [dz[r] + dl2[r] for r in range(n)]
        dctx = reduce_scatter_cols([dy1[r] @ sh["wo"][r].T for r in range(n)], d1, d2, 2, log, "bwd", "out")
        dql = [core_softmax_bwd(dctx[r], Rk(fw["qkv"][r], k), hl, seq, causal) for r in range(n)]
        dqkv = all_gather_cols(dql, d1, d2, 2, log, "bwd", "qkv")
        da = all_reduce([dqkv[r] @ sh["wqkv"][r].T for r in range(n)], d1, d2, 1, log, "bwd", "qkv")
        x = [Rk(sh["x"][r], k) for r in range(n)]
        dl1, dg1, dbe1 = _ln_sharded_bwd(da, x, sh["g1"], [Rk(fw["mu1"][r], k) for r in range(n)],
                                         [Rk(fw["rs1"][r], k) for r in range(n)], h, d1, d2, log, "ln1")
        for r in range(n):
            for key, v in (("dh", dh[r]), ("du", du[r]), ("dbn", dbn[r]), ("dy1", dy1[r]), ("dctx_loc", dctx[r]),
                           ("dqkv_loc", dql[r]), ("dqkv", dqkv[r]), ("da", da[r]), ("dx", dy1[r] + dl1[r])):
                gr[key][r][k] = v
            accum("dw2", r, Rk(fw["h"][r], k).T @ dz[r])
            accum("dw1", r, Rk(fw["bn"][r], k).T @ du[r])
            accum("dwo", r, Rk(fw["ctx"][r], k).T @ dy1[r])
            accum("dwqkv", r, Rk(fw["a"][r], k).T @ dqkv[r])
            for key, v in (("dg2", dg2[r]), ("dbe2", dbe2[r]), ("dg1", dg1[r]), ("dbe1", dbe1[r])):
                accum(key, r, v)
    out = {key: [np.concatenate(v[r], axis=0) for r in range(n)] for key, v in gr.items()}
    out.update(acc)
    out["db2"] = [dz_loc[r].sum(axis=0) for r in range(n)]
    out["db1"] = [out["du"][r].sum(axis=0) for r in range(n)]
    out["dbo"] = [out["dy1"][r].sum(axis=0) for r in range(n)]
    out["dbqkv"] = [out["dqkv_loc"][r].sum(axis=0) for r in range(n)]
    return out


# Placements of the full layer's per-rank tensors (for unsharding).
SPECS = {"x": ACT, "y1": ACT, "z": ACT, "dz": ACT, "dy1": ACT, "dx": ACT, "a": ACT, "bn": ACT,
         "dbn": ACT, "da": ACT, "ctx": (_sh.S1, _sh.R), "u": (_sh.S1, _sh.R), "h": (_sh.S1, _sh.R),
         "dh": (_sh.S1, _sh.R), "du": (_sh.S1, _sh.R), "dqkv": (_sh.S1, _sh.R),
         "wqkv": COL_W, "w1": COL_W, "dwqkv": COL_W, "dw1": COL_W,
         "wo": ROW_W, "w2": ROW_W, "dwo": ROW_W, "dw2": ROW_W}
HEAD_SHARDED = ("qkv", "ctx_loc", "dctx_loc", "dqkv_loc", "bqkv", "dbqkv")
ROW_VECTORS = ("bo", "b2", "dbo", "db2", "g1", "be1", "g2", "be2", "dg1", "dbe1", "dg2", "dbe2")


def unshard_named(name: str, locals_: list, d1: int, d2: int) -> np.ndarray:
    if name in HEAD_SHARDED:
        return np.concatenate(locals_, axis=-1)
    if name in ROW_VECTORS:
        return _sh.unshard([l[None, :] for l in locals_], (_sh.R, _sh.S1), d1, d2)[0]
    if name in ("b1", "db1"):
        return _sh.unshard([l[None, :] for l in locals_], (_sh.S1, _sh.R), d1, d2)[0]
    return _sh.unshard(locals_, SPECS[name], d1, d2)


def run_gpt(g: dict, d1: int, d2: int, heads: int, seq: int, chunks: int = 1, causal=True):
    """Shard, forward, backward; returns (shards, fwd, bwd, log)."""
    g = {k: np.asarray(v, dtype=np.float64) for k, v in g.items()}
    sh = shard_gpt(g, d1, d2)
    log = CommLog()
    fw = spmd_forward(sh, d1, d2, heads, seq, chunks, causal, log)
    bw = spmd_backward(sh, fw, sh["dz"], d1, d2, heads, seq, chunks, causal, log)
    return sh, fw, bw, log
