"""Pins for oracle.layer: the dense block, the sharded SPMD simulation, chunking.

Pins: closed-form GeLU values; a hand-worked forward
(golden); special cases (zero weights -> residual identity); finite
differences for the analytic backward; sharded == dense;
column-first == row-first; chunked == unchunked; (N,1) == textbook
Megatron; collective counts.
"""
import json
import os

import numpy as np
import pytest

import datagen
from oracle import costmodel, layer, mesh, sharding
from oracle.sharding import R, S0, S1

from conftest import GOLDEN


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


# ------------------------------------------------------------------ GeLU
def test_gelu_closed_form_values():
    # S:49-50 / textbook: GeLU(0) = 0, GeLU(1) = Phi(1) = 0.8413447461, GeLU(-10) ~ 0
    assert layer.gelu(np.array(0.0)) == 0.0
    assert abs(layer.gelu(np.array(1.0)) - 0.8413447460685429) < 1e-15
    assert abs(layer.gelu(np.array(-10.0))) < 1e-8
    assert abs(layer.gelu(np.array(2.0)) - 2 * 0.9772498680518208) < 1e-15
    # large positive -> identity
    assert abs(layer.gelu(np.array(10.0)) - 10.0) < 1e-12


def test_gelu_grad_matches_finite_difference():
    x = np.linspace(-6, 6, 241)
    eps = 1e-6
    fd = (layer.gelu(x + eps) - layer.gelu(x - eps)) / (2 * eps)
    assert np.max(np.abs(fd - layer.gelu_grad(x))) < 1e-8
    assert abs(layer.gelu_grad(np.array(0.0)) - 0.5) < 1e-15


# ------------------------------------------------------------------ dense layer
def test_hand_worked_forward():
    g = json.load(open(os.path.join(GOLDEN, "tiny_layer_hand.json")))
    t = {k: np.array(g[k], dtype=np.float64) for k in ("x", "wqkv", "bqkv", "wo", "bo", "w1", "b1", "w2", "b2")}
    out = layer.dense_forward(t, g["heads"])
    for k, v in g["expect"].items():
        np.testing.assert_allclose(out[k], np.array(v), rtol=0, atol=1e-15, err_msg=k)


def test_core_head_interleaved_layout():
    # G19/G20: column = head*3d + s*d + j; ctx[:, head*d + j] = sum_s qkv[:, head*3d + s*d + j]
    T, heads, d = 3, 2, 4
    qkv = np.arange(T * 3 * heads * d, dtype=np.float64).reshape(T, 3 * heads * d)
    ctx = layer.core_fwd(qkv, heads)
    for t in range(T):
        for hd in range(heads):
            for j in range(d):
                want = sum(qkv[t, hd * 3 * d + s * d + j] for s in range(3))
                assert ctx[t, hd * d + j] == want
    # core_bwd is the adjoint of core_fwd: <core(q), c> == <q, core^T(c)>
    c = np.random.default_rng(1).standard_normal(ctx.shape)
    assert abs(np.sum(ctx * c) - np.sum(qkv * layer.core_bwd(c, heads))) < 1e-9


def _globals(T, h, F, seed=7):
    return {k: v.astype(np.float64) for k, v in datagen.layer_globals(T, h, F, seed=seed).items()}


def test_zero_weights_reduce_to_residual_identity():
    T, h, F, a = 8, 16, 64, 2
    g = _globals(T, h, F)
    for w in ("wqkv", "wo", "w1", "w2"):
        g[w] = np.zeros_like(g[w])
    c = layer.dense_forward(g, a)
    # Y1 = X + bo, U = b1, Z = Y1 + GeLU(b1)*0 + b2
    np.testing.assert_allclose(c["y1"], g["x"] + g["bo"], atol=0)
    np.testing.assert_allclose(c["z"], g["x"] + g["bo"] + g["b2"], atol=0)


def test_backward_matches_finite_differences():
    T, h, F, a = 4, 8, 32, 2
    g = _globals(T, h, F, seed=11)
    g["wqkv"] *= 20; g["wo"] *= 20; g["w1"] *= 20; g["w2"] *= 20  # make every path O(1)
    dz = g["dz"]
    c = layer.dense_forward(g, a)
    grads = layer.dense_backward(g, c, dz, a)
    loss = lambda gg: float(np.sum(layer.dense_forward(gg, a)["z"] * dz))
    rng = np.random.default_rng(3)
    names = [("x", "dx"), ("wqkv", "dwqkv"), ("bqkv", "dbqkv"), ("wo", "dwo"), ("bo", "dbo"),
             ("w1", "dw1"), ("b1", "db1"), ("w2", "dw2"), ("b2", "db2")]
    n_checked = 0
    for p, dp in names:
        for _ in range(3):
            idx = tuple(int(rng.integers(s)) for s in g[p].shape)
            eps = 1e-5
            gp = {k: v.copy() for k, v in g.items()}
            gp[p][idx] += eps
            gm = {k: v.copy() for k, v in g.items()}
            gm[p][idx] -= eps
            fd = (loss(gp) - loss(gm)) / (2 * eps)
            an = grads[dp][idx]
            assert abs(fd - an) <= 1e-4 * max(1.0, abs(an)), (p, idx, fd, an)
            n_checked += 1
    assert n_checked >= 20


# ------------------------------------------------------------------ SPMD == dense
ALL_MESHES = [m for n in (1, 2, 4, 8) for m in mesh.enumerate_meshes(n)]


def _check_layer(T, h, F, heads, d1, d2, chunks, tol=1e-12, seed=5):
    g = _globals(T, h, F, seed=seed)
    dense = layer.dense_forward(g, heads)
    dgr = layer.dense_backward(g, dense, g["dz"], heads)
    sh, fw, bw, log = layer.run_layer(g, d1, d2, heads, chunks)
    for k in ("qkv", "ctx", "y1", "u", "h", "z"):
        assert rel(layer.unshard_named(k, fw[k], d1, d2), dense[k]) <= tol, k
    for k in ("dx", "dy1", "du", "dh", "dctx", "dqkv", "dwqkv", "dwo", "dw1", "dw2",
              "dbqkv", "dbo", "db1", "db2"):
        assert rel(layer.unshard_named(k, bw[k], d1, d2), dgr[k]) <= tol, k
    return log


def test_cfg1_mlp_2x2_matches_dense():
    # BASELINE.json configs[0]: h=64, ffn=256, tokens=32 on a 2x2 virtual mesh
    _check_layer(32, 64, 256, 4, 2, 2, 1)


@pytest.mark.parametrize("d1,d2", ALL_MESHES)
@pytest.mark.parametrize("chunks", [1, 2, 4])
def test_every_mesh_matches_dense(d1, d2, chunks):
    # SPEC acceptance 5 shape (h=64, b=2, s=8); heads=8 so that heads % d1 == 0 at d1=8
    log = _check_layer(16, 64, 256, 8, d1, d2, chunks)
    # the simulation's executed collectives are exactly the closed-form list
    assert log.calls == costmodel.comm_volume(d1, d2, 16, 64, chunks)


def test_unit_mesh_makes_no_collective():
    # mesh (1,1) invokes zero collectives
    assert _check_layer(16, 64, 256, 8, 1, 1, 2).calls == []


@pytest.mark.parametrize("d1,d2", [(2, 2), (4, 2), (2, 4)])
def test_chunked_equals_unchunked(d1, d2):
    g = _globals(32, 64, 256, seed=9)
    _, f1, b1, _ = layer.run_layer(g, d1, d2, 8, 1)
    _, f4, b4, _ = layer.run_layer(g, d1, d2, 8, 4)
    for k in ("z", "y1"):
        for r in range(d1 * d2):
            assert np.max(np.abs(f1[k][r] - f4[k][r])) <= 1e-12
    for k in ("dx", "dw1", "dw2", "dwo", "dwqkv"):
        for r in range(d1 * d2):
            assert rel(b4[k][r], b1[k][r]) <= 1e-12


@pytest.mark.parametrize("d1,d2", ALL_MESHES)
def test_colfirst_equals_rowfirst_single_linear(d1, d2):
    rng = np.random.default_rng(d1 * 10 + d2)
    b, h1, h2 = 16, 32, 48
    x = rng.standard_normal((b, h1))
    w = rng.standard_normal((h1, h2))
    dense = x @ w
    yc = layer.colfirst_forward(sharding.shard(x, layer.ACT, d1, d2),
                                sharding.shard(w, layer.COL_W, d1, d2), d1, d2)
    yr = layer.rowfirst_forward(sharding.shard(x, (S1, R), d1, d2),
                                sharding.shard(w, layer.ROW_W, d1, d2), d1, d2)
    gc = sharding.unshard(yc, layer.COL_OUT, d1, d2)
    gr = sharding.unshard(yr, layer.ACT, d1, d2)
    assert rel(gc, dense) <= 1e-13 and rel(gr, dense) <= 1e-13 and rel(gc, gr) <= 1e-13


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_mesh_n1_is_textbook_megatron(n):
    """P:89-95 / P:254: DeviceMesh(N,1) is Megatron 1-D TP: A split by columns,
    B by rows, Z = reduce(GeLU(X A_i) B_i); two all-reduces in each of forward
    and backward per layer, each of the full [b,s,h] activation."""
    T, h, F, heads = 16, 64, 256, 8
    g = _globals(T, h, F, seed=13)
    sh, fw, bw, log = layer.run_layer(g, n, 1, heads, 1)
    y1 = layer.unshard_named("y1", fw["y1"], n, 1)
    A = np.split(g["w1"], n, axis=1)
    Bm = np.split(g["w2"], n, axis=0)
    ba = np.split(g["b1"], n)
    z_meg = y1 + sum(layer.gelu(y1 @ A[i] + ba[i]) @ Bm[i] for i in range(n)) + g["b2"]
    assert rel(layer.unshard_named("z", fw["z"], n, 1), z_meg) <= 1e-12
    if n > 1:
        assert [(c[0], c[2], c[4]) for c in log.calls] == [
            ("fwd", 1, T * h), ("fwd", 1, T * h), ("bwd", 1, T * h), ("bwd", 1, T * h)]
    else:
        assert log.calls == []


def test_per_rank_index_map_matches_specs():
    """SURVEY §8(c) index map: X cols blk(h,d2,i2); Wqkv [blk(h,d2,i2), blk(3h,d1,i1)];
    Wo [blk(h,d1,i1), blk(h,d2,i2)] — derived from P:218/P:234 placements."""
    T, h, F = 8, 24, 96
    g = _globals(T, h, F)
    for d1, d2 in [(2, 2), (4, 2), (2, 4), (3, 1), (1, 3)]:
        sh = layer.shard_layer(g, d1, d2)
        for r in range(d1 * d2):
            i1, i2 = mesh.coords(d1, d2, r)
            blk = lambda n, parts, i: slice(i * n // parts, (i + 1) * n // parts)
            np.testing.assert_array_equal(sh["x"][r], g["x"][:, blk(h, d2, i2)])
            np.testing.assert_array_equal(sh["wqkv"][r], g["wqkv"][blk(h, d2, i2), blk(3 * h, d1, i1)])
            np.testing.assert_array_equal(sh["wo"][r], g["wo"][blk(h, d1, i1), blk(h, d2, i2)])
            np.testing.assert_array_equal(sh["w1"][r], g["w1"][blk(h, d2, i2), blk(F, d1, i1)])
            np.testing.assert_array_equal(sh["w2"][r], g["w2"][blk(F, d1, i1), blk(h, d2, i2)])
            np.testing.assert_array_equal(sh["b1"][r], g["b1"][blk(F, d1, i1)])
            np.testing.assert_array_equal(sh["bo"][r], g["bo"][blk(h, d2, i2)])
