"""Pins of oracle/gpt.py (full GPT layer) against things
other than itself: closed forms, invariants, central finite differences,
independent library routines (torch CPU float64: scaled_dot_product_attention,
layer_norm, autograd through a torch re-statement of the layer), and
sharded == dense on every mesh of N in {1, 2, 4, 8}."""
import math

import numpy as np
import pytest
import torch

import datagen
from oracle import gpt
from oracle.layer import CommLog

RNG = np.random.default_rng(2301)


def _t(a):
    return torch.tensor(a, dtype=torch.float64, requires_grad=True)


# ---------------------------------------------------------------- attention core
@pytest.mark.parametrize("causal", [True, False])
def test_attention_fwd_matches_torch_sdpa(causal):
    """Eq. 1 vs torch's scaled_dot_product_attention (float64, CPU)."""
    s, d = 37, 16
    q, k, v = (RNG.standard_normal((s, d)) for _ in range(3))
    o, lse = gpt.attention_fwd(q, k, v, causal)
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.tensor(q)[None, None], torch.tensor(k)[None, None], torch.tensor(v)[None, None], is_causal=causal)
    np.testing.assert_allclose(o, ref[0, 0].numpy(), rtol=0, atol=1e-12)
    sc = (torch.tensor(q) @ torch.tensor(k).T) / math.sqrt(d)
    if causal:
        sc = sc.masked_fill(~torch.ones(s, s, dtype=torch.bool).tril(), float("-inf"))
    np.testing.assert_allclose(lse, torch.logsumexp(sc, dim=1).numpy(), rtol=0, atol=1e-12)


def test_attention_closed_forms():
    """q = 0: every visible key has weight 1/(t+1) -> O_t = mean(v[0..t]),
    lse_t = log(t+1) (causal); a sequence of one token returns v itself."""
    s, d = 9, 4
    q = np.zeros((s, d))
    k, v = RNG.standard_normal((s, d)), RNG.standard_normal((s, d))
    o, lse = gpt.attention_fwd(q, k, v, causal=True)
    for t in range(s):
        np.testing.assert_allclose(o[t], v[:t + 1].mean(axis=0), atol=1e-14)
        assert abs(lse[t] - math.log(t + 1)) < 1e-14
    o1, _ = gpt.attention_fwd(RNG.standard_normal((1, d)), RNG.standard_normal((1, d)), v[:1], causal=True)
    np.testing.assert_allclose(o1, v[:1], atol=1e-15)
    # row 0 of a causal sequence sees only key 0
    o, _ = gpt.attention_fwd(RNG.standard_normal((s, d)), k, v, causal=True)
    np.testing.assert_allclose(o[0], v[0], atol=1e-14)


@pytest.mark.parametrize("causal", [True, False])
def test_attention_bwd_matches_autograd_and_fd(causal):
    s, d = 11, 8
    q, k, v, do = (RNG.standard_normal((s, d)) for _ in range(4))
    dq, dk, dv = gpt.attention_bwd(do, q, k, v, causal)
    tq, tk, tv = _t(q), _t(k), _t(v)
    o = torch.nn.functional.scaled_dot_product_attention(tq[None, None], tk[None, None], tv[None, None],
                                                         is_causal=causal)[0, 0]
    (o * torch.tensor(do)).sum().backward()
    for mine, ref in ((dq, tq.grad), (dk, tk.grad), (dv, tv.grad)):
        np.testing.assert_allclose(mine, ref.numpy(), rtol=0, atol=1e-12)
    # central finite differences of <dO, O> at a few coordinates
    eps = 1e-6
    for arr, grad in ((q, dq), (k, dk), (v, dv)):
        for _ in range(4):
            i, j = RNG.integers(s), RNG.integers(d)
            old = arr[i, j]
            arr[i, j] = old + eps
            fp = (gpt.attention_fwd(q, k, v, causal)[0] * do).sum()
            arr[i, j] = old - eps
            fm = (gpt.attention_fwd(q, k, v, causal)[0] * do).sum()
            arr[i, j] = old
            assert abs((fp - fm) / (2 * eps) - grad[i, j]) < 1e-6


def test_core_head_interleaving_and_sequences():
    """core_softmax_fwd applies Eq. 1 per head (G19 column order) and per
    sequence (rows of different sequences never attend to each other)."""
    seq, heads, d = 5, 3, 4
    T = 2 * seq
    qkv = RNG.standard_normal((T, 3 * heads * d))
    ctx, lse = gpt.core_softmax_fwd(qkv, heads, seq)
    for n in range(2):
        r = slice(n * seq, (n + 1) * seq)
        for j in range(heads):
            b = 3 * j * d
            q, k, v = (torch.tensor(qkv[r, b + i * d:b + (i + 1) * d])[None, None] for i in range(3))
            ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)[0, 0].numpy()
            np.testing.assert_allclose(ctx[r, j * d:(j + 1) * d], ref, atol=1e-12)
    # the second sequence is unaffected by the first
    qkv2 = qkv.copy()
    qkv2[:seq] = RNG.standard_normal((seq, 3 * heads * d))
    np.testing.assert_array_equal(gpt.core_softmax_fwd(qkv2, heads, seq)[0][seq:], ctx[seq:])


# ---------------------------------------------------------------- LayerNorm
def test_layernorm_matches_torch_and_invariants():
    T, h = 7, 24
    x = RNG.standard_normal((T, h)) * 3 + 1.5
    gam, bet = 1 + 0.1 * RNG.standard_normal(h), 0.1 * RNG.standard_normal(h)
    y, mu, rs = gpt.layernorm_fwd(x, gam, bet)
    tx, tg, tb = _t(x), _t(gam), _t(bet)
    ty = torch.nn.functional.layer_norm(tx, (h,), tg, tb, eps=gpt.LN_EPS)
    np.testing.assert_allclose(y, ty.detach().numpy(), atol=1e-12)
    dy = RNG.standard_normal((T, h))
    (ty * torch.tensor(dy)).sum().backward()
    dx, dg, db = gpt.layernorm_bwd(dy, x, gam, mu, rs)
    for mine, ref in ((dx, tx.grad), (dg, tg.grad), (db, tb.grad)):
        np.testing.assert_allclose(mine, ref.numpy(), atol=1e-11)
    # identity affine: rows have mean 0 and (biased) variance var/(var+eps)
    y0, _, _ = gpt.layernorm_fwd(x, np.ones(h), np.zeros(h))
    np.testing.assert_allclose(y0.mean(axis=1), 0, atol=1e-13)
    var = x.var(axis=1)
    np.testing.assert_allclose(y0.var(axis=1), var / (var + gpt.LN_EPS), atol=1e-13)
    # gamma = 1: the gradient has no component along the constant direction, and
    # along xhat only the eps leak: sum(dx*xhat) = rstd * sum(dy*xhat) * eps/(var+eps)
    dx0, _, _ = gpt.layernorm_bwd(dy, x, np.ones(h), mu, rs)
    np.testing.assert_allclose(dx0.sum(axis=1), 0, atol=1e-12)
    xhat = (x - mu[:, None]) * rs[:, None]
    np.testing.assert_allclose((dx0 * xhat).sum(axis=1),
                               rs * (dy * xhat).sum(axis=1) * gpt.LN_EPS / (var + gpt.LN_EPS), atol=1e-13)


# ---------------------------------------------------------------- dense layer vs torch autograd
def _torch_layer(g, heads, seq, causal=True):
    """The layer re-stated in torch ops (layer_norm, SDPA, erf GeLU); autograd
    gives an independent backward."""
    tg = {k: _t(v) for k, v in g.items() if k != "dz"}
    x = tg["x"]
    T, h = x.shape
    d = h // heads
    a = torch.nn.functional.layer_norm(x, (h,), tg["g1"], tg["be1"], eps=gpt.LN_EPS)
    qkv = (a @ tg["wqkv"] + tg["bqkv"]).view(T // seq, seq, heads, 3, d)
    q, k, v = (qkv[:, :, :, i].permute(0, 2, 1, 3) for i in range(3))
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=causal)
    ctx = o.permute(0, 2, 1, 3).reshape(T, h)
    y1 = x + ctx @ tg["wo"] + tg["bo"]
    bn = torch.nn.functional.layer_norm(y1, (h,), tg["g2"], tg["be2"], eps=gpt.LN_EPS)
    z = y1 + torch.nn.functional.gelu(bn @ tg["w1"] + tg["b1"]) @ tg["w2"] + tg["b2"]
    (z * torch.tensor(g["dz"])).sum().backward()
    return z.detach().numpy(), {k: v.grad.numpy() for k, v in tg.items()}


def _globals(T, h, F, seed=5, scale_up=True):
    g = {k: v.astype(np.float64) for k, v in datagen.gpt_globals(T, h, F, seed, bf16=False).items()}
    if scale_up:  # larger weights so that attention is far from uniform
        for w in ("wqkv",):
            g[w] = g[w] * 20.0
    return g


@pytest.mark.parametrize("causal", [True, False])
def test_dense_layer_matches_torch_autograd(causal):
    T, h, F, heads, seq = 24, 32, 64, 4, 8
    g = _globals(T, h, F)
    fw = gpt.dense_forward(g, heads, seq, causal)
    bw = gpt.dense_backward(g, fw, g["dz"], heads, seq, causal)
    z, grads = _torch_layer(g, heads, seq, causal)
    np.testing.assert_allclose(fw["z"], z, atol=1e-12)
    names = {"x": "dx", "wqkv": "dwqkv", "bqkv": "dbqkv", "wo": "dwo", "bo": "dbo", "w1": "dw1", "b1": "db1",
             "w2": "dw2", "b2": "db2", "g1": "dg1", "be1": "dbe1", "g2": "dg2", "be2": "dbe2"}
    for tn, on in names.items():
        np.testing.assert_allclose(bw[on], grads[tn], atol=1e-10, err_msg=on)


def test_dense_layer_finite_differences():
    T, h, F, heads, seq = 16, 16, 32, 2, 8
    g = _globals(T, h, F, seed=9)
    fw = gpt.dense_forward(g, heads, seq)
    bw = gpt.dense_backward(g, fw, g["dz"], heads, seq)
    f = lambda: float((gpt.dense_forward(g, heads, seq)["z"] * g["dz"]).sum())
    eps = 1e-5
    for name, gname in (("x", "dx"), ("wqkv", "dwqkv"), ("g1", "dg1"), ("be2", "dbe2"), ("w1", "dw1")):
        a = g[name]
        for _ in range(4):
            idx = tuple(RNG.integers(n) for n in a.shape)
            old = a[idx]
            a[idx] = old + eps
            fp = f()
            a[idx] = old - eps
            fm = f()
            a[idx] = old
            assert abs((fp - fm) / (2 * eps) - bw[gname][idx]) < 1e-5 * max(1.0, abs(bw[gname][idx]))


# ---------------------------------------------------------------- sharded == dense
MESHES = [(1, 1), (2, 1), (1, 2), (4, 1), (2, 2), (1, 4), (8, 1), (4, 2), (2, 4), (1, 8)]


@pytest.mark.parametrize("d1,d2", MESHES)
@pytest.mark.parametrize("chunks", [1, 2])
def test_sharded_equals_dense(d1, d2, chunks):
    T, h, F, heads, seq = 32, 64, 128, 8, 8
    g = _globals(T, h, F, seed=11)
    dfw = gpt.dense_forward(g, heads, seq)
    dbw = gpt.dense_backward(g, dfw, g["dz"], heads, seq)
    sh, fw, bw, log = gpt.run_gpt(g, d1, d2, heads, seq, chunks)
    for name in ("z", "y1", "ctx", "u", "h", "a", "bn"):
        np.testing.assert_allclose(gpt.unshard_named(name, fw[name], d1, d2), dfw[name], atol=1e-12, err_msg=name)
    np.testing.assert_allclose(gpt.unshard_named("qkv", fw["qkv"], d1, d2), dfw["qkv"], atol=1e-12)
    np.testing.assert_allclose(gpt.unshard_named("ctx_loc", fw["ctx_loc"], d1, d2), dfw["ctx"], atol=1e-12)
    for name in ("dx", "dy1", "du", "dqkv", "dwqkv", "dwo", "dw1", "dw2", "dbqkv", "dbo", "db1", "db2",
                 "dg1", "dbe1", "dg2", "dbe2"):
        np.testing.assert_allclose(gpt.unshard_named(name, bw[name], d1, d2), dbw[name], atol=1e-11, err_msg=name)
    np.testing.assert_allclose(gpt.unshard_named("dqkv_loc", bw["dqkv_loc"], d1, d2), dbw["dqkv"], atol=1e-11)


def test_comm_log_closed_forms():
    """Executed collectives of the full layer (G4): on dim 2 the attention moves
    fwd RS(3h/d1) + AG(h/d1) and bwd RS(h/d1) + AG(3h/d1) = 8 T h/d1 elements;
    LN statistics are [rows, 2] all-reduces on dim 2, one forward and one
    backward per LayerNorm per chunk; a size-1 dimension issues nothing (G7)."""
    T, h, F, heads, seq = 32, 64, 128, 8, 8
    g = _globals(T, h, F, seed=3)
    for d1, d2, c in ((4, 2, 2), (2, 4, 1), (8, 1, 2), (1, 1, 1)):
        _, _, _, log = gpt.run_gpt(g, d1, d2, heads, seq, c)
        att = sum(e for ph, nm, dim, p, e in log.calls if nm.endswith((":rs", ":ag")))
        stats = [(ph, nm, e) for ph, nm, dim, p, e in log.calls if nm.endswith(":stats")]
        if d2 > 1:
            assert att == 8 * T * h // d1
            assert all(dim == 2 for ph, nm, dim, p, e in log.calls if nm.endswith((":rs", ":ag", ":stats")))
            assert len(stats) == 4 * c and sum(e for *_, e in stats) == 4 * 2 * T
        else:
            assert att == 0 and not stats
        fc = sum(e for ph, nm, dim, p, e in log.calls if nm in ("fc1", "fc2", "out") or nm == "qkv")
        exp = 0
        if d2 > 1:
            exp += 2 * T * F // d1            # fc1 fwd + fc2-dX bwd on dim 2
        if d1 > 1:
            exp += 2 * T * h // d2 * 2        # out/fc2 fwd + fc1-dX/qkv-dX bwd on dim 1
        assert fc == exp


def test_sharded_rejects_bad_shapes():
    g = _globals(16, 32, 64, seed=1)
    with pytest.raises(ValueError):
        gpt.run_gpt(g, 2, 2, 2, 8, 1)      # 2 heads over 4 ranks
    with pytest.raises(ValueError):
        gpt.run_gpt(g, 1, 1, 4, 8, 4)      # chunks of half sequences
