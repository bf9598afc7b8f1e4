"""Full-size parity of the full GPT layer in the launch
configurations bench.py --layer gpt times.

The layer is sequence-local (attention mixes tokens only within a sequence,
G34), so the outputs of one sampled sequence are exactly the oracle's dense
layer evaluated on that sequence alone (float32 BLAS; the oracle code is
dtype-agnostic).  Weight gradients sum over all sequences; for them a property
that holds at any size is checked: dW2 = H^T dZ  ==>  dW2 1 = H^T (dZ 1) with
the GPU's own saved H, and db2 = column sums of dZ.
"""
import numpy as np
import pytest

import datagen
from oracle import gpt

from gpu_util import rel, to_np

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _seq_globals(seq_idx, seq, h, F, seed, T):
    rows = np.arange(seq_idx * seq, (seq_idx + 1) * seq)
    g = {}
    for k, s in datagen.gpt_shapes(T, h, F).items():
        if k in ("x", "dz"):
            g[k] = datagen.tensor(k, s, seed=seed, rows=rows).astype(np.float32)
        else:
            g[k] = datagen.tensor(k, s, seed=seed).astype(np.float32)
    return g


def _check_sequence(bufs_slice, g, heads, seq):
    fw = gpt.dense_forward(g, heads, seq)
    bw = gpt.dense_backward(g, fw, g["dz"], heads, seq)
    for k, ref in (("a", fw["a"]), ("y1", fw["y1"]), ("bn", fw["bn"]), ("z", fw["z"]), ("dx", bw["dx"])):
        e = rel(bufs_slice(k), ref)
        assert e <= TOL, (k, e)
    return fw, bw


def test_fullsize_gpt_mesh11_sampled_sequences():
    import torch
    import paper_2301_08658_b200 as atp

    b, seq, h, heads, seed = 4, 2048, 4096, 32, 2301
    T, F = b * seq, 4 * h
    uid = atp.atp_get_unique_id()
    mesh = atp.Mesh.distributed(1, 1, 0, uid, 0)
    try:
        bufs = atp.alloc_gpt_rank(1, 1, 0, T, h, F, heads, "cuda", seed)
        atp.GptCall(mesh, [bufs], T, h, F, heads, seq, 1, True)()
        torch.cuda.synchronize()
    finally:
        mesh.destroy()
    for sidx in (0, b - 1):
        g = _seq_globals(sidx, seq, h, F, seed, T)
        fw, _ = _check_sequence(lambda k: to_np(bufs[k])[sidx * seq:(sidx + 1) * seq], g, heads, seq)
        got_ctx = to_np(bufs["ctx"])[sidx * seq:(sidx + 1) * seq]
        assert rel(got_ctx, fw["ctx"]) <= TOL
    # weight-gradient properties at full size
    H, dz = bufs["h"].double(), datagen.torch_block("dz", (T, h), 0, T, 0, h, "cuda", seed=seed).double()
    lhs = bufs["dw2"].double() @ torch.ones(h, dtype=torch.float64, device="cuda")
    rhs = H.t() @ (dz @ torch.ones(h, dtype=torch.float64, device="cuda"))
    assert rel(lhs.cpu().numpy(), rhs.cpu().numpy()) <= TOL
    assert rel(bufs["db2"].double().cpu().numpy(), dz.sum(0).cpu().numpy()) <= 1e-4


def test_fullsize_gpt_cfg4_mesh42_chunked():
    """cfg 4 (h=5120, 40 heads) per-rank shapes on a virtual DeviceMesh(4,2), chunks 2
    (bench --layer gpt's N>1 default): sequence 0's outputs on every rank."""
    import torch
    import paper_2301_08658_b200 as atp

    b, seq, h, heads, seed, d1, d2 = 4, 2048, 5120, 40, 7, 4, 2
    T, F = b * seq, 4 * h
    mesh = atp.Mesh.virtual(d1, d2)
    try:
        bufs = [atp.alloc_gpt_rank(d1, d2, r, T, h, F, heads, "cuda", seed) for r in range(d1 * d2)]
        atp.GptCall(mesh, bufs, T, h, F, heads, seq, 2, True)()
        torch.cuda.synchronize()
    finally:
        mesh.destroy()
    g = _seq_globals(0, seq, h, F, seed, T)
    fw = gpt.dense_forward(g, heads, seq)
    bw = gpt.dense_backward(g, fw, g["dz"], heads, seq)
    hc = h // d2
    for r, bb in enumerate(bufs):
        i2 = r % d2
        for k, ref in (("z", fw["z"]), ("dx", bw["dx"]), ("y1", fw["y1"])):
            got = to_np(bb[k])[:seq]
            e = rel(got, ref[:, i2 * hc:(i2 + 1) * hc])
            assert e <= TOL, (r, k, e)
