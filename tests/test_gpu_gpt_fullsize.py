"""Full-size parity of the full GPT layer in the launch
configurations bench.py --layer gpt times.

At N=1 (DeviceMesh(1,1)) every output of the layer is compared with the
dense oracle evaluated on the whole batch with float32 BLAS (the oracle code
is dtype-agnostic), element-wise through a global and a per-tile bound, after
NaN-poisoning the outputs.  On the chunked cfg-4 mesh the layer is
sequence-local (attention mixes tokens only within a sequence, G34), so the
outputs of one sampled sequence are exactly the oracle's dense layer
evaluated on that sequence alone.
"""
import numpy as np
import pytest

import datagen
from oracle import gpt

from gpu_util import assert_close, to_np

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


def test_fullsize_gpt_mesh11_every_output():
    """bench.py --layer gpt at N=1 (h=4096, 32 heads, b4 s2048, causal): every
    activation, dX and every weight / bias / LayerNorm gradient against the
    dense oracle (float32 BLAS), global and per-tile bound, outputs poisoned."""
    import torch
    import paper_2301_08658_b200 as atp
    from test_gpu_gpt import NAMES, _expected

    b, seq, h, heads, seed = 4, 2048, 4096, 32, 2301
    T, F = b * seq, 4 * h
    mesh = atp.Mesh.distributed(1, 1, 0, atp.atp_get_unique_id(), 0)
    try:
        bufs = atp.alloc_gpt_rank(1, 1, 0, T, h, F, heads, "cuda", seed)
        for k in NAMES:
            bufs[k].fill_(float("nan"))
        atp.GptCall(mesh, [bufs], T, h, F, heads, seq, 1, True)()
        torch.cuda.synchronize()
    finally:
        mesh.destroy()
    g = {k: datagen.tensor(k, s, seed=seed).astype(np.float32) for k, s in datagen.gpt_shapes(T, h, F).items()}
    fw = gpt.dense_forward(g, heads, seq)
    bw = gpt.dense_backward(g, fw, g["dz"], heads, seq)
    for name in NAMES:
        exp = _expected(name, fw, bw, 1, 1, 0, h, F)
        assert_close(name, to_np(bufs[name]).reshape(exp.shape), exp, TOL)


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
        for bb in bufs:
            for k in ("a", "y1", "bn", "u", "h", "z", "dx"):
                bb[k].fill_(float("nan"))
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
        i1, F1 = r // d2, F // d1
        for k, ref in (("z", fw["z"]), ("dx", bw["dx"]), ("y1", fw["y1"]), ("a", fw["a"]), ("bn", fw["bn"])):
            assert_close((r, k), to_np(bb[k])[:seq], ref[:, i2 * hc:(i2 + 1) * hc], TOL)
        for k in ("u", "h"):
            assert_close((r, k), to_np(bb[k])[:seq], fw[k][:, i1 * F1:(i1 + 1) * F1], TOL)
        # the other sequences were written too (no NaN left anywhere)
        for k in ("z", "dx", "h"):
            assert bool(torch.isfinite(bb[k]).all()), (r, k)
