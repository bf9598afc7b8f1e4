"""Runs first in a -m gpu session (conftest orders it): one tiny layer
forward+backward on a virtual DeviceMesh(2,2) with host-generated inputs, i.e.
libatp's GEMM / elementwise / group-sum kernels are the session's first
launches, checked against the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_libatp_kernels_first():
    import torch

    import datagen
    import paper_2301_08658_b200 as atp
    from oracle import layer as olayer

    T, h, F, heads, d1, d2, chunks, seed = 128, 128, 512, 4, 2, 2, 2, 7
    g = {k: v.astype(np.float64) for k, v in datagen.layer_globals(T, h, F, seed=seed).items()}
    _, fw, bw, _ = olayer.run_layer(g, d1, d2, heads, chunks)
    mesh = atp.Mesh.virtual(d1, d2, 0)
    try:
        bufs = [atp.alloc_layer_rank(d1, d2, r, T, h, F, "cuda:0", seed, host_inputs=True) for r in range(d1 * d2)]
        atp.atp_layer_fwd_bwd(mesh, bufs, T, h, F, heads, chunks, True)
        torch.cuda.synchronize()
    finally:
        mesh.destroy()
    for r, b in enumerate(bufs):
        for k, ref in (("z", fw["z"][r]), ("dx", bw["dx"][r]), ("dw1", bw["dw1"][r])):
            got = b[k].float().cpu().numpy().astype(np.float64)
            assert np.linalg.norm(got - ref) <= 2e-2 * np.linalg.norm(ref), (r, k)
