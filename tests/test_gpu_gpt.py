"""GPU parity of the full pre-LN GPT layer on virtual
meshes: every rank's shards vs the fp64 dense oracle (oracle/gpt.py) on the
same seeded inputs, through the C ABI (atp_gpt_layer_fwd_bwd)."""
import numpy as np
import pytest

from gpu_util import rel

pytestmark = pytest.mark.gpu

TOL = 2e-2


def _oracle(T, h, F, heads, seq, seed, causal=True):
    import datagen
    from oracle import gpt

    g = {k: v.astype(np.float64) for k, v in datagen.gpt_globals(T, h, F, seed, bf16=True).items()}
    fw = gpt.dense_forward(g, heads, seq, causal)
    bw = gpt.dense_backward(g, fw, g["dz"], heads, seq, causal)
    return g, fw, bw


def _expected(name, fw, bw, d1, d2, r, h, F):
    i1, i2 = r // d2, r % d2
    hc, h1, q1, F1 = h // d2, h // d1, 3 * h // d1, F // d1
    n = d1 * d2
    c = lambda a, w, i: a[..., i * w:(i + 1) * w]
    if name in ("z", "y1", "a", "bn"):
        return c(fw[name], hc, i2)
    if name == "dx":
        return c(bw["dx"], hc, i2)
    if name == "ctx":
        return c(fw["ctx"], h1, i1)
    if name in ("u", "h"):
        return c(fw[name], F1, i1)
    if name == "qkv":
        return c(fw["qkv"], 3 * h // n, r)
    if name == "dwqkv":
        return bw["dwqkv"][i2 * hc:(i2 + 1) * hc, i1 * q1:(i1 + 1) * q1]
    if name == "dbqkv":
        return c(bw["dbqkv"], q1, i1)
    if name == "dwo":
        return bw["dwo"][i1 * h1:(i1 + 1) * h1, i2 * hc:(i2 + 1) * hc]
    if name == "dw1":
        return bw["dw1"][i2 * hc:(i2 + 1) * hc, i1 * F1:(i1 + 1) * F1]
    if name == "db1":
        return c(bw["db1"], F1, i1)
    if name == "dw2":
        return bw["dw2"][i1 * F1:(i1 + 1) * F1, i2 * hc:(i2 + 1) * hc]
    if name in ("dbo", "db2", "dg1", "dbe1", "dg2", "dbe2"):
        return c(bw[name], hc, i2)
    raise KeyError(name)


NAMES = ("a", "qkv", "ctx", "y1", "bn", "u", "h", "z", "dx", "dwqkv", "dbqkv", "dwo", "dbo", "dw1", "db1", "dw2",
         "db2", "dg1", "dbe1", "dg2", "dbe2")


def run_gpt(d1, d2, chunks, T=512, h=1024, F=2048, heads=8, seq=256, seed=29, causal=True):
    import torch
    import paper_2301_08658_b200 as atp

    mesh = atp.Mesh.virtual(d1, d2)
    try:
        bufs = [atp.alloc_gpt_rank(d1, d2, r, T, h, F, heads, "cuda", seed) for r in range(d1 * d2)]
        call = atp.GptCall(mesh, bufs, T, h, F, heads, seq, chunks, causal)
        call()
        call()  # repeated calls must give the same results
        torch.cuda.synchronize()
    finally:
        mesh.destroy()
    return bufs


@pytest.mark.parametrize("d1,d2,chunks", [(1, 1, 1), (1, 1, 2), (2, 1, 2), (1, 2, 1), (2, 2, 2), (4, 2, 1),
                                          (2, 4, 2), (8, 1, 1), (1, 8, 2)])
def test_gpt_layer_matches_oracle(d1, d2, chunks):
    T, h, F, heads, seq = 512, 1024, 2048, 8, 256
    g, fw, bw = _oracle(T, h, F, heads, seq, 29)
    bufs = run_gpt(d1, d2, chunks, T, h, F, heads, seq, 29)
    worst = {}
    for r, b in enumerate(bufs):
        for name in NAMES:
            got = b[name].float().cpu().numpy()
            exp = _expected(name, fw, bw, d1, d2, r, h, F)
            worst[name] = max(worst.get(name, 0.0), rel(got.reshape(exp.shape), exp))
    bad = {k: v for k, v in worst.items() if not v < TOL}
    assert not bad, bad
    # replicas: z and dx are bit-identical across each dim-1 group (same i2)
    for i2 in range(d2):
        ranks = [i1 * d2 + i2 for i1 in range(d1)]
        for name in ("z", "dx", "dg1", "dbe2"):
            ref = bufs[ranks[0]][name]
            for r in ranks[1:]:
                assert bool((bufs[r][name] == ref).all()), (name, r)


@pytest.mark.parametrize("h,heads,d1", [(1536, 12, 1), (1536, 12, 2), (640, 5, 1)])
def test_gpt_layer_layernorm_widths(h, heads, d1):
    """d2 = 1 LayerNorm paths at other widths: the register-resident row
    kernels with 96 threads per row (h = 1536) and the warp-per-row fallback
    (h = 640, not a multiple of 512)."""
    T, F, seq = 512, 2 * h, 256
    g, fw, bw = _oracle(T, h, F, heads, seq, 37)
    bufs = run_gpt(d1, 1, 1, T, h, F, heads, seq, 37)
    for r, b in enumerate(bufs):
        for name in NAMES:
            got = b[name].float().cpu().numpy()
            exp = _expected(name, fw, bw, d1, 1, r, h, F)
            assert rel(got.reshape(exp.shape), exp) < TOL, (name, r)


def test_gpt_layer_noncausal_and_long_sequence():
    T, h, F, heads, seq = 1024, 512, 2048, 4, 512
    g, fw, bw = _oracle(T, h, F, heads, seq, 5, causal=False)
    bufs = run_gpt(2, 2, 2, T, h, F, heads, seq, 5, causal=False)
    for r, b in enumerate(bufs):
        for name in ("z", "dx", "dwqkv", "dwo", "dg1"):
            exp = _expected(name, fw, bw, 2, 2, r, h, F)
            assert rel(b[name].float().cpu().numpy().reshape(exp.shape), exp) < TOL, name


def test_gpt_layer_shape_errors():
    import torch
    import paper_2301_08658_b200 as atp
    from paper_2301_08658_b200._abi import AtpError

    mesh = atp.Mesh.virtual(2, 2)
    try:
        bufs = [atp.alloc_gpt_rank(2, 2, r, 512, 1024, 2048, 8, "cuda", 1) for r in range(4)]
        with pytest.raises(AtpError):
            atp.GptCall(mesh, bufs, 512, 1024, 2048, 8, 256, 4)()   # chunks of half sequences
        with pytest.raises(AtpError):
            atp.GptCall(mesh, bufs, 512, 1024, 2048, 6, 256, 1)()   # head dim != 128 / heads % 4
        with pytest.raises(AtpError):
            atp.GptCall(mesh, bufs, 512, 1024, 2048, 8, 200, 1)()   # seq % 128
        torch.cuda.synchronize()
    finally:
        mesh.destroy()


@pytest.mark.parametrize("gated", [False, True])
def test_gpt_layer_signalled_stages_with_cap(gated):
    """Chunked all-reduce stages of the full layer run as signalled stages (one GEMM per stage);
    with a GEMM CTA cap and gating on, the stages after LayerNorm must not gate on stale chunk gates."""
    import torch
    import paper_2301_08658_b200 as atp

    T, h, F, heads, seq, d1, d2, chunks = 1024, 1024, 2048, 8, 256, 2, 2, 4
    g, fw, bw = _oracle(T, h, F, heads, seq, 17)
    mesh = atp.Mesh.virtual(d1, d2)
    try:
        mesh.set_gemm_ctas(32)
        mesh.set_gating(gated)
        bufs = [atp.alloc_gpt_rank(d1, d2, r, T, h, F, heads, "cuda", 17) for r in range(d1 * d2)]
        call = atp.GptCall(mesh, bufs, T, h, F, heads, seq, chunks, True)
        for _ in range(2):
            call()
        torch.cuda.synchronize()
    finally:
        mesh.destroy()
    for r, b in enumerate(bufs):
        for name in ("z", "dx", "dwqkv", "dw1", "dg2"):
            exp = _expected(name, fw, bw, d1, d2, r, h, F)
            assert rel(b[name].float().cpu().numpy().reshape(exp.shape), exp) < TOL, (name, r)
