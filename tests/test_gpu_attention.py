"""GPU parity of the attention core against the fp64
oracle (oracle/gpt.py: Eq. 1), through the C ABI."""
import numpy as np
import pytest

from gpu_util import rel
from paper_2301_08658_b200._abi import AtpError

pytestmark = pytest.mark.gpu

TOL = 2e-2  # bf16 inputs / P, fp32 accumulation (north_star bf16 bar)


def _qkv(T, heads, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    import datagen

    return datagen.round_bf16((rng.standard_normal((T, 3 * heads * 128)) * scale).astype(np.float32))


@pytest.mark.parametrize("T,seq,heads,causal", [
    (256, 128, 1, True), (512, 256, 3, True), (768, 384, 2, True), (1024, 512, 2, False),
    (2048, 2048, 1, True), (256, 256, 2, False)])
def test_attn_fwd_matches_oracle(T, seq, heads, causal):
    import torch
    import paper_2301_08658_b200 as atp
    from oracle import gpt

    q = _qkv(T, heads, seed=T + heads, scale=1.5)
    qd = torch.from_numpy(q).to("cuda", torch.bfloat16)
    ctx = torch.zeros(T, heads * 128, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(heads, T, device="cuda", dtype=torch.float32)
    atp.atp_attn_core_fwd(qd, ctx, lse, seq, heads, causal)
    torch.cuda.synchronize()
    ref, ref_lse = gpt.core_softmax_fwd(q.astype(np.float64), heads, seq, causal)
    got = ctx.float().cpu().numpy()
    assert rel(got, ref) < TOL
    assert np.abs(lse.cpu().numpy() - ref_lse).max() < 2e-2


@pytest.mark.parametrize("T,seq,heads,causal,scale", [
    (8192, 2048, 8, True, 1.5), (24576, 384, 4, True, 4.0), (8192, 1024, 6, False, 1.5)])
def test_attn_fwd_many_items(T, seq, heads, causal, scale):
    """Grids larger than the GPU (256-768 query-tile pairs on 148 SMs): the
    persistent forward's work stealing, phases across items, an odd number of
    query blocks (seq 384: the last pair has one tile), and the lazy rescale
    restarting per item (scale 4)."""
    import torch
    import paper_2301_08658_b200 as atp
    from oracle import gpt

    q = _qkv(T, heads, seed=T + 3 * heads, scale=scale)
    qd = torch.from_numpy(q).to("cuda", torch.bfloat16)
    ctx = torch.full((T, heads * 128), float("nan"), device="cuda", dtype=torch.bfloat16)
    lse = torch.full((heads, T), float("nan"), device="cuda", dtype=torch.float32)
    atp.atp_attn_core_fwd(qd, ctx, lse, seq, heads, causal)
    torch.cuda.synchronize()
    ref, ref_lse = gpt.core_softmax_fwd(q.astype(np.float64), heads, seq, causal)
    got = ctx.float().cpu().numpy()
    assert np.isfinite(got).all() and np.isfinite(lse.cpu().numpy()).all()
    assert rel(got, ref) < TOL
    # every 128-row query tile of every head (a wrong or skipped item fails here)
    for h in range(heads):
        for r0 in range(0, T, 128):
            blk = slice(r0, r0 + 128), slice(h * 128, h * 128 + 128)
            assert rel(got[blk], ref[blk]) < TOL, (h, r0)
    assert np.abs(lse.cpu().numpy() - ref_lse).max() < 5e-2


def test_attn_fwd_peaked_scores():
    """Large logits (one key dominates): exercises the lazy rescaling path."""
    import torch
    import paper_2301_08658_b200 as atp
    from oracle import gpt

    T, seq, heads = 1024, 1024, 2
    q = _qkv(T, heads, seed=7, scale=4.0)
    qd = torch.from_numpy(q).to("cuda", torch.bfloat16)
    ctx = torch.zeros(T, heads * 128, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(heads, T, device="cuda", dtype=torch.float32)
    atp.atp_attn_core_fwd(qd, ctx, lse, seq, heads, True)
    torch.cuda.synchronize()
    ref, ref_lse = gpt.core_softmax_fwd(q.astype(np.float64), heads, seq, True)
    assert rel(ctx.float().cpu().numpy(), ref) < TOL
    assert np.abs(lse.cpu().numpy() - ref_lse).max() < 5e-2


def test_attn_shape_errors():
    import torch
    import paper_2301_08658_b200 as atp

    qd = torch.zeros(256, 3 * 128, device="cuda", dtype=torch.bfloat16)
    ctx = torch.zeros(256, 128, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(1, 256, device="cuda", dtype=torch.float32)
    with pytest.raises(AtpError):
        atp.atp_attn_core_fwd(qd, ctx, lse, 100, 1)   # seq not a multiple of 128
    with pytest.raises(AtpError):
        atp.atp_attn_core_fwd(qd[:200], ctx, lse, 128, 1)  # T not whole sequences


@pytest.mark.parametrize("T,seq,heads,causal", [
    (256, 128, 1, True), (512, 256, 3, True), (768, 384, 2, True), (1024, 512, 2, False), (2048, 1024, 1, True),
    # grids larger than the GPU (the persistent backward's work stealing and cross-item rings)
    (8192, 2048, 4, True), (12288, 384, 16, True), (4096, 1024, 12, False)])
def test_attn_bwd_matches_oracle(T, seq, heads, causal):
    import torch
    import paper_2301_08658_b200 as atp
    from oracle import gpt

    q = _qkv(T, heads, seed=3 * T + heads, scale=1.5)
    rng = np.random.default_rng(T)
    import datagen

    do = datagen.round_bf16(rng.standard_normal((T, heads * 128)).astype(np.float32))
    qd = torch.from_numpy(q).to("cuda", torch.bfloat16)
    dod = torch.from_numpy(do).to("cuda", torch.bfloat16)
    ctx = torch.zeros(T, heads * 128, device="cuda", dtype=torch.bfloat16)
    lse = torch.zeros(heads, T, device="cuda", dtype=torch.float32)
    dqkv = torch.full((T, 3 * heads * 128), float("nan"), device="cuda", dtype=torch.bfloat16)
    atp.atp_attn_core_fwd(qd, ctx, lse, seq, heads, causal)
    atp.atp_attn_core_bwd(qd, ctx, lse, dod, dqkv, seq, heads, causal)
    torch.cuda.synchronize()
    ref = gpt.core_softmax_bwd(do.astype(np.float64), q.astype(np.float64), heads, seq, causal)
    got = dqkv.float().cpu().numpy()
    assert np.isfinite(got).all()
    for part in range(3):  # q, k, v columns of every head
        cols = np.concatenate([np.arange(128) + (3 * j + part) * 128 for j in range(heads)])
        assert rel(got[:, cols], ref[:, cols]) < TOL, ("qkv"[part], rel(got[:, cols], ref[:, cols]))
    if T >= 4096:  # every 128-key block of every head and part (a wrong or skipped item fails here)
        for j in range(heads):
            for part in range(3):
                c = slice((3 * j + part) * 128, (3 * j + part + 1) * 128)
                for r0 in range(0, T, 128):
                    assert rel(got[r0:r0 + 128, c], ref[r0:r0 + 128, c]) < TOL, (j, part, r0)
