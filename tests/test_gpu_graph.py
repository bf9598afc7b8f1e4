"""CUDA-graph capture and replay of whole layer steps (atp_graph_begin / end /
launch): a replay must reproduce the direct call bit for bit, repeatedly (the
chunk counters restart at zero every call), on virtual meshes with signalled
and chunk-gated stages, on a 1-rank NCCL mesh (the bench's N=1 path) and for
the full GPT layer; the fused peer-memory mesh and profiling refuse capture."""
import pytest

from gpu_util import oracle_layer

pytestmark = pytest.mark.gpu

OUTS = ("qkv", "ctx", "y1", "u", "h", "z", "dy1", "dx", "dwqkv", "dbqkv", "dwo", "dbo", "dw1", "db1", "dw2", "db2")


def _replay_matches(mesh, bufs, call, keys, stream, n_replays=3):
    import torch
    import paper_2301_08658_b200 as atp

    call(stream)
    stream.synchronize()
    ref = [{k: b[k].clone() for k in keys} for b in bufs]
    g = atp.Graph.capture(mesh, call, stream)
    try:
        for _ in range(n_replays):
            for b in bufs:
                for k in keys:
                    b[k].fill_(float("nan"))
            torch.cuda.synchronize()  # the fills (default stream) must land before the replay (its own stream)
            g(stream)
            stream.synchronize()
            for b, r in zip(bufs, ref):
                for k in keys:
                    assert torch.equal(b[k], r[k]), k
    finally:
        g.destroy()


@pytest.mark.parametrize("d1,d2,chunks,gated", [(1, 1, 1, False), (2, 2, 2, False), (4, 2, 4, False),
                                                (2, 2, 4, True), (1, 4, 2, True)])
def test_layer_graph_replay(d1, d2, chunks, gated):
    import numpy as np
    import torch
    import paper_2301_08658_b200 as atp

    T, h, F, heads, seed = 1024, 512, 2048, 8, 53
    mesh = atp.Mesh.virtual(d1, d2)
    try:
        if gated:
            mesh.set_gemm_ctas(16)
            mesh.set_gating(True)
        bufs = [atp.alloc_layer_rank(d1, d2, r, T, h, F, "cuda", seed) for r in range(d1 * d2)]
        call = atp.LayerCall(mesh, bufs, T, h, F, heads, chunks, True)
        stream = torch.cuda.Stream()
        _replay_matches(mesh, bufs, call, OUTS, stream)
    finally:
        mesh.destroy()
    # and the replayed values are the oracle's
    from gpu_util import BWD_MAP, FWD_MAP, rel, to_np

    _, _, fw, bw, _ = oracle_layer(T, h, F, heads, d1, d2, chunks, seed)
    for r, b in enumerate(bufs):
        for k, ok in list(FWD_MAP.items()) + list(BWD_MAP.items()):
            src = fw if k in FWD_MAP else bw
            got = to_np(b[k])
            assert np.isfinite(got).all() and rel(got, src[ok][r]) <= 2e-2, k


def test_layer_graph_nccl_single_rank():
    """The bench's N=1 path: a 1-rank NCCL mesh (atp_mesh_init), graph replay."""
    import torch
    import paper_2301_08658_b200 as atp

    T, h, F, heads, seed = 2048, 1024, 4096, 8, 59
    mesh = atp.Mesh.distributed(1, 1, 0, atp.atp_get_unique_id(), torch.cuda.current_device())
    try:
        bufs = [atp.alloc_layer_rank(1, 1, 0, T, h, F, "cuda", seed)]
        call = atp.LayerCall(mesh, bufs, T, h, F, heads, 1, True)
        _replay_matches(mesh, bufs, call, OUTS, torch.cuda.Stream())
    finally:
        mesh.destroy()


@pytest.mark.parametrize("d1,d2,chunks", [(1, 1, 1), (2, 2, 2)])
def test_gpt_graph_replay(d1, d2, chunks):
    import torch
    import paper_2301_08658_b200 as atp

    T, h, F, heads, seq, seed = 512, 1024, 2048, 8, 256, 61
    mesh = atp.Mesh.virtual(d1, d2)
    try:
        bufs = [atp.alloc_gpt_rank(d1, d2, r, T, h, F, heads, "cuda", seed) for r in range(d1 * d2)]
        call = atp.GptCall(mesh, bufs, T, h, F, heads, seq, chunks, True)
        _replay_matches(mesh, bufs, call, ("z", "dx", "dwqkv", "dw1", "dg1", "dbe2"), torch.cuda.Stream())
    finally:
        mesh.destroy()


def test_graph_refusals():
    import torch
    import paper_2301_08658_b200 as atp
    from paper_2301_08658_b200 import AtpError, _abi

    mesh = atp.Mesh.virtual(2, 1)
    st = torch.cuda.Stream()
    try:
        _abi.check(_abi.lib().atp_profile_begin(mesh.handle))
        with pytest.raises(AtpError):
            atp.Graph.capture(mesh, lambda s: None, st)
        prof = _abi.Profile()
        _abi.check(_abi.lib().atp_profile_end(mesh.handle, prof))
        mesh.enable_fused_ar(1 << 20)
        with pytest.raises(AtpError):
            atp.Graph.capture(mesh, lambda s: None, st)
    finally:
        mesh.destroy()


def test_profile_trace_timeline():
    """atp_profile_trace: one record per bracketed launch, in enqueue order,
    non-negative durations, and the per-class totals equal atp_profile_end's."""
    import ctypes as C
    import torch
    import paper_2301_08658_b200 as atp
    from paper_2301_08658_b200 import _abi

    T, h, F, heads = 1024, 512, 2048, 8
    mesh = atp.Mesh.virtual(2, 2)
    try:
        bufs = [atp.alloc_layer_rank(2, 2, r, T, h, F, "cuda", 5) for r in range(4)]
        call = atp.LayerCall(mesh, bufs, T, h, F, heads, 2, True)
        call()
        torch.cuda.synchronize()
        lib = _abi.lib()
        _abi.check(lib.atp_profile_begin(mesh.handle))
        call()
        torch.cuda.synchronize()
        recs = (_abi.TraceRec * 4096)()
        n = C.c_int()
        _abi.check(lib.atp_profile_trace(mesh.handle, recs, 4096, C.byref(n)))
        prof = _abi.Profile()
        _abi.check(lib.atp_profile_end(mesh.handle, C.byref(prof)))
    finally:
        mesh.destroy()
    rs = list(recs[: n.value])
    assert n.value == sum(prof.launches) and n.value > 0
    assert all(r.t1_ms >= r.t0_ms >= 0.0 for r in rs)
    assert sum(1 for r in rs if r.kind == 0) == prof.launches[0]  # GEMMs
    for cls in range(4):  # event timestamps have ~0.5 us resolution: per-record slack
        sel = [r for r in rs if r.cls == cls]
        tot = sum(r.t1_ms - r.t0_ms for r in sel)
        assert abs(tot - prof.ms[cls]) <= 2e-3 * (len(sel) + 1) + 1e-2 * prof.ms[cls], cls
