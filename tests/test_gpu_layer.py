"""Sharded ATP layer on the GPU vs the oracle, element by element per rank.

Virtual meshes run every rank of DeviceMesh(d1, d2) on one B200 with the same
schedule (chunk pipeline, events, epilogues) the distributed mesh uses; the
grouped all-reduce is a library kernel.  Every forward activation, the input
gradient and every weight/bias gradient of every rank is compared with the
oracle's shard: relative Frobenius <= 2e-2 (north_star, bf16).  Ranks of one
all-reduce group must hold bit-identical replicas."""
import numpy as np
import pytest

from gpu_util import BWD_MAP, FWD_MAP, oracle_layer, rel, to_np

pytestmark = pytest.mark.gpu

TOL = 2e-2
MESHES = [(1, 1), (2, 1), (1, 2), (4, 1), (2, 2), (1, 4), (8, 1), (4, 2), (2, 4), (1, 8)]


def run_gpu_layer(d1, d2, T, h, F, heads, chunks, seed, backward=True, fp32=False):
    import torch
    import paper_2301_08658_b200 as atp

    mesh = atp.Mesh.virtual(d1, d2, 0)
    try:
        bufs = [atp.alloc_layer_rank(d1, d2, r, T, h, F, "cuda", seed, fp32=fp32) for r in range(d1 * d2)]
        for b in bufs:  # poison outputs so unwritten elements show up
            for k in ("qkv", "ctx", "y1", "u", "h", "z", "dy1", "dx", "dwqkv", "dbqkv", "dwo", "dbo",
                      "dw1", "db1", "dw2", "db2"):
                b[k].fill_(float("nan"))
        atp.atp_layer_fwd_bwd(mesh, bufs, T, h, F, heads, chunks, backward)
        torch.cuda.synchronize()
    finally:
        mesh.destroy()
    return bufs


def compare(bufs, fw, bw, d1, d2, backward=True, tol=TOL):
    worst = {}
    for r, b in enumerate(bufs):
        for k, ok in FWD_MAP.items():
            got = to_np(b[k])
            assert np.isfinite(got).all(), (r, k)
            e = rel(got, fw[ok][r])
            worst[k] = max(worst.get(k, 0), e)
            assert e <= tol, (d1, d2, r, k, e)
        if backward:
            for k, ok in BWD_MAP.items():
                got = to_np(b[k])
                assert np.isfinite(got).all(), (r, k)
                e = rel(got, bw[ok][r])
                worst[k] = max(worst.get(k, 0), e)
                assert e <= tol, (d1, d2, r, k, e)
    return worst


def check_replicas(bufs, d1, d2):
    import torch
    from oracle import mesh as omesh

    # QKV, U, H, dU-derived grads are replicated over dim 2; Y1, Z, dY1, dX over dim 1
    for dim, keys in ((2, ("qkv", "ctx", "u", "h", "db1", "dbqkv")),
                      (1, ("y1", "z", "dy1", "dx", "db2", "dbo"))):
        for grp in omesh.groups(d1, d2, dim):
            for k in keys:
                for r in grp[1:]:
                    assert torch.equal(bufs[r][k], bufs[grp[0]][k]), (dim, grp, k)


@pytest.mark.parametrize("d1,d2", MESHES)
@pytest.mark.parametrize("chunks", [1, 2, 4])
def test_layer_every_mesh(d1, d2, chunks):
    T, h, F, heads, seed = 256, 256, 1024, 8, 17
    g, sh, fw, bw, log = oracle_layer(T, h, F, heads, d1, d2, chunks, seed)
    bufs = run_gpu_layer(d1, d2, T, h, F, heads, chunks, seed)
    compare(bufs, fw, bw, d1, d2)
    check_replicas(bufs, d1, d2)


@pytest.mark.parametrize("d1,d2", [(2, 2), (4, 2), (2, 4), (8, 1), (1, 8)])
def test_layer_signalled_stages(d1, d2):
    """T/chunks = 256 rows: every communicating stage runs as ONE GEMM with
    per-chunk completion counters gating the all-reduces (signalled stages)."""
    T, h, F, heads, chunks, seed = 1024, 512, 2048, 8, 4, 23
    g, sh, fw, bw, _ = oracle_layer(T, h, F, heads, d1, d2, chunks, seed)
    bufs = run_gpu_layer(d1, d2, T, h, F, heads, chunks, seed)
    compare(bufs, fw, bw, d1, d2)
    check_replicas(bufs, d1, d2)
    # a second call reuses the counters (cumulative targets) and must agree bit for bit
    bufs2 = run_gpu_layer(d1, d2, T, h, F, heads, chunks, seed)
    import torch
    for b1, b2 in zip(bufs, bufs2):
        for k in ("z", "dx", "dw1", "dwqkv"):
            assert torch.equal(b1[k], b2[k]), k


FP32_TOL = 1e-4  # north_star fp32 check mode


@pytest.mark.parametrize("d1,d2", MESHES)
@pytest.mark.parametrize("chunks", [1, 4])
def test_layer_fp32_check_mode(d1, d2, chunks):
    """ATP_FP32: the same sharded schedule in fp32 (FFMA GEMMs, fp32
    all-reduces) on unrounded fp32 inputs, every tensor of every rank within
    1e-4 relative Frobenius of the fp64 oracle."""
    from gpu_util import oracle_layer_fp32

    T, h, F, heads, seed = 512, 256, 1024, 8, 41
    g, sh, fw, bw, _ = oracle_layer_fp32(T, h, F, heads, d1, d2, chunks, seed)
    bufs = run_gpu_layer(d1, d2, T, h, F, heads, chunks, seed, fp32=True)
    worst = compare(bufs, fw, bw, d1, d2, tol=FP32_TOL)
    assert max(worst.values()) < FP32_TOL


def test_cfg1_mlp_2x2():
    """BASELINE.json configs[0]: h=64, ffn=256, tokens=32 on a 2x2 mesh."""
    import torch
    import paper_2301_08658_b200 as atp

    T, h, F, heads, seed, d1, d2 = 32, 64, 256, 2, 5, 2, 2
    g, sh, fw, bw, _ = oracle_layer(T, h, F, heads, d1, d2, 1, seed)
    mesh = atp.Mesh.virtual(d1, d2)
    bufs = [atp.alloc_layer_rank(d1, d2, r, T, h, F, "cuda", seed) for r in range(4)]
    # the MLP alone, fed the oracle's Y1 shards
    for r, b in enumerate(bufs):
        b["y1"].copy_(torch.from_numpy(fw["y1"][r]).to(torch.bfloat16))
    atp.atp_mlp_fwd(mesh, bufs, T, h, F, 1)
    torch.cuda.synchronize()
    mesh.destroy()
    for r, b in enumerate(bufs):
        assert rel(to_np(b["z"]), fw["z"][r]) <= TOL


@pytest.mark.parametrize("chunks", [1, 2])
def test_cfg1_fp32_check_mode_2x2(chunks):
    """BASELINE.json configs[0] in its own precision: h=64, ffn=256, tokens=32,
    fp32, DeviceMesh(2,2) -- the whole layer (fwd+bwd) and the MLP block alone
    in the ATP_FP32 check mode, every tensor of every rank <= 1e-4 relF
    against the fp64 oracle on the same unrounded fp32 inputs."""
    import torch
    import paper_2301_08658_b200 as atp
    from gpu_util import assert_close, oracle_layer_fp32

    T, h, F, heads, seed, d1, d2 = 32, 64, 256, 2, 5, 2, 2
    g, sh, fw, bw, _ = oracle_layer_fp32(T, h, F, heads, d1, d2, chunks, seed)
    bufs = run_gpu_layer(d1, d2, T, h, F, heads, chunks, seed, fp32=True)
    for r, b in enumerate(bufs):
        for k, ok in list(FWD_MAP.items()) + list(BWD_MAP.items()):
            src = fw if k in FWD_MAP else bw
            assert_close((r, k), to_np(b[k]), src[ok][r], FP32_TOL, tile=(32, 32))
    check_replicas(bufs, d1, d2)
    # the MLP block alone (atp_mlp_fwd / atp_mlp_bwd), fed the oracle's Y1 shards
    mesh = atp.Mesh.virtual(d1, d2)
    try:
        mb = [atp.alloc_layer_rank(d1, d2, r, T, h, F, "cuda", seed, fp32=True) for r in range(4)]
        for r, b in enumerate(mb):
            b["y1"].copy_(torch.from_numpy(fw["y1"][r]).to(torch.float32))
            for k in ("u", "h", "z", "dy1", "dw1", "db1", "dw2", "db2"):
                b[k].fill_(float("nan"))
        atp.atp_mlp_fwd(mesh, mb, T, h, F, chunks)
        atp.atp_mlp_bwd(mesh, mb, T, h, F, chunks)
        torch.cuda.synchronize()
    finally:
        mesh.destroy()
    for r, b in enumerate(mb):
        for k in ("u", "h", "z"):
            assert_close((r, k), to_np(b[k]), fw[k][r], FP32_TOL, tile=(32, 32))
        for k in ("dw1", "db1", "dw2", "db2"):
            assert_close((r, k), to_np(b[k]), bw[k][r], FP32_TOL, tile=(32, 32))
        # dY1 from the MLP alone = dZ + dU W1^T (the attention block's input gradient comes later)
        assert_close((r, "dy1"), to_np(b["dy1"]), bw["dy1"][r], FP32_TOL, tile=(32, 32))


@pytest.mark.parametrize("d1,d2", [(2, 2), (4, 2), (1, 1)])
def test_ragged_chunk_and_odd_sizes(d1, d2):
    # T/chunks = 72 rows (not a multiple of the 128-row tile), head dim 16
    T, h, F, heads, chunks, seed = 216, 192, 320, 12, 3, 29
    if heads % d1:
        pytest.skip("heads % d1")
    g, sh, fw, bw, _ = oracle_layer(T, h, F, heads, d1, d2, chunks, seed)
    bufs = run_gpu_layer(d1, d2, T, h, F, heads, chunks, seed)
    compare(bufs, fw, bw, d1, d2)


@pytest.mark.parametrize("colfirst", [True, False])
@pytest.mark.parametrize("d1,d2", [(2, 2), (4, 2), (2, 4), (1, 1)])
@pytest.mark.parametrize("chunks", [1, 4])
def test_single_linear(colfirst, d1, d2, chunks):
    """atp_linear_{colfirst,rowfirst}_{fwd,bwd} vs the oracle's sharded linear."""
    import torch
    import datagen
    import paper_2301_08658_b200 as atp
    from oracle import layer as olayer, sharding as osh
    from oracle.sharding import R, S1

    M, K, N, seed = 256, 384, 512, 3
    X = datagen.tensor("lin_x", (M, K), seed).astype(np.float64)
    W = datagen.tensor("lin_w", (K, N), seed).astype(np.float64) * 20
    W = datagen.round_bf16(W.astype(np.float32)).astype(np.float64)
    bvec = datagen.tensor("lin_b", (N,), seed).astype(np.float64)
    dY = datagen.tensor("lin_dy", (M, N), seed).astype(np.float64)
    xs = (olayer.ACT if colfirst else (S1, R))
    ws = olayer.COL_W if colfirst else olayer.ROW_W
    ys = olayer.COL_OUT if colfirst else olayer.ACT
    Xl, Wl, dYl = osh.shard(X, xs, d1, d2), osh.shard(W, ws, d1, d2), osh.shard(dY, ys, d1, d2)
    bl = [osh.local(bvec[None, :], ys, d1, d2, r)[0] for r in range(d1 * d2)]
    fwd = olayer.colfirst_forward if colfirst else olayer.rowfirst_forward
    Yl = fwd(Xl, Wl, d1, d2)
    Yl = [y + b for y, b in zip(Yl, bl)]
    dXl, dWl = olayer.linear_backward("col" if colfirst else "row", Xl, Wl, dYl, d1, d2)
    mesh = atp.Mesh.virtual(d1, d2)
    T_ = lambda a, dt=torch.bfloat16: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)
    fa = [dict(x=T_(Xl[r]), w=T_(Wl[r]), bias=T_(bl[r]), y=torch.empty(Yl[r].shape, dtype=torch.bfloat16, device="cuda"))
          for r in range(d1 * d2)]
    atp.atp_linear_fwd(mesh, colfirst, fa, M, K, N, chunks)
    ba = [dict(x=fa[r]["x"], w=fa[r]["w"], dy=T_(dYl[r]), dx=torch.empty(Xl[r].shape, dtype=torch.bfloat16, device="cuda"),
               dw=torch.empty(Wl[r].shape, dtype=torch.float32, device="cuda"),
               dbias=torch.empty(bl[r].shape, dtype=torch.float32, device="cuda")) for r in range(d1 * d2)]
    atp.atp_linear_bwd(mesh, colfirst, ba, M, K, N, chunks)
    torch.cuda.synchronize()
    mesh.destroy()
    for r in range(d1 * d2):
        assert rel(to_np(fa[r]["y"]), Yl[r]) <= TOL
        assert rel(to_np(ba[r]["dx"]), dXl[r]) <= TOL
        assert rel(to_np(ba[r]["dw"]), dWl[r]) <= TOL
        assert rel(to_np(ba[r]["dbias"]), dYl[r].sum(axis=0)) <= TOL


def test_shape_errors_before_enqueue():
    import paper_2301_08658_b200 as atp

    mesh = atp.Mesh.virtual(2, 2)
    try:
        bufs = [atp.alloc_layer_rank(2, 2, r, 64, 64, 256, "cuda", 1) for r in range(4)]
        with pytest.raises(atp.AtpError) as e:
            atp.atp_layer_fwd_bwd(mesh, bufs, 64, 64, 256, 3, 1)  # heads % d1 != 0
        assert e.value.status == 2
        with pytest.raises(atp.AtpError):
            atp.atp_layer_fwd_bwd(mesh, bufs, 64, 64, 256, 4, 3)  # T % chunks != 0
    finally:
        mesh.destroy()


def test_probe_single_rank_and_local_mesh():
    """atp_probe_hcm on a 1-rank NCCL mesh (the only size this box has): no
    pairs, no groups, one calibration entry with NoComm on both dimensions;
    and a local dry-run mesh runs a schedule with its collectives elided."""
    import torch
    import paper_2301_08658_b200 as atp

    uid = atp.atp_get_unique_id()
    mesh = atp.Mesh.distributed(1, 1, 0, uid, 0)
    try:
        scratch = torch.empty(1 << 20, dtype=torch.bfloat16, device="cuda")
        layers, matrix, calib = atp.atp_probe_hcm(mesh, scratch, msg_bytes=(1 << 20,), calib_bytes=1 << 20, iters=2)
        assert [(l.ranks) for l in layers] == [1] and matrix == [[0.0]]
        assert calib == {(1, 1): (None, None)}
        plan = atp.atp_search(layers, calibration=calib)
        assert plan["chosen"] == (1, 1)
    finally:
        mesh.destroy()
    loc = atp.Mesh.local(4, 2, 3)
    try:
        b = atp.alloc_layer_rank(4, 2, 3, 256, 256, 1024, "cuda", 3)
        atp.atp_layer_fwd_bwd(loc, [b], 256, 256, 1024, 8, 2, True)
        torch.cuda.synchronize()
        assert torch.isfinite(b["z"].float()).all() and torch.isfinite(b["dw1"]).all()
        with pytest.raises(atp.AtpError):
            atp.atp_probe_hcm(loc, scratch, msg_bytes=(1 << 20,))
    finally:
        loc.destroy()


@pytest.mark.isolated(timeout=240, retries=1)
@pytest.mark.parametrize("d1,d2", [(2, 1), (1, 2), (2, 2), (4, 2), (2, 4), (8, 1), (1, 8)])
@pytest.mark.parametrize("chunks", [1, 4])
def test_layer_fused_peer_allreduce(d1, d2, chunks):
    """Fused stages: signalled GEMM into the peer-visible buffer + one kernel
    per chunk doing the grouped all-reduce over peer memory with the
    elementwise step fused; parity, replicas and a repeated call."""
    import torch
    import paper_2301_08658_b200 as atp

    T, h, F, heads, seed = 1024, 512, 2048, 8, 31
    g, sh, fw, bw, _ = oracle_layer(T, h, F, heads, d1, d2, chunks, seed)
    mesh = atp.Mesh.virtual(d1, d2)
    try:
        mesh.enable_fused_ar(T * F * 2)
        bufs = [atp.alloc_layer_rank(d1, d2, r, T, h, F, "cuda", seed) for r in range(d1 * d2)]
        call = atp.LayerCall(mesh, bufs, T, h, F, heads, chunks, True)
        call()
        torch.cuda.synchronize()
        snap = [{k: b[k].clone() for k in ("z", "dx", "dw1", "dwqkv")} for b in bufs]
        call()
        torch.cuda.synchronize()
    finally:
        mesh.destroy()
    compare(bufs, fw, bw, d1, d2)
    check_replicas(bufs, d1, d2)
    for b, s in zip(bufs, snap):
        for k, v in s.items():
            assert torch.equal(b[k], v), k


def _fused_launches(mesh, call):
    """Run `call` under the executor's per-launch trace; returns the number of
    fused all-reduce kernels (op kind 4) and of ordinary collectives (kind 2)."""
    import ctypes as C

    import torch
    from paper_2301_08658_b200 import _abi

    lib = _abi.lib()
    _abi.check(lib.atp_profile_begin(mesh.handle))
    call()
    torch.cuda.synchronize()
    recs = (_abi.TraceRec * 65536)()
    n = C.c_int()
    _abi.check(lib.atp_profile_trace(mesh.handle, recs, 65536, C.byref(n)))
    _abi.check(lib.atp_profile_end(mesh.handle, C.byref(_abi.Profile())))
    kinds = [r.kind for r in recs[: n.value]]
    return kinds.count(4), kinds.count(2)


@pytest.mark.isolated(timeout=240, retries=1)
@pytest.mark.parametrize("d1,d2", [(4, 2), (2, 4), (8, 1), (1, 8)])
def test_layer_fused_push_every_stage(d1, d2):
    """Fused GEMM -> reduce-scatter (TMA stores into the slice owners' receive
    slots) -> pull all-gather with the elementwise step, at a size where every
    communicating stage of the layer qualifies (slices of whole 128-row tiles):
    all 8 stages x 4 chunks run as fused kernels on every rank (no collective
    falls back), outputs poisoned with NaN beforehand, every output of every
    rank vs the oracle, bit-identical replicas, a second call identical."""
    import torch
    import paper_2301_08658_b200 as atp

    T, h, F, heads, chunks, seed = 4096, 512, 2048, 8, 4, 53
    g, sh, fw, bw, _ = oracle_layer(T, h, F, heads, d1, d2, chunks, seed)
    mesh = atp.Mesh.virtual(d1, d2)
    try:
        mesh.enable_fused_ar(T * F * 2)
        bufs = [atp.alloc_layer_rank(d1, d2, r, T, h, F, "cuda", seed) for r in range(d1 * d2)]
        for b in bufs:
            for k in ("qkv", "ctx", "y1", "u", "h", "z", "dx", "dwqkv", "dbqkv", "dwo", "dbo", "dw1", "db1", "dw2",
                      "db2"):
                b[k].fill_(float("nan"))
        call = atp.LayerCall(mesh, bufs, T, h, F, heads, chunks, True)
        n_fused, n_coll = _fused_launches(mesh, call)
        snap = [{k: b[k].clone() for k in ("z", "dx", "dw1", "dwqkv", "u", "h")} for b in bufs]
        call()
        torch.cuda.synchronize()
    finally:
        mesh.destroy()
    comm_stages = 4 * (d1 > 1) + 4 * (d2 > 1)  # a size-1 mesh dimension has no collective (G7)
    assert n_coll == 0 and n_fused == comm_stages * chunks * d1 * d2, (n_fused, n_coll)
    compare(bufs, fw, bw, d1, d2)
    check_replicas(bufs, d1, d2)
    for b, s in zip(bufs, snap):
        for k, v in s.items():
            assert torch.equal(b[k], v), k


@pytest.mark.isolated(timeout=240, retries=1)
@pytest.mark.parametrize("d1,d2,cap", [(2, 2, 32), (4, 2, 16), (2, 4, 16), (8, 1, 16)])
@pytest.mark.parametrize("fused", [False, True])
def test_layer_chunk_gated(d1, d2, cap, fused):
    """Chunk-gated GEMMs: with a GEMM CTA cap that leaves SMs for the
    communication kernels, each stage's GEMM waits per chunk for the previous
    stage's chunk gate instead of its last all-reduce (NCCL-path or fused)."""
    import torch
    import paper_2301_08658_b200 as atp

    T, h, F, heads, chunks, seed = 1024, 512, 2048, 8, 4, 37
    g, sh, fw, bw, _ = oracle_layer(T, h, F, heads, d1, d2, chunks, seed)
    mesh = atp.Mesh.virtual(d1, d2)
    try:
        mesh.set_gemm_ctas(cap)
        mesh.set_gating(True)
        if fused:
            mesh.enable_fused_ar(T * F * 2)
        bufs = [atp.alloc_layer_rank(d1, d2, r, T, h, F, "cuda", seed) for r in range(d1 * d2)]
        call = atp.LayerCall(mesh, bufs, T, h, F, heads, chunks, True)
        for _ in range(3):
            call()
        torch.cuda.synchronize()
    finally:
        mesh.destroy()
    compare(bufs, fw, bw, d1, d2)
    check_replicas(bufs, d1, d2)


@pytest.mark.isolated(timeout=240, retries=1)
@pytest.mark.gpu
@pytest.mark.parametrize("fused", [False, True])
def test_layer_gated_chunk_count_changes(fused):
    """One mesh serving schedules with different chunk counts: counter and gate
    slots change role between calls (gates hold the call's epoch, tile counters
    cumulative totals), so every call must still complete and match the oracle."""
    import torch
    import paper_2301_08658_b200 as atp

    d1, d2, cap = 2, 2, 32
    T, h, F, heads, seed = 1024, 512, 2048, 8, 41
    mesh = atp.Mesh.virtual(d1, d2)
    try:
        mesh.set_gemm_ctas(cap)
        mesh.set_gating(True)
        if fused:
            mesh.enable_fused_ar(T * F * 2)
        for chunks in (2, 4, 1, 8, 2):
            g, sh, fw, bw, _ = oracle_layer(T, h, F, heads, d1, d2, chunks, seed)
            bufs = [atp.alloc_layer_rank(d1, d2, r, T, h, F, "cuda", seed) for r in range(d1 * d2)]
            atp.LayerCall(mesh, bufs, T, h, F, heads, chunks, True)()
            torch.cuda.synchronize()
            compare(bufs, fw, bw, d1, d2)
    finally:
        mesh.destroy()


@pytest.mark.gpu
def test_mesh_from_borrowed_comms():
    """atp_mesh_init_from_comms: a mesh over caller-created NCCL
    communicators (here 1-rank ones from the same libnccl libatp links) runs
    the linear block like atp_mesh_init, and is destroyed without touching them."""
    import ctypes as C
    import os
    import torch
    import paper_2301_08658_b200 as atp
    from paper_2301_08658_b200 import build as B

    class UniqueId(C.Structure):  # ncclUniqueId, passed by value
        _fields_ = [("internal", C.c_char * 128)]

    nccl = C.CDLL(os.path.join(B.nccl_dir(), "lib", "libnccl.so.2"))
    nccl.ncclGetUniqueId.argtypes = [C.POINTER(UniqueId)]
    nccl.ncclCommInitRank.argtypes = [C.POINTER(C.c_void_p), C.c_int, UniqueId, C.c_int]
    nccl.ncclCommCount.argtypes = [C.c_void_p, C.POINTER(C.c_int)]
    nccl.ncclCommDestroy.argtypes = [C.c_void_p]
    torch.cuda.set_device(0)
    uid = UniqueId()
    assert nccl.ncclGetUniqueId(C.byref(uid)) == 0
    comm = C.c_void_p()
    assert nccl.ncclCommInitRank(C.byref(comm), 1, uid, 0) == 0
    T, h, F, heads, seed = 512, 256, 1024, 2, 3
    g, sh, fw, bw, _ = oracle_layer(T, h, F, heads, 1, 1, 1, seed)
    mesh = atp.Mesh.from_comms(1, 1, 0, comm.value, comm.value, 0)
    try:
        bufs = atp.alloc_layer_rank(1, 1, 0, T, h, F, "cuda", seed)
        atp.LayerCall(mesh, [bufs], T, h, F, heads, 1, True)()
        torch.cuda.synchronize()
    finally:
        mesh.destroy()
    compare([bufs], fw, bw, 1, 1)
    cnt = C.c_int()
    assert nccl.ncclCommCount(comm, C.byref(cnt)) == 0 and cnt.value == 1  # still alive
    nccl.ncclCommDestroy(comm)
    from paper_2301_08658_b200._abi import AtpError
    with pytest.raises(AtpError):
        atp.Mesh.from_comms(2, 1, 0, None, None, 0)


@pytest.mark.parametrize("d1,d2,chunks", [(1, 1, 1), (2, 2, 2), (4, 2, 2), (1, 4, 2)])
def test_layer_stack(d1, d2, chunks):
    """atp_layer_stack_fwd_bwd: 3 layers as ONE pipeline (forward 0..2, backward
    2..0; SURVEY §8(d) L_bench) vs the oracle run layer by layer: layer l's
    input is the oracle's Z of layer l-1 and its upstream gradient the oracle's
    dX of layer l+1.  Every output of every layer and rank is compared (all
    outputs poisoned with NaN first), replicas bit-identical."""
    import torch
    import datagen
    import paper_2301_08658_b200 as atp
    from oracle import layer as olayer

    L, T, h, F, heads, seed = 3, 512, 256, 1024, 4, 61
    gs = [{k: v.astype(np.float64) for k, v in datagen.layer_globals(T, h, F, seed=seed + l).items()}
          for l in range(L)]
    xs = [gs[0]["x"]]
    for l in range(L - 1):  # dense forward chain
        xs.append(olayer.dense_forward(dict(gs[l], x=xs[l]), heads)["z"])
    dzs = [None] * L
    dzs[L - 1] = gs[L - 1]["dz"]
    for l in range(L - 1, 0, -1):  # dense backward chain
        gl = dict(gs[l], x=xs[l])
        dzs[l - 1] = olayer.dense_backward(gl, olayer.dense_forward(gl, heads), dzs[l], heads)["dx"]
    ref = [olayer.run_layer(dict(gs[l], x=xs[l], dz=dzs[l]), d1, d2, heads, chunks) for l in range(L)]

    mesh = atp.Mesh.virtual(d1, d2)
    try:
        per_rank = [atp.alloc_layer_stack(d1, d2, r, T, h, F, "cuda", seed, L) for r in range(d1 * d2)]
        stack = [[per_rank[r][l] for r in range(d1 * d2)] for l in range(L)]
        for layer in stack:
            for b in layer:
                for k in ("qkv", "ctx", "y1", "u", "h", "z", "dy1", "dx", "dwqkv", "dbqkv", "dwo", "dbo", "dw1",
                          "db1", "dw2", "db2"):
                    b[k].fill_(float("nan"))
        atp.LayerStackCall(mesh, stack, T, h, F, heads, chunks)()
        torch.cuda.synchronize()
    finally:
        mesh.destroy()
    for l in range(L):
        _, fw, bw, _ = ref[l]
        compare(stack[l], fw, bw, d1, d2)
        check_replicas(stack[l], d1, d2)


@pytest.mark.isolated(timeout=240, retries=1)
@pytest.mark.parametrize("d1,d2,fused,gated", [(2, 2, True, False), (4, 2, True, True), (2, 2, False, True)])
def test_layer_stack_fused_and_gated(d1, d2, fused, gated):
    """The layer stack with the fused GEMM -> RS -> AG stages (receive regions
    alternate across all 8 x L stages of the pipeline) and / or chunk-gated
    GEMMs (layer l+1's first GEMM gated on layer l's last stage), against the
    oracle run layer by layer; replicas bit-identical."""
    import torch
    import datagen
    import paper_2301_08658_b200 as atp
    from oracle import layer as olayer

    L, T, h, F, heads, chunks, seed = 2, 1024, 256, 1024, 4, 4, 67
    gs = [{k: v.astype(np.float64) for k, v in datagen.layer_globals(T, h, F, seed=seed + l).items()}
          for l in range(L)]
    xs = [gs[0]["x"], olayer.dense_forward(dict(gs[0], x=gs[0]["x"]), heads)["z"]]
    g1 = dict(gs[1], x=xs[1])
    dzs = [olayer.dense_backward(g1, olayer.dense_forward(g1, heads), gs[1]["dz"], heads)["dx"], gs[1]["dz"]]
    ref = [olayer.run_layer(dict(gs[l], x=xs[l], dz=dzs[l]), d1, d2, heads, chunks) for l in range(L)]
    mesh = atp.Mesh.virtual(d1, d2)
    try:
        if gated:
            mesh.set_gemm_ctas(16)
            mesh.set_gating(True)
        if fused:
            mesh.enable_fused_ar(T * F * 2)
        per_rank = [atp.alloc_layer_stack(d1, d2, r, T, h, F, "cuda", seed, L) for r in range(d1 * d2)]
        stack = [[per_rank[r][l] for r in range(d1 * d2)] for l in range(L)]
        call = atp.LayerStackCall(mesh, stack, T, h, F, heads, chunks)
        for _ in range(2):
            call()
        torch.cuda.synchronize()
    finally:
        mesh.destroy()
    for l in range(L):
        _, fw, bw, _ = ref[l]
        compare(stack[l], fw, bw, d1, d2)
        check_replicas(stack[l], d1, d2)
