"""One rank of a real multi-process NCCL mesh whose ranks SHARE one GPU.

Launched by tests/test_gpu_nccl_multiproc.py (torch.multiprocessing.spawn).
NCCL refuses two ranks on one device of one host ("Duplicate GPU"), so each
rank sets a distinct NCCL_HOSTID: NCCL then treats the ranks as separate hosts
and moves data over its socket transport on 127.0.0.1.  That is slow, but it
drives the exact code the multi-GPU job runs -- atp_mesh_init's communicator
split, the communication stream, the per-chunk event handoff, signalled stages
(cuStreamWaitValue32 on tile counters), NCCL all-reduce / reduce-scatter /
all-gather on the dim-1 / dim-2 communicators -- through the C ABI, one process
per rank, and each rank's shards are compared with the oracle's.

Test infrastructure only: the oracle is imported here, never by the product."""
from __future__ import annotations

import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def _layer(atp, mesh, d1, d2, rank, chunks, seed, graph=False):
    import numpy as np
    import torch

    from gpu_util import BWD_MAP, FWD_MAP, oracle_layer, rel, to_np

    T, h, F, heads = 512, 256, 1024, 8
    _, _, fw, bw, _ = oracle_layer(T, h, F, heads, d1, d2, chunks, seed)
    b = atp.alloc_layer_rank(d1, d2, rank, T, h, F, "cuda:0", seed)
    call = atp.LayerCall(mesh, [b], T, h, F, heads, chunks, True)
    call()
    torch.cuda.synchronize()
    snap = {k: b[k].clone() for k in ("z", "dx", "dw1", "dwqkv", "db1")}
    call()  # a repeated call gives the same bits
    torch.cuda.synchronize()
    worst = 0.0
    for k, ok in list(FWD_MAP.items()) + list(BWD_MAP.items()):
        src = fw if k in FWD_MAP else bw
        got = to_np(b[k])
        assert np.isfinite(got).all(), k
        e = rel(got, src[ok][rank])
        assert e <= 2e-2, (k, e)
        worst = max(worst, e)
    for k, v in snap.items():
        assert torch.equal(b[k], v), k
    if graph:  # CUDA-graph capture of the step (NCCL collectives as graph nodes), replayed twice
        st = torch.cuda.Stream()
        g = atp.Graph.capture(mesh, call, st)
        try:
            for _ in range(2):
                for k in snap:
                    b[k].fill_(float("nan"))
                g(st)
                st.synchronize()
                for k, v in snap.items():
                    assert torch.equal(b[k], v), ("graph replay", k)
        finally:
            g.destroy()
    # replicas: digests of the tensors replicated over each dim must agree in the group
    return worst, {k: float(b[k].double().sum().item()) for k in ("qkv", "u", "db1", "y1", "z", "dx", "db2")}


def _gpt(atp, mesh, d1, d2, rank, chunks, seed):
    import numpy as np
    import torch

    from gpu_util import rel
    from test_gpu_gpt import NAMES, _expected, _oracle

    T, h, F, heads, seq = 512, 1024, 2048, 8, 256
    _, fw, bw = _oracle(T, h, F, heads, seq, seed)
    b = atp.alloc_gpt_rank(d1, d2, rank, T, h, F, heads, "cuda:0", seed)
    atp.GptCall(mesh, [b], T, h, F, heads, seq, chunks, True)()
    torch.cuda.synchronize()
    worst = 0.0
    for k in NAMES:
        got = b[k].detach().float().cpu().numpy().astype(np.float64)
        ref = _expected(k, fw, bw, d1, d2, rank, h, F)
        e = rel(got, ref)
        assert e <= 2e-2, (k, e)
        worst = max(worst, e)
    return worst


def _probe_search(atp, mesh, world):
    """S1 -> S2 ("run S" of SURVEY §8(d)): atp_probe_hcm on the world mesh, its
    HCM written as SPEC's topology document plus the calibration
    table, read back, and ranked by libatp's atp_search and by the oracle's
    search on the SAME parsed numbers: rankings and doubles must agree bit for
    bit, with and without the calibration."""
    import json

    import torch
    from oracle import costmodel as cm

    scratch = torch.empty((4 << 20) + 64, dtype=torch.uint8, device="cuda:0")
    layers, matrix, calib = atp.atp_probe_hcm(mesh, scratch, msg_bytes=(1 << 20, 4 << 20), calib_bytes=1 << 20,
                                              iters=3)
    doc = json.dumps({"name": f"probe-{world}", "layers": [{"ranks": l.ranks, "p2p_gbps": l.p2p_gbps,
                                                            "group_gbps": l.group_gbps} for l in layers],
                      "calibration": [[d1, d2, b1, b2] for (d1, d2), (b1, b2) in sorted(calib.items())]})
    d = json.loads(doc)
    lay = [atp.HcmLayer(l["ranks"], l["p2p_gbps"], l["group_gbps"]) for l in d["layers"]]
    cal = {(c[0], c[1]): (c[2], c[3]) for c in d["calibration"]}
    hcm = cm.Hcm([cm.HcmLayer(l["ranks"], l["p2p_gbps"], l["group_gbps"]) for l in d["layers"]])
    assert hcm.n_devices == world and len(matrix) == world
    assert all(matrix[i][j] > 0 for i in range(world) for j in range(world) if i != j)
    n_cmp = 0
    for h, heads in ((4096, 32), (5120, 40), (12288, 96)):
        m = cm.Model(L=1, b=4, s=2048, h=h, a=heads)
        for c in (None, cal):
            lib_plan = atp.atp_search(lay, 1, 4, 2048, h, heads, 2, calibration=c)
            o = cm.search(hcm, m, c)
            assert [(r["d1"], r["d2"]) for r in lib_plan["ranked"]] == [(r.d1, r.d2) for r in o.ranked]
            for a_, b_ in zip(lib_plan["ranked"], o.ranked):
                assert a_["t_comm"] == b_.t_comm and a_["t_f"] == list(b_.t), (a_, b_)
            assert lib_plan["chosen"] == (o.chosen.d1, o.chosen.d2)
            n_cmp += 1
    return 0.0, {"plans_compared": n_cmp, "group_gbps": layers[0].group_gbps, "n_calib": len(cal)}


def worker(rank: int, world: int, port: int, jobs: list, results) -> None:
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["NCCL_HOSTID"] = f"atp-shared-gpu-rank{rank}"  # defeat the duplicate-GPU check
    os.environ.setdefault("NCCL_SOCKET_IFNAME", "lo")
    os.environ.setdefault("NCCL_IB_DISABLE", "1")
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    out = {}
    try:
        import torch
        import torch.distributed as dist

        import paper_2301_08658_b200 as atp

        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)  # host-side plumbing only
        for job in jobs:
            kind, d1, d2, chunks, opts = job
            uid = atp.atp_get_unique_id() if rank == 0 else bytes(128)
            obj = [uid]
            dist.broadcast_object_list(obj, src=0)
            mesh = atp.Mesh.distributed(d1, d2, rank, obj[0], 0)
            try:
                if opts.get("gemm_ctas"):
                    mesh.set_gemm_ctas(opts["gemm_ctas"])
                if opts.get("gated"):
                    mesh.set_gating(True)
                if opts.get("fused"):
                    mesh.enable_fused_ar(opts["fused"])  # CUDA IPC peer buffers, opened across processes
                if kind == "probe":
                    worst, dig = _probe_search(atp, mesh, world)
                elif kind == "layer":
                    worst, dig = _layer(atp, mesh, d1, d2, rank, chunks, 43, bool(opts.get("graph")))
                else:
                    worst, dig = _gpt(atp, mesh, d1, d2, rank, chunks, 47), {}
            finally:
                mesh.destroy()
            digs = [None] * world
            dist.all_gather_object(digs, dig)
            out[str(job[:4])] = {"worst": worst, "digests": digs}
        dist.destroy_process_group()
    except BaseException as e:  # noqa: BLE001
        out["error"] = f"{type(e).__name__}: {e}\n{traceback.format_exc()}"
    results[rank] = out
