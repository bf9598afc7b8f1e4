"""Device timeline of one layer step (atp_profile_trace): every GEMM /
elementwise / collective launch with its stream and start / end on the device.

    python scripts/trace_step.py --h 5120 --mesh 4x2 --chunks 1,4 [--local] [--gemm-ctas 132]

With --local (default) the mesh is rank 0 of DeviceMesh(d1, d2) with the
collectives elided (atp_mesh_init_local), i.e. the per-rank compute of the
multi-GPU step on one GPU.  Prints the ops and, per stream, busy time and the
compute stream's idle gaps."""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

EW = ["gelu", "dgelu", "add", "core_fwd", "core_bwd", "colsum", "ln_stats", "ln_apply", "ln_bwd_stats",
      "ln_bwd_apply", "ln_param_grad", "pack", "unpack", "attn_fwd", "attn_bwd", "ln_fwd", "ln_bwd"]
EPI = ["bf16", "f32", "resid", "bias_gelu", "dgelu"]
KIND = {0: "gemm", 1: "ew", 2: "coll", 4: "fused_ar"}


def name(r):
    if r.kind == 0:
        return f"gemm[{EPI[r.sub]}]"
    if r.kind == 1:
        return EW[r.sub] if r.sub < len(EW) else f"ew{r.sub}"
    return KIND.get(r.kind, str(r.kind)) + f"[{r.sub}]"


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--h", type=int, default=5120)
    p.add_argument("--heads", type=int, default=40)
    p.add_argument("--T", type=int, default=8192)
    p.add_argument("--mesh", default="4x2")
    p.add_argument("--chunks", default="1,4")
    p.add_argument("--gemm-ctas", type=int, default=132)
    p.add_argument("--layer", default="linear", choices=["linear", "gpt"])
    p.add_argument("--seq", type=int, default=2048)
    p.add_argument("--ops", action="store_true", help="print every op")
    p.add_argument("--fused-ar", action="store_true",
                   help="fused GEMM -> reduce-scatter -> all-gather stages (dry run: every peer is this rank)")
    a = p.parse_args()
    import torch
    import paper_2301_08658_b200 as atp
    from paper_2301_08658_b200 import _abi

    d1, d2 = (int(v) for v in a.mesh.split("x"))
    h, T, F = a.h, a.T, 4 * a.h
    mesh = atp.Mesh.local(d1, d2, 0) if d1 * d2 > 1 else atp.Mesh.virtual(1, 1)
    mesh.set_gemm_ctas(a.gemm_ctas if d1 * d2 > 1 else 0)
    if a.fused_ar:
        mesh.enable_fused_ar(T * max(3 * h // d1, 4 * h // d1, h // d2) * 2)
    if a.layer == "gpt":
        bufs = atp.alloc_gpt_rank(d1, d2, 0, T, h, F, a.heads, "cuda", 2301)
    else:
        bufs = atp.alloc_layer_rank(d1, d2, 0, T, h, F, "cuda", 2301)
    lib = _abi.lib()
    for c in [int(x) for x in a.chunks.split(",")]:
        if a.layer == "gpt":
            call = atp.GptCall(mesh, [bufs], T, h, F, a.heads, a.seq, c, True)
        else:
            call = atp.LayerCall(mesh, [bufs], T, h, F, a.heads, c, True)
        for _ in range(5):
            call()
        torch.cuda.synchronize()
        # host enqueue cost per call (schedule build + launches), no device sync inside
        import time
        t0 = time.perf_counter()
        for _ in range(20):
            call()
        host_us = (time.perf_counter() - t0) / 20 * 1e6
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            call()
        e1.record()
        e1.synchronize()
        dev_ms = e0.elapsed_time(e1) / 20
        _abi.check(lib.atp_profile_begin(mesh.handle))
        call()
        torch.cuda.synchronize()
        cap = 4096
        recs = (_abi.TraceRec * cap)()
        n = C.c_int()
        _abi.check(lib.atp_profile_trace(mesh.handle, recs, cap, C.byref(n)))
        prof = _abi.Profile()
        _abi.check(lib.atp_profile_end(mesh.handle, C.byref(prof)))
        rs = list(recs[: n.value])
        end = max(r.t1_ms for r in rs)
        busy = {}
        for r in rs:
            busy[r.stream] = busy.get(r.stream, 0.0) + (r.t1_ms - r.t0_ms)
        comp = sorted((r for r in rs if r.stream == 0), key=lambda r: r.t0_ms)
        gaps, t = [], 0.0
        for r in comp:
            if r.t0_ms - t > 0.002:
                gaps.append((round(t, 4), round(r.t0_ms - t, 4), name(r)))
            t = max(t, r.t1_ms)
        by = {}
        for r in rs:
            k = (r.stream, name(r))
            by.setdefault(k, [0, 0.0])
            by[k][0] += 1
            by[k][1] += r.t1_ms - r.t0_ms
        print(json.dumps({"mesh": [d1, d2], "h": h, "chunks": c, "host_enqueue_us_per_call": round(host_us, 1),
                          "device_ms_per_call": round(dev_ms, 4), "span_ms": round(end, 4),
                          "busy_ms_per_stream": {k: round(v, 4) for k, v in busy.items()},
                          "compute_idle_ms": round(sum(g[1] for g in gaps), 4),
                          "by_op": {f"s{k[0]}:{k[1]}": [v[0], round(v[1], 4)] for k, v in sorted(by.items())},
                          "largest_compute_gaps": sorted(gaps, key=lambda g: -g[1])[:8]}), flush=True)
        if a.ops:
            for r in rs:
                print(f"  s{r.stream} {name(r):16s} {r.t0_ms:8.4f} {r.t1_ms:8.4f} {1e3 * (r.t1_ms - r.t0_ms):8.1f} us")
    mesh.destroy()


if __name__ == "__main__":
    main()
