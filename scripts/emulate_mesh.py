"""Per-rank compute of the multi-GPU configurations, measured on ONE GPU.

Runs rank 0's schedule of DeviceMesh(d1, d2) (atp_mesh_init_local: collectives
elided) for the BASELINE configs at N=8 and reports the per-rank compute time
and TFLOP/s.  This is the compute side of the 8-GPU step; the communication and
its overlap need the 8 GPUs themselves (bench.py under torchrun).

    python scripts/emulate_mesh.py [--cfg 3,4,5] [--chunks 1,2,4,8] [--steps 20]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CFGS = {3: (4096, 32), 4: (5120, 40), 5: (12288, 96)}


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--cfg", default="3,4,5")
    p.add_argument("--chunks", default="1,2,4,8")
    p.add_argument("--meshes", default="8x1,4x2,2x4,1x8")
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--tokens", type=int, default=8192)
    p.add_argument("--gemm-ctas", type=int, default=132)
    p.add_argument("--gated", action="store_true", help="chunk-gated GEMMs")
    p.add_argument("--layer", default="linear", choices=["linear", "gpt"],
                   help="gpt: the full pre-LN layer (chunks = whole sequences of --seq tokens)")
    p.add_argument("--seq", type=int, default=2048)
    p.add_argument("--fused-ar", action="store_true",
                   help="fused peer-memory all-reduce stages (run against the rank's own buffer)")
    a = p.parse_args()
    import torch
    import paper_2301_08658_b200 as atp

    T = a.tokens
    for cfg in [int(c) for c in a.cfg.split(",")]:
        h, heads = CFGS[cfg]
        F = 4 * h
        for m in a.meshes.split(","):
            d1, d2 = (int(v) for v in m.split("x"))
            if heads % d1 or (a.layer == "gpt" and heads % (d1 * d2)):
                continue
            mesh = atp.Mesh.local(d1, d2, 0)
            mesh.set_gemm_ctas(a.gemm_ctas)  # the N>1 default of bench.py: SMs left for the communication kernels
            mesh.set_gating(a.gated)
            if a.fused_ar:
                mesh.enable_fused_ar(T * max(3 * h // d1, F // d1, h // d2) * 2)
            if a.layer == "gpt":
                bufs = atp.alloc_gpt_rank(d1, d2, 0, T, h, F, heads, "cuda", 2301)
            else:
                bufs = atp.alloc_layer_rank(d1, d2, 0, T, h, F, "cuda", 2301)
            for c in [int(x) for x in a.chunks.split(",")]:
                if a.layer == "gpt":
                    if T % (c * a.seq):
                        continue
                    call = atp.GptCall(mesh, [bufs], T, h, F, heads, a.seq, c, True)
                else:
                    call = atp.LayerCall(mesh, [bufs], T, h, F, heads, c, True)
                for _ in range(3):
                    call()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.steps):
                    call()
                e1.record()
                e1.synchronize()
                ms = e0.elapsed_time(e1) / a.steps
                fl = (72.0 * T * h * h + (7.0 * (a.seq + 1) * T * h if a.layer == "gpt" else 0.0)) / (d1 * d2)
                print(json.dumps({"cfg": cfg, "h": h, "mesh": [d1, d2], "chunks": c, "ms_compute_per_rank": round(ms, 4),
                                  "tflops_per_rank": round(fl / ms / 1e9, 1), "fused_ar": a.fused_ar,
                                  "gated": a.gated, "layer": a.layer}), flush=True)
            del bufs
            mesh.destroy()
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
