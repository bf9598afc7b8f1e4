"""Predicted N-GPU step time per (mesh, chunks) — a MODEL, not a measurement.

Compute side: measured on one GPU by running rank 0's schedule with the
collectives elided (scripts/emulate_mesh.py output, JSON lines).  Communication
side: each stage's executed all-reduce bytes (atp_comm_volume, reading G4) at a
bus bandwidth (default 725 GB/s: the 8-rank NCCL all-reduce measured on this
pool, /opt/skills/guides/B200_PROFILING.md).  Per-stage compute is the
measured total split in proportion to the stage's GEMM FLOPs; the stages are
then run through atp_overlap_estimate (signalled schedule: chunk k's all-reduce
overlaps the GEMM's later chunks and the dW GEMM).

    python scripts/predict_multi_gpu.py profiles/r01_emulate_per_rank_v2_signalled.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def stages_for(h, d1, d2, T, F, t_compute_ms, busbw_gbs):
    import paper_2301_08658_b200 as atp

    hc, h1, q1, F1 = h // d2, h // d1, 3 * h // d1, F // d1
    # (name, gemm flops, dW flops, reducing dim, all-reduce elements per rank)
    fl = lambda m, n, k: 2.0 * m * n * k
    st = [
        ("qkv", fl(T, q1, hc), 0.0, 2, T * q1), ("out", fl(T, hc, h1), 0.0, 1, T * hc),
        ("fc1", fl(T, F1, hc), 0.0, 2, T * F1), ("fc2", fl(T, hc, F1), 0.0, 1, T * hc),
        ("fc2_b", fl(T, F1, hc), fl(F1, hc, T), 2, T * F1), ("fc1_b", fl(T, hc, F1), fl(hc, F1, T), 1, T * hc),
        ("out_b", fl(T, h1, hc), fl(h1, hc, T), 2, T * h1), ("qkv_b", fl(T, hc, q1), fl(hc, q1, T), 1, T * hc),
    ]
    tot = sum(s[1] + s[2] for s in st)
    out = []
    for name, g, w, dim, elems in st:
        p = d1 if dim == 1 else d2
        comm = (2.0 * (p - 1) / p * elems * 2) / (busbw_gbs * 1e9) * 1e3 if p > 1 else 0.0
        out.append((t_compute_ms * g / tot, t_compute_ms * w / tot, comm))
    return out


def main():
    import paper_2301_08658_b200 as atp

    path = sys.argv[1]
    busbw = float(sys.argv[2]) if len(sys.argv) > 2 else 725.0
    try:
        pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                         "MEASURED_PEAKS.json")))
        burst, sustained = pk["bf16_tflops"], pk["bf16_tflops_sustained"]
    except (OSError, KeyError, ValueError):
        burst, sustained = 1590.0, 1400.0  # B200_PROFILING.md fallback
    T = 8192
    for line in open(path):
        r = json.loads(line)
        h, (d1, d2), c = r["h"], r["mesh"], r["chunks"]
        F = 4 * h
        st = stages_for(h, d1, d2, T, F, r["ms_compute_per_rank"], busbw)
        mk, ex = atp.atp_overlap_estimate(st, c, "signalled")
        comm = sum(s[2] for s in st)
        fl = 72.0 * T * h * h / (d1 * d2)
        nvl = comm * busbw / 900.0  # the same ring bytes at NVLink's 900 GB/s per direction
        roof = {  # ms: max(tensor time, NVLink time) -- SURVEY §8(d)'s definition, three tensor peaks
            "survey_2.25PF": max(fl / 2.25e12, nvl), "burst": max(fl / (burst * 1e9), nvl),
            "sustained": max(fl / (sustained * 1e9), nvl)}
        print(json.dumps({"cfg": r["cfg"], "h": h, "mesh": [d1, d2], "chunks": c,
                          "compute_ms": r["ms_compute_per_rank"], "comm_ms": round(comm, 4),
                          "predicted_ms": round(mk, 4), "predicted_exposed_ms": round(ex, 4),
                          "predicted_exposed_share": round(ex / mk, 3),
                          "predicted_roofline_frac": {k: round(v / mk, 3) for k, v in roof.items()},
                          "model": f"overlap model, busBW {busbw} GB/s"}))


if __name__ == "__main__":
    main()
