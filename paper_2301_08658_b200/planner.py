"""Chunk-count planner: predicted step time of the chunk
pipeline for a mesh, from a measured compute-side time and a bus bandwidth,
through libatp's overlap model (atp_overlap_estimate, §4.1/§4.2).

Per-stage compute is the measured total split in proportion to the stage's
GEMM FLOPs (dX GEMM = the stage GEMM, dW GEMM = the extra compute overlapping
the stage's all-reduces); per-stage communication is the executed ring bytes
of its all-reduces (atp_comm_volume, reading G4) at `busbw_gbs`.
"""
from __future__ import annotations


def layer_stages(T: int, h: int, F: int, d1: int, d2: int, compute_ms: float, busbw_gbs: float):
    """[(comp_ms, dw_ms, comm_ms)] for the 8 stages of one layer fwd+bwd (schedule order)."""
    hc, h1, q1, F1 = h // d2, h // d1, 3 * h // d1, F // d1
    fl = lambda m, n, k: 2.0 * m * n * k
    st = [  # (gemm flops, dW flops, reducing dim, all-reduce elements per rank)
        (fl(T, q1, hc), 0.0, 2, T * q1), (fl(T, hc, h1), 0.0, 1, T * hc),
        (fl(T, F1, hc), 0.0, 2, T * F1), (fl(T, hc, F1), 0.0, 1, T * hc),
        (fl(T, F1, hc), fl(F1, hc, T), 2, T * F1), (fl(T, hc, F1), fl(hc, F1, T), 1, T * hc),
        (fl(T, h1, hc), fl(h1, hc, T), 2, T * h1), (fl(T, hc, q1), fl(hc, q1, T), 1, T * hc),
    ]
    tot = sum(g + w for g, w, _, _ in st)
    out = []
    for g, w, dim, elems in st:
        p = d1 if dim == 1 else d2
        comm = (2.0 * (p - 1) / p * elems * 2) / (busbw_gbs * 1e9) * 1e3 if p > 1 else 0.0
        out.append((compute_ms * g / tot, compute_ms * w / tot, comm))
    return out


def predict_step(T, h, F, d1, d2, compute_ms, busbw_gbs, chunks, mode="signalled"):
    """(predicted step ms, predicted exposed-communication ms)."""
    from .api import atp_overlap_estimate

    return atp_overlap_estimate(layer_stages(T, h, F, d1, d2, compute_ms, busbw_gbs), chunks, mode)


def choose_chunks(T, h, F, d1, d2, compute_ms_by_c: dict, busbw_gbs: float):
    """Chunk count with the smallest predicted step; ties -> fewer chunks.
    Returns (chosen c, {c: predicted ms})."""
    pred = {c: predict_step(T, h, F, d1, d2, t, busbw_gbs, c)[0] for c, t in sorted(compute_ms_by_c.items())}
    best = min(pred, key=lambda c: (pred[c], c))
    return best, pred
