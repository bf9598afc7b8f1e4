"""Chunk-overlap timing model — PAPER.md §4.1 (Fig. 7) and §4.2
(P:341-345); SPEC.md's overlap module for the single-block form.

One compute stream and one communication stream (the paper's single
communication channel).  A stage is one linear: compute time `comp`
(the GEMM of all chunks), optional extra compute `dw` that follows it on the
compute stream and does not feed the collective (the dW GEMM of §4.2), and
the all-reduce time `comm` of all chunks.  Chunks split `comp` and `comm`
evenly (c equal chunks).

Two dependency structures between consecutive stages:
  "per_chunk"  Fig. 7 reading G14: chunk k of stage s+1 starts after chunk k's
               all-reduce of stage s (and after the compute stream is free);
  "signalled"  the library's signalled stages: the whole GEMM of stage s+1
               starts after the LAST all-reduce of stage s.
"""
from __future__ import annotations


def simulate_block(t_comp: float, t_comm: float, c: int) -> float:
    """makespan = t_comp/c + (c-1)/c * max(t_comp, t_comm) + t_comm/c."""
    return t_comp / c + (c - 1) / c * max(t_comp, t_comm) + t_comm / c


def simulate(stages, c: int, mode: str = "signalled"):
    """Event simulation; stages = [(comp, dw, comm), ...] in schedule order.

    Returns (makespan, exposed) with exposed = makespan - total compute.
    """
    if c < 1:
        raise ValueError("chunks >= 1")
    if mode not in ("signalled", "per_chunk"):
        raise ValueError(mode)
    t_cmp = 0.0   # compute stream free at
    t_com = 0.0   # comm stream free at
    prev_comm_end = [0.0] * c  # per chunk: end of the previous stage's all-reduce
    total_compute = 0.0
    for comp, dw, comm in stages:
        gk = comp / c
        ak = comm / c
        comp_end = [0.0] * c
        if mode == "signalled":
            start = max(t_cmp, prev_comm_end[c - 1])
            for k in range(c):
                comp_end[k] = start + (k + 1) * gk
            t_cmp = comp_end[c - 1]
        else:
            for k in range(c):
                start = max(t_cmp, prev_comm_end[k])
                comp_end[k] = start + gk
                t_cmp = comp_end[k]
        t_cmp = t_cmp + dw
        for k in range(c):
            if comm > 0.0:
                start = max(t_com, comp_end[k])
                t_com = start + ak
                prev_comm_end[k] = t_com
            else:
                prev_comm_end[k] = comp_end[k]
        total_compute += comp + dw
    makespan = max(t_cmp, t_com)
    return makespan, makespan - total_compute


# ------------------------------------------------------- chunk-count planner
# The paper fixes the chunk count by hand ("2 or 4 is usually enough", P:332;
# Table 3, P:449 shows the best count depends on the interconnect).  The
# planner closes the loop: one measured number, the
# compute-side time of the layer at each candidate chunk count (collectives
# elided), and one probed number, the all-reduce bus bandwidth, are split
# into the layer's eight stages and run through `simulate`.
#
# Stage decomposition (schedule order, reading G36):
#   the compute of stage s is the measured total split in proportion to its
#   GEMM FLOPs 2*M*N*K (the dX GEMM = the stage GEMM; in backward the dW GEMM
#   2*N*K*T is the extra compute that overlaps the stage's all-reduces, §4.2);
#   the communication of stage s is its executed ring all-reduce bytes
#   2(p-1)/p * elements * bytes (costmodel.comm_volume, reading G4) at the bus
#   bandwidth.  Evaluation order is fixed so libatp's atp_plan_chunks produces
#   the same doubles.
def layer_stages(T: int, h: int, F: int, d1: int, d2: int, compute_ms: float, busbw_gbps: float,
                 bytes_per_elem: int = 2):
    """[(comp_ms, dw_ms, comm_ms)] of the 8 linear stages of one layer fwd+bwd."""
    hc, h1, q1, F1 = h // d2, h // d1, 3 * h // d1, F // d1
    # (GEMM N, GEMM K, dW?, reducing mesh dim, all-reduce width per row)
    st = [(q1, hc, False, 2, q1), (hc, h1, False, 1, hc), (F1, hc, False, 2, F1), (hc, F1, False, 1, hc),
          (F1, hc, True, 2, F1), (hc, F1, True, 1, hc), (h1, hc, True, 2, h1), (hc, q1, True, 1, hc)]
    g = [2.0 * T * n * k for (n, k, _, _, _) in st]
    w = [(2.0 * n * k * T if dw else 0.0) for (n, k, dw, _, _) in st]
    tot = 0.0
    for i in range(len(st)):
        tot = tot + (g[i] + w[i])
    out = []
    for i, (_, _, _, dim, width) in enumerate(st):
        p = d1 if dim == 1 else d2
        elems = T * width
        comm = (2.0 * (p - 1) / p * elems * bytes_per_elem) / (busbw_gbps * 1e9) * 1e3 if p > 1 else 0.0
        out.append((compute_ms * g[i] / tot, compute_ms * w[i] / tot, comm))
    return out


def plan_chunks(T: int, h: int, F: int, d1: int, d2: int, compute_ms_by_c: dict, busbw_gbps: float,
                mode: str = "signalled", bytes_per_elem: int = 2):
    """Chunk count with the smallest predicted makespan (ties -> fewer chunks).
    Returns (chosen c, {c: (makespan_ms, exposed_ms)})."""
    pred = {}
    for c in sorted(compute_ms_by_c):
        pred[c] = simulate(layer_stages(T, h, F, d1, d2, compute_ms_by_c[c], busbw_gbps, bytes_per_elem), c, mode)
    best = None
    for c in sorted(pred):
        if best is None or pred[c][0] < pred[best][0]:
            best = c
    return best, pred
