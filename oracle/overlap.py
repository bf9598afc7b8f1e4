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
