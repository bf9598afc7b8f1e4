"""ATP cost model and search — PAPER.md §3.3-§3.5 (Eq. 2, 3, 4) and §5.4.

Bandwidths are GB/s per direction (reading G26).  ``None`` is the NoComm value
of a size-1 mesh dimension (Eq. 4 divides by d-1 = 0, reading G7).

Canonical evaluation order (the C++ search reproduces these
doubles bit for bit, so only this exact order may be used):
    Bk  = (dk * B'k) / (2.0 * (dk - 1))                        Eq. 4
    t1  = (3h) / (d1 * B2 * 1e9)    t2 = h / (d2 * B1 * 1e9)   Eq. 2
    t3  = (4h) / (d1 * B2 * 1e9)    t4 = h / (d2 * B1 * 1e9)
    T   = (2 L b s bytes) * (((t1 + t2) + t3) + t4)
"""
from __future__ import annotations

from dataclasses import dataclass, field

from .mesh import enumerate_meshes


# ------------------------------------------------------------------ HCM (§3.4)
@dataclass
class HcmLayer:
    """One layer of the hierarchical communication matrix: R_j ranks,
    the P2P bandwidth between two layer-j ranks and each rank's group bandwidth."""
    ranks: int
    p2p_gbps: float
    group_gbps: float


@dataclass
class Hcm:
    layers: list  # outermost first ("layers 1 to i" for mesh dim 1)
    name: str = ""

    @property
    def n_devices(self) -> int:
        n = 1
        for l in self.layers:
            n *= l.ranks
        return n


@dataclass
class Model:
    """ModelConfig (Table 2; b=4, s=2048, FP16 by default)."""
    L: int = 1
    b: int = 4
    s: int = 2048
    h: int = 4096
    a: int = 32
    bytes_per_elem: int = 2


class Misaligned(ValueError):
    pass


def dim_spans(hcm: Hcm, d1: int, d2: int):
    """How many layer-j ranks each mesh dimension spans (reading G5).

    Mesh dim 2 is innermost (rank = i1*d2 + i2), so it occupies the innermost
    layers: whole layers first, then an even divisor of the next layer.
    Returns (k1, k2): per-layer participant counts (1 = layer not spanned).
    """
    if d1 * d2 != hcm.n_devices:
        raise ValueError("mesh size != HCM device count")
    L = len(hcm.layers)
    k2 = [1] * L
    rem = d2
    for j in range(L - 1, -1, -1):
        Rj = hcm.layers[j].ranks
        if rem == 1:
            break
        if rem >= Rj:
            if rem % Rj:
                raise Misaligned(f"d2={d2} does not align with layer {j + 1}")
            k2[j] = Rj
            rem //= Rj
        else:
            if Rj % rem:
                raise Misaligned(f"d2={d2} does not evenly split layer {j + 1}")
            k2[j] = rem
            rem = 1
    k1 = [hcm.layers[j].ranks // k2[j] for j in range(L)]
    return k1, k2


def effective_bandwidths(hcm: Hcm, d1: int, d2: int):
    """Eq. 3 with the P2P correction and the /d2 sharing (G5, G6).

    For each layer j spanned by a dimension with k_j > 1 participants:
        B'_j = min(GroupBW_j, (k_j - 1) * P2P_j) / share_j
    share_j = min(d2, devices per layer-j rank) for dim 1 ("d2 groups of
    all-reduce share the interconnection bandwidth") and 1 for dim 2.
    B' = min over spanned layers (outermost first); None if d = 1.
    """
    k1, k2 = dim_spans(hcm, d1, d2)
    L = len(hcm.layers)
    per_rank_devices = []
    for j in range(L):
        n = 1
        for jj in range(j + 1, L):
            n *= hcm.layers[jj].ranks
        per_rank_devices.append(n)
    b1 = None
    b2 = None
    for j in range(L):
        lay = hcm.layers[j]
        if k1[j] > 1:
            v = min(lay.group_gbps, (k1[j] - 1) * lay.p2p_gbps) / min(d2, per_rank_devices[j])
            b1 = v if b1 is None else min(b1, v)
        if k2[j] > 1:
            v = min(lay.group_gbps, (k2[j] - 1) * lay.p2p_gbps) / 1
            b2 = v if b2 is None else min(b2, v)
    return (b1 if d1 > 1 else None), (b2 if d2 > 1 else None)


def algo_bandwidth(b_prime, d: int):
    """Eq. 4, Rabenseifner: B = d / (2(d-1)) * B'; NoComm at d = 1."""
    if d == 1 or b_prime is None:
        return None
    return (d * b_prime) / (2.0 * (d - 1))


@dataclass
class CostReport:
    d1: int
    d2: int
    b1p: float | None
    b2p: float | None
    b1: float | None
    b2: float | None
    t: tuple  # (t_f1, t_f2, t_f3, t_f4) in seconds, already x 2Lbs*bytes
    t_comm: float
    calibrated: bool = False


def comm_time(m: Model, d1: int, d2: int, b1, b2):
    """Eq. 2: T = 2Lbs (3h/(d1 B2) + h/(d2 B1) + 4h/(d1 B2) + h/(d2 B1)).

    Bandwidths in GB/s; a None (NoComm) bandwidth contributes 0 (G7).
    Element terms are multiplied by the element size (G3).
    """
    h = float(m.h)
    t1 = (3.0 * h) / (d1 * (b2 * 1e9)) if b2 is not None else 0.0
    t2 = h / (d2 * (b1 * 1e9)) if b1 is not None else 0.0
    t3 = (4.0 * h) / (d1 * (b2 * 1e9)) if b2 is not None else 0.0
    t4 = h / (d2 * (b1 * 1e9)) if b1 is not None else 0.0
    scale = 2.0 * m.L * m.b * m.s * m.bytes_per_elem
    total = scale * (((t1 + t2) + t3) + t4)
    return (scale * t1, scale * t2, scale * t3, scale * t4), total


def closed_form_factor(d1: int, d2: int) -> float:
    """§5.4: T_comm / (2Lbsh/GroupBW) = (14 d2 + 4 d1 - 18) / (d1 d2)."""
    return (14 * d2 + 4 * d1 - 18) / (d1 * d2)


def model_divisible(m: Model, d1: int, d2: int) -> str | None:
    """Shard divisibility of the layer on (d1, d2) (G19)."""
    if m.h % d2:
        return "h % d2 != 0"
    if m.h % d1:
        return "h % d1 != 0"
    if m.a % d1:
        return "heads % d1 != 0"
    if m.h % m.a:
        return "h % heads != 0"
    return None


@dataclass
class Plan:
    ranked: list = field(default_factory=list)   # CostReports, ascending t_comm
    rejected: list = field(default_factory=list)  # (d1, d2, reason)
    chosen: CostReport | None = None


def search(hcm: Hcm, m: Model, calibration: dict | None = None) -> Plan:
    """ATP selection: argmin of T_comm over all 2-D meshes.

    ``calibration`` maps (d1, d2) -> (B1, B2) algorithm bandwidths measured
    (reading G11); it overrides Eq. 3/4 for the meshes it names.
    Ties (exact double equality) go to the larger d1 (G8): candidates are
    scanned by descending d1 and only a strictly smaller time replaces.
    """
    plan = Plan()
    reps = []
    for d1, d2 in enumerate_meshes(hcm.n_devices):
        why = model_divisible(m, d1, d2)
        if why:
            plan.rejected.append((d1, d2, why))
            continue
        cal = calibration.get((d1, d2)) if calibration else None
        if cal is not None:
            b1p = b2p = None
            b1, b2 = cal
            b1 = b1 if d1 > 1 else None
            b2 = b2 if d2 > 1 else None
        else:
            try:
                b1p, b2p = effective_bandwidths(hcm, d1, d2)
            except Misaligned as e:
                plan.rejected.append((d1, d2, str(e)))
                continue
            b1 = algo_bandwidth(b1p, d1)
            b2 = algo_bandwidth(b2p, d2)
        terms, total = comm_time(m, d1, d2, b1, b2)
        reps.append(CostReport(d1, d2, b1p, b2p, b1, b2, terms, total, cal is not None))
    if not reps:
        raise ValueError("no candidate mesh")
    best = None
    for rep in reps:
        if best is None or rep.t_comm < best.t_comm:
            best = rep
    # stable sort keeps descending-d1 order among equal times
    plan.ranked = sorted(reps, key=lambda r: r.t_comm)
    plan.chosen = best
    return plan


# ------------------------------------------------------- communication volume
def comm_volume(d1: int, d2: int, T: int, h: int, chunks: int = 1, F: int | None = None):
    """Executed collective list of one layer fwd+bwd (reading G4).

    One entry per NCCL call per rank: (phase, name, dim, p, elements).
    Size-1 dimensions make no call (G7).  The forward follows Eq. 2's f1..f4
    (P:264); the backward reduces the dX partials on the conjugate dimension
    (P:343): FC2-dX width F/d1 on dim 2, FC1-dX h/d2 on dim 1, Out-dX h/d1 on
    dim 2 (the stand-in core keeps ctx replicated over dim 2, G4/G20), QKV-dX
    h/d2 on dim 1.  Order = the schedule order (block by block, chunk by chunk).
    """
    F = 4 * h if F is None else F
    M = T // chunks
    seq = [
        ("fwd", "qkv", 2, 3 * h // d1), ("fwd", "out", 1, h // d2),
        ("fwd", "fc1", 2, F // d1), ("fwd", "fc2", 1, h // d2),
        ("bwd", "fc2", 2, F // d1), ("bwd", "fc1", 1, h // d2),
        ("bwd", "out", 2, h // d1), ("bwd", "qkv", 1, h // d2),
    ]
    calls = []
    for phase, name, dim, width in seq:
        p = d1 if dim == 1 else d2
        if p == 1:
            continue
        for _ in range(chunks):
            calls.append((phase, name, dim, p, M * width))
    return calls


def ring_bytes_per_gpu(calls, bytes_per_elem: int = 2) -> float:
    """Bytes each GPU sends in ring all-reduces: 2(p-1)/p * elements * bytes."""
    return sum(2.0 * (p - 1) / p * e * bytes_per_elem for (_, _, _, p, e) in calls)


def eq2_elements(d1: int, d2: int, T: int, h: int):
    """Eq. 2's per-rank element counts per layer (fwd+bwd: the 2x of 2Lbs):
    dim 2: 2T(3h+4h)/d1, dim 1: 2T(h+h)/d2; zero on size-1 dimensions."""
    dim2 = 2 * T * 7 * h // d1 if d2 > 1 else 0
    dim1 = 2 * T * 2 * h // d2 if d1 > 1 else 0
    return dim1, dim2


def layer_flops(T: int, h: int) -> int:
    """Hot-path FLOPs of one layer fwd+bwd: 72 T h^2 (fwd 24, bwd 48; G24)."""
    return 72 * T * h * h


def table2_tflops(b: int, s: int, h: int) -> float:
    """Table 2 "#TFLOPs per layer": (72bsh^2 + 12bs^2h) / 2^40 (G23)."""
    return (72 * b * s * h * h + 12 * b * s * s * h) / 2 ** 40


def table2_bparams(h: int) -> float:
    """Table 2 "#billion params per layer": 12 h^2 / (1000 * 2^20) (G23)."""
    return 12 * h * h / (1000 * 2 ** 20)
