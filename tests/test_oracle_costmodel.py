"""Pins for oracle.costmodel: Eq. 2/3/4, the §5.4 closed form, search, volumes,
Table 2 FLOP/param formulas."""
import json
import os
import random

import pytest

from oracle import costmodel as cm
from oracle import mesh

from conftest import GOLDEN


def hcm_from(layers):
    return cm.Hcm([cm.HcmLayer(l["ranks"], l["p2p_gbps"], l["group_gbps"]) for l in layers])


def flat(n, bw):
    return cm.Hcm([cm.HcmLayer(n, bw, bw)])


def test_eq3_fig9a_anchor_p307():
    g = json.load(open(os.path.join(GOLDEN, "hcm_fig9.json")))
    hcm = hcm_from(g["fig9a"]["layers"])
    assert hcm.n_devices == 16
    b1p, b2p = cm.effective_bandwidths(hcm, 8, 2)
    assert b2p == g["fig9a"]["mesh_8_2"]["B2_prime"]
    assert b1p == g["fig9a"]["mesh_8_2"]["B1_prime"]
    # further readings of Eq. 3 on the same topology (G5): (16,1) and (4,4)
    assert cm.effective_bandwidths(hcm, 16, 1) == (25.0, None)
    assert cm.effective_bandwidths(hcm, 4, 4) == (6.25, 600.0)


def test_eq3_fig9b_torus_equals_groupbw_p488():
    g = json.load(open(os.path.join(GOLDEN, "hcm_fig9.json")))
    hcm = hcm_from(g["fig9b"]["layers"])
    b1p, b2p = cm.effective_bandwidths(hcm, 4, 4)
    assert (b1p, b2p) == (g["fig9b"]["mesh_4_4"]["B1_prime"], g["fig9b"]["mesh_4_4"]["B2_prime"])


def test_eq3_misalignment():
    hcm = cm.Hcm([cm.HcmLayer(4, 25, 25), cm.HcmLayer(4, 200, 600)])
    with pytest.raises(cm.Misaligned):
        cm.effective_bandwidths(cm.Hcm([cm.HcmLayer(2, 1, 1), cm.HcmLayer(3, 1, 1)]), 3, 2)
    with pytest.raises(ValueError):
        cm.effective_bandwidths(hcm, 4, 2)


def test_eq4_rabenseifner():
    # B = d/(2(d-1)) B'
    assert cm.algo_bandwidth(200.0, 2) == 200.0
    assert cm.algo_bandwidth(600.0, 4) == 400.0
    assert cm.algo_bandwidth(123.0, 1) is None
    for d in range(2, 200):
        b = cm.algo_bandwidth(1.0, d)
        assert 0.5 < b <= 1.0


def test_megatron_cost_p151():
    # Megatron TP costs 4Lbsh/B per step (q is a typo for h, G2); Eq. 2 at (N,1)
    m = cm.Model(L=3, b=4, s=2048, h=4096, bytes_per_elem=1)
    for n in (2, 4, 8):
        _, t = cm.comm_time(m, n, 1, 100.0, None)
        assert t == pytest.approx(4 * m.L * m.b * m.s * m.h / (100.0 * 1e9), rel=1e-14)
    _, t = cm.comm_time(m, 1, 1, None, None)
    assert t == 0.0


def test_calibration_anchor_p482():
    g = json.load(open(os.path.join(GOLDEN, "calibration_p482.json")))
    m = cm.Model()
    cal = {tuple(e["mesh"]): (e["B1"], e["B2"]) for e in g["calibration"]}
    _, t24 = cm.comm_time(m, 2, 4, *cal[(2, 4)])
    _, t81 = cm.comm_time(m, 8, 1, *cal[(8, 1)])
    ratio = t24 / t81
    assert abs(ratio - (1 - g["reduction_percent"] / 100)) <= g["ratio_tolerance"]
    # the planner restricted to the calibrated meshes picks ATP-4 = (2,4)
    hcm = flat(8, 1.0)
    plan = cm.search(hcm, m, cal)
    chosen = min((r for r in plan.ranked if r.calibrated), key=lambda r: r.t_comm)
    assert (chosen.d1, chosen.d2) == (2, 4)


@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64])
def test_pipeline_equals_closed_form_p490(n):
    # single-layer topology, B1' = B2' = GroupBW
    bw = 50.0
    m = cm.Model(L=2, b=4, s=2048, h=4096, bytes_per_elem=2)
    delta = 2 * m.L * m.b * m.s * m.h * m.bytes_per_elem / (bw * 1e9)
    for d1, d2 in mesh.enumerate_meshes(n):
        b1p, b2p = cm.effective_bandwidths(flat(n, bw), d1, d2)
        _, t = cm.comm_time(m, d1, d2, cm.algo_bandwidth(b1p, d1), cm.algo_bandwidth(b2p, d2))
        want = delta * cm.closed_form_factor(d1, d2)
        assert abs(t - want) <= 1e-12 * max(want, 1e-30), (d1, d2, t, want)


def test_search_fully_connected_p478():
    m = cm.Model()
    # ATP-1 when the number of devices is less than 8, ATP-2 at 16
    for n in (2, 4):
        assert (cm.search(flat(n, 600.0), m).chosen.d1, cm.search(flat(n, 600.0), m).chosen.d2) == (n, 1)
    c16 = cm.search(flat(16, 600.0), cm.Model(a=32)).chosen
    assert (c16.d1, c16.d2) == (8, 2)
    assert cm.closed_form_factor(8, 2) == 2.625
    # N=8: the formula gives (4,2)=3.25 < (8,1)=3.5 (reading G9: follow the formula)
    c8 = cm.search(flat(8, 900.0), m).chosen
    assert (c8.d1, c8.d2) == (4, 2)
    assert [cm.closed_form_factor(*mm) for mm in [(8, 1), (4, 2), (2, 4), (1, 8)]] == [3.5, 3.25, 5.75, 12.25]


def test_fig12_trends_p492():
    # cost increases with scaling in ATP-1, decreases in ATP-2 and ATP-4
    f1 = [cm.closed_form_factor(n, 1) for n in (2, 4, 8, 16, 32, 64)]
    f2 = [cm.closed_form_factor(n // 2, 2) for n in (4, 8, 16, 32, 64)]
    f4 = [cm.closed_form_factor(n // 4, 4) for n in (8, 16, 32, 64)]
    assert all(a < b for a, b in zip(f1, f1[1:]))
    assert all(a > b for a, b in zip(f2, f2[1:]))
    assert all(a > b for a, b in zip(f4, f4[1:]))
    # N = 16 row of the sweep: ATP-1/2/4/8 = 3.75/2.625/3.375/6.375
    assert [cm.closed_form_factor(16 // i, i) for i in (1, 2, 4, 8)] == [3.75, 2.625, 3.375, 6.375]


def test_tcomm_decreases_with_mesh_size_p268():
    m = cm.Model()
    for d1 in (1, 2, 4):
        for d2 in (1, 2, 4):
            _, t = cm.comm_time(m, d1, d2, 10.0, 10.0)
            _, t_more1 = cm.comm_time(m, 2 * d1, d2, 10.0, 10.0)
            _, t_more2 = cm.comm_time(m, d1, 2 * d2, 10.0, 10.0)
            if d1 * d2 > 1 or True:
                assert t_more1 <= t and t_more2 <= t


def test_scale_invariance_and_determinism():
    rnd = random.Random(5)
    m = cm.Model(a=64)
    for _ in range(100):
        layers = [cm.HcmLayer(rnd.choice([2, 4]), rnd.choice([12.5, 25.0, 50.0, 200.0]),
                              rnd.choice([25.0, 50.0, 100.0, 600.0])) for _ in range(rnd.choice([1, 2, 3]))]
        hcm = cm.Hcm(layers)
        alpha = rnd.choice([0.25, 0.5, 2.0, 4.0, 8.0])
        hcm2 = cm.Hcm([cm.HcmLayer(l.ranks, l.p2p_gbps * alpha, l.group_gbps * alpha) for l in layers])
        p1, p2 = cm.search(hcm, m), cm.search(hcm2, m)
        assert (p1.chosen.d1, p1.chosen.d2) == (p2.chosen.d1, p2.chosen.d2)
        assert repr(cm.search(hcm, m)) == repr(p1)
        for r in p1.ranked:
            assert p1.chosen.t_comm <= r.t_comm


TIE_CAL = {(4, 1): (64.0, None), (2, 2): (64.0, 224.0), (1, 4): (1e-3, 1e-3)}


def test_tie_break_larger_d1():
    """G8 (P:316 is silent): exact double ties go to the larger d1.

    The calibrated bandwidths are chosen so the two Eq. 2 sums tie bit for bit:
    (4,1) with B1 = 64 GB/s gives 2Lbs*2h/B1; (2,2) with B1 = 64, B2 = 224 =
    3.5*64 gives 2Lbs(3h/(2B2) + h/(2B1) + 4h/(2B2) + h/(2B1)) = the same value
    mathematically, and (with h = 4096, scale 2Lbs*2 = 2^15, B1 doubled exactly)
    the same double (asserted, not assumed).  A strictly faster (2,2) must win.
    """
    m = cm.Model()
    hcm = flat(4, 1e9)
    _, t41 = cm.comm_time(m, 4, 1, 64.0, None)
    _, t22 = cm.comm_time(m, 2, 2, 64.0, 224.0)
    assert t22 == t41  # an exact tie in float64
    plan = cm.search(hcm, m, TIE_CAL)
    assert (plan.chosen.d1, plan.chosen.d2) == (4, 1)
    assert [(r.d1, r.d2) for r in plan.ranked][:2] == [(4, 1), (2, 2)]
    # break the tie by a hair in (2,2)'s favour: it must now be chosen
    faster = dict(TIE_CAL)
    faster[(2, 2)] = (64.0, 225.0)
    _, t22f = cm.comm_time(m, 2, 2, 64.0, 225.0)
    assert t22f < t41
    plan = cm.search(hcm, m, faster)
    assert (plan.chosen.d1, plan.chosen.d2) == (2, 2)


def test_table2_formulas_p386():
    g = json.load(open(os.path.join(GOLDEN, "table2.json")))
    for row in g["rows"]:
        assert round(cm.table2_tflops(g["b"], g["s"], row["h"]), 3) == row["tflops"]
        assert round(cm.table2_bparams(row["h"]), 3) == row["bparams"]


@pytest.mark.parametrize("d1,d2", [(8, 1), (4, 2), (2, 4), (1, 8), (2, 2), (1, 1)])
@pytest.mark.parametrize("chunks", [1, 2, 4, 8])
def test_comm_volume_closed_forms(d1, d2, chunks):
    T, h = 8192, 4096
    calls = cm.comm_volume(d1, d2, T, h, chunks)
    dim2 = sum(e for (_, _, dim, _, e) in calls if dim == 2)
    dim1 = sum(e for (_, _, dim, _, e) in calls if dim == 1)
    # executed: 12 T h / d1 on dim 2 (fwd 3h+4h, bwd 4h+h) and 4 T h / d2 on dim 1 (G4)
    assert dim2 == (12 * T * h // d1 if d2 > 1 else 0)
    assert dim1 == (4 * T * h // d2 if d1 > 1 else 0)
    e1, e2 = cm.eq2_elements(d1, d2, T, h)
    assert e1 == dim1 and (e2 == 14 * T * h // d1 if d2 > 1 else e2 == 0)
    n_calls = (4 * chunks if d1 > 1 else 0) + (4 * chunks if d2 > 1 else 0)
    assert len(calls) == n_calls
    # ring bytes per GPU: 2B * T h [24(d2-1) + 8(d1-1)] / (d1 d2)
    want = 2 * T * h * (24 * (d2 - 1) + 8 * (d1 - 1)) / (d1 * d2)
    assert cm.ring_bytes_per_gpu(calls) == pytest.approx(want, rel=1e-12)


def test_layer_flops():
    # 72 T h^2 = the Table-2 formula minus the attention-core term 12 b s^2 h (G24)
    b, s, h = 4, 2048, 4096
    assert cm.layer_flops(b * s, h) == 72 * b * s * h * h
    assert abs(cm.table2_tflops(b, s, h) * 2 ** 40 - cm.layer_flops(b * s, h) - 12 * b * s * s * h) < 1
