"""CPU-side tests of the C-ABI library (no GPU needed): it loads, exports every
symbol include/atp.h declares, and its host-only entry points (mesh groups,
cost model, search, communication volume) equal the oracle exactly."""
import ctypes
import os
import random
import re

import pytest

from conftest import ROOT

import paper_2301_08658_b200 as atp
from paper_2301_08658_b200 import _abi, build
from oracle import costmodel as cm
from oracle import mesh as omesh


@pytest.fixture(scope="module", autouse=True)
def built():
    build.build()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "atp.h")).read()
    return sorted(set(re.findall(r"^(?:atp_status|const char\*|size_t)\s+(atp_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    names = declared_symbols()
    assert len(names) >= 20
    L = ctypes.CDLL(_abi.LIB_PATH)
    for n in names:
        assert hasattr(L, n), n
    assert set(names) == set(_abi.SIGNATURES), set(names) ^ set(_abi.SIGNATURES)
    assert _abi.lib().atp_version().decode() == "0.1.0"


@pytest.mark.parametrize("d1,d2", [(1, 1), (2, 2), (4, 2), (2, 4), (8, 1), (1, 8), (3, 5)])
def test_mesh_groups_match_oracle(d1, d2):
    for dim in (1, 2):
        assert atp.atp_mesh_groups(d1, d2, dim) == omesh.groups(d1, d2, dim)
    with pytest.raises(atp.AtpError):
        atp.atp_mesh_groups(2, 2, 3)


def _oracle_plan(layers, m, cal=None):
    return cm.search(cm.Hcm([cm.HcmLayer(l.ranks, l.p2p_gbps, l.group_gbps) for l in layers]), m, cal)


def _same_plan(lib_plan, o):
    assert len(lib_plan["ranked"]) == len(o.ranked)
    for a, b in zip(lib_plan["ranked"], o.ranked):
        assert (a["d1"], a["d2"]) == (b.d1, b.d2)
        assert a["t_comm"] == b.t_comm  # bit-exact
        assert a["t_f"] == list(b.t)
        assert a["b1"] == (b.b1 or 0.0) and a["b2"] == (b.b2 or 0.0)
    assert lib_plan["chosen"] == (o.chosen.d1, o.chosen.d2)


def test_search_fig9a_and_flat_bit_exact():
    layers = [atp.HcmLayer(4, 25.0, 25.0), atp.HcmLayer(4, 200.0, 600.0)]
    assert atp.atp_effective_bandwidth(layers, 8, 2) == (12.5, 200.0)
    m = cm.Model(L=1, b=4, s=2048, h=4096, a=32)
    _same_plan(atp.atp_search(layers, 1, 4, 2048, 4096, 32, 2), _oracle_plan(layers, m))
    flat8 = [atp.HcmLayer(8, 900.0, 900.0)]
    p = atp.atp_search(flat8, 1, 4, 2048, 5120, 40, 2)
    assert p["chosen"] == (4, 2)
    _same_plan(p, _oracle_plan(flat8, cm.Model(h=5120, a=40)))


def test_search_random_hcms_bit_exact():
    rnd = random.Random(1234)
    for _ in range(300):
        layers = [atp.HcmLayer(rnd.choice([1, 2, 3, 4, 8]), rnd.choice([12.5, 25.0, 50.0, 100.0, 200.0, 300.0, 777.7]),
                               rnd.choice([25.0, 50.0, 100.0, 600.0, 900.0, 1.2345])) for _ in range(rnd.choice([1, 2, 3]))]
        n = 1
        for l in layers:
            n *= l.ranks
        h = rnd.choice([2048, 4096, 5120, 12288])
        heads = rnd.choice([16, 32, 40, 96])
        if h % heads:
            continue
        m = cm.Model(L=rnd.choice([1, 24]), b=4, s=2048, h=h, a=heads)
        try:
            o = _oracle_plan(layers, m)
        except ValueError:
            with pytest.raises(atp.AtpError):
                atp.atp_search(layers, m.L, m.b, m.s, h, heads, 2)
            continue
        _same_plan(atp.atp_search(layers, m.L, m.b, m.s, h, heads, 2), o)


def test_search_calibration_p482():
    cal = {(2, 4): (1.20, 4.95), (8, 1): (0.97, None)}
    layers = [atp.HcmLayer(8, 1e3, 1e3)]
    p = atp.atp_search(layers, calibration=cal)
    o = _oracle_plan(layers, cm.Model(), cal)
    _same_plan(p, o)
    t = {(r["d1"], r["d2"]): r["t_comm"] for r in p["ranked"]}
    assert abs(t[(2, 4)] / t[(8, 1)] - 0.545) < 0.001


def test_search_exact_tie_break():
    """G8: the C++ search resolves the exact (4,1)/(2,2) tie like the oracle (larger d1)."""
    layers = [atp.HcmLayer(4, 1e9, 1e9)]
    cal = {(4, 1): (64.0, None), (2, 2): (64.0, 224.0), (1, 4): (1e-3, 1e-3)}
    p = atp.atp_search(layers, calibration=cal)
    _same_plan(p, _oracle_plan(layers, cm.Model(), cal))
    t = {(r["d1"], r["d2"]): r["t_comm"] for r in p["ranked"]}
    assert t[(4, 1)] == t[(2, 2)] and p["chosen"] == (4, 1)
    cal[(2, 2)] = (64.0, 225.0)
    assert atp.atp_search(layers, calibration=cal)["chosen"] == (2, 2)


def test_search_errors():
    with pytest.raises(atp.AtpError) as e:
        atp.atp_search([atp.HcmLayer(4, -1.0, 1.0)])
    assert e.value.status == _abi.ATP_ERR_INVALID
    with pytest.raises(atp.AtpError) as e:
        atp.atp_search([atp.HcmLayer(8, 1.0, 1.0)], h=4096, heads=3)  # h % heads != 0 everywhere
    assert e.value.status == _abi.ATP_ERR_EMPTY


@pytest.mark.parametrize("d1,d2", [(1, 1), (2, 1), (1, 2), (2, 2), (4, 2), (2, 4), (8, 1), (1, 8)])
@pytest.mark.parametrize("chunks", [1, 2, 4, 8])
def test_comm_volume_matches_oracle(d1, d2, chunks):
    T, h = 8192, 4096
    calls, e1, e2 = atp.atp_comm_volume(d1, d2, T, h, 4 * h, chunks)
    assert calls == cm.comm_volume(d1, d2, T, h, chunks)
    assert e1 == sum(c[4] for c in calls if c[2] == 1)
    assert e2 == sum(c[4] for c in calls if c[2] == 2)


def test_workspace_size_matches_argument_shapes():
    """atp_workspace_size reports exactly the bf16 workspace buffers the op structs name."""
    import paper_2301_08658_b200 as atp
    from paper_2301_08658_b200 import api

    T, h, F = 512, 256, 1024
    for d1, d2 in ((1, 1), (2, 1), (2, 4), (4, 2)):
        assert api.atp_workspace_size(api.ATP_OP_MLP_BWD, d1, d2, T, h, F) == [T * F // d1 * 2, 0, 0, 0]
        assert api.atp_workspace_size(api.ATP_OP_ATTN_BWD, d1, d2, T, h, F) == [T * h // d1 * 2, T * 3 * h // d1 * 2, 0, 0]
        assert api.atp_workspace_size(api.ATP_OP_LAYER, d1, d2, T, h, F) == [T * F // d1 * 2, T * h // d1 * 2,
                                                                             T * 3 * h // d1 * 2, 0]
        g = api.atp_workspace_size(api.ATP_OP_GPT_LAYER, d1, d2, T, h, F, 8, 256, 2)
        assert g[0] == atp._abi.lib().atp_gpt_workspace(d1, d2, T, h, F, 8, 256, 2) > 0 and g[1:] == [0, 0, 0]
    with pytest.raises(atp._abi.AtpError):
        api.atp_workspace_size(9, 1, 1, T, h, F)
