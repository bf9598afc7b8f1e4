"""Pins for oracle.overlap (PAPER §4.1/§4.2) and bit-exactness
of the library's atp_overlap_estimate against it."""
import random

import pytest

from oracle import overlap as ov


def test_spec_examples():
    # S:570-572
    assert ov.simulate_block(10, 10, 1) == 20
    assert ov.simulate_block(10, 10, 2) == 15
    for c in (1, 2, 4, 8):
        assert ov.simulate_block(10, 0, c) == 10


@pytest.mark.parametrize("mode", ["signalled", "per_chunk"])
def test_single_stage_equals_closed_form(mode):
    # one stage, no dW: the event simulation is exactly SPEC's closed form
    for comp, comm in [(10.0, 10.0), (8.0, 2.0), (2.0, 8.0), (6.0, 6.0), (16.0, 4.0)]:
        for c in (1, 2, 4, 8):
            mk, ex = ov.simulate([(comp, 0.0, comm)], c, mode)
            assert mk == ov.simulate_block(comp, comm, c), (comp, comm, c)
    rnd = random.Random(3)
    for _ in range(500):
        comp, comm, c = rnd.uniform(0, 5), rnd.uniform(0, 5), rnd.choice([1, 2, 3, 4, 8, 16])
        assert abs(ov.simulate([(comp, 0.0, comm)], c, mode)[0] - ov.simulate_block(comp, comm, c)) < 1e-12
        # SPEC invariant: non-increasing in c, bounded by max and sum
        assert ov.simulate_block(comp, comm, 2 * c) <= ov.simulate_block(comp, comm, c) + 1e-12


def _random_stages(rnd, n):
    return [(rnd.uniform(0.1, 2), rnd.choice([0.0, rnd.uniform(0, 1)]), rnd.choice([0.0, rnd.uniform(0, 2)]))
            for _ in range(n)]


def test_bounds_serial_and_orderings():
    rnd = random.Random(11)
    for _ in range(300):
        st = _random_stages(rnd, rnd.randint(1, 8))
        comp = sum(s[0] + s[1] for s in st)
        comm = sum(s[2] for s in st)
        for c in (1, 2, 4, 8):
            for mode in ("signalled", "per_chunk"):
                mk, ex = ov.simulate(st, c, mode)
                assert max(comp, comm) - 1e-12 <= mk <= comp + comm + 1e-12
                assert abs(ex - (mk - comp)) < 1e-12
            # fewer dependencies can only help: per-chunk <= signalled
            assert ov.simulate(st, c, "per_chunk")[0] <= ov.simulate(st, c, "signalled")[0] + 1e-12
        # c = 1 without dW: fully serial
        st0 = [(s[0], 0.0, s[2]) for s in st]
        assert abs(ov.simulate(st0, 1)[0] - sum(s[0] + s[2] for s in st0)) < 1e-12


def test_dw_overlap_strictly_helps_p345():
    # the dX all-reduce overlaps the dW GEMM
    for c in (1, 2, 4):
        overlapped = ov.simulate([(4.0, 3.0, 2.0)], c)[0]
        serial = ov.simulate([(4.0, 0.0, 2.0), (3.0, 0.0, 0.0)], c)[0]
        assert overlapped < serial


def test_library_estimate_bit_exact():
    import paper_2301_08658_b200 as atp
    from paper_2301_08658_b200 import build

    build.build()
    rnd = random.Random(5)
    for _ in range(300):
        st = _random_stages(rnd, rnd.randint(1, 12))
        c = rnd.choice([1, 2, 3, 4, 8, 16])
        for mode in ("signalled", "per_chunk"):
            assert atp.atp_overlap_estimate(st, c, mode) == ov.simulate(st, c, mode)


def test_chunk_planner_oracle_pins():
    """oracle.overlap.layer_stages / plan_chunks against independent facts:
    the split conserves the measured compute; forward = 1/3 of the GEMM FLOPs
    (fwd 24Th^2 of 72Th^2 at F = 4h, P:375 / G24); the communication equals
    the executed ring bytes of costmodel.comm_volume (another function) at the
    bus bandwidth; with no communication the makespan is the compute and
    nothing is exposed; more chunks win when compute is chunk-invariant."""
    from oracle import costmodel as cm

    T, h, F = 8192, 4096, 16384
    for d1, d2 in [(8, 1), (4, 2), (2, 4), (1, 8), (1, 1), (2, 2)]:
        st = ov.layer_stages(T, h, F, d1, d2, 2.0, 725.0)
        assert len(st) == 8
        assert abs(sum(s[0] + s[1] for s in st) - 2.0) < 1e-12
        assert abs(sum(s[0] for s in st[:4]) - 2.0 / 3.0) < 1e-12
        assert all(s[1] == 0.0 for s in st[:4]) and all(s[1] == s[0] for s in st[4:])  # dW = dX GEMM FLOPs
        ring = cm.ring_bytes_per_gpu(cm.comm_volume(d1, d2, T, h, 1))
        assert abs(sum(s[2] for s in st) - ring / 725e9 * 1e3) < 1e-9
        # size-1 dimensions move nothing
        assert all(s[2] == 0.0 for i, s in enumerate(st) if (d2 == 1 and i in (0, 2, 4, 6)) or
                   (d1 == 1 and i in (1, 3, 5, 7)))
    c, pred = ov.plan_chunks(T, h, F, 4, 2, {1: 1.3, 2: 1.3, 4: 1.3, 8: 1.3}, 725.0)
    assert c == 8 and pred[8][0] <= pred[4][0] <= pred[2][0] <= pred[1][0]
    c, pred = ov.plan_chunks(T, h, F, 4, 2, {1: 1.2, 2: 1.25, 4: 1.6, 8: 2.5}, 725.0)
    assert c == 2
    c, pred = ov.plan_chunks(T, h, F, 1, 1, {1: 1.0, 2: 1.0, 4: 0.9}, 725.0)
    assert c == 4 and pred[1][0] == pytest.approx(1.0, rel=1e-12) and pred[4][0] == pytest.approx(0.9, rel=1e-12)
    assert abs(pred[1][1]) < 1e-12 and abs(pred[4][1]) < 1e-12
    c, pred = ov.plan_chunks(T, h, F, 1, 1, {1: 1.0, 2: 1.0}, 725.0)
    assert c == 1  # tie -> fewer chunks


def test_chunk_planner_library_bit_exact():
    """libatp atp_layer_stages / atp_plan_chunks == the oracle, bit for bit."""
    import paper_2301_08658_b200 as atp
    from paper_2301_08658_b200 import build

    build.build()
    rnd = random.Random(8)
    for _ in range(200):
        h = rnd.choice([1024, 4096, 5120, 12288])
        F = rnd.choice([4 * h, 2 * h])
        T = rnd.choice([2048, 8192])
        d1, d2 = rnd.choice([(8, 1), (4, 2), (2, 4), (1, 8), (2, 2), (1, 1), (4, 1), (1, 2)])
        bw = rnd.choice([725.0, 900.0, 1.2, 0.97, 333.3])
        comp = rnd.uniform(0.1, 50.0)
        for bpe in (2, 4):
            assert atp.atp_layer_stages(T, h, F, d1, d2, comp, bw, bpe) == ov.layer_stages(T, h, F, d1, d2, comp,
                                                                                             bw, bpe)
        cands = {c: rnd.uniform(0.5, 3.0) for c in rnd.sample([1, 2, 4, 8], rnd.randint(1, 4))}
        for mode in ("signalled", "per_chunk"):
            assert atp.atp_plan_chunks(T, h, F, d1, d2, cands, bw, mode) == ov.plan_chunks(T, h, F, d1, d2, cands,
                                                                                          bw, mode)
    with pytest.raises(atp.AtpError):
        atp.atp_plan_chunks(8192, 4096, 16384, 3, 1, {1: 1.0}, 900.0)  # 4096 % 3
    with pytest.raises(atp.AtpError):
        atp.atp_plan_chunks(8192, 4096, 16384, 2, 1, {3: 1.0}, 900.0)  # 8192 % 3
    with pytest.raises(atp.AtpError):
        atp.atp_plan_chunks(8192, 4096, 16384, 2, 1, {1: 1.0}, 0.0)
