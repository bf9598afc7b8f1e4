"""N>1 host logic on CPU: two processes over torch.distributed (gloo, 127.0.0.1).

Covers what bench.py does before any GPU work at N>1 — unique-id broadcast,
every rank reaching the same atp_search decision, each rank's shard boxes
(paper_2301_08658_b200.layout) tiling the global tensors exactly — and uses
libatp's mesh groups (the same member lists the NCCL split produces) to run
the sharded column-/row-first linears as a real 2-process SPMD program, whose
gathered result must equal the dense product."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2301_08658_b200 as atp
        from paper_2301_08658_b200 import layout

        # (a) unique-id broadcast exactly as bench.py does it
        uid = bytes(range(128)) if rank == 0 else bytes(128)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == bytes(range(128))

        # (b) every rank reaches the same search decision
        plan = atp.atp_search([atp.HcmLayer(world, 900.0, 900.0)], 1, 4, 2048, 4096, 32, 2)
        got = [None] * world
        dist.all_gather_object(got, plan["chosen"])
        assert all(g == got[0] for g in got)

        out = {"chosen": plan["chosen"]}
        for d1, d2 in ((world, 1), (1, world)):
            # (c) shard boxes tile the global tensors
            T, h, F = 16, 32, 128
            boxes = [None] * world
            dist.all_gather_object(boxes, layout.shard_boxes(d1, d2, rank, T, h, F))
            for name, shape in (("wqkv", (h, 3 * h)), ("wo", (h, h)), ("w1", (h, F)), ("w2", (F, h)), ("x", (T, h))):
                cover = np.zeros(shape, dtype=np.int32)
                for b in boxes:
                    r0, nr, c0, nc = b[name]
                    cover[r0:r0 + nr, c0:c0 + nc] += 1
                # weights are partitioned exactly once; activations are replicated over dim 1
                want = 1 if name != "x" else d1
                assert (cover == want).all(), (name, d1, d2)

            # (d) sharded linears as a 2-process SPMD program with libatp's groups
            groups = {dim: atp.atp_mesh_groups(d1, d2, dim) for dim in (1, 2)}
            pg = {}
            for dim in (1, 2):
                for members in groups[dim]:
                    g = dist.new_group(members)  # every rank creates every group, in the same order
                    if rank in members:
                        pg[dim] = g
            rng = np.random.default_rng(7)
            M, K, N = 8, 24, 40
            X = rng.standard_normal((M, K))
            W = rng.standard_normal((K, N))
            i1, i2 = rank // d2, rank % d2
            # column-first: X [R, S1] (cols by i2), W [S1, S0] (rows by i2, cols by i1), AR on dim 2
            xl = X[:, i2 * K // d2:(i2 + 1) * K // d2]
            wl = W[i2 * K // d2:(i2 + 1) * K // d2, i1 * N // d1:(i1 + 1) * N // d1]
            y = torch.from_numpy(xl @ wl)
            if d2 > 1:
                dist.all_reduce(y, group=pg[2])
            np.testing.assert_allclose(y.numpy(), (X @ W)[:, i1 * N // d1:(i1 + 1) * N // d1], rtol=1e-12, atol=1e-12)
            # row-first: X [S1, R] (cols by i1), W [S0, S1] (rows by i1, cols by i2), AR on dim 1
            xl = X[:, i1 * K // d1:(i1 + 1) * K // d1]
            wl = W[i1 * K // d1:(i1 + 1) * K // d1, i2 * N // d2:(i2 + 1) * N // d2]
            y = torch.from_numpy(xl @ wl)
            if d1 > 1:
                dist.all_reduce(y, group=pg[1])
            np.testing.assert_allclose(y.numpy(), (X @ W)[:, i2 * N // d2:(i2 + 1) * N // d2], rtol=1e-12, atol=1e-12)
        results[rank] = out
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_process_host_logic(world):
    from paper_2301_08658_b200 import build

    build.build()
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
    assert len(results) == world
    assert results[0]["chosen"] == (2, 1)  # N <= 4 on a flat HCM -> (N, 1)
