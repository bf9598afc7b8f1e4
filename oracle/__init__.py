"""CPU oracle for ATP (arXiv 2301.08658) — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct NumPy (float64) implementation of what the
hot path computes, written from PAPER.md (cited as ``P:<line>``, section /
equation named).  It simulates the N virtual devices of a DeviceMesh(d1, d2),
holds every rank's shards and performs every group reduction explicitly.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package.  The product path (``paper_2301_08658_b200``)
never imports it and shares no code with it; the only shared module is
``datagen`` (seeded counter-based inputs, no method arithmetic).

Modules
    mesh       DeviceMesh, rank <-> coordinates, communication groups (§3.1)
    sharding   placements Shard/Replicate/Partial, shard/unshard (§3.1, Table 1)
    layer      dense layer, ATP row/column-first linears, sharded
               attention-projection + MLP blocks fwd/bwd with chunking (§3.2, §4)
    costmodel  Eq. 2 / Eq. 3 / Eq. 4, closed form (§5.4), search, comm volume

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py``; none is
"parity unpinned".
"""
