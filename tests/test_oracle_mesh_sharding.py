"""Pins for oracle.mesh and oracle.sharding (§3.1, §3.2)."""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import mesh, sharding
from oracle.sharding import P, R, S0, S1

from conftest import GOLDEN


def test_enumerate_four_devices_p161():
    # "a device mesh with four devices can be represented ... 2D: [1,4], [2,2], [4,1]"
    assert sorted(mesh.enumerate_meshes(4)) == [(1, 4), (2, 2), (4, 1)]
    assert mesh.enumerate_meshes(4) == [(4, 1), (2, 2), (1, 4)]  # descending d1


@pytest.mark.parametrize("n", range(0, 9))
def test_power_of_two_has_n_plus_1_meshes_p252(n):
    # "if we have 2^n devices, then we will have n+1 kinds of 2D device meshes"
    assert len(mesh.enumerate_meshes(2 ** n)) == n + 1


def test_enumerate_divisor_count():
    for n in range(1, 65):
        assert len(mesh.enumerate_meshes(n)) == sum(1 for k in range(1, n + 1) if n % k == 0)
    with pytest.raises(ValueError):
        mesh.enumerate_meshes(0)


def test_groups_2x2_p175():
    # [Replicate, Shard(0)] -> "rank-0 and rank-2" hold the same block => dim-1 group {0,2}
    assert mesh.groups(2, 2, 1) == [[0, 2], [1, 3]]
    assert mesh.groups(2, 2, 2) == [[0, 1], [2, 3]]
    assert mesh.groups(4, 1, 2) == [[0], [1], [2], [3]]
    with pytest.raises(ValueError):
        mesh.groups(2, 2, 3)


@pytest.mark.parametrize("d1,d2", [(1, 1), (2, 2), (4, 2), (2, 4), (8, 1), (1, 8), (8, 2), (3, 5)])
def test_groups_partition_and_intersect(d1, d2):
    n = d1 * d2
    for dim in (1, 2):
        gs = mesh.groups(d1, d2, dim)
        assert sorted(itertools.chain(*gs)) == list(range(n))
        assert len(gs) == (d2 if dim == 1 else d1)
    for g1 in mesh.groups(d1, d2, 1):
        for g2 in mesh.groups(d1, d2, 2):
            assert len(set(g1) & set(g2)) == 1
    for r in range(n):
        i1, i2 = mesh.coords(d1, d2, r)
        assert mesh.rank_of(d1, d2, i1, i2) == r
    assert mesh.coords(8, 2, 5) == (2, 1)
    assert mesh.coords(2, 2, 3) == (1, 1)


def test_sharding_worked_example_p175():
    g = json.load(open(os.path.join(GOLDEN, "sharding_example_p175.json")))
    t = np.array(g["tensor"])
    d1, d2 = g["mesh"]
    for r, want in g["replicate_shard0"].items():
        np.testing.assert_array_equal(sharding.local(t, (R, S0), d1, d2, int(r)), np.array(want))
    # [Shard(1), Shard(0)]: ranks {0,1} share the left column half, {2,3} the right half
    left = [sharding.local(t, (S1, S0), d1, d2, r) for r in g["shard1_shard0_column_pairs"]["ranks_sharing_left_columns"]]
    right = [sharding.local(t, (S1, S0), d1, d2, r) for r in g["shard1_shard0_column_pairs"]["ranks_sharing_right_columns"]]
    np.testing.assert_array_equal(np.concatenate(left, 0), t[:, :2])
    np.testing.assert_array_equal(np.concatenate(right, 0), t[:, 2:])


def test_shard_unshard_roundtrip_random():
    rng = np.random.default_rng(0)
    specs = [(a, b) for a in (S0, S1, R) for b in (S0, S1, R)]
    meshes = [(1, 1), (2, 1), (1, 2), (2, 2), (4, 2), (2, 4), (3, 2)]
    for _ in range(1000):
        d1, d2 = meshes[rng.integers(len(meshes))]
        spec = specs[rng.integers(len(specs))]
        shp = [int(rng.integers(1, 4)) * 24, int(rng.integers(1, 4)) * 24]
        t = rng.standard_normal(shp)
        locs = sharding.shard(t, spec, d1, d2)
        assert locs[0].shape == sharding.local_shape(shp, spec, d1, d2)
        np.testing.assert_array_equal(sharding.unshard(locs, spec, d1, d2), t)


def test_local_shapes_p220():
    # row-first X [b, h1/d1], W [h1/d1, h2/d2], Y [b, h2/d2]; column-first comm [b, h2/d1]
    b, h1, h2, d1, d2 = 8, 24, 36, 2, 3
    assert sharding.local_shape((b, h1), (S1, R), d1, d2) == (b, h1 // d1)
    assert sharding.local_shape((h1, h2), (S0, S1), d1, d2) == (h1 // d1, h2 // d2)
    assert sharding.local_shape((h1, h2), (S1, S0), d1, d2) == (h1 // d2, h2 // d1)
    assert sharding.local_shape((b, h1), (R, S1), d1, d2) == (b, h1 // d2)


def test_partial_has_no_local_split():
    with pytest.raises(ValueError):
        sharding.local(np.zeros((2, 2)), (P, R), 2, 1, 0)
