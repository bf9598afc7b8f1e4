"""The parity helpers themselves (CPU): the per-tile bound catches what the
global relative Frobenius norm misses."""
import numpy as np

from gpu_util import assert_close, rel, tile_rel_max


def test_tile_bound_catches_one_bad_tile():
    rng = np.random.default_rng(0)
    ref = rng.standard_normal((4096, 4096))
    got = ref + 3e-3 * rng.standard_normal(ref.shape)
    assert tile_rel_max(got, ref) < 5e-3
    bad = got.copy()
    bad[256:384, 512:768] *= 1.3  # one tile of 512 wrong by 30%
    assert rel(bad, ref) < 2e-2  # the global norm passes ...
    assert tile_rel_max(bad, ref) > 0.29  # ... the tile bound does not
    ref2 = ref[:1000, :1000]
    bad2 = got[:1000, :1000].copy()
    bad2[896:, 768:] = 0.0  # the ragged corner block (104 x 232) zeroed
    assert tile_rel_max(bad2, ref2) > 0.99


def test_tile_bound_1d_and_nan():
    ref = np.linspace(1.0, 2.0, 1000)
    got = ref.copy()
    got[768:] *= 1.1
    assert abs(tile_rel_max(got, ref) - 0.1) < 1e-9
    import pytest

    got2 = ref.copy()
    got2[3] = np.nan
    with pytest.raises(AssertionError):
        assert_close("x", got2, ref, 2e-2)
