"""Pins for the counter-based N(0,1) generator the method draws from."""
import numpy as np

from oracle import rng


def test_splitmix64_reference_values():
    """splitmix64 of 0 (state += golden gamma, then mix) is the published first
    output of Vigna's splitmix64 seeded with 0: 0xE220A8397B1DCDAF."""
    assert rng._sm64_int(0) == 0xE220A8397B1DCDAF
    arr = rng._sm64_arr(np.array([0, 1, 12345], dtype=np.uint64))
    assert [int(x) for x in arr] == [rng._sm64_int(0), rng._sm64_int(1), rng._sm64_int(12345)]


def test_gaussian_moments_and_determinism():
    z = rng.gaussian_column(7, rng.TAG_Q0, 3, 0, 1, 200_000)
    assert np.array_equal(z, rng.gaussian_column(7, rng.TAG_Q0, 3, 0, 1, 200_000))
    assert abs(z.mean()) < 0.01
    assert abs(z.var() - 1.0) < 0.01
    assert abs(np.mean(np.abs(z) < 1.0) - 0.6827) < 0.005
    assert abs(np.mean(np.abs(z) < 2.0) - 0.9545) < 0.003
    assert np.all(z == z.astype(np.float32))


def test_keys_give_independent_columns():
    a = rng.gaussian_column(7, rng.TAG_Q0, 3, 0, 1, 10_000)
    for other in [(8, 1, 3, 0, 1), (7, 2, 3, 0, 1), (7, 1, 4, 0, 1), (7, 1, 3, 1, 1),
                  (7, 1, 3, 0, 2)]:
        b = rng.gaussian_column(*other, 10_000)
        assert abs(np.corrcoef(a, b)[0, 1]) < 0.05
    # a prefix of a longer column is the shorter column (counter-based)
    np.testing.assert_array_equal(rng.gaussian_column(7, 1, 3, 0, 1, 50), a[:50])
