"""bench.py draws the reference timer's inputs exactly: std::mt19937_64(7), each component
(rng() >> 11) * 2^-53 - 0.5, x, f, n per point (tools/bench_kernels.cpp:46-50)."""
import os

import numpy as np
import pytest


def test_mt19937_64_standard_value():
    import bench

    rng = bench.Mt19937_64()  # default seed 5489
    v = [rng() for _ in range(10000)]
    assert v[0] == 14514284786278117030
    assert v[-1] == 9981545732273789042  # the C++ standard's required 10000th output


def test_inputs_match_reference_draws():
    import bench
    from oracle.pyoracle import LIB_PATHS, Oracle

    if not os.path.exists(LIB_PATHS["ref"]):
        pytest.skip("oracle/_ref not built")
    ref = Oracle("ref")
    n = 257
    x, f, t = bench.synthetic_inputs(n, 7)
    want = ref.random_draws(7, 0, 9 * n) - 0.5  # uniform(0, 1) = (rng() >> 11) * 2^-53
    assert np.array_equal(np.stack([x, f, t], axis=1).reshape(-1), want)


def test_inputs_match_golden_mrs1k():
    import bench

    path = os.path.join(os.path.dirname(__file__), "golden", "golden.npz")
    g = np.load(path)
    x, f, t = bench.synthetic_inputs(1024, 7)
    assert np.array_equal(x, g["mrs1k_x"]) and np.array_equal(f, g["mrs1k_f"]) and np.array_equal(t, g["mrs1k_n"])
