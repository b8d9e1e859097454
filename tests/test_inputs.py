"""The seeded input generators: deterministic, normalised, the configs' shapes."""
import numpy as np
import pytest

import mmot_inputs as mi


def test_configs_match_baseline():
    c = mi.CONFIGS
    assert (c["C1"].l, c["C1"].N, c["C1"].eta, c["C1"].iters) == (3, 64, 0.05, 200)
    assert (c["C2"].l, c["C2"].N, c["C2"].eta, c["C2"].iters, c["C2"].tol) == (4, 1000, 0.01, 2000, 1e-9)
    assert (c["C3"].l, c["C3"].N, c["C3"].eta, c["C3"].iters) == (6, 100_000, 1e-3, 500)
    assert (c["C4"].l, c["C4"].N, c["C4"].eta, c["C4"].iters) == (4, 100_000_000, 1e-4, 100)
    assert (c["C5"].l, c["C5"].N, c["C5"].batch, c["C5"].iters) == (5, 4096, 8192, 300)


@pytest.mark.parametrize("name,N", [("C1", 64), ("C2", 1000), ("C3", 5000), ("C4", 20000), ("C5", 4096)])
def test_generators(name, N):
    a = mi.make_marginals(name, 0, N)
    b = mi.make_marginals(name, 0, N)
    assert a.shape == (mi.CONFIGS[name].l, N)
    assert np.array_equal(a, b)
    np.testing.assert_allclose(a.sum(axis=1), 1.0, rtol=1e-12)
    assert np.all(a >= 0)
    c = mi.make_marginals(name, 1, N)
    assert not np.array_equal(a, c)


def test_c1_floor_and_c5_etas():
    a = mi.c1_marginals(0)
    assert a.min() > 5e-7
    etas = mi.c5_etas(64)
    assert np.all((etas >= 1e-3) & (etas <= 1e-1))
    assert mi.c5_etas(4)[2] == mi.c5_etas(8)[2]


def test_c5_batch_generator_matches_per_instance():
    """The vectorised C5 generator (bench) gives bit-identical values to the per-instance one."""
    a = mi.c5_batch_marginals(5, 3, 256, 5)
    for i in range(3):
        assert np.array_equal(a[:, i, :], mi.c5_marginals(5 + i, 256, 5))
