"""Seeded synthetic inputs (BASELINE.json configs)."""
import numpy as np

from paper_1311_5614_b200 import configs


def test_c1_equal_arclength_ellipse():
    p = configs.config1()
    assert p.N == 64 and p.nb == [128] and p.kappa == [1e2] and p.dt == 1e-2
    L = 128 * p.ds[0]
    assert abs(L - 1.4532672331) < 1e-9  # SURVEY §8d perimeter
    r = (p.X[:, 0] - 0.5) ** 2 / 0.3 ** 2 + (p.X[:, 1] - 0.5) ** 2 / 0.15 ** 2
    assert np.allclose(r, 1.0, atol=1e-13)


def test_c2_c5_shapes():
    for k in (1e2, 1e4, 1e6):
        p = configs.config2(k)
        assert p.N == 256 and p.npts == 512 and p.kappa == [k] and p.dt == 1e-3
    q = configs.config5_problem(7)
    assert q.N == 256 and q.npts == 512 and 10 <= q.kappa[0] <= 1e6
    assert np.array_equal(q.X, configs.config5_problem(7).X)


def test_c3_reproducible_and_separated():
    a, b = configs.config3(), configs.config3()
    assert np.array_equal(a.X, b.X) and a.nb == b.nb and len(a.nb) == 16
    h = 1.0 / 1024
    for nb, ds in zip(a.nb, a.ds):
        assert abs(ds - h / 2) < 0.01 * h  # spacing h/2
    assert all(1e3 <= k <= 1e6 for k in a.kappa)
