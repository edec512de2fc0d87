"""SPEC invariants of the CPU oracle itself (the GPU path is checked against it
in test_gpu_parity.py): SPEC.md KATs and properties re-expressed for the
periodic, backward-Euler system."""
import numpy as np
import pytest

from helpers import rand, rel
from paper_1311_5614_b200 import configs
import oracle as O


@pytest.fixture(scope="module")
def small():
    prob = configs.small_problem(N=32, nb=64, kappa=1e3, dt=1e-2)
    return prob, O.Oracle(prob)


def test_levels_and_sizes(small):
    prob, o = small
    assert [o.level_n(l) for l in range(o.nlevels)] == [32, 16, 8, 4]  # SPEC.md:346 (32 -> 4: 4 levels)


def test_operator_symmetric_fine_level(small):
    """Fine A = [A_mom G; G^T 0] with SPD momentum."""
    prob, o = small
    m = 3 * prob.N ** 2
    rng = np.random.default_rng(1)
    x, y = rng.uniform(-1, 1, m), rng.uniform(-1, 1, m)
    assert abs(x @ o.apply(y) - y @ o.apply(x)) < 1e-10 * abs(x @ o.apply(x))
    v = np.zeros(m)
    v[: 2 * prob.N ** 2] = x[: 2 * prob.N ** 2]
    assert v @ o.apply(v) > 0


def test_constant_pressure_nullspace(small):
    prob, o = small
    w = np.zeros(3 * prob.N ** 2)
    w[2 * prob.N ** 2:] = 3.7
    assert np.abs(o.apply(w)).max() < 1e-10


def test_spread_interp_adjoint_and_conservation(small):
    """<S F, u> h^2 = <F, S* u> ds^2 (ds^2 in both weights) and
    sum_faces f h^2 = sum_k F ds^2."""
    prob, o = small
    n, h, ds = prob.N, 1.0 / prob.N, prob.ds[0]
    rng = np.random.default_rng(2)
    F = rng.uniform(-1, 1, (prob.npts, 2))
    u = rng.uniform(-1, 1, 2 * n * n)
    f = o.spread(F)
    U = o.interp(u)
    assert abs((f @ u) * h * h - np.sum(F * U) * ds * ds / (h * h) * h * h) < 1e-12 * abs(f @ u) * h * h
    assert np.allclose([f[: n * n].sum() * h * h, f[n * n:].sum() * h * h], F.sum(0) * ds * ds, rtol=1e-12)


def test_interp_reproduces_constants(small):
    prob, o = small
    n = prob.N
    u = np.concatenate([np.full(n * n, 1.5), np.full(n * n, -0.25)])
    U = o.interp(u)
    assert np.allclose(U[:, 0], 1.5, atol=1e-13) and np.allclose(U[:, 1], -0.25, atol=1e-13)


def test_transfers_constants_and_restrict_kat():
    n = 16
    rf = np.ones(3 * n * n)
    assert np.allclose(O.restrict(n, rf), 1.0)  # weights sum to 1
    wf = O.prolong_add(n, np.ones(3 * (n // 2) ** 2), np.zeros(3 * n * n))
    assert np.allclose(wf, 1.0)  # prolongation reproduces constants
    # 2x2 fine pressure [1,2;3,4] -> 2.5
    rf = np.zeros(3 * 4)
    rf[8:] = [1, 2, 3, 4]
    assert np.isclose(O.restrict(2, rf)[2], 2.5)


def test_sweep_noop_on_exact_solution(small):
    """w exact -> sweep is a no-op to round-off."""
    prob, o = small
    w = rand(3 * prob.N ** 2, 3)
    w[2 * prob.N ** 2:] -= w[2 * prob.N ** 2:].mean()
    b = o.apply(w)
    assert rel(o.sweep(b, w), w) < 1e-12


def test_sweep_is_affine(small):
    """w' = w + C (b - A w), linear in (w, b)."""
    prob, o = small
    m = 3 * prob.N ** 2
    b1, b2, w1, w2 = rand(m, 4), rand(m, 5), rand(m, 6), rand(m, 7)
    lhs = o.sweep(b1 + 2 * b2, w1 + 2 * w2)
    rhs = o.sweep(b1, w1) + 2 * o.sweep(b2, w2)
    assert rel(lhs, rhs) < 1e-12


def test_coarse_solve_round_trip(small):
    """b = A w -> recovers w up to the pressure constant."""
    prob, o = small
    nc = o.level_n(o.nlevels - 1)
    w = rand(3 * nc * nc, 8)
    w[2 * nc * nc:] -= w[2 * nc * nc:].mean()
    b = o.apply(w, level=o.nlevels - 1)
    assert rel(o.coarse_solve(b), w) < 1e-10


def test_vcycle_contracts(small):
    """One V-cycle from zero reduces the residual (PAPER Fig. 4 regime)."""
    prob, o = small
    b = o.rhs(np.zeros(2 * prob.N ** 2))
    z = o.vcycle(b)
    assert np.linalg.norm(b - o.apply(z)) < 0.5 * np.linalg.norm(b)
    assert abs(z[2 * prob.N ** 2:].mean()) < 1e-13  # mean-zero pressure


def test_fgmres_monotone_and_converged(small):
    """residual history non-increasing; true residual <= 1e-10."""
    prob, o = small
    b = o.rhs(np.zeros(2 * prob.N ** 2))
    x, st, hist = o.solve(b, hist_len=200)
    assert st["converged"] and st["relres"] <= 1e-10
    assert np.all(np.diff(hist) <= 1e-14)
    assert rel(o.apply(x), b) <= 1.0001e-10


def test_threads_do_not_change_results():
    """Boxes of one pass are independent: the OpenMP oracle is bitwise equal to
    the sequential one (the schedule, not the thread count, defines the result)."""
    prob = configs.small_problem(N=64, nb=128, kappa=1e4, dt=1e-2)
    b = O.Oracle(prob).rhs(np.zeros(2 * 64 * 64))
    z1 = O.Oracle(prob, threads=1).vcycle(b)
    z4 = O.Oracle(prob, threads=4).vcycle(b)
    assert np.array_equal(z1, z4)


def test_big_blocks_cover_the_structure():
    prob = configs.config1()
    o = O.Oracle(prob)
    big = o.big_blocks(0)
    n = prob.N
    ij = np.floor(prob.X * n).astype(int) % n
    assert all(big[j // 4, i // 4] for i, j in ij)
    assert big.sum() < big.size // 2


def test_step_c1_converges_and_moves_structure():
    prob = configs.config1()
    o = O.Oracle(prob)
    u, p, X, st = o.step(np.zeros(2 * prob.N ** 2), prob.X)
    assert st["converged"] and st["iters"] <= 20
    # the stretched membrane relaxes: the ellipse contracts along its long axis
    assert np.ptp(X[:, 0]) < np.ptp(prob.X[:, 0])
    # discrete incompressibility of the solved velocity: -D u = 0 rows of A x = b
    w = np.concatenate([u, p])
    r = o.apply(w) - o.rhs(np.zeros(2 * prob.N ** 2)) * 0
    assert np.abs(r[2 * prob.N ** 2:]).max() < 1e-8 * np.abs(r[: 2 * prob.N ** 2]).max()
