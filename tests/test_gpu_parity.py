"""GPU (C-ABI) vs CPU oracle parity on identical seeded inputs.

Bars (BASELINE.json north_star): operators to round-off (1e-12 relative);
solves/steps u, p, X^{n+1} within 1e-8 relative when both converge to 1e-10,
FGMRES iteration counts within +2 of the oracle.
"""
import numpy as np
import pytest

from helpers import rand, rel
from paper_1311_5614_b200 import configs
from paper_1311_5614_b200.ibmg import SaddleSystem
import oracle as O

pytestmark = pytest.mark.gpu


def pair(prob, **kw):
    return SaddleSystem.from_problem(prob, **kw), O.Oracle(prob, threads=4)


@pytest.fixture(scope="module")
def c1():
    return pair(configs.config1())


def test_apply_all_levels(c1):
    g, o = c1
    for l in range(g.num_levels):
        n = g.level_n(l)
        w = rand(3 * n * n, seed=l)
        assert rel(g.apply(w, level=l), o.apply(w, level=l)) < 1e-12, l


def test_residual(c1):
    g, o = c1
    n = g.N
    b, w = rand(3 * n * n, 1), rand(3 * n * n, 2)
    r, nrm = g.residual(b, w)
    ro = o.residual(b, w)
    assert rel(r, ro) < 1e-12
    assert abs(nrm - np.linalg.norm(ro)) < 1e-10 * np.linalg.norm(ro)


def test_transfers(c1):
    g, o = c1
    n = g.N
    rf = rand(3 * n * n, 3)
    assert rel(g.restrict_saddle(rf), O.restrict(n, rf)) < 1e-14
    ec = rand(3 * (n // 2) ** 2, 4)
    wf = rand(3 * n * n, 5)
    assert rel(g.prolong_saddle_add(ec, wf.copy()), O.prolong_add(n, ec, wf)) < 1e-14


def _dense(trip, m):
    r, c, v = trip
    D = np.zeros((m, m))
    np.add.at(D, (r, c), v)
    return D


def test_elasticity_matrices(c1):
    """GPU E'_l (factored windows -> assembled rows) == oracle R*E*P sparse products."""
    g, o = c1
    for l in range(g.num_levels):
        n = g.level_n(l)
        Dg, Do = _dense(g.elasticity(l), 2 * n * n), _dense(o.elasticity(l), 2 * n * n)
        assert np.abs(Dg - Do).max() <= 1e-12 * np.abs(Do).max(), l


def test_big_blocks_match(c1):
    g, o = c1
    for l in range(g.num_levels - 1):
        assert np.array_equal(g.big_blocks(l), o.big_blocks(l)), l


def test_rhs_interp_spread(c1):
    g, o = c1
    prob = configs.config1()
    n = prob.N
    u = rand(2 * n * n, 6)
    assert rel(g.build_rhs(u), o.rhs(u)) < 1e-13
    assert rel(g.interpolate(u).reshape(-1, 2), o.interp(u)) < 1e-13
    F = rand(2 * prob.npts, 7)
    assert rel(g.spread(F), o.spread(F)) < 1e-13


def test_sweep_level0(c1):
    g, o = c1
    n = g.N
    b, w = rand(3 * n * n, 8), rand(3 * n * n, 9)
    wg = g.sweep(b, w.copy())
    wo = o.sweep(b, w)
    assert rel(wg, wo) < 1e-11


def test_coarse_solve(c1):
    g, o = c1
    nc = g.level_n(g.num_levels - 1)
    b = rand(3 * nc * nc, 10)
    b[2 * nc * nc:] -= b[2 * nc * nc:].mean()
    assert rel(g.coarsest_solve(b), o.coarse_solve(b)) < 1e-11


@pytest.mark.parametrize("N", [16, 32, 64])
def test_vcycle(N):
    prob = configs.small_problem(N=N, nb=2 * N, kappa=1e3)
    g, o = pair(prob)
    b = rand(3 * N * N, 11)
    b[2 * N * N:] -= b[2 * N * N:].mean()
    assert rel(g.v_cycle(b), o.vcycle(b)) < 1e-10


def test_vcycle_deterministic(c1):
    g, _ = c1
    b = rand(3 * g.N * g.N, 12)
    z1, z2 = g.v_cycle(b), g.v_cycle(b)
    assert np.array_equal(z1, z2)


def test_solve_c1(c1):
    g, o = c1
    prob = configs.config1()
    u0 = np.zeros(2 * prob.N ** 2)
    b = o.rhs(u0)
    xg, sg = g.gmres_solve(b)
    xo, so, _ = o.solve(b)
    assert sg["converged"] and so["converged"]
    assert sg["iters"] <= so["iters"] + 2
    assert rel(xg, xo) < 1e-8


def test_step_c1():
    prob = configs.config1()
    g, o = pair(prob)
    n = prob.N
    u = np.zeros(2 * n * n)
    p = np.zeros(n * n)
    X = prob.X.reshape(-1).copy()
    sg = g.step_implicit(u, p, X)
    uo, po, Xo, so = o.step(np.zeros(2 * n * n), prob.X)
    assert sg["converged"] and so["converged"]
    assert abs(sg["iters"] - so["iters"]) <= 2
    assert rel(u, uo) < 1e-8
    assert rel(p, po) < 1e-8
    assert rel(X.reshape(-1, 2), Xo) < 1e-8


def test_solve_c2_stiff():
    """kappa = 1e6 (the stiff regime the big boxes target): parity at rtol 1e-10."""
    prob = configs.config2(1e6)
    g, o = pair(prob)
    b = o.rhs(np.zeros(2 * prob.N ** 2))
    xg, sg = g.gmres_solve(b)
    xo, so, _ = o.solve(b)
    assert sg["converged"] and so["converged"]
    assert sg["iters"] <= so["iters"] + 2
    assert rel(xg, xo) < 1e-8


def test_step_c3():
    """C3: 16 membranes (seed 0), N = 1024, one implicit step."""
    prob = configs.config3()
    g = SaddleSystem.from_problem(prob)
    o = O.Oracle(prob, threads=16)
    n = prob.N
    u, p, X = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
    sg = g.step_implicit(u, p, X)
    uo, po, Xo, so = o.step(np.zeros(2 * n * n), prob.X)
    assert sg["converged"] and so["converged"]
    assert abs(sg["iters"] - so["iters"]) <= 2
    assert rel(u, uo) < 1e-8 and rel(p, po) < 1e-8
    assert rel(X.reshape(-1, 2), Xo) < 1e-8


def test_context_reuse_across_batch_problems():
    """C5 path: one context, structures swapped between problems (buffers reused
    without reallocation) — each step still matches the oracle."""
    g = SaddleSystem(256, 1.0, 1.0, 1e-3)
    for i in (0, 3):
        prob = configs.config5_problem(i)
        g.set_structures(prob.nb, prob.kappa, prob.ds, prob.X)
        n = prob.N
        u, p, X = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
        sg = g.step_implicit(u, p, X)
        uo, po, Xo, so = O.Oracle(prob, threads=16).step(np.zeros(2 * n * n), prob.X)
        assert sg["converged"] and so["converged"], i
        assert abs(sg["iters"] - so["iters"]) <= 2, i
        assert rel(u, uo) < 1e-8 and rel(X.reshape(-1, 2), Xo) < 1e-8, i


def test_no_structures_pure_stokes():
    """n_mem = 0 (kappa-free Stokes): the whole path runs without IB data."""
    from paper_1311_5614_b200.configs import Problem
    prob = Problem("stokes", 64, 1.0, 1.0, 1e-2, [], [], [], np.zeros((0, 2)))
    g, o = pair(prob)
    b = rand(3 * 64 * 64, 21)
    b[2 * 64 * 64:] = 0.0
    xg, sg = g.gmres_solve(b)
    xo, so, _ = o.solve(b)
    assert sg["converged"] and so["converged"] and abs(sg["iters"] - so["iters"]) <= 2
    assert rel(xg, xo) < 1e-8


def test_consecutive_steps_track_oracle():
    """Three implicit steps (lagged rebuild at the moving X^n each step)."""
    prob = configs.config2(1e4, N=64, nb=128)
    g, o = pair(prob)
    n = prob.N
    u, p, X = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
    uo, Xo = np.zeros(2 * n * n), prob.X.copy()
    for s in range(3):
        sg = g.step_implicit(u, p, X)
        uo, po, Xo, so = o.step(uo, Xo)
        assert sg["converged"] and so["converged"], s
        assert abs(sg["iters"] - so["iters"]) <= 2, s
    assert rel(u, uo) < 1e-8 and rel(p, po) < 1e-8
    assert rel(X.reshape(-1, 2), Xo) < 1e-8


def test_membrane_across_periodic_boundary():
    """An ellipse centred near the corner: windows, face lists and big blocks wrap."""
    prob = configs.small_problem(N=64, nb=160, kappa=1e4, dt=1e-2, a=0.2, b=0.12, cx=0.03, cy=0.97, rot=0.4)
    g, o = pair(prob)
    for l in range(g.num_levels - 1):
        assert np.array_equal(g.big_blocks(l), o.big_blocks(l)), l
    n = prob.N
    u, p, X = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
    sg = g.step_implicit(u, p, X)
    uo, po, Xo, so = o.step(np.zeros(2 * n * n), prob.X)
    assert sg["converged"] and so["converged"] and abs(sg["iters"] - so["iters"]) <= 2
    assert rel(u, uo) < 1e-8 and rel(X.reshape(-1, 2), Xo) < 1e-8


def test_not_converged_is_a_flag():
    """hitting max_iters returns the best iterate flagged, no error."""
    prob = configs.config1()
    g = SaddleSystem.from_problem(prob, max_iters=3)
    b = g.build_rhs(np.zeros(2 * prob.N ** 2))
    x, st = g.gmres_solve(b)
    assert st["converged"] == 0 and st["iters"] == 3 and 0 < st["relres"] < 1


def test_step_bitwise_deterministic():
    prob = configs.config2(1e6, N=128, nb=256)
    outs = []
    for _ in range(2):
        g = SaddleSystem.from_problem(prob)
        n = prob.N
        u, p, X = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
        g.step_implicit(u, p, X)
        outs.append((u, p, X))
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


def test_invalid_arguments_raise_value_error():
    with pytest.raises(RuntimeError):
        SaddleSystem(12)  # not a power of two -> ibmg_create status 1
    prob = configs.config1()
    g = SaddleSystem.from_problem(prob)
    with pytest.raises(ValueError):
        g.set_structures([2], [1.0], [0.01], np.zeros((2, 2)))  # FiberMesh: m1 >= 3
    with pytest.raises(ValueError):
        g.sweep(np.zeros(3 * 64 * 64), np.zeros(3 * 64 * 64), level=3)  # coarse-kernel level



def test_run_simulation_equals_repeated_steps():
    """ibmg_run_simulation (run_simulation): the state stays on the device between
    the steps; results are bit for bit those of n calls of ibmg_step, with host arrays and with
    device tensors."""
    import torch
    prob = configs.config2(1e4, N=64, nb=128)
    n = prob.N
    g = SaddleSystem.from_problem(prob)
    u, p, X = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
    its = [g.step_implicit(u, p, X)["iters"] for _ in range(3)]
    g2 = SaddleSystem.from_problem(prob)
    u2, p2, X2 = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
    sts = g2.run_simulation(3, u2, p2, X2)
    assert [s["iters"] for s in sts] == its and all(s["converged"] for s in sts)
    assert np.array_equal(u, u2) and np.array_equal(p, p2) and np.array_equal(X, X2)
    g3 = SaddleSystem.from_problem(prob)
    ud = torch.zeros(2 * n * n, dtype=torch.float64, device="cuda")
    pd = torch.zeros(n * n, dtype=torch.float64, device="cuda")
    Xd = torch.tensor(prob.X.reshape(-1), dtype=torch.float64, device="cuda")
    sts = g3.run_simulation(3, ud, pd, Xd)
    assert len(sts) == 3 and np.array_equal(ud.cpu().numpy(), u) and np.array_equal(Xd.cpu().numpy(), X)
    assert g3.run_simulation(0, ud, pd, Xd) == []
