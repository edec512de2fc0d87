"""Slab partition of one problem vs the one-context solver.

The group runs the single-GPU colour-pass schedule over y-slabs with a seam
merge and a halo push after every pass, so a distributed sweep must equal the
one-context sweep to round-off, and V-cycles / solves / steps (whose FGMRES
dots are summed per slab, then over slabs) must match to the north_star bar.
Slabs share the one GPU here (host-ordered exchanges, no cross-slab waits).
"""
import numpy as np
import pytest

from helpers import rand, rel
from paper_1311_5614_b200 import configs
from paper_1311_5614_b200.ibmg import SaddleSystem, SlabGroup

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2():
    prob = configs.config2(kappa=1e4)
    return prob, SaddleSystem.from_problem(prob)


@pytest.mark.parametrize("P", [2, 4])
def test_group_sweep_matches_single(c2, P):
    prob, s = c2
    g = SlabGroup.from_problem(prob, P, min_cells=0)
    assert g.distributed_levels >= 1
    for l in range(g.distributed_levels):
        n = s.level_n(l)
        b, w = rand(3 * n * n, 20 + l), rand(3 * n * n, 30 + l)
        ws = s.sweep(b, w.copy(), level=l)
        wg = g.sweep(b, w, level=l)
        # same passes, same per-box arithmetic: bitwise equal (measured on B200)
        assert np.array_equal(wg, ws), (P, l, rel(wg, ws))


def test_group_sweep_tiles_level_bitwise():
    """N=1024 (C3 geometry): the one-context fine sweep is the same tile-colour
    and big-colour passes, so the slab sweep reproduces it exactly."""
    prob = configs.config3()
    s = SaddleSystem.from_problem(prob)
    g = SlabGroup.from_problem(prob, 4, min_cells=0)
    n = prob.N
    b, w = rand(3 * n * n, 40), rand(3 * n * n, 41)
    ws = s.sweep(b, w.copy(), level=0)
    wg = g.sweep(b, w, level=0)
    assert np.array_equal(wg, ws), rel(wg, ws)


@pytest.mark.parametrize("P", [2, 4])
def test_group_vcycle_matches_single(c2, P):
    prob, s = c2
    g = SlabGroup.from_problem(prob, P, min_cells=0)
    n = prob.N
    b = rand(3 * n * n, 50)
    zg, zs = g.v_cycle(b), s.v_cycle(b)
    assert rel(zg, zs) < 1e-13  # only the pressure-mean reduction order differs
    assert g.exchanges > 0


def test_group_vcycle_nothing_distributed(c2):
    """Too few rows per slab: every level agglomerated, Krylov rows still split."""
    prob, s = c2
    g = SlabGroup.from_problem(prob, 8, min_cells=0)
    assert g.distributed_levels == 0
    b = rand(3 * prob.N ** 2, 51)
    assert rel(g.v_cycle(b), s.v_cycle(b)) < 1e-10


def test_group_vcycle_deterministic(c2):
    prob, _ = c2
    g = SlabGroup.from_problem(prob, 2, min_cells=0)
    b = rand(3 * prob.N ** 2, 52)
    assert np.array_equal(g.v_cycle(b), g.v_cycle(b))


def test_group_solve_matches_single(c2):
    prob, s = c2
    g = SlabGroup.from_problem(prob, 2, min_cells=0)
    u0 = rand(2 * prob.N ** 2, 53)
    b = s.build_rhs(u0)
    xs, ss = s.gmres_solve(b)
    xg, sg = g.gmres_solve(b)
    assert ss["converged"] and sg["converged"]
    assert abs(sg["iters"] - ss["iters"]) <= 1
    assert rel(xg, xs) < 1e-8


@pytest.mark.parametrize("P", [2, 4])
def test_group_steps_match_single(P):
    prob = configs.config2(kappa=1e6)
    s = SaddleSystem.from_problem(prob)
    g = SlabGroup.from_problem(prob, P, min_cells=0)
    n = prob.N
    us, ps, Xs = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
    ug, pg, Xg = us.copy(), ps.copy(), Xs.copy()
    for _ in range(2):
        ss = s.step_implicit(us, ps, Xs)
        sg = g.step_implicit(ug, pg, Xg)
        assert ss["converged"] and sg["converged"]
        assert abs(sg["iters"] - ss["iters"]) <= 1
    assert rel(ug, us) < 1e-8 and rel(pg, ps) < 1e-8 and rel(Xg, Xs) < 1e-8
    assert g.kernel_launches > 0


@pytest.mark.parametrize("transport", ["inprocess", "nccl"])
def test_one_slab_test_mode_exchanges_with_itself(c2, transport):
    """min_rows < 0 distributes levels even for one slab: every seam, halo,
    allgather and allreduce then targets the slab itself (NCCL: self send/recv,
    world-size-1 collectives).  Results must equal the one-context solver."""
    prob, s = c2
    kw = dict(min_rows=-1, min_cells=0)
    if transport == "nccl":
        g = SlabGroup(prob.N, 1, nccl=(0, 0, SlabGroup.nccl_unique_id()), rho=prob.rho, mu=prob.mu, dt=prob.dt, **kw)
        g.set_structures(prob.nb, prob.kappa, prob.ds, prob.X)
    else:
        g = SlabGroup.from_problem(prob, 1, **kw)
    assert g.distributed_levels == 3  # 256, 128, 64
    n = prob.N
    for l in range(3):
        m = s.level_n(l)
        b, w = rand(3 * m * m, 60 + l), rand(3 * m * m, 70 + l)
        assert np.array_equal(g.sweep(b, w, level=l), s.sweep(b, w.copy(), level=l)), l
    b = rand(3 * n * n, 80)
    assert rel(g.v_cycle(b), s.v_cycle(b)) < 1e-13
    rhs = s.build_rhs(rand(2 * n * n, 81))
    xs, ss = s.gmres_solve(rhs)
    xg, sg = g.gmres_solve(rhs)
    assert sg["converged"] and sg["iters"] == ss["iters"]
    assert rel(xg, xs) < 1e-10


def test_group_three_sweep_cgs2_still_matches(c2):
    """IBMG_CGS2=1 keeps the three-sweep CGS2 over the slabs (fgmres_group); the default is the
    two-pass lagged CGS2 with the pass-1 sums reduced across the slabs (fgmres_group2).  Both
    solve to the one-context result with the same iteration count (+-1)."""
    import os
    prob, s = c2
    n = prob.N
    rhs = s.build_rhs(rand(2 * n * n, 91))
    xs, ss = s.gmres_solve(rhs)
    for env in ("1", None):
        old = os.environ.get("IBMG_CGS2")
        if env is None:
            os.environ.pop("IBMG_CGS2", None)
        else:
            os.environ["IBMG_CGS2"] = env
        try:
            g = SlabGroup.from_problem(prob, 2, min_cells=0)
        finally:
            if old is None:
                os.environ.pop("IBMG_CGS2", None)
            else:
                os.environ["IBMG_CGS2"] = old
        xg, sg = g.gmres_solve(rhs)
        assert sg["converged"] and abs(sg["iters"] - ss["iters"]) <= 1, (env, sg, ss)
        assert rel(xg, xs) < 1e-8
        g.close()
