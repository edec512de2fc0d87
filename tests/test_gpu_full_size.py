"""Parity and size-independent properties at BASELINE.json's full sizes.

* C2 at full size against the CPU oracle: every kappa block, 10 consecutive
  implicit steps each (BASELINE configs[1]), u, p, X^{n+1} within 1e-8 and
  iteration counts within +-2 at every step.
* C3 at full size against the oracle: the 5 consecutive steps of configs[2],
  each on identical inputs.
* C4 (N = 8192, 256 membranes, 222k points) is out of the oracle's reach (it
  needs > 110 GB of host RAM), so it is checked through properties that do not
  depend on size: the converged step's true residual recomputed through
  ibmg_residual against the right-hand side built at X^n, X^{n+1} - X^n equal to
  dt * S*(X^n) u^{n+1}, the spread/interpolate adjoint identity
  (SPEC.md:166), force conservation of the closed membranes and
  bitwise repeatability.
* C5: all 512 problems of the batch through one context, each converged to
  1e-10 with the same X-update identity.
"""
import numpy as np
import pytest

from helpers import rel
from paper_1311_5614_b200 import configs
from paper_1311_5614_b200.ibmg import SaddleSystem
import oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kappa", [1e2, 1e4, 1e6])
def test_c2_full_block_tracks_oracle(kappa):
    prob = configs.config2(kappa)
    g = SaddleSystem.from_problem(prob)
    o = O.Oracle(prob, threads=16)
    n = prob.N
    u, p, X = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
    uo, Xo = np.zeros(2 * n * n), prob.X.copy()
    for s in range(10):
        sg = g.step_implicit(u, p, X)
        uo, po, Xo, so = o.step(uo, Xo)
        assert sg["converged"] and so["converged"], s
        assert sg["relres"] <= 1e-10, s
        assert abs(sg["iters"] - so["iters"]) <= 2, (s, sg["iters"], so["iters"])
        assert rel(u, uo) < 1e-8, s
        assert rel(p, po) < 1e-8, s
        assert rel(X.reshape(-1, 2), Xo) < 1e-8, s


def test_c3_five_steps_match_oracle():
    """C3 as BASELINE configs[2] runs it: 5 consecutive implicit steps at N = 1024.
    Each step is compared on identical inputs (the oracle steps from the GPU's
    u^n, X^n): the north_star bar is per solve.  Free-running trajectories, each
    step converged only to 1e-10, drift apart by about 1e-8 after 4 steps
    (1.2e-8 in u measured on B200), so they are not held to the per-solve bar."""
    prob = configs.config3()
    g = SaddleSystem.from_problem(prob)
    o = O.Oracle(prob, threads=16)
    n = prob.N
    u, p, X = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
    for s in range(5):
        u_in, X_in = u.copy(), X.reshape(-1, 2).copy()
        sg = g.step_implicit(u, p, X)
        uo, po, Xo, so = o.step(u_in, X_in)
        assert sg["converged"] and so["converged"], s
        assert abs(sg["iters"] - so["iters"]) <= 2, (s, sg["iters"], so["iters"])
        assert rel(u, uo) < 1e-8 and rel(p, po) < 1e-8, s
        assert rel(X.reshape(-1, 2), Xo) < 1e-8, s
    g.close()


@pytest.fixture(scope="module")
def c4():
    prob = configs.config4()
    g = SaddleSystem.from_problem(prob)
    yield prob, g
    g.close()


def test_c4_spread_interp_adjoint_and_conservation(c4):
    """<S F, u> h^2 = sum_k ds_k^2 F_k . (S* u)_k / h^2 * h^2 (ds^2 in both
    weights, as the oracle's small-size test), and sum_faces f h^2 = sum_k F_k ds_k^2."""
    prob, g = c4
    n, h = prob.N, 1.0 / prob.N
    rng = np.random.default_rng(7)
    F = rng.uniform(-1, 1, (prob.npts, 2))
    u = rng.uniform(-1, 1, 2 * n * n)
    ds2 = np.repeat(np.asarray(prob.ds) ** 2, prob.nb)
    f = g.spread(F.reshape(-1))
    U = g.interpolate(u).reshape(-1, 2)
    lhs = (f @ u) * h * h
    rhs = np.sum(ds2[:, None] * F * U)
    assert abs(lhs - rhs) <= 1e-11 * np.sum(np.abs(ds2[:, None] * F * U))
    tot = (F * ds2[:, None]).sum(0)
    scale = np.abs(F * ds2[:, None]).sum(0)
    assert np.all(np.abs([f[: n * n].sum() * h * h, f[n * n:].sum() * h * h] - tot) <= 1e-11 * scale)


def test_c4_step_residual_and_position_update(c4):
    prob, g = c4
    n = prob.N
    nn = n * n
    X0 = prob.X.reshape(-1).copy()
    u0 = np.zeros(2 * nn)
    g.set_structures(prob.nb, prob.kappa, prob.ds, prob.X)
    b = g.build_rhs(u0)                      # RHS at X^n
    u, p, X = u0.copy(), np.zeros(nn), X0.copy()
    st = g.step_implicit(u, p, X)
    assert st["converged"] and st["relres"] <= 1e-10
    assert 5 <= st["iters"] <= 60
    assert np.all(np.isfinite(u)) and np.all(np.isfinite(p))
    assert abs(p.mean()) < 1e-12 * max(np.abs(p).max(), 1e-300)
    # the operators are still those at X^n after the step (lagged)
    _, rnorm = g.residual(b, np.concatenate([u, p]))
    assert rnorm <= 2e-10 * np.linalg.norm(b), (rnorm, np.linalg.norm(b))
    dX = X - X0
    ref = prob.dt * g.interpolate(u)
    # X^{n+1} - X^n cancels: allow a few ulps of |X^n| on top of 1e-12 of dt U
    assert np.max(np.abs(dX - ref)) <= 1e-12 * np.max(np.abs(ref)) + 4 * np.finfo(float).eps
    # bitwise repeatable
    u2, p2, X2 = u0.copy(), np.zeros(nn), X0.copy()
    st2 = g.step_implicit(u2, p2, X2)
    assert st2["iters"] == st["iters"]
    assert np.array_equal(u, u2) and np.array_equal(p, p2) and np.array_equal(X, X2)


def test_c5_full_batch_converges():
    g = SaddleSystem(256, 1.0, 1.0, 1e-3)
    n = 256
    iters = []
    for i in range(512):
        prob = configs.config5_problem(i)
        g.set_structures(prob.nb, prob.kappa, prob.ds, prob.X)
        u, p, X = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
        st = g.step_implicit(u, p, X)
        assert st["converged"] and st["relres"] <= 1e-10, i
        ref = prob.dt * g.interpolate(u)
        dX = X - prob.X.reshape(-1)
        assert np.max(np.abs(dX - ref)) <= 1e-12 * np.max(np.abs(ref)) + 4 * np.finfo(float).eps, i
        iters.append(st["iters"])
    assert max(iters) <= 60
    g.close()
