"""Explicit IB scheme and the explicit stability limit (PAPER.md
§4.1, Table 1): step_explicit against the oracle (spring forces spread on the
right, Stokes(+mass) solve, X update), and estimate_alpha_exp (power iteration
on M X = S^T L^{-1} S A_f X) against the same power iteration on the oracle's
operators."""
import copy

import numpy as np
import pytest

from helpers import rel
from paper_1311_5614_b200 import configs
from paper_1311_5614_b200.ibmg import SaddleSystem, estimate_alpha_exp, fiber_force_unit
import oracle as O

pytestmark = pytest.mark.gpu


def no_springs(prob):
    q = copy.copy(prob)
    q.kappa = [0.0] * len(prob.kappa)
    return q


def test_step_explicit_matches_oracle():
    prob = configs.small_problem(N=64, nb=128, kappa=1e2, dt=1e-3)
    g = SaddleSystem.from_problem(prob)
    ok, o0 = O.Oracle(prob), O.Oracle(no_springs(prob))   # forces with kappa; E' = 0 solve
    n = prob.N
    u = np.zeros(2 * n * n)
    p = np.zeros(n * n)
    X = prob.X.reshape(-1).copy()
    st = g.step_explicit(u, p, X)
    b = ok.rhs(np.zeros(2 * n * n))
    xo, so, _ = o0.solve(b)
    Xo = prob.X + prob.dt * o0.interp(xo)
    assert st["converged"] and so["converged"] and abs(st["iters"] - so["iters"]) <= 2
    assert rel(u, xo[: 2 * n * n]) < 1e-8 and rel(X.reshape(-1, 2), Xo) < 1e-8
    # the implicit scheme is restored on the next implicit step
    u2, p2, X2 = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
    g.step_implicit(u2, p2, X2)
    uo, _, Xoi, _ = ok.step(np.zeros(2 * n * n), prob.X)
    assert rel(u2, uo) < 1e-8 and rel(X2.reshape(-1, 2), Xoi) < 1e-8


def oracle_alpha_exp(prob, tol=1e-6, seed=0):
    o0 = O.Oracle(no_springs(prob))
    n = prob.N
    x = np.random.default_rng(seed).uniform(-1.0, 1.0, (prob.npts, 2))
    x /= np.linalg.norm(x)
    lam_prev = None
    for it in range(1, 1001):
        f = o0.spread(fiber_force_unit(x, prob.nb, prob.ds).reshape(-1))
        u, _, _ = o0.solve(np.concatenate([f, np.zeros(n * n)]))
        y = o0.interp(u)
        lam = float(np.sum(x * y))
        x = y / np.linalg.norm(y)
        if lam_prev is not None and abs(lam - lam_prev) <= tol * abs(lam):
            return 2.0 / abs(lam), lam, it
        lam_prev = lam
    raise RuntimeError("no convergence")


def test_alpha_exp_matches_oracle_power_iteration():
    prob = configs.small_problem(N=32, nb=64, kappa=1e2, dt=1e-2)
    g = SaddleSystem.from_problem(prob)
    a, lam, it = estimate_alpha_exp(g, tol=1e-8)
    ao, lamo, ito = oracle_alpha_exp(prob, tol=1e-8)
    assert lam < 0.0  # S^T L^-1 S A_f is negative semidefinite
    assert abs(it - ito) <= 2
    assert abs(a - ao) <= 1e-6 * ao, (a, ao)


def test_explicit_stability_limit():
    """dt * kappa slightly below alpha_exp: the stiffest mode decays; above: it grows
    (SPEC.md:546-547)."""
    base = configs.small_problem(N=32, nb=64, kappa=1.0, dt=1e-2)
    g = SaddleSystem.from_problem(base)
    a, _, _ = estimate_alpha_exp(g, tol=1e-8)
    growth = {}
    for f in (0.8, 1.25):
        prob = configs.small_problem(N=32, nb=64, kappa=f * a / base.dt, dt=base.dt)
        s = SaddleSystem.from_problem(prob)
        n = prob.N
        u, p = np.zeros(2 * n * n), np.zeros(n * n)
        X = prob.X.reshape(-1).copy()
        X += 1e-6 * np.random.default_rng(1).uniform(-1, 1, X.size)  # seed every mode
        e0 = np.linalg.norm(fiber_force_unit(X, prob.nb, prob.ds))
        for _ in range(60):
            s.step_explicit(u, p, X)
        growth[f] = np.linalg.norm(fiber_force_unit(X, prob.nb, prob.ds)) / e0
    assert growth[1.25] > 10.0 * growth[0.8], growth
    assert growth[1.25] > 1.0
