"""FGMRES orthogonalisation variants on the GPU: the default two-pass lagged
CGS2 (k_ortho_dots / k_ortho_update) against the three-sweep CGS2
(IBMG_CGS2=1) and the oracle (whose fgmres() is CGS2), on stiff C2-class
steps and on a restarted solve."""
import numpy as np
import pytest

from helpers import rel
from paper_1311_5614_b200 import configs
from paper_1311_5614_b200.ibmg import SaddleSystem
import oracle as O

pytestmark = pytest.mark.gpu


def step(prob, monkeypatch, **env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = SaddleSystem.from_problem(prob)
    for k in env:
        monkeypatch.delenv(k)
    n = prob.N
    u, p, X = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
    st = g.step_implicit(u, p, X)
    return u, p, X, st


@pytest.mark.parametrize("kappa", [1e2, 1e6])
def test_two_pass_matches_cgs2_and_oracle(kappa, monkeypatch):
    prob = configs.config2(kappa, N=128, nb=256)
    u2, p2, X2, s2 = step(prob, monkeypatch)
    u3, p3, X3, s3 = step(prob, monkeypatch, IBMG_CGS2="1")
    assert s2["converged"] and s3["converged"]
    assert abs(s2["iters"] - s3["iters"]) <= 1
    assert rel(u2, u3) < 1e-9 and rel(p2, p3) < 1e-9 and rel(X2, X3) < 1e-12
    o = O.Oracle(prob, threads=8)
    n = prob.N
    uo, po, Xo, so = o.step(np.zeros(2 * n * n), prob.X)
    assert abs(s2["iters"] - so["iters"]) <= 2
    assert rel(u2, uo) < 1e-8 and rel(p2, po) < 1e-8


def test_two_pass_across_restarts(monkeypatch):
    """restart 5 forces several FGMRES cycles (q_0 = r / |r| each time)."""
    prob = configs.config2(1e4, N=64, nb=128)
    g2 = SaddleSystem.from_problem(prob, restart=5)
    monkeypatch.setenv("IBMG_CGS2", "1")
    g3 = SaddleSystem.from_problem(prob, restart=5)
    monkeypatch.delenv("IBMG_CGS2")
    n = prob.N
    outs = []
    for g in (g2, g3):
        u, p, X = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
        st = g.step_implicit(u, p, X)
        outs.append((u, p, st))
    (u2, p2, s2), (u3, p3, s3) = outs
    assert s2["converged"] and s3["converged"] and s2["restarts"] >= 2
    assert abs(s2["iters"] - s3["iters"]) <= 2
    assert rel(u2, u3) < 1e-8 and rel(p2, p3) < 1e-8
