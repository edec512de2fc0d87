"""Bandwidth-regime kernels (levels n > 512) against the oracle and against
their simpler launch variants, on the C3 geometry (N = 1024, 16 membranes):

* the band-major plain dataflow phase (k_plain_df) runs the same tile tasks
  as the four tile-colour launches (IBMG_PLAIN_DF=0): bitwise equal sweeps;
* the tiled residual + restriction (k_residual_restrict_t) evaluates the
  same expressions as the one-thread-per-component kernel (IBMG_RR_TILED=0);
* both paths match the oracle's sweep / V-cycle to round-off.
"""
import numpy as np
import pytest

from helpers import rand, rel
from paper_1311_5614_b200 import configs
from paper_1311_5614_b200.ibmg import SaddleSystem
import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3():
    return configs.config3()


def system(prob, monkeypatch, **env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    g = SaddleSystem.from_problem(prob)
    for k in env:
        monkeypatch.delenv(k)
    return g


def test_plain_df_sweep_bitwise_and_oracle(c3, monkeypatch):
    n = c3.N
    b, w = rand(3 * n * n, 31), rand(3 * n * n, 32)
    g_df = system(c3, monkeypatch, IBMG_PLAIN_DF="1")
    g_4 = system(c3, monkeypatch, IBMG_PLAIN_DF="0")
    w_df = g_df.sweep(b, w.copy())
    w_4 = g_4.sweep(b, w.copy())
    assert np.array_equal(w_df, w_4)
    # repeated sweeps (epochs advance) stay identical
    assert np.array_equal(g_df.sweep(b, w_df.copy()), g_4.sweep(b, w_4.copy()))
    o = O.Oracle(c3, threads=16)
    assert rel(w_df, o.sweep(b, w)) < 1e-11


def test_tiled_restriction_matches(c3, monkeypatch):
    n = c3.N
    b = rand(3 * n * n, 33)
    b[2 * n * n:] -= b[2 * n * n:].mean()
    g_t = system(c3, monkeypatch, IBMG_RR_TILED="1")
    g_u = system(c3, monkeypatch, IBMG_RR_TILED="0")
    z_t, z_u = g_t.v_cycle(b), g_u.v_cycle(b)
    assert rel(z_t, z_u) < 1e-13
    o = O.Oracle(c3, threads=16)
    assert rel(z_t, o.vcycle(b)) < 1e-10


@pytest.mark.parametrize("which", ["c3", "dense"])
def test_restriction_from_assembled_rows(c3, which, monkeypatch):
    """Point-dense levels take E' w from the assembled rows (IBMG_RR_CSR):
    same V-cycle as the factored point-force path to round-off, and the
    oracle's.  'dense': 4096 points on one ellipse at N = 128, so even the
    fine level's restriction uses the rows."""
    prob = c3 if which == "c3" else configs.small_problem(N=128, nb=4096, kappa=1e4)
    n = prob.N
    b = rand(3 * n * n, 34)
    b[2 * n * n:] -= b[2 * n * n:].mean()
    g_r = system(prob, monkeypatch, IBMG_RR_CSR="1")
    g_p = system(prob, monkeypatch, IBMG_RR_CSR="0")
    z_r, z_p = g_r.v_cycle(b), g_p.v_cycle(b)
    assert rel(z_r, z_p) < 1e-12
    o = O.Oracle(prob, threads=16)
    assert rel(z_r, o.vcycle(b)) < 1e-10


def test_tiled_apply_matches(c3, monkeypatch):
    """k_stokes_apply_t (64 x 16 cell tiles) = the cell-per-thread apply
    (IBMG_AP_TILED=0) = the oracle's operator, on the C3 fine level."""
    n = c3.N
    w = rand(3 * n * n, 35)
    g_t = system(c3, monkeypatch, IBMG_AP_TILED="1")
    g_u = system(c3, monkeypatch, IBMG_AP_TILED="0")
    a_t, a_u = g_t.apply(w), g_u.apply(w)
    assert rel(a_t, a_u) < 1e-14
    o = O.Oracle(c3, threads=16)
    assert rel(a_t, o.apply(w)) < 1e-12


def test_canonical_inverses_bitwise(c3, monkeypatch):
    """Box inverses computed in block-id order during the colouring and moved to
    list order (IBMG_CANON_INV) equal the list-order inverses: two consecutive
    steps (the first sizes the canonical buffers) are bitwise identical."""
    outs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("IBMG_CANON_INV", flag)
        g = SaddleSystem.from_problem(c3)
        monkeypatch.delenv("IBMG_CANON_INV")
        n = c3.N
        u, p, X = np.zeros(2 * n * n), np.zeros(n * n), c3.X.reshape(-1).copy()
        for _ in range(2):
            g.step_implicit(u, p, X)
        outs.append((u, p, X))
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
