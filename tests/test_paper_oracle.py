"""Paper-reproduction mode, CPU side.

1. The Dirichlet oracle (oracle/paper_oracle.cpp) against the REFERENCE's own
   code, walls included: golden fixture tests/golden/ref_dirichlet.npz written
   by tests/golden/make_golden_dirichlet.py from oracle/_ref (assembled saddle
   matrix with the thick annulus, Galerkin elasticity, build_rhs with the lid
   data, spread/interpolate, restriction and prolongation).
2. Its solver semantics (box relaxation in lexicographic order, V(nu1,nu2),
   coarsest solve, MG and MG-GMRES) against the PUBLISHED iteration counts:
   Table 2, §5.1 and Table 1
   (PAPER.md:664-670), with the acceptance bands of SPEC.md:683-690.
"""
import os

import numpy as np
import pytest
import scipy.sparse as sp

from helpers import rel
from paper_1311_5614_b200 import configs
import oracle as O

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_dirichlet.npz"))
n = int(G["n"])
nu = nv = n * (n - 1)
nvel, ntot = nu + nv, nu + nv + n * n


@pytest.fixture(scope="module")
def orc32():
    return O.PaperOracle(n, box=1, alpha=float(G["alpha"]), mesh=configs.paper_annulus(n))


def csr(t, shape):
    return sp.coo_matrix((t[2], (t[0], t[1])), shape=shape).tocsr()


def test_saddle_matrix_matches_reference(orc32):
    A = csr(orc32.saddle(0), (ntot, ntot))
    R = csr((G["Ar"], G["Ac"], G["Av"]), (ntot, ntot))
    d = abs(A - R).max()
    assert d <= 1e-12 * abs(R).max(), d
    # and the matrix-free rows agree with it
    w = np.random.default_rng(1).uniform(-1, 1, ntot)
    assert rel(orc32.apply(w), R @ w) < 1e-13


@pytest.mark.parametrize("lev", [1, 2])
def test_galerkin_elasticity_matches_reference(orc32, lev):
    nc = n >> lev
    nuc, nvelc = nc * (nc - 1), 2 * nc * (nc - 1)
    E = csr(orc32.elasticity(lev), (nvelc, nvelc))
    R = csr((G[f"E{lev}r"], G[f"E{lev}c"], G[f"E{lev}v"]), (nvelc, nvelc))
    # E is block diagonal in (u, v); the u block is exact in the reference, the v block
    # goes through the wrong packed v weight (transfers.cpp:202), which the oracle fixes
    du = abs(E[:nuc, :nuc] - R[:nuc, :nuc]).max()
    assert du <= 1e-12 * abs(R).max(), du
    assert abs(E[:nuc, nuc:]).max() == 0 and abs(E[nuc:, :nuc]).max() == 0
    assert abs(E[nuc:, nuc:] - R[nuc:, nuc:]).max() > 1e-3 * abs(R).max()  # the documented bug


def test_galerkin_identity(orc32):
    """E_{l+1} = R E_l P with the oracle's own transfers, column by column."""
    nc = n // 2
    nvelc = 2 * nc * (nc - 1)
    E0 = csr(orc32.elasticity(0), (nvel, nvel))
    E1 = csr(orc32.elasticity(1), (nvelc, nvelc))
    rng = np.random.default_rng(3)
    for _ in range(3):
        e = np.concatenate([rng.uniform(-1, 1, nvelc), np.zeros(nc * nc)])
        pe = O.paper_prolong_add(n, e, np.zeros(ntot))
        f = np.concatenate([E0 @ pe[:nvel], np.zeros(n * n)])
        assert rel(O.paper_restrict(n, f)[:nvelc], E1 @ e[:nvelc]) < 1e-12


def test_rhs_spread_interp_match_reference(orc32):
    assert rel(orc32.rhs(True, float(G["alpha"])), G["rhs"]) < 1e-13
    assert rel(orc32.rhs(True, 0.0), G["rhs0"]) < 1e-14
    assert rel(orc32.spread(G["Fr"]), G["f_spread"]) < 1e-13
    assert rel(orc32.interp(G["velr"]).reshape(-1), G["U"]) < 1e-13


def test_transfers_match_reference():
    assert rel(O.paper_restrict(n, G["rf"]), G["rc"]) < 1e-15
    wf = O.paper_prolong_add(n, G["ec"], np.zeros(ntot))
    assert rel(wf[:nu], G["wf"][:nu]) < 1e-15            # u: packed prolongation
    assert rel(wf[nvel:], G["wf"][nvel:]) < 1e-15        # p
    assert rel(wf[nu:nvel], G["wf"][nu:nvel]) > 1e-2     # v: line 202's weight differs
    # v against the reference's correct field-level weights (transfers.cpp:67-105); that routine
    # clamps the tangential ghost where the packed one reflects it, so compare off the side walls
    v, vf = wf[nu:nvel].reshape(n - 1, n), G["wf_field"][nu:].reshape(n - 1, n)
    assert rel(v[:, 1:-1], vf[:, 1:-1]) < 1e-15
    # at the side walls: v is the transpose of the (pinned) u prolongation
    nc = n // 2
    ecu = G["ec"][nc * (nc - 1):2 * nc * (nc - 1)].reshape(nc - 1, nc).T  # coarse v(I,J) -> u(J,I)
    et = np.concatenate([ecu.reshape(-1), np.zeros(nc * (nc - 1) + nc * nc)])
    ut = O.paper_prolong_add(n, et, np.zeros(ntot))[:nu].reshape(n, n - 1)
    assert rel(v, ut.T) < 1e-15


def test_whole_box_sweep_is_exact_solve():
    o = O.PaperOracle(8, box=8, alpha=0.0)
    w = np.random.default_rng(5).uniform(-1, 1, o.level_dofs(0))
    w[2 * 8 * 7:] -= w[2 * 8 * 7:].mean()
    b = o.apply(w)
    assert rel(o.sweep(b, np.zeros_like(w)), w) < 1e-10


def test_vcycle_linear_and_zero():
    o = O.PaperOracle(16, box=4, alpha=30.0, mesh=configs.paper_annulus(32))
    rng = np.random.default_rng(7)
    a, b = rng.uniform(-1, 1, (2, o.level_dofs(0)))
    assert np.all(o.vcycle(np.zeros_like(a)) == 0)
    assert rel(o.vcycle(2 * a - 3 * b), 2 * o.vcycle(a) - 3 * o.vcycle(b)) < 1e-11


# ---- published counts -----------------------------------------------------------------

TABLE2 = {  # (b, nu1, nu2): iterations at relative stiffness 10, 100, 500 (100 = cap reached)
    (1, 1, 0): (16, 53, 100), (1, 1, 1): (9, 33, 80), (1, 2, 1): (7, 21, 55), (1, 2, 2): (6, 17, 44),
    (4, 1, 0): (10, 20, 53), (4, 1, 1): (6, 11, 23), (4, 2, 1): (5, 9, 18), (4, 2, 2): (5, 7, 15),
    (8, 1, 0): (8, 14, 28), (8, 1, 1): (5, 8, 15), (8, 2, 1): (5, 7, 12), (8, 2, 2): (4, 6, 10),
}


def within(got, want):  # +-2 iterations or +-15%, whichever is larger
    return abs(got - want) <= max(2, 0.15 * want)


def paper_iters(N, box, nu1, nu2, rel_stiff, solver="gmres"):
    alpha = rel_stiff * configs.PAPER_ALPHA_EXP[N]
    o = O.PaperOracle(N, box, nu1, nu2, alpha=alpha, mesh=configs.paper_annulus(N))
    b = o.rhs(True, alpha)
    _, st, hist = (o.gmres_solve if solver == "gmres" else o.mg_solve)(b, 1e-6, 100)
    return st, hist


@pytest.mark.parametrize("cell", sorted(TABLE2))
def test_table2_counts(cell):
    """MG-GMRES iterations at h = 2^-6 to a 1e-6 reduction (Table 2)."""
    for rel_stiff, want in zip((10, 100, 500), TABLE2[cell]):
        st, hist = paper_iters(64, *cell, rel_stiff)
        assert within(st["iters"], want), (cell, rel_stiff, st["iters"], want)
        assert st["converged"] or want >= 100
        assert np.all(np.diff(hist) <= 1e-12)  # GMRES residuals never grow


def test_table2_bold_pattern():
    """V(1,1) has the lowest work (nu1+nu2+1) x iterations for boxes 4 and 8.
    One cell departs: b = 4 at relative stiffness 500, where V(2,2) takes 13 iterations here
    against the paper's 15 (inside the +-2 band) and so costs 65 against V(1,1)'s 69."""
    ties = 0
    for box in (4, 8):
        for rel_stiff in (10, 100, 500):
            work = {(a, b): (a + b + 1) * paper_iters(64, box, a, b, rel_stiff)[0]["iters"]
                    for a, b in ((1, 0), (1, 1), (2, 1), (2, 2))}
            assert work[(1, 1)] <= 1.1 * min(work.values()), (box, rel_stiff, work)
            ties += work[(1, 1)] == min(work.values())
    assert ties >= 5


def test_section_5_1_counts():
    """h = 2^-5, single-cell boxes, V(1,1)."""
    for rel_stiff in (0, 1, 10):
        assert abs(paper_iters(32, 1, 1, 1, rel_stiff, "mg")[0]["iters"] - 9) <= 2
        assert abs(paper_iters(32, 1, 1, 1, rel_stiff, "gmres")[0]["iters"] - 8) <= 2
    assert within(paper_iters(32, 1, 1, 1, 100, "mg")[0]["iters"], 62)
    assert within(paper_iters(32, 1, 1, 1, 100, "gmres")[0]["iters"], 30)
    st = paper_iters(32, 1, 1, 1, 200, "mg")[0]   # "fails to converge" near 160
    assert not st["converged"]
    assert paper_iters(32, 1, 1, 1, 800, "mg")[0]["diverged"]
    st = paper_iters(32, 1, 1, 1, 800, "gmres")[0]  # cap reached near 800 (+-2x in stiffness)
    assert st["iters"] >= 80
    assert not paper_iters(32, 1, 1, 1, 1600, "gmres")[0]["converged"]


def test_big_box_robustness():
    """Fig. 5: at relative stiffness 500, iterations(box 8) < (box 4) < (box 1)."""
    it = [paper_iters(32, b, 1, 1, 500)[0]["iters"] for b in (1, 4, 8)]
    assert it[2] < it[1] < it[0], it


@pytest.mark.parametrize("N", [32, 64])
def test_alpha_exp_table1(N):
    """Table 1: alpha_exp = 6.09 (h = 2^-5), 3.93 (2^-6) within 5%."""
    o = O.PaperOracle(N, box=1, alpha=0.0, mesh=configs.paper_annulus(N))
    a, _ = o.alpha_exp(1e-5)
    assert abs(a / configs.PAPER_ALPHA_EXP[N] - 1) < 0.05, a


@pytest.mark.parametrize("rel_stiff,want", [(0, 0.24), (1, 0.22), (10, 0.30), (100, 0.85)])
def test_fig4_spectral_radii(rel_stiff, want):
    """Fig. 4: spectral radius of the V(1,1) iteration matrix at
    32^2 with single-cell boxes, constant-pressure mode excluded, within +-0.05 (0.241, 0.217,
    0.303, 0.854 here)."""
    o = O.PaperOracle(32, 1, 1, 1, alpha=rel_stiff * configs.PAPER_ALPHA_EXP[32], mesh=configs.paper_annulus(32))
    ritz, H = o.iteration_matrix_spectrum(m=60, seed=1)
    assert abs(abs(ritz[0]) - want) <= 0.05, abs(ritz[0])
    # rho predicts the stand-alone multigrid count log(1e-6) / log(rho): within 30% up to
    # stiffness 10; at 100 the asymptotic rate is an upper bound (56 cycles against 87: the lid data
    # excites the slow structure modes only weakly)
    if rel_stiff:
        alpha = rel_stiff * configs.PAPER_ALPHA_EXP[32]
        it = o.mg_solve(o.rhs(True, alpha), 1e-6, 200)[1]["iters"]
        pred = np.log(1e-6) / np.log(abs(ritz[0]))
        assert abs(it / pred - 1) < 0.3 if rel_stiff <= 10 else 0.5 * pred < it <= pred


def test_multicolour_ordering_keeps_the_counts():
    """The opt-in multicolour box ordering (colours (bx mod (R+1), by mod (R+1)) with R the
    coupling reach in boxes) against the paper's lexicographic one, Table 2's V(1,1) rows at h = 2^-6:
    the same MG-GMRES counts (+-1) for boxes 4 and 8, no more iterations for single-cell boxes (9 / 24 / 60
    against 9 / 33 / 74).  This is the ordering family of the production path's smoother (D12)."""
    mesh = configs.paper_annulus(64)
    for box in (1, 4, 8):
        for rel_stiff in (10, 100, 500):
            alpha = rel_stiff * configs.PAPER_ALPHA_EXP[64]
            its = []
            for order in (0, 1):
                o = O.PaperOracle(64, box, 1, 1, alpha=alpha, mesh=mesh, order=order)
                its.append(o.gmres_solve(o.rhs(True, alpha))[1]["iters"])
            assert its[1] <= its[0] + 1, (box, rel_stiff, its)
            if box > 1:
                assert abs(its[1] - its[0]) <= 1, (box, rel_stiff, its)
    o = O.PaperOracle(64, 1, 1, 1, alpha=393.0, mesh=mesh, order=1)
    assert [o.level_reach(l) for l in range(o.nlevels)] == [5, 4, 3, 3, 1]


def test_fig5_standalone_mg_failure_thresholds():
    """Fig. 5(a): the stand-alone multigrid solver with boxes 2 and 4 fails
    at about the same relative stiffness as single-cell boxes (between 100 and 200), with fewer iterations
    before that; boxes 8 and 16 converge an order of magnitude further (still at 1000, not at 2000) with
    very similar counts."""
    mesh = configs.paper_annulus(32)

    def mg(box, rel_stiff):
        alpha = rel_stiff * configs.PAPER_ALPHA_EXP[32]
        o = O.PaperOracle(32, box, 1, 1, alpha=alpha, mesh=mesh)
        return o.mg_solve(o.rhs(True, alpha), 1e-6, 100)[1]

    at100 = {b: mg(b, 100) for b in (1, 2, 4, 8, 16)}
    assert all(s["converged"] for s in at100.values())
    assert at100[1]["iters"] > at100[2]["iters"] > at100[4]["iters"] > at100[8]["iters"] >= at100[16]["iters"]
    for b in (1, 2, 4):
        assert not mg(b, 200)["converged"]
    for b in (8, 16):
        assert mg(b, 1000)["converged"] and not mg(b, 2000)["converged"]
    assert abs(mg(8, 500)["iters"] - mg(16, 500)["iters"]) <= 5


def test_fig6_grid_refinement():
    """Fig. 6: MG-GMRES counts at fixed alpha on 32^2, 64^2, 128^2.
    Non-stiff and mildly stiff (alpha = 6, 60): independent of the grid for every box size; moderately
    stiff (alpha = 600): growing for single-cell boxes (29, 42, 49), nearly independent for box 8 (9, 10, 11)."""
    def counts(alpha, box):
        out = []
        for N in (32, 64, 128):
            o = O.PaperOracle(N, box, 1, 1, alpha=alpha, mesh=configs.paper_annulus(N))
            st = o.gmres_solve(o.rhs(True, alpha), 1e-6, 100)[1]
            assert st["converged"]
            out.append(st["iters"])
        return out

    for alpha in (6.0, 60.0):
        for box in (1, 4, 8):
            c = counts(alpha, box)
            assert max(c) - min(c) <= 3, (alpha, box, c)
    small, big = counts(600.0, 1), counts(600.0, 8)
    assert small[2] - small[0] >= 10 and big[2] - big[0] <= 3, (small, big)


def test_elasticity_symmetry_semidefiniteness_and_adjointness(orc32):
    """SPEC.md:690 property suite on the thick annulus: the fine E = S A_f S* is symmetric and negative
    semidefinite (A_f is a periodic second difference), spread and interpolate are adjoint with their
    ds^2 / h^2 weights, and E applied as a matrix equals spread(A_f interpolate(.)) h^2 ds^2-consistently."""
    E = csr(orc32.elasticity(0), (nvel, nvel))
    assert abs(E - E.T).max() <= 1e-12 * abs(E).max()
    rng = np.random.default_rng(17)
    for _ in range(20):
        x = rng.uniform(-1, 1, nvel)
        assert x @ (E @ x) <= 1e-10 * abs(E).max()
    mesh = configs.paper_annulus(n)
    F = rng.uniform(-1, 1, 2 * mesh.m1 * mesh.m2)
    vel = rng.uniform(-1, 1, nvel)
    lhs = orc32.spread(F) @ vel * (1.0 / n) ** 2
    rhs = F @ orc32.interp(vel).reshape(-1) * mesh.ds ** 2
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    # matrix-free twin (elasticity.cpp:109-117): E vel = spread(second difference(interpolate(vel)))
    U = orc32.interp(vel).reshape(mesh.m2, mesh.m1, 2)
    D = (np.roll(U, 1, axis=1) + np.roll(U, -1, axis=1) - 2 * U) / mesh.ds ** 2
    assert rel(orc32.spread(D.reshape(-1)), E @ vel) < 1e-12
