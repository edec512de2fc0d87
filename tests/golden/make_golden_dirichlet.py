"""Generate tests/golden/ref_dirichlet.npz from the REFERENCE's own code: the
Dirichlet cavity operators of the paper-reproduction mode,
walls included, with the thick annulus mesh of PAPER.md Eq. 21.

Runs oracle/_ref/libibmg_ref.so (reference TUs compiled in place by
oracle/Makefile.ref).  The fixture is committed; this script needs
/root/reference and is run in the build container only:
    python tests/golden/make_golden_dirichlet.py
"""
import ctypes as C
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
from make_golden import P, load, trip  # noqa: E402
from paper_1311_5614_b200 import configs  # noqa: E402


def main():
    L = load()
    for f in ("ref_assemble_saddle_m2", "ref_galerkin_elasticity_m2"):
        getattr(L, f).restype = C.c_long
    n = 32
    mesh = configs.paper_annulus(n)
    X = np.ascontiguousarray(mesh.X).reshape(-1)
    m = (n, mesh.m1, mesh.m2, C.c_double(mesh.ds), P(X))
    alpha = 60.9
    rng = np.random.default_rng(20131121)
    nvel, ntot = 2 * n * (n - 1), 2 * n * (n - 1) + n * n
    A = trip(L, L.ref_assemble_saddle_m2, *m, C.c_double(alpha))
    E1 = trip(L, L.ref_galerkin_elasticity_m2, *m, 1)
    E2 = trip(L, L.ref_galerkin_elasticity_m2, *m, 2)
    rhs = np.zeros(ntot)
    assert L.ref_build_rhs_lid(*m, C.c_double(alpha), P(rhs)) == 0
    rhs0 = np.zeros(ntot)
    assert L.ref_build_rhs_lid(*m, C.c_double(0.0), P(rhs0)) == 0
    Fr = rng.uniform(-1, 1, X.size)
    f_spread = np.zeros(nvel)
    assert L.ref_spread_m2(*m, P(Fr), P(f_spread)) == 0
    velr = rng.uniform(-1, 1, nvel)
    U = np.zeros(X.size)
    assert L.ref_interpolate_m2(*m, P(velr), P(U)) == 0
    # transfers on full random vectors (walls included)
    nc = n // 2
    ntc = 2 * nc * (nc - 1) + nc * nc
    rf = rng.uniform(-1, 1, ntot)
    rc = np.zeros(ntc)
    assert L.ref_restrict_saddle(n, P(rf), P(rc)) == 0
    ec = rng.uniform(-1, 1, ntc)
    wf = np.zeros(ntot)  # packed prolongation: u and p exact, v through line 202's weight
    assert L.ref_prolong_saddle_add(n, P(ec), P(wf)) == 0
    wf_field = np.zeros(nvel)  # field-level prolongation (correct weights, transfers.cpp:67-105)
    assert L.ref_prolong_velocity(n, P(np.ascontiguousarray(ec[: 2 * nc * (nc - 1)])), P(wf_field)) == 0
    out = os.path.join(HERE, "ref_dirichlet.npz")
    np.savez_compressed(out, n=n, alpha=alpha, Ar=A[0], Ac=A[1], Av=A[2], E1r=E1[0], E1c=E1[1], E1v=E1[2],
                        E2r=E2[0], E2c=E2[1], E2v=E2[2], rhs=rhs, rhs0=rhs0, Fr=Fr, f_spread=f_spread, velr=velr, U=U,
                        rf=rf, rc=rc, ec=ec, wf=wf, wf_field=wf_field)
    print("wrote", out, os.path.getsize(out))


if __name__ == "__main__":
    main()
