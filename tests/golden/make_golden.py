"""Generate tests/golden/ref_ops.npz from the REFERENCE's own operator code.

Runs oracle/_ref/libibmg_ref.so — the reference TUs of
/root/reference/proj/core/src compiled in place by oracle/Makefile.ref (with the
test-only Eigen shim) — on seeded, interior-supported inputs, and stores
inputs + outputs.  The fixture is committed; this script needs /root/reference
and is run in the build container only:  python tests/golden/make_golden.py
"""
import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
LIB = os.path.join(ROOT, "oracle", "_ref", "libibmg_ref.so")


def load():
    if not os.path.exists(LIB):
        subprocess.check_call(["make", "-s", "-f", os.path.join(ROOT, "oracle", "Makefile.ref")])
    L = C.CDLL(LIB)
    L.ref_delta_1d.restype = C.c_double
    L.ref_delta_1d.argtypes = [C.c_double, C.c_double]
    L.ref_adjointness_check.restype = C.c_double
    L.ref_adjointness_check.argtypes = [C.c_int, C.c_int, C.c_ulonglong]
    L.ref_assemble_elasticity.restype = C.c_long
    L.ref_galerkin_elasticity.restype = C.c_long
    L.ref_galerkin_elasticity_fixed_p.restype = C.c_long
    return L


def P(a):
    return a.ctypes.data_as(C.c_void_p)


def trip(L, fn, *args):
    nnz = fn(*args, None, None, None, C.c_long(0))
    r = np.zeros(nnz, np.int32)
    c = np.zeros(nnz, np.int32)
    v = np.zeros(nnz)
    fn(*args, P(r), P(c), P(v), C.c_long(nnz))
    return r, c, v


def main():
    L = load()
    n = 32
    rng = np.random.default_rng(20131115)
    nu = (n - 1) * n
    nv = n * (n - 1)
    npr = n * n
    nvel = nu + nv
    # interior-supported fields: zero within 4 cells of the walls
    def interior_u():
        u = np.zeros((n, n - 1))  # [j, i-1], i in 1..n-1
        u[4:n - 4, 3:n - 5] = rng.uniform(-1, 1, (n - 8, n - 8))
        return u.reshape(-1)
    def interior_v():
        v = np.zeros((n - 1, n))  # [j-1, i]
        v[3:n - 5, 4:n - 4] = rng.uniform(-1, 1, (n - 8, n - 8))
        return v.reshape(-1)
    vel = np.concatenate([interior_u(), interior_v()])
    p = np.zeros((n, n))
    p[4:n - 4, 4:n - 4] = rng.uniform(-1, 1, (n - 8, n - 8))
    p = p.reshape(-1)
    lap = np.zeros(nvel); grad = np.zeros(nvel); div = np.zeros(npr)
    assert L.ref_laplacian_hom(n, P(vel), P(lap)) == 0
    assert L.ref_gradient_hom(n, P(p), P(grad)) == 0
    assert L.ref_divergence_hom(n, P(vel), P(div)) == 0
    # one closed fiber: circle r = 0.2 at the centre, m1 = 64 (interior supports)
    m1 = 64
    th = 2 * np.pi * np.arange(m1) / m1
    X = np.stack([0.5 + 0.2 * np.cos(th), 0.5 + 0.2 * np.sin(th)], 1).copy()
    ds = 2 * np.pi * 0.2 / m1
    gamma = 1e3
    F = np.zeros(2 * m1)
    assert L.ref_fiber_force(m1, C.c_double(ds), C.c_double(gamma), P(X), P(F)) == 0
    f_force = np.zeros(nvel)
    assert L.ref_spread(n, m1, C.c_double(ds), P(X), P(F), P(f_force)) == 0
    Fr = rng.uniform(-1, 1, 2 * m1)
    f_spread = np.zeros(nvel)
    assert L.ref_spread(n, m1, C.c_double(ds), P(X), P(Fr), P(f_spread)) == 0
    velr = rng.uniform(-1, 1, nvel)
    U = np.zeros(2 * m1)
    assert L.ref_interpolate(n, m1, C.c_double(ds), P(X), P(velr), P(U)) == 0
    args = (n, m1, C.c_double(ds), P(X), C.c_double(gamma))
    E0 = trip(L, L.ref_assemble_elasticity, *args)
    E1 = trip(L, L.ref_galerkin_elasticity, *args, 1)
    E1f = trip(L, L.ref_galerkin_elasticity_fixed_p, *args)
    Emf = np.zeros(nvel)
    assert L.ref_elasticity_apply_matrix_free(n, m1, C.c_double(ds), P(X), P(velr), P(Emf)) == 0
    # transfers on interior-supported vectors
    rf = np.concatenate([vel, p])
    nc = n // 2
    rc = np.zeros((nc - 1) * nc * 2 + nc * nc)
    assert L.ref_restrict_saddle(n, P(rf), P(rc)) == 0
    ec_u = np.zeros((nc, nc - 1)); ec_u[3:nc - 3, 2:nc - 4] = rng.uniform(-1, 1, (nc - 6, nc - 6))
    ec_v = np.zeros((nc - 1, nc)); ec_v[2:nc - 4, 3:nc - 3] = rng.uniform(-1, 1, (nc - 6, nc - 6))
    ec_p = np.zeros((nc, nc)); ec_p[3:nc - 3, 3:nc - 3] = rng.uniform(-1, 1, (nc - 6, nc - 6))
    ec = np.concatenate([ec_u.reshape(-1), ec_v.reshape(-1), ec_p.reshape(-1)])
    wf = np.zeros(nvel + npr)
    assert L.ref_prolong_saddle_add(n, P(ec), P(wf)) == 0
    wf_field = np.zeros(nvel)
    nvc = (nc - 1) * nc * 2
    assert L.ref_prolong_velocity(n, P(np.ascontiguousarray(ec[:nvc])), P(wf_field)) == 0
    # the survey's P4 probe: constant coarse v prolongs to 0.625 / 1.25 (transfers.cpp:202)
    ec_const = np.concatenate([np.zeros((nc - 1) * nc), np.ones(nc * (nc - 1)), np.zeros(nc * nc)])
    wf_const = np.zeros(nvel + npr)
    assert L.ref_prolong_saddle_add(n, P(ec_const), P(wf_const)) == 0
    # composite saddle apply with alpha = dt * gamma
    alpha = 1e-2 * gamma
    w = np.concatenate([vel, p])
    Aw = np.zeros(nvel + npr)
    assert L.ref_saddle_apply(n, m1, C.c_double(ds), P(X), C.c_double(gamma), C.c_double(alpha), P(w), P(Aw)) == 0
    h = 1.0 / n
    deltas = np.array([L.ref_delta_1d(r, h) for r in (0.0, 2 * h, -2 * h, 0.3 * h, 1.7 * h)])
    adj = np.array([L.ref_adjointness_check(k, 10, 0x1B2D3C4D) for k in (8, 16, 32)])
    np.savez_compressed(
        os.path.join(HERE, "ref_ops.npz"), n=n, vel=vel, p=p, lap=lap, grad=grad, div=div, X=X, ds=ds,
        gamma=gamma, F=F, f_force=f_force, Fr=Fr, f_spread=f_spread, velr=velr, U=U, E0r=E0[0], E0c=E0[1], E0v=E0[2],
        E1r=E1[0], E1c=E1[1], E1v=E1[2], E1fr=E1f[0], E1fc=E1f[1], E1fv=E1f[2], Emf=Emf, rf=rf, rc=rc, ec=ec, wf=wf, wf_field=wf_field, wf_const=wf_const, alpha=alpha,
        w=w, Aw=Aw, deltas=deltas, adj=adj)
    print("wrote", os.path.join(HERE, "ref_ops.npz"))


if __name__ == "__main__":
    main()
