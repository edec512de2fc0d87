"""ctypes binding of the CPU oracle (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg import this module.  It is the checker, never the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class OrcParams(C.Structure):
    _fields_ = [("N", C.c_int), ("rho", C.c_double), ("mu", C.c_double), ("dt", C.c_double),
                ("nu1", C.c_int), ("nu2", C.c_int), ("restart", C.c_int), ("max_iters", C.c_int),
                ("rtol", C.c_double), ("coarsest_n", C.c_int), ("threads", C.c_int)]


class OrcStats(C.Structure):
    _fields_ = [("iters", C.c_int), ("restarts", C.c_int), ("converged", C.c_int),
                ("relres", C.c_double), ("setup_ms", C.c_double), ("solve_ms", C.c_double),
                ("total_ms", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class PorcParams(C.Structure):
    _fields_ = [("N", C.c_int), ("box", C.c_int), ("nu1", C.c_int), ("nu2", C.c_int), ("coarsest_n", C.c_int),
                ("alpha", C.c_double), ("order", C.c_int)]


class PorcStats(C.Structure):
    _fields_ = [("iters", C.c_int), ("converged", C.c_int), ("diverged", C.c_int), ("relres", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def build():
    subprocess.check_call(["make", "-s", "-C", _HERE])


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libibmg_oracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        dp = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        ip = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
        L.orc_create.restype = C.c_void_p
        L.orc_create.argtypes = [C.POINTER(OrcParams), C.c_char_p, C.c_int]
        L.orc_destroy.argtypes = [C.c_void_p]
        L.orc_last_error.restype = C.c_char_p
        L.orc_last_error.argtypes = [C.c_void_p]
        L.orc_set_structures.argtypes = [C.c_void_p, C.c_int, ip, dp, dp, dp]
        L.orc_num_levels.argtypes = [C.c_void_p]
        L.orc_level_n.argtypes = [C.c_void_p, C.c_int]
        L.orc_apply.argtypes = [C.c_void_p, C.c_int, dp, dp]
        L.orc_residual.argtypes = [C.c_void_p, C.c_int, dp, dp, dp]
        L.orc_sweep.argtypes = [C.c_void_p, C.c_int, dp, dp]
        L.orc_vcycle.argtypes = [C.c_void_p, dp, dp]
        L.orc_coarse_solve.argtypes = [C.c_void_p, dp, dp]
        L.orc_restrict.argtypes = [C.c_int, dp, dp]
        L.orc_prolong_add.argtypes = [C.c_int, dp, dp]
        L.orc_elasticity_triplets.restype = C.c_long
        L.orc_elasticity_triplets.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_long]
        L.orc_big_blocks.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
        L.orc_rhs.argtypes = [C.c_void_p, dp, dp]
        L.orc_interp.argtypes = [C.c_void_p, dp, dp]
        L.orc_spread.argtypes = [C.c_void_p, dp, dp]
        L.orc_solve.argtypes = [C.c_void_p, dp, dp, C.POINTER(OrcStats), C.c_void_p, C.c_int]
        L.orc_step.argtypes = [C.c_void_p, dp, dp, dp, C.POINTER(OrcStats)]
        # paper-reproduction mode (paper_oracle.h)
        L.porc_create.restype = C.c_void_p
        L.porc_create.argtypes = [C.POINTER(PorcParams), C.c_char_p, C.c_int]
        L.porc_destroy.argtypes = [C.c_void_p]
        L.porc_last_error.restype = C.c_char_p
        L.porc_last_error.argtypes = [C.c_void_p]
        L.porc_set_mesh.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_void_p]
        for f in ("porc_num_levels",):
            getattr(L, f).argtypes = [C.c_void_p]
        for f in ("porc_level_n", "porc_level_dofs", "porc_level_boxes", "porc_level_reach"):
            getattr(L, f).argtypes = [C.c_void_p, C.c_int]
        L.porc_apply.argtypes = [C.c_void_p, C.c_int, dp, dp]
        L.porc_residual.argtypes = [C.c_void_p, C.c_int, dp, dp, dp]
        L.porc_sweep.argtypes = [C.c_void_p, C.c_int, dp, dp]
        L.porc_vcycle.argtypes = [C.c_void_p, dp, dp]
        L.porc_restrict.argtypes = [C.c_int, dp, dp]
        L.porc_prolong_add.argtypes = [C.c_int, dp, dp]
        for f in ("porc_elasticity_triplets", "porc_saddle_triplets"):
            getattr(L, f).restype = C.c_long
            getattr(L, f).argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_long]
        L.porc_rhs.argtypes = [C.c_void_p, C.c_int, C.c_double, dp]
        L.porc_spread.argtypes = [C.c_void_p, dp, dp]
        L.porc_interp.argtypes = [C.c_void_p, dp, dp]
        for f in ("porc_mg_solve", "porc_gmres_solve"):
            getattr(L, f).argtypes = [C.c_void_p, dp, dp, C.c_double, C.c_int, C.POINTER(PorcStats), C.c_void_p, C.c_int]
        L.porc_vcycle_spectrum.argtypes = [C.c_void_p, C.c_int, C.c_ulonglong, dp, C.POINTER(C.c_int)]
        L.porc_alpha_exp.argtypes = [C.c_void_p, C.c_double, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_int)]
        _LIB = L
    return _LIB


class Oracle:
    """CPU oracle context for one problem (periodic MAC grid + membranes)."""

    def __init__(self, prob, restart=30, max_iters=600, rtol=1e-10, nu1=1, nu2=1, threads=1):
        self.prob = prob
        self.N = prob.N
        p = OrcParams(prob.N, prob.rho, prob.mu, prob.dt, nu1, nu2, restart, max_iters, rtol, 4, threads)
        err = C.create_string_buffer(512)
        self._ctx = lib().orc_create(C.byref(p), err, 512)
        if not self._ctx:
            raise ValueError(err.value.decode())
        self.set_structures(prob.X)

    def __del__(self):
        if getattr(self, "_ctx", None):
            lib().orc_destroy(self._ctx)
            self._ctx = None

    def _chk(self, rc, ok=(0,)):
        if rc not in ok:
            raise RuntimeError(lib().orc_last_error(self._ctx).decode())
        return rc

    def set_structures(self, X):
        p = self.prob
        self._chk(lib().orc_set_structures(self._ctx, len(p.nb), np.asarray(p.nb, np.int32),
                                           np.asarray(p.kappa, np.float64), np.asarray(p.ds, np.float64),
                                           np.ascontiguousarray(X, np.float64).reshape(-1)))

    @property
    def nlevels(self):
        return lib().orc_num_levels(self._ctx)

    def level_n(self, l):
        return lib().orc_level_n(self._ctx, l)

    def apply(self, w, level=0):
        out = np.empty_like(w)
        self._chk(lib().orc_apply(self._ctx, level, np.ascontiguousarray(w), out))
        return out

    def residual(self, b, w, level=0):
        r = np.empty_like(w)
        self._chk(lib().orc_residual(self._ctx, level, np.ascontiguousarray(b), np.ascontiguousarray(w), r))
        return r

    def sweep(self, b, w, level=0):
        w = np.array(w, dtype=np.float64, copy=True)
        self._chk(lib().orc_sweep(self._ctx, level, np.ascontiguousarray(b), w))
        return w

    def vcycle(self, b):
        z = np.empty_like(b)
        self._chk(lib().orc_vcycle(self._ctx, np.ascontiguousarray(b), z))
        return z

    def coarse_solve(self, b):
        x = np.empty_like(b)
        self._chk(lib().orc_coarse_solve(self._ctx, np.ascontiguousarray(b), x))
        return x

    def elasticity(self, level=0):
        """E'_level as a scipy-free (rows, cols, vals) triplet tuple."""
        cnt = lib().orc_elasticity_triplets(self._ctx, level, None, None, None, 0)
        r = np.empty(cnt, np.int32)
        c = np.empty(cnt, np.int32)
        v = np.empty(cnt, np.float64)
        lib().orc_elasticity_triplets(self._ctx, level, r.ctypes.data, c.ctypes.data, v.ctypes.data, cnt)
        return r, c, v

    def big_blocks(self, level=0):
        n = self.level_n(level)
        f = np.zeros((n // 4) * (n // 4), np.int32)
        lib().orc_big_blocks(self._ctx, level, f.ctypes.data)
        return f.reshape(n // 4, n // 4)

    def rhs(self, u_n):
        b = np.empty(3 * self.N * self.N)
        self._chk(lib().orc_rhs(self._ctx, np.ascontiguousarray(u_n, np.float64), b))
        return b

    def interp(self, u):
        U = np.empty(2 * self.prob.npts)
        self._chk(lib().orc_interp(self._ctx, np.ascontiguousarray(u[: 2 * self.N * self.N]), U))
        return U.reshape(-1, 2)

    def spread(self, F):
        f = np.empty(2 * self.N * self.N)
        self._chk(lib().orc_spread(self._ctx, np.ascontiguousarray(F, np.float64).reshape(-1), f))
        return f

    def solve(self, b, hist_len=0):
        x = np.empty_like(b)
        st = OrcStats()
        hist = np.zeros(max(hist_len, 1))
        rc = lib().orc_solve(self._ctx, np.ascontiguousarray(b), x, C.byref(st),
                             hist.ctypes.data if hist_len else None, hist_len)
        self._chk(rc, ok=(0, 2))
        return x, st.as_dict(), hist[:st.iters] if hist_len else None

    def step(self, u, X):
        """One implicit step; returns (u^{n+1}, p^{n+1}, X^{n+1}, stats)."""
        u = np.array(u, np.float64, copy=True)
        X = np.array(X, np.float64, copy=True).reshape(-1)
        p = np.empty(self.N * self.N)
        st = OrcStats()
        rc = lib().orc_step(self._ctx, u, p, X, C.byref(st))
        self._chk(rc, ok=(0, 2))
        return u, p, X.reshape(-1, 2), st.as_dict()


def restrict(nf, rf):
    rc = np.empty(3 * (nf // 2) ** 2)
    if lib().orc_restrict(nf, np.ascontiguousarray(rf), rc):
        raise ValueError("restrict: bad size")
    return rc


def prolong_add(nf, ec, wf):
    wf = np.array(wf, np.float64, copy=True)
    if lib().orc_prolong_add(nf, np.ascontiguousarray(ec), wf):
        raise ValueError("prolong: bad size")
    return wf


class PaperOracle:
    """CPU oracle of the Dirichlet paper-reproduction mode (paper_oracle.h): cavity
    walls, thick fiber mesh, b x b box relaxation in lexicographic order."""

    def __init__(self, N, box=1, nu1=1, nu2=1, alpha=0.0, mesh=None, coarsest_n=4, order=0):
        self.N = N
        p = PorcParams(N, box, nu1, nu2, coarsest_n, alpha, order)
        err = C.create_string_buffer(512)
        self._ctx = lib().porc_create(C.byref(p), err, 512)
        if not self._ctx:
            raise ValueError(err.value.decode())
        self.mesh = None
        if mesh is not None:
            self.set_mesh(mesh)

    def __del__(self):
        if getattr(self, "_ctx", None):
            lib().porc_destroy(self._ctx)
            self._ctx = None

    def _chk(self, rc):
        if rc:
            raise ValueError(lib().porc_last_error(self._ctx).decode())

    def set_mesh(self, mesh):
        X = np.ascontiguousarray(mesh.X, np.float64).reshape(-1)
        self._chk(lib().porc_set_mesh(self._ctx, mesh.m1, mesh.m2, mesh.ds, X.ctypes.data))
        self.mesh = mesh

    @property
    def nlevels(self):
        return lib().porc_num_levels(self._ctx)

    def level_n(self, l):
        return lib().porc_level_n(self._ctx, l)

    def level_dofs(self, l=0):
        return lib().porc_level_dofs(self._ctx, l)

    def level_boxes(self, l=0):
        return lib().porc_level_boxes(self._ctx, l)

    def level_reach(self, l=0):
        return lib().porc_level_reach(self._ctx, l)

    def apply(self, w, level=0):
        out = np.empty_like(w)
        self._chk(lib().porc_apply(self._ctx, level, np.ascontiguousarray(w), out))
        return out

    def residual(self, b, w, level=0):
        r = np.empty_like(w)
        self._chk(lib().porc_residual(self._ctx, level, np.ascontiguousarray(b), np.ascontiguousarray(w), r))
        return r

    def sweep(self, b, w, level=0):
        w = np.array(w, np.float64, copy=True)
        self._chk(lib().porc_sweep(self._ctx, level, np.ascontiguousarray(b), w))
        return w

    def vcycle(self, b):
        z = np.empty_like(b)
        self._chk(lib().porc_vcycle(self._ctx, np.ascontiguousarray(b), z))
        return z

    def _trips(self, fn, level):
        cnt = fn(self._ctx, level, None, None, None, 0)
        r, c, v = np.empty(cnt, np.int32), np.empty(cnt, np.int32), np.empty(cnt, np.float64)
        fn(self._ctx, level, r.ctypes.data, c.ctypes.data, v.ctypes.data, cnt)
        return r, c, v

    def elasticity(self, level=0):
        return self._trips(lib().porc_elasticity_triplets, level)

    def saddle(self, level=0):
        return self._trips(lib().porc_saddle_triplets, level)

    def rhs(self, lid=True, gamma=0.0):
        b = np.empty(self.level_dofs(0))
        self._chk(lib().porc_rhs(self._ctx, int(lid), gamma, b))
        return b

    def spread(self, F):
        n = self.N
        f = np.empty(2 * n * (n - 1))
        self._chk(lib().porc_spread(self._ctx, np.ascontiguousarray(F, np.float64).reshape(-1), f))
        return f

    def interp(self, vel):
        U = np.empty(2 * self.mesh.m1 * self.mesh.m2)
        self._chk(lib().porc_interp(self._ctx, np.ascontiguousarray(vel, np.float64), U))
        return U.reshape(-1, 2)

    def _solve(self, fn, b, rtol, max_iter):
        x = np.empty_like(b)
        st = PorcStats()
        hist = np.zeros(max_iter + 1)
        self._chk(fn(self._ctx, np.ascontiguousarray(b), x, rtol, max_iter, C.byref(st), hist.ctypes.data, max_iter + 1))
        return x, st.as_dict(), hist[: st.iters + 1]

    def mg_solve(self, b, rtol=1e-6, max_iter=100):
        return self._solve(lib().porc_mg_solve, b, rtol, max_iter)

    def gmres_solve(self, b, rtol=1e-6, max_iter=100):
        return self._solve(lib().porc_gmres_solve, b, rtol, max_iter)

    def iteration_matrix_spectrum(self, m=60, seed=1):
        """(Ritz values by descending modulus, Hessenberg (m+1) x m) of the V-cycle's error propagator."""
        H = np.zeros((m + 1) * m)
        k = C.c_int()
        self._chk(lib().porc_vcycle_spectrum(self._ctx, m, seed, H, C.byref(k)))
        H = H.reshape(m + 1, m)
        ritz = np.linalg.eigvals(H[: k.value, : k.value])
        return ritz[np.argsort(-np.abs(ritz))], H

    def alpha_exp(self, tol=1e-4, max_steps=1000):
        a, k = C.c_double(), C.c_int()
        self._chk(lib().porc_alpha_exp(self._ctx, tol, max_steps, C.byref(a), C.byref(k)))
        return a.value, k.value


def paper_restrict(nf, rf):
    nc = nf // 2
    rc = np.empty(2 * nc * (nc - 1) + nc * nc)
    lib().porc_restrict(nf, np.ascontiguousarray(rf), rc)
    return rc


def paper_prolong_add(nf, ec, wf):
    wf = np.array(wf, np.float64, copy=True)
    lib().porc_prolong_add(nf, np.ascontiguousarray(ec), wf)
    return wf
