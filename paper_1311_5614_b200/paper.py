"""Paper-reproduction mode over the C ABI include/ibmg_paper.h.

Host-side mirror of the reference's names for the Dirichlet cavity problem of
arXiv 1311.5614 §4-§6: SaddleSystem.apply / .residual (saddle.hpp:32-38),
restrict_saddle / prolong_saddle_add (transfers.hpp:25-28), spread / interpolate
(fiber.hpp:80-83), build_rhs (saddle.hpp:46) and the SPEC-only sweep, v_cycle,
mg_solve, gmres_solve and estimate_alpha_exp.
Vectors use the reference's packed interior ordering (geometry.hpp:54-76).
Status 1 -> ValueError (std::invalid_argument), 3 -> RuntimeError.  There is no CPU
fallback: everything runs in libibmg_b200.so's sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import ibmg as _ibmg


class PaperParams(C.Structure):
    _fields_ = [("N", C.c_int), ("box", C.c_int), ("nu1", C.c_int), ("nu2", C.c_int), ("coarsest_n", C.c_int),
                ("alpha", C.c_double), ("device", C.c_int), ("order", C.c_int)]


class PaperStats(C.Structure):
    _fields_ = [("iters", C.c_int), ("converged", C.c_int), ("diverged", C.c_int), ("relres", C.c_double),
                ("setup_ms", C.c_double), ("solve_ms", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


EXPORTS = ["ibmg_paper_create", "ibmg_paper_destroy", "ibmg_paper_last_error", "ibmg_paper_set_mesh",
           "ibmg_paper_num_levels", "ibmg_paper_level_n", "ibmg_paper_level_dofs", "ibmg_paper_level_boxes",
           "ibmg_paper_level_reach", "ibmg_paper_apply", "ibmg_paper_residual", "ibmg_paper_restrict",
           "ibmg_paper_prolong_add", "ibmg_paper_sweep", "ibmg_paper_vcycle", "ibmg_paper_elasticity_triplets",
           "ibmg_paper_build_rhs", "ibmg_paper_spread", "ibmg_paper_interpolate", "ibmg_paper_mg_solve",
           "ibmg_paper_gmres_solve", "ibmg_paper_alpha_exp", "ibmg_paper_vcycle_spectrum", "ibmg_paper_kernel_launches"]

_BOUND = False


def lib():
    global _BOUND
    L = _ibmg.lib()
    if not _BOUND:
        vp, ip, d = C.c_void_p, C.c_int, C.c_double
        L.ibmg_paper_create.argtypes = [C.POINTER(PaperParams), C.POINTER(C.c_void_p)]
        L.ibmg_paper_destroy.argtypes = [vp]
        L.ibmg_paper_last_error.restype = C.c_char_p
        L.ibmg_paper_last_error.argtypes = [vp]
        L.ibmg_paper_set_mesh.argtypes = [vp, ip, ip, d, vp]
        L.ibmg_paper_num_levels.argtypes = [vp]
        for f in ("level_n", "level_dofs", "level_boxes", "level_reach"):
            getattr(L, "ibmg_paper_" + f).argtypes = [vp, ip]
        L.ibmg_paper_apply.argtypes = [vp, ip, vp, vp]
        L.ibmg_paper_residual.argtypes = [vp, ip, vp, vp, vp, C.POINTER(d)]
        L.ibmg_paper_restrict.argtypes = [vp, ip, vp, vp]
        L.ibmg_paper_prolong_add.argtypes = [vp, ip, vp, vp]
        L.ibmg_paper_sweep.argtypes = [vp, ip, vp, vp]
        L.ibmg_paper_vcycle.argtypes = [vp, vp, vp]
        L.ibmg_paper_elasticity_triplets.restype = C.c_long
        L.ibmg_paper_elasticity_triplets.argtypes = [vp, ip, vp, vp, vp, C.c_long]
        L.ibmg_paper_build_rhs.argtypes = [vp, ip, d, vp]
        L.ibmg_paper_spread.argtypes = [vp, vp, vp]
        L.ibmg_paper_interpolate.argtypes = [vp, vp, vp]
        for f in ("mg_solve", "gmres_solve"):
            getattr(L, "ibmg_paper_" + f).argtypes = [vp, vp, vp, d, ip, C.POINTER(PaperStats), vp, ip]
        L.ibmg_paper_alpha_exp.argtypes = [vp, d, ip, C.POINTER(d), C.POINTER(ip)]
        L.ibmg_paper_vcycle_spectrum.argtypes = [vp, ip, C.c_ulonglong, vp, C.POINTER(ip)]
        L.ibmg_paper_kernel_launches.restype = C.c_longlong
        L.ibmg_paper_kernel_launches.argtypes = [vp]
        _BOUND = True
    return L


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, np.float64)


class PaperSystem:
    """The cavity SaddleSystem with its hierarchy and box smoothers on one GPU."""

    def __init__(self, N, box=1, nu1=1, nu2=1, alpha=0.0, mesh=None, coarsest_n=4, device=0, order=0):
        """order 0: the paper's lexicographic sweep; 1: the multicolour ordering (SPEC.md:452 opt-in)."""
        self.N = N
        self._h = C.c_void_p()
        rc = lib().ibmg_paper_create(C.byref(PaperParams(N, box, nu1, nu2, coarsest_n, alpha, device, order)),
                                     C.byref(self._h))
        if rc == 1:
            raise ValueError("ibmg_paper_create: invalid parameters")
        if rc:
            raise RuntimeError("ibmg_paper_create: CUDA error")
        self.mesh = None
        if mesh is not None:
            self.set_mesh(mesh)

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().ibmg_paper_destroy(self._h)
            self._h = C.c_void_p()

    def _chk(self, rc):
        if rc == 0:
            return
        msg = lib().ibmg_paper_last_error(self._h).decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)

    def set_mesh(self, mesh):
        """FiberMesh of m1 x m2 nodes (fiber.hpp:36-50); None clears the structure."""
        if mesh is None:
            self._chk(lib().ibmg_paper_set_mesh(self._h, 0, 0, 0.0, None))
        else:
            X = _f64(mesh.X).reshape(-1)
            self._chk(lib().ibmg_paper_set_mesh(self._h, mesh.m1, mesh.m2, mesh.ds, _p(X)))
        self.mesh = mesh

    @property
    def nlevels(self):
        return lib().ibmg_paper_num_levels(self._h)

    def level_n(self, l):
        return lib().ibmg_paper_level_n(self._h, l)

    def level_dofs(self, l=0):
        return lib().ibmg_paper_level_dofs(self._h, l)

    def level_boxes(self, l=0):
        return lib().ibmg_paper_level_boxes(self._h, l)

    def level_reach(self, l=0):
        return lib().ibmg_paper_level_reach(self._h, l)

    @property
    def kernel_launches(self):
        return lib().ibmg_paper_kernel_launches(self._h)

    def _vec(self, a, l):
        a = _f64(a)
        if a.shape != (self.level_dofs(l),):
            raise ValueError("size mismatch")  # SaddleSystem::apply: size mismatch (saddle.cpp:20-21)
        return a

    def apply(self, w, level=0):
        w = self._vec(w, level)
        out = np.empty_like(w)
        self._chk(lib().ibmg_paper_apply(self._h, level, _p(w), _p(out)))
        return out

    def residual(self, b, w, level=0, with_norm=False):
        b, w = self._vec(b, level), self._vec(w, level)
        r = np.empty_like(w)
        nrm = C.c_double()
        self._chk(lib().ibmg_paper_residual(self._h, level, _p(b), _p(w), _p(r), C.byref(nrm)))
        return (r, nrm.value) if with_norm else r

    def restrict_saddle(self, rf, level=0):
        rf = self._vec(rf, level)
        rc = np.empty(self.level_dofs(level + 1))
        self._chk(lib().ibmg_paper_restrict(self._h, level, _p(rf), _p(rc)))
        return rc

    def prolong_saddle_add(self, ec, wf, level=0):
        ec = self._vec(ec, level + 1)
        wf = np.array(self._vec(wf, level), copy=True)
        self._chk(lib().ibmg_paper_prolong_add(self._h, level, _p(ec), _p(wf)))
        return wf

    def sweep(self, b, w, level=0):
        b = self._vec(b, level)
        w = np.array(self._vec(w, level), copy=True)
        self._chk(lib().ibmg_paper_sweep(self._h, level, _p(b), _p(w)))
        return w

    def v_cycle(self, b):
        b = self._vec(b, 0)
        z = np.empty_like(b)
        self._chk(lib().ibmg_paper_vcycle(self._h, _p(b), _p(z)))
        return z

    def elasticity(self, level=0):
        L = lib()
        cnt = L.ibmg_paper_elasticity_triplets(self._h, level, None, None, None, 0)
        if cnt < 0:
            self._chk(3)
        r, c, v = np.empty(cnt, np.int32), np.empty(cnt, np.int32), np.empty(cnt, np.float64)
        if cnt:
            L.ibmg_paper_elasticity_triplets(self._h, level, _p(r), _p(c), _p(v), cnt)
        return r, c, v

    def build_rhs(self, lid=True, gamma=0.0):
        b = np.empty(self.level_dofs(0))
        self._chk(lib().ibmg_paper_build_rhs(self._h, int(lid), gamma, _p(b)))
        return b

    def spread(self, F):
        F = _f64(F).reshape(-1)
        f = np.empty(2 * self.N * (self.N - 1))
        self._chk(lib().ibmg_paper_spread(self._h, _p(F), _p(f)))
        return f

    def interpolate(self, vel):
        vel = _f64(vel)
        U = np.empty(2 * self.mesh.m1 * self.mesh.m2)
        self._chk(lib().ibmg_paper_interpolate(self._h, _p(vel), _p(U)))
        return U.reshape(-1, 2)

    def _solve(self, fn, b, rtol, max_iter):
        b = self._vec(b, 0)
        x = np.empty_like(b)
        st = PaperStats()
        hist = np.zeros(max_iter + 1)
        self._chk(fn(self._h, _p(b), _p(x), rtol, max_iter, C.byref(st), _p(hist), max_iter + 1))
        return x, st.as_dict(), hist[: st.iters + 1]

    def mg_solve(self, b, rtol=1e-6, max_iter=100):
        return self._solve(lib().ibmg_paper_mg_solve, b, rtol, max_iter)

    def gmres_solve(self, b, rtol=1e-6, max_iter=100):
        return self._solve(lib().ibmg_paper_gmres_solve, b, rtol, max_iter)

    def iteration_matrix_spectrum(self, m=60, seed=1):
        """(Ritz values by descending modulus, Hessenberg (m+1) x m) of the V-cycle's error
        propagator E = I - v_cycle(0, A .) on mean-zero pressure."""
        H = np.zeros((m + 1) * m)
        k = C.c_int()
        self._chk(lib().ibmg_paper_vcycle_spectrum(self._h, m, seed, _p(H), C.byref(k)))
        H = H.reshape(m + 1, m)
        ritz = np.linalg.eigvals(H[: k.value, : k.value])
        return ritz[np.argsort(-np.abs(ritz))], H

    def estimate_alpha_exp(self, tol=1e-4, max_steps=1000):
        a, k = C.c_double(), C.c_int()
        self._chk(lib().ibmg_paper_alpha_exp(self._h, tol, max_steps, C.byref(a), C.byref(k)))
        return a.value, k.value
