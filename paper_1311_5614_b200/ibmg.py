"""Host-side mirror of the reference's ibmg:: solver interface over the C ABI.

The reference is C++ (proj/core/include/ibmg/*.hpp); its solver path is
reached here through include/ibmg_gpu.h (libibmg_b200.so, hand-written sm_100a
kernels).  Names follow the reference: SaddleSystem.apply / .residual
(saddle.hpp:32-38), restrict_saddle / prolong_saddle_add (transfers.hpp:25-28),
spread / interpolate (fiber.hpp:80-83), build_rhs (saddle.hpp:46), v_cycle /
gmres_solve / step_implicit.  Errors map back to the
reference's exception types: status 1 -> ValueError (std::invalid_argument),
3 -> RuntimeError (std::runtime_error).  Non-convergence is a flag, not an
error.

Arrays may be numpy (host; copied inside the call) or CUDA torch tensors on
the context's device (zero-copy).  There is no CPU fallback: if the CUDA
library is missing this module raises on import of the context.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

IBMG_PTR_HOST, IBMG_PTR_DEVICE = 0, 1
_LIB = None


class Params(C.Structure):
    _fields_ = [("N", C.c_int), ("rho", C.c_double), ("mu", C.c_double), ("dt", C.c_double),
                ("nu1", C.c_int), ("nu2", C.c_int), ("restart", C.c_int), ("max_iters", C.c_int),
                ("rtol", C.c_double), ("coarsest_n", C.c_int), ("device", C.c_int)]


class Stats(C.Structure):
    _fields_ = [("iters", C.c_int), ("restarts", C.c_int), ("converged", C.c_int), ("relres", C.c_double),
                ("setup_ms", C.c_double), ("solve_ms", C.c_double), ("total_ms", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


EXPORTS = ["ibmg_create", "ibmg_destroy", "ibmg_last_error", "ibmg_set_structures", "ibmg_num_levels",
           "ibmg_level_n", "ibmg_apply", "ibmg_residual", "ibmg_restrict", "ibmg_prolong_add", "ibmg_sweep",
           "ibmg_vcycle", "ibmg_coarse_solve", "ibmg_big_blocks", "ibmg_build_rhs", "ibmg_interpolate",
           "ibmg_spread", "ibmg_solve", "ibmg_step", "ibmg_kernel_launches", "ibmg_stream", "ibmg_profile",
           "ibmg_profile_report", "ibmg_elasticity_triplets", "ibmg_debug_sweep_trace", "ibmg_set_grid_limit",
           "ibmg_debug_coarse_trace", "ibmg_slab_plan", "ibmg_group_create", "ibmg_group_destroy",
           "ibmg_group_last_error", "ibmg_group_distributed_levels", "ibmg_group_kernel_launches",
           "ibmg_group_exchanges", "ibmg_group_set_structures", "ibmg_group_sweep", "ibmg_group_vcycle",
           "ibmg_group_solve", "ibmg_group_step", "ibmg_nccl_unique_id", "ibmg_group_create_nccl",
           "ibmg_vcycle_spectrum", "ibmg_set_scheme", "ibmg_set_input_stream", "ibmg_debug_cluster_trace",
           "ibmg_cluster_level", "ibmg_batch_create", "ibmg_batch_destroy", "ibmg_batch_last_error",
           "ibmg_batch_kernel_launches", "ibmg_batch_stream", "ibmg_batch_set_structures", "ibmg_batch_step",
           "ibmg_batch_prepare", "ibmg_batch_solve", "ibmg_run_simulation"]


def lib_path() -> str:
    # IBMG_LIB: another build of the same library (A/B of compile-time variants)
    return os.environ.get("IBMG_LIB", _build.LIB)


def lib(build_if_missing: bool = True):
    """Load libibmg_b200.so (building it in-tree if absent and nvcc is present)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        if not build_if_missing:
            raise RuntimeError(f"CUDA library missing: {path}")
        _build.build_cuda()
    L = C.CDLL(path)
    vp, ip, dp = C.c_void_p, C.c_int, C.c_void_p
    L.ibmg_create.argtypes = [C.POINTER(Params), C.POINTER(C.c_void_p)]
    L.ibmg_destroy.argtypes = [vp]
    L.ibmg_last_error.restype = C.c_char_p
    L.ibmg_last_error.argtypes = [vp]
    L.ibmg_set_structures.argtypes = [vp, ip, vp, vp, vp, vp, ip]
    L.ibmg_num_levels.argtypes = [vp]
    L.ibmg_level_n.argtypes = [vp, ip]
    L.ibmg_apply.argtypes = [vp, ip, dp, dp, ip]
    L.ibmg_residual.argtypes = [vp, ip, dp, dp, dp, C.POINTER(C.c_double), ip]
    L.ibmg_restrict.argtypes = [vp, ip, dp, dp, ip]
    L.ibmg_prolong_add.argtypes = [vp, ip, dp, dp, ip]
    L.ibmg_sweep.argtypes = [vp, ip, dp, dp, ip]
    L.ibmg_vcycle.argtypes = [vp, dp, dp, ip]
    L.ibmg_coarse_solve.argtypes = [vp, dp, dp, ip]
    L.ibmg_big_blocks.argtypes = [vp, ip, vp]
    L.ibmg_build_rhs.argtypes = [vp, dp, dp, ip]
    L.ibmg_interpolate.argtypes = [vp, dp, dp, ip]
    L.ibmg_spread.argtypes = [vp, dp, dp, ip]
    L.ibmg_solve.argtypes = [vp, dp, dp, C.POINTER(Stats), ip]
    L.ibmg_step.argtypes = [vp, dp, dp, dp, C.POINTER(Stats), ip]
    L.ibmg_run_simulation.argtypes = [vp, ip, dp, dp, dp, vp, C.POINTER(C.c_int), ip]
    L.ibmg_kernel_launches.restype = C.c_longlong
    L.ibmg_kernel_launches.argtypes = [vp]
    L.ibmg_stream.restype = C.c_void_p
    L.ibmg_stream.argtypes = [vp]
    L.ibmg_set_input_stream.argtypes = [vp, vp]
    L.ibmg_debug_cluster_trace.restype = C.c_long
    L.ibmg_debug_cluster_trace.argtypes = [vp, vp, vp, vp, C.c_long]
    L.ibmg_cluster_level.argtypes = [vp]
    L.ibmg_batch_create.argtypes = [C.POINTER(Params), ip, C.POINTER(C.c_void_p)]
    L.ibmg_batch_destroy.argtypes = [vp]
    L.ibmg_batch_last_error.restype = C.c_char_p
    L.ibmg_batch_last_error.argtypes = [vp]
    L.ibmg_batch_kernel_launches.restype = C.c_longlong
    L.ibmg_batch_kernel_launches.argtypes = [vp]
    L.ibmg_batch_stream.restype = C.c_void_p
    L.ibmg_batch_stream.argtypes = [vp]
    L.ibmg_batch_set_structures.argtypes = [vp, ip, ip, vp, vp, vp, vp]
    L.ibmg_batch_step.argtypes = [vp, ip, vp, vp, vp, vp, ip]
    L.ibmg_batch_prepare.argtypes = [vp, ip, vp, vp, ip]
    L.ibmg_batch_solve.argtypes = [vp, ip, vp, vp, vp, vp, ip]
    L.ibmg_debug_sweep_trace.restype = C.c_long
    L.ibmg_debug_sweep_trace.argtypes = [vp, ip, vp, vp, vp, C.c_long]
    L.ibmg_elasticity_triplets.restype = C.c_long
    L.ibmg_elasticity_triplets.argtypes = [vp, ip, vp, vp, vp, C.c_long]
    L.ibmg_set_grid_limit.argtypes = [vp, ip]
    L.ibmg_debug_coarse_trace.restype = C.c_long
    L.ibmg_debug_coarse_trace.argtypes = [vp, vp, vp, vp, C.c_long]
    L.ibmg_profile.argtypes = [vp, ip]
    L.ibmg_profile_report.argtypes = [vp, C.c_char_p, ip]
    L.ibmg_slab_plan.argtypes = [ip, ip, ip, ip, C.c_long, vp]
    L.ibmg_vcycle_spectrum.argtypes = [vp, ip, C.c_ulonglong, vp, C.POINTER(C.c_int)]
    L.ibmg_set_scheme.argtypes = [vp, ip]
    L.ibmg_group_create.argtypes = [C.POINTER(Params), ip, vp, ip, C.c_long, C.POINTER(C.c_void_p)]
    L.ibmg_group_create_nccl.argtypes = [C.POINTER(Params), ip, ip, vp, ip, C.c_long, C.POINTER(C.c_void_p)]
    L.ibmg_nccl_unique_id.argtypes = [vp]
    L.ibmg_group_destroy.argtypes = [vp]
    L.ibmg_group_last_error.restype = C.c_char_p
    L.ibmg_group_last_error.argtypes = [vp]
    L.ibmg_group_distributed_levels.argtypes = [vp]
    L.ibmg_group_kernel_launches.restype = C.c_longlong
    L.ibmg_group_kernel_launches.argtypes = [vp]
    L.ibmg_group_exchanges.restype = C.c_longlong
    L.ibmg_group_exchanges.argtypes = [vp]
    L.ibmg_group_set_structures.argtypes = [vp, ip, vp, vp, vp, vp]
    L.ibmg_group_sweep.argtypes = [vp, ip, dp, dp]
    L.ibmg_group_vcycle.argtypes = [vp, dp, dp]
    L.ibmg_group_solve.argtypes = [vp, dp, dp, C.POINTER(Stats)]
    L.ibmg_group_step.argtypes = [vp, dp, dp, dp, C.POINTER(Stats)]
    _LIB = L
    return L


def _ptr(a):
    """(pointer, kind) of a numpy array or a CUDA torch tensor."""
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
            raise ValueError("arrays must be C-contiguous float64")
        return a.ctypes.data, IBMG_PTR_HOST
    if hasattr(a, "data_ptr") and getattr(a, "is_cuda", False):
        import torch
        if a.dtype != torch.float64 or not a.is_contiguous():
            raise ValueError("tensors must be contiguous float64")
        return a.data_ptr(), IBMG_PTR_DEVICE
    raise TypeError(f"unsupported array type {type(a)}")


def _empty_like(a, n):
    if isinstance(a, np.ndarray):
        return np.empty(n, np.float64)
    import torch
    return torch.empty(n, dtype=torch.float64, device=a.device)


class SaddleSystem:
    """Periodic backward-Euler IB-Stokes saddle system on a MAC grid, with its
    multigrid hierarchy and FGMRES solver, resident on one GPU.

    Mirrors ibmg::SaddleSystem (saddle.hpp:19-39) extended per SURVEY §9:
    periodic geometry (D1), rho/dt and mu (D2), sign (D3), per-membrane kappa.
    """

    def __init__(self, N, rho=1.0, mu=1.0, dt=1e-2, nu1=1, nu2=1, restart=30, max_iters=600, rtol=1e-10,
                 device=0):
        self._L = lib()
        p = Params(N, rho, mu, dt, nu1, nu2, restart, max_iters, rtol, 4, device)
        h = C.c_void_p()
        rc = self._L.ibmg_create(C.byref(p), C.byref(h))
        if rc != 0 or not h.value:
            raise RuntimeError(f"ibmg_create failed (status {rc}); is a CUDA device available?")
        self._h = h
        self._in_stream = 0
        self.N, self.rho, self.mu, self.dt = N, rho, mu, dt
        self.npts = 0

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._L.ibmg_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def _p(self, a):
        """(pointer, kind) of `a`; for a CUDA tensor the context is first told the
        caller's current torch stream (ibmg_set_input_stream), so its inputs are
        read after their producers on that stream."""
        ptr, kind = _ptr(a)
        if kind == IBMG_PTR_DEVICE:
            import torch
            sp = torch.cuda.current_stream(a.device).cuda_stream
            if sp != self._in_stream:
                self._chk(self._L.ibmg_set_input_stream(self._h, C.c_void_p(sp)))
                self._in_stream = sp
        return ptr, kind

    def _chk(self, rc, ok=(0,)):
        if rc in ok:
            return rc
        msg = self._L.ibmg_last_error(self._h).decode()
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)

    # -- structure (FiberMesh + assemble_elasticity + Galerkin hierarchy)
    def set_structures(self, nb, kappa, ds, X):
        nb = np.ascontiguousarray(nb, np.int32)
        kappa = np.ascontiguousarray(kappa, np.float64)
        ds = np.ascontiguousarray(ds, np.float64)
        if isinstance(X, np.ndarray):
            X = np.ascontiguousarray(X, np.float64).reshape(-1)
        xp, kind = self._p(X)
        self._chk(self._L.ibmg_set_structures(self._h, len(nb), nb.ctypes.data, kappa.ctypes.data,
                                              ds.ctypes.data, xp, kind))
        self.npts = int(nb.sum())
        self._nb, self._ds = nb.astype(np.int64), ds
        self._X_host = np.array(X.detach().cpu().numpy() if hasattr(X, "detach") else X, np.float64).reshape(-1)
        return self

    @classmethod
    def from_problem(cls, prob, **kw):
        s = cls(prob.N, prob.rho, prob.mu, prob.dt, **kw)
        s.set_structures(prob.nb, prob.kappa, prob.ds, prob.X)
        return s

    def set_scheme(self, implicit=True):
        """implicit=True: E' = dt S K S^T on the left (step_implicit); False: the
        explicit IB scheme: pure Stokes(+mass) on the left,
        spread spring forces S F(X^n) on the right."""
        self._chk(self._L.ibmg_set_scheme(self._h, int(bool(implicit))))
        self._implicit = bool(implicit)

    @property
    def num_levels(self):
        return self._L.ibmg_num_levels(self._h)

    def level_n(self, level):
        return self._L.ibmg_level_n(self._h, level)

    def _size(self, level):
        n = self.level_n(level)
        return 3 * n * n

    def apply(self, w, out=None, level=0):
        out = _empty_like(w, self._size(level)) if out is None else out
        (wp, k), (op, _) = self._p(w), self._p(out)
        self._chk(self._L.ibmg_apply(self._h, level, wp, op, k))
        return out

    def residual(self, b, w, level=0):
        r = _empty_like(w, self._size(level))
        nrm = C.c_double()
        (bp, k), (wp, _), (rp, _) = self._p(b), self._p(w), self._p(r)
        self._chk(self._L.ibmg_residual(self._h, level, bp, wp, rp, C.byref(nrm), k))
        return r, nrm.value

    def sweep(self, b, w, level=0):
        """One multicolour box sweep, in place on w (returns w)."""
        (bp, k), (wp, _) = self._p(b), self._p(w)
        self._chk(self._L.ibmg_sweep(self._h, level, bp, wp, k))
        return w

    def v_cycle(self, b):
        z = _empty_like(b, self._size(0))
        (bp, k), (zp, _) = self._p(b), self._p(z)
        self._chk(self._L.ibmg_vcycle(self._h, bp, zp, k))
        return z

    def coarsest_solve(self, b):
        x = _empty_like(b, self._size(self.num_levels - 1))
        (bp, k), (xp, _) = self._p(b), self._p(x)
        self._chk(self._L.ibmg_coarse_solve(self._h, bp, xp, k))
        return x

    def restrict_saddle(self, rf, level=0):
        rc = _empty_like(rf, self._size(level + 1))
        (fp, k), (cp, _) = self._p(rf), self._p(rc)
        self._chk(self._L.ibmg_restrict(self._h, level, fp, cp, k))
        return rc

    def prolong_saddle_add(self, ec, wf, level=0):
        (ep, k), (wp, _) = self._p(ec), self._p(wf)
        self._chk(self._L.ibmg_prolong_add(self._h, level, ep, wp, k))
        return wf

    def big_blocks(self, level=0):
        n = self.level_n(level)
        f = np.zeros((n // 4) * (n // 4), np.int32)
        cnt = self._L.ibmg_big_blocks(self._h, level, f.ctypes.data)
        if cnt < 0:
            raise ValueError("big_blocks: bad level")
        return f.reshape(n // 4, n // 4)

    def elasticity(self, level=0):
        """Assembled E'_level velocity block as (rows, cols, vals) host triplets."""
        nnz = self._L.ibmg_elasticity_triplets(self._h, level, None, None, None, 0)
        if nnz < 0:
            raise ValueError("elasticity: bad level")
        r = np.empty(nnz, np.int32)
        c = np.empty(nnz, np.int32)
        v = np.empty(nnz, np.float64)
        if nnz:
            self._L.ibmg_elasticity_triplets(self._h, level, r.ctypes.data, c.ctypes.data, v.ctypes.data, nnz)
        return r, c, v

    def build_rhs(self, u_n):
        b = _empty_like(u_n, 3 * self.N * self.N)
        (up, k), (bp, _) = self._p(u_n), self._p(b)
        self._chk(self._L.ibmg_build_rhs(self._h, up, bp, k))
        return b

    def interpolate(self, u):
        U = _empty_like(u, 2 * self.npts)
        (up, k), (Up, _) = self._p(u), self._p(U)
        self._chk(self._L.ibmg_interpolate(self._h, up, Up, k))
        return U

    def spread(self, F):
        f = _empty_like(F, 2 * self.N * self.N)
        (Fp, k), (fp, _) = self._p(F), self._p(f)
        self._chk(self._L.ibmg_spread(self._h, Fp, fp, k))
        return f

    def gmres_solve(self, b, x=None):
        """FGMRES(restart) with one V-cycle right preconditioner; returns (x, stats)."""
        x = _empty_like(b, self._size(0)) if x is None else x
        st = Stats()
        (bp, k), (xp, _) = self._p(b), self._p(x)
        self._chk(self._L.ibmg_solve(self._h, bp, xp, C.byref(st), k), ok=(0, 2))
        return x, st.as_dict()

    def step_explicit(self, u, p, X):
        """One explicit IB step in place on (u, p, X): forces at
        X^n spread to the right-hand side, Stokes(+mass) solve, X^{n+1} = X^n +
        dt S^T u^{n+1}."""
        if getattr(self, "_implicit", True):
            self.set_scheme(False)
        return self._step(u, p, X)

    def step_implicit(self, u, p, X):
        """One backward-Euler implicit step in place on (u, p, X); returns stats."""
        if not getattr(self, "_implicit", True):
            self.set_scheme(True)
        return self._step(u, p, X)

    def run_simulation(self, n_steps, u, p, X):
        """n_steps consecutive steps in place on (u, p, X) with the state resident on the device
        between them (run_simulation); returns the per-step stats of the steps taken."""
        st = (Stats * max(n_steps, 1))()
        done = C.c_int()
        (up, k), (pp, _), (Xp, _) = self._p(u), self._p(p), self._p(X)
        self._chk(self._L.ibmg_run_simulation(self._h, n_steps, up, pp, Xp, st, C.byref(done), k), ok=(0, 2))
        return [st[i].as_dict() for i in range(done.value)]

    def _step(self, u, p, X):
        st = Stats()
        (up, k), (pp, _), (Xp, _) = self._p(u), self._p(p), self._p(X)
        self._chk(self._L.ibmg_step(self._h, up, pp, Xp, C.byref(st), k), ok=(0, 2))
        return st.as_dict()

    def iteration_matrix_spectrum(self, m=30, seed=1):
        """Arnoldi probe of E = I - V(0, A .): returns (ritz, H),
        Ritz values sorted by decreasing modulus; rho = abs(ritz[0])."""
        H = np.zeros((m + 1) * m)
        done = C.c_int()
        self._chk(self._L.ibmg_vcycle_spectrum(self._h, m, seed, H.ctypes.data, C.byref(done)))
        k = done.value
        Hm = H.reshape(m + 1, m)[:k, :k]
        ritz = np.linalg.eigvals(Hm)  # host: eigenvalues of the k x k Hessenberg matrix
        return ritz[np.argsort(-np.abs(ritz))], H.reshape(m + 1, m)[: k + 1, :k]

    @property
    def cluster_level(self):
        """First level run by the 16-CTA cluster kernel, or -1 (cluster path off)."""
        return self._L.ibmg_cluster_level(self._h)

    @property
    def kernel_launches(self):
        return int(self._L.ibmg_kernel_launches(self._h))

    def set_grid_limit(self, max_ctas):
        """Cap the persistent kernels' grids (0 = all SMs) for concurrent contexts."""
        self._chk(self._L.ibmg_set_grid_limit(self._h, int(max_ctas)))

    def profile(self, enable=True):
        """Start (and clear) / stop live per-kernel CUDA-event timing."""
        self._chk(self._L.ibmg_profile(self._h, int(enable)))

    def profile_report(self):
        """{kernel: (total_ms, launches)} accumulated since profile(True)."""
        import json
        n = self._L.ibmg_profile_report(self._h, None, 0)
        buf = C.create_string_buffer(n + 1)
        self._L.ibmg_profile_report(self._h, buf, n + 1)
        return {k: tuple(v) for k, v in json.loads(buf.value.decode()).items()}

    @property
    def stream(self):
        return self._L.ibmg_stream(self._h)


class BatchSystem:
    """`nslots` independent problems of one grid size (64 <= N <= 512) stepped in
    lockstep (C ABI ibmg_batch_*): per slot its own structures;
    step_implicit runs the rebuilds per slot, then one launch per smoother /
    transfer / Krylov phase for all slots.  Each problem's result equals the
    single-context step_implicit's."""

    def __init__(self, N, nslots, rho=1.0, mu=1.0, dt=1e-2, nu1=1, nu2=1, restart=30, max_iters=600,
                 rtol=1e-10, device=0):
        self._L = lib()
        p = Params(N, rho, mu, dt, nu1, nu2, restart, max_iters, rtol, 4, device)
        h = C.c_void_p()
        rc = self._L.ibmg_batch_create(C.byref(p), int(nslots), C.byref(h))
        if rc != 0 or not h.value:
            raise RuntimeError(f"ibmg_batch_create failed (status {rc})")
        self._h = h
        self.N, self.nslots = N, nslots
        self._in_stream = 0

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._L.ibmg_batch_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def _chk(self, rc, ok=(0,)):
        if rc in ok:
            return rc
        msg = self._L.ibmg_batch_last_error(self._h).decode()
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)

    def set_structures(self, slot, nb, kappa, ds, X):
        nb = np.ascontiguousarray(nb, np.int32)
        kappa = np.ascontiguousarray(kappa, np.float64)
        ds = np.ascontiguousarray(ds, np.float64)
        X = np.ascontiguousarray(X, np.float64).reshape(-1)
        self._chk(self._L.ibmg_batch_set_structures(self._h, int(slot), len(nb), nb.ctypes.data, kappa.ctypes.data,
                                                    ds.ctypes.data, X.ctypes.data))

    @staticmethod
    def _arrays(*lists):
        n = len(lists[0])
        if any(len(x) != n for x in lists):
            raise ValueError("one array of each kind per problem")
        ptrs = [[_ptr(a) for a in arrs] for arrs in lists]
        kinds = {k for arr in ptrs for _, k in arr}
        if len(kinds) != 1:
            raise ValueError("all arrays host or all device")
        return n, kinds.pop(), [(C.c_void_p * n)(*[pt for pt, _ in a]) for a in ptrs]

    def step_implicit(self, us, ps, Xs):
        """One implicit step of slots 0..len(us)-1 in place on the per-problem
        (u, p, X) arrays (all numpy, or all CUDA tensors); returns the stats."""
        n, kind, arr = self._arrays(us, ps, Xs)
        st = (Stats * n)()
        self._chk(self._L.ibmg_batch_step(self._h, n, arr[0], arr[1], arr[2], st, kind), ok=(0, 2))
        return [s.as_dict() for s in st]

    def prepare(self, us, Xs):
        """Phase 1 of step_implicit (upload, rebuild at X^n, RHS); releases the
        GIL, so another thread can solve another batch meanwhile."""
        n, kind, arr = self._arrays(us, Xs)
        self._prep = (arr, kind)
        self._chk(self._L.ibmg_batch_prepare(self._h, n, arr[0], arr[1], kind))

    def solve(self, us, ps, Xs):
        """Phase 2 of step_implicit for the prepared slots; returns the stats."""
        n, kind, arr = self._arrays(us, ps, Xs)
        st = (Stats * n)()
        self._chk(self._L.ibmg_batch_solve(self._h, n, arr[0], arr[1], arr[2], st, kind), ok=(0, 2))
        return [s.as_dict() for s in st]

    @property
    def kernel_launches(self):
        return int(self._L.ibmg_batch_kernel_launches(self._h))


def slab_plan(N, nslabs, min_rows=64, min_cells=1 << 16, coarsest_n=4):
    """(la, rows) of the slab partition (host-only, no GPU): la = number of
    distributed levels, rows[r][l] = (y0, y1) owned by slab r on level l."""
    L = lib()
    nlev = int(np.log2(N // coarsest_n)) + 1
    rows = np.zeros((nslabs, nlev, 2), np.int32)
    la = L.ibmg_slab_plan(N, coarsest_n, nslabs, min_rows, min_cells, rows.ctypes.data)
    if la < 0:
        raise ValueError("slab_plan: invalid arguments")
    return la, rows


class SlabGroup:
    """One problem slab-partitioned over `nslabs` contexts:
    y-slabs of the fine grid on `devices` (slabs may share a GPU), halo
    exchange + seam merge after every colour pass, agglomerated coarse levels,
    FGMRES dots allreduced in rank order.  Host (numpy) whole-grid vectors."""

    def __init__(self, N, nslabs, devices=None, rho=1.0, mu=1.0, dt=1e-2, nu1=1, nu2=1, restart=30,
                 max_iters=600, rtol=1e-10, min_rows=64, min_cells=1 << 16, nccl=None):
        """nccl=(rank, device, unique_id bytes): this process holds slab `rank`
        of an NCCL group of `nslabs` ranks (see nccl_group); otherwise all
        slabs live in this process on `devices` (default: all on GPU 0)."""
        self._L = lib()
        h = C.c_void_p()
        if nccl is not None:
            rank, device, uid = nccl
            p = Params(N, rho, mu, dt, nu1, nu2, restart, max_iters, rtol, 4, device)
            buf = C.create_string_buffer(bytes(uid), 128)
            rc = self._L.ibmg_group_create_nccl(C.byref(p), rank, nslabs, buf, min_rows, min_cells, C.byref(h))
        else:
            p = Params(N, rho, mu, dt, nu1, nu2, restart, max_iters, rtol, 4, 0 if devices is None else devices[0])
            dev = (C.c_int * nslabs)(*(devices if devices is not None else [0] * nslabs))
            rc = self._L.ibmg_group_create(C.byref(p), nslabs, dev, min_rows, min_cells, C.byref(h))
        if rc != 0 or not h.value:
            raise RuntimeError(f"slab group creation failed (status {rc})")
        self._h = h
        self.N, self.nslabs, self.npts = N, nslabs, 0

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._L.ibmg_group_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def _chk(self, rc, ok=(0,)):
        if rc in ok:
            return rc
        msg = self._L.ibmg_group_last_error(self._h).decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)

    @staticmethod
    def nccl_unique_id():
        buf = C.create_string_buffer(128)
        if lib().ibmg_nccl_unique_id(buf) != 0:
            raise RuntimeError("ncclGetUniqueId failed")
        return buf.raw

    @classmethod
    def nccl_group(cls, N, device=None, **kw):
        """One slab per torch.distributed rank (torchrun): rank 0 makes the NCCL
        id, every rank receives it through the process group's broadcast."""
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        obj = [cls.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        dev = int(os.environ.get("LOCAL_RANK", "0")) if device is None else device
        return cls(N, world, nccl=(rank, dev, obj[0]), **kw)

    @property
    def distributed_levels(self):
        return self._L.ibmg_group_distributed_levels(self._h)

    @property
    def cluster_level(self):
        """First level run by the 16-CTA cluster kernel, or -1 (cluster path off)."""
        return self._L.ibmg_cluster_level(self._h)

    @property
    def kernel_launches(self):
        return int(self._L.ibmg_group_kernel_launches(self._h))

    @property
    def exchanges(self):
        return int(self._L.ibmg_group_exchanges(self._h))

    def set_structures(self, nb, kappa, ds, X):
        nb = np.ascontiguousarray(nb, np.int32)
        kappa = np.ascontiguousarray(kappa, np.float64)
        ds = np.ascontiguousarray(ds, np.float64)
        X = np.ascontiguousarray(X, np.float64).reshape(-1)
        self._chk(self._L.ibmg_group_set_structures(self._h, len(nb), nb.ctypes.data, kappa.ctypes.data,
                                                    ds.ctypes.data, X.ctypes.data))
        self.npts = int(nb.sum())
        return self

    @classmethod
    def from_problem(cls, prob, nslabs, **kw):
        g = cls(prob.N, nslabs, rho=prob.rho, mu=prob.mu, dt=prob.dt, **kw)
        return g.set_structures(prob.nb, prob.kappa, prob.ds, prob.X)

    def sweep(self, b, w, level=0):
        b = np.ascontiguousarray(b, np.float64)
        w = np.array(w, np.float64)
        self._chk(self._L.ibmg_group_sweep(self._h, level, b.ctypes.data, w.ctypes.data))
        return w

    def v_cycle(self, b):
        b = np.ascontiguousarray(b, np.float64)
        z = np.empty_like(b)
        self._chk(self._L.ibmg_group_vcycle(self._h, b.ctypes.data, z.ctypes.data))
        return z

    def gmres_solve(self, b):
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty_like(b)
        st = Stats()
        self._chk(self._L.ibmg_group_solve(self._h, b.ctypes.data, x.ctypes.data, C.byref(st)), ok=(0, 2))
        return x, st.as_dict()

    def step_implicit(self, u, p, X):
        st = Stats()
        for a in (u, p, X):
            if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]):
                raise ValueError("group step: C-contiguous float64 numpy arrays")
        self._chk(self._L.ibmg_group_step(self._h, u.ctypes.data, p.ctypes.data, X.ctypes.data, C.byref(st)),
                  ok=(0, 2))
        return st.as_dict()


def fiber_force_unit(X, nb, ds):
    """A_f X per unit stiffness (fiber.cpp:34-55): (X_{k+1} - 2 X_k + X_{k-1}) / ds_m^2
    on each closed membrane; X is (npts, 2)."""
    X = np.asarray(X, np.float64).reshape(-1, 2)
    F = np.empty_like(X)
    o = 0
    for m, d in zip(nb, ds):
        Xm = X[o:o + m]
        F[o:o + m] = (np.roll(Xm, -1, axis=0) - 2.0 * Xm + np.roll(Xm, 1, axis=0)) / (d * d)
        o += m
    return F


def estimate_alpha_exp(sys_, tol=1e-6, max_iter=1000, seed=0):
    """alpha_exp = 2 / |lambda_max| of M X = interpolate(stokes_solve(spread(A_f X)))
    by power iteration (§4.1, Table 1): the critical
    dt * kappa of the explicit IB scheme.  The Stokes(+mass) solves are FGMRES on
    the GPU with E' off; A_f is the unit-stiffness spring operator at the
    context's current X.  Returns (alpha_exp, lambda_max, iterations)."""
    was = getattr(sys_, "_implicit", True)
    sys_.set_scheme(False)
    try:
        nb, ds = sys_._nb, sys_._ds
        X0 = sys_._X_host.reshape(-1, 2)
        N = sys_.N
        rng = np.random.default_rng(seed)
        x = rng.uniform(-1.0, 1.0, X0.shape)
        x /= np.linalg.norm(x)
        lam_prev = None
        for it in range(1, max_iter + 1):
            F = fiber_force_unit(x, nb, ds)
            f = sys_.spread(F.reshape(-1))
            b = np.concatenate([f, np.zeros(N * N)])
            u, _ = sys_.gmres_solve(b)
            y = sys_.interpolate(u[: 2 * N * N]).reshape(-1, 2)
            lam = float(np.sum(x * y))
            nrm = np.linalg.norm(y)
            if nrm == 0.0:
                raise RuntimeError("estimate_alpha_exp: zero operator")
            x = y / nrm
            if lam_prev is not None and abs(lam - lam_prev) <= tol * abs(lam):
                return 2.0 / abs(lam), lam, it
            lam_prev = lam
        raise RuntimeError("estimate_alpha_exp: power iteration did not converge")
    finally:
        sys_.set_scheme(was)
