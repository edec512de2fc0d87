"""Mesh and field text formats (reference fiber.cpp:142-166,
SPEC.md:203, 666): checkpoints and external verification.

FiberMesh: a header line "m1 m2 ds periodic_s1" then one line "k l x y" per
node, l-major (write_fiber_mesh / read_fiber_mesh, fiber.cpp:142-166), numbers
at 17 significant digits.  A structure set (several closed membranes) is the
concatenation of one such block per membrane.  Field snapshot:
one line "field i j value" per DOF (field 0 u, 1 v, 2 p; x fastest), after a
header "N".  A checkpoint is a field snapshot of (u, p) plus the mesh blocks
of X.  Host-side only; nothing here touches the device.
"""
from __future__ import annotations

import numpy as np


def _g(x: float) -> str:
    return "%.17g" % x  # std::ostream precision(17), default float format


def write_fiber_mesh(f, X, ds, periodic=True):
    """One closed membrane (m2 = 1): X (m1, 2)."""
    X = np.asarray(X, np.float64).reshape(-1, 2)
    f.write(f"{X.shape[0]} 1 {_g(ds)} {1 if periodic else 0}\n")
    for k, (x, y) in enumerate(X):
        f.write(f"{k} 0 {_g(x)} {_g(y)}\n")


class _Stop(Exception):
    pass


def read_fiber_mesh(f, stop=None):
    """Next mesh block of a stream: (X (m1 * m2, 2), ds, periodic, m1, m2), or None at EOF
    (or at a line equal to `stop`, which is consumed)."""
    head = ""
    while not head.strip():
        head = f.readline()
        if head == "":
            return None
    if stop is not None and head.strip() == stop:
        raise _Stop
    parts = head.split()
    if len(parts) != 4:
        raise RuntimeError("read_fiber_mesh: bad header")
    m1, m2, ds, per = int(parts[0]), int(parts[1]), float(parts[2]), int(parts[3])
    X = np.empty((m1 * m2, 2))
    for _ in range(m1 * m2):
        t = f.readline().split()
        if len(t) != 4:
            raise RuntimeError("read_fiber_mesh: bad node line")
        k, l = int(t[0]), int(t[1])
        if not (0 <= k < m1 and 0 <= l < m2):
            raise RuntimeError("read_fiber_mesh: node index out of range")
        X[l * m1 + k] = (float(t[2]), float(t[3]))
    return X, ds, per != 0, m1, m2


def write_structures(f, nb, ds, X):
    X = np.asarray(X, np.float64).reshape(-1, 2)
    o = 0
    for m, d in zip(nb, ds):
        write_fiber_mesh(f, X[o:o + m], d)
        o += m


def read_structures(f, stop=None):
    """Mesh blocks until EOF (or until a `stop` line, consumed; then
    f.stopped is not set but the caller knows the section that follows)."""
    nb, ds, Xs = [], [], []
    while True:
        try:
            blk = read_fiber_mesh(f, stop)
        except _Stop:
            break
        if blk is None:
            break
        X, d, _, m1, m2 = blk
        nb.append(m1 * m2)
        ds.append(d)
        Xs.append(X)
    return nb, ds, (np.concatenate(Xs) if Xs else np.zeros((0, 2)))


def write_field(f, x, N):
    """Saddle vector [u | v | p] (3 N^2) as 'field i j value' lines."""
    x = np.asarray(x, np.float64).reshape(3, N, N)
    f.write(f"{N}\n")
    for fld in range(3):
        for j in range(N):
            for i in range(N):
                f.write(f"{fld} {i} {j} {_g(x[fld, j, i])}\n")


def read_field(f):
    N = int(f.readline())
    x = np.empty((3, N, N))
    for _ in range(3 * N * N):
        t = f.readline().split()
        fld, i, j = int(t[0]), int(t[1]), int(t[2])
        x[fld, j, i] = float(t[3])
    return x.reshape(-1), N


def save_checkpoint(path, u, p, X, nb, ds, N, kappa=None, rho=None, mu=None, dt=None):
    """Field, then the membranes in the reference write_fiber_mesh format (byte-
    identical blocks), then a trailing 'params' section with what a restart
    needs beyond the meshes: the solver parameters rho, mu, dt and one kappa
    per membrane ('nan' where not given).  The reference format has no such
    section; read_fiber_mesh stops at it (not a mesh header)."""
    nmem = len(nb)
    kap = [float("nan")] * nmem if kappa is None else [float(k) for k in np.asarray(kappa).reshape(-1)]
    if len(kap) != nmem:
        raise ValueError("one kappa per membrane")
    with open(path, "w") as f:
        write_field(f, np.concatenate([np.asarray(u).reshape(-1), np.asarray(p).reshape(-1)]), N)
        write_structures(f, nb, ds, X)
        f.write("params\n")
        f.write(" ".join(_g(float("nan") if v is None else float(v)) for v in (rho, mu, dt)) + "\n")
        f.write(f"{nmem}\n")
        for k in kap:
            f.write(_g(k) + "\n")


def load_checkpoint(path, with_params=False):
    """(u, p, X, nb, ds, N), plus {'kappa', 'rho', 'mu', 'dt'} when with_params."""
    with open(path) as f:
        x, N = read_field(f)
        nb, ds, X = read_structures(f, stop="params")
        prm = {"kappa": None, "rho": None, "mu": None, "dt": None}
        rest = f.readline()
        if rest.strip():  # the params section follows (its header line was consumed)
            rho, mu, dt = (float(t) for t in rest.split())
            nmem = int(f.readline())
            prm = {"kappa": np.array([float(f.readline()) for _ in range(nmem)]), "rho": rho, "mu": mu, "dt": dt}
    out = (x[: 2 * N * N].copy(), x[2 * N * N:].copy(), X, nb, ds, N)
    return out + (prm,) if with_params else out
