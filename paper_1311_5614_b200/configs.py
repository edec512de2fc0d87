"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference ships no inputs; these generators are the
single source of the structures both the GPU path and the CPU oracle consume.
Decisions: D4 ds^2 quadrature, D5 equal-arclength ellipse
points, D9 min-separation r_i + r_j + 4h (periodic distance), C4 orientation
U[0, pi), C5 per-problem seed 5 + index.  numpy's default_rng (PCG64) stands
in for the survey's mt19937_64 suggestion; the draw order is documented in
each function.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Problem:
    name: str
    N: int
    rho: float
    mu: float
    dt: float
    nb: list = field(default_factory=list)      # points per membrane
    kappa: list = field(default_factory=list)   # stiffness per membrane
    ds: list = field(default_factory=list)      # Lagrangian spacing per membrane
    X: np.ndarray = None                        # (sum nb, 2) float64, membrane-major
    steps: int = 1

    @property
    def npts(self) -> int:
        return int(sum(self.nb))

    @property
    def dof(self) -> int:
        return 3 * self.N * self.N


def _arclength_series(a: float, b: float, modes: int = 64):
    """Fourier series of s'(t) = sqrt(a^2 sin^2 t + b^2 cos^2 t) (even, pi-periodic)."""
    m = 4 * modes
    t = 2 * np.pi * np.arange(m) / m
    sp = np.sqrt((a * np.sin(t)) ** 2 + (b * np.cos(t)) ** 2)
    c = np.fft.rfft(sp) / m
    return c[: modes + 1]


def ellipse_points(cx, cy, a, b, nb, theta0=0.0, rot=0.0):
    """nb points at equal arclength on an ellipse (D5); returns (X (nb,2), ds, L).

    The arclength s(t) = int_0^t sqrt(a^2 sin^2 + b^2 cos^2) is evaluated from
    its Fourier series (spectrally accurate) and s(t_q) = q L / nb is solved by
    vectorised Newton iteration to machine precision."""
    c = _arclength_series(a, b)
    k = np.arange(1, len(c))
    L = 2 * np.pi * c[0].real
    target = np.arange(nb) * (L / nb)
    t = 2 * np.pi * np.arange(nb) / nb
    coef = 2 * c[1:] / (1j * k)
    for _ in range(60):
        e = np.exp(1j * np.outer(t, k))
        S = c[0].real * t + ((e - 1.0) @ coef).real
        f = S - target
        t = t - f / np.sqrt((a * np.sin(t)) ** 2 + (b * np.cos(t)) ** 2)
        if np.max(np.abs(f)) < 1e-15 * max(1.0, L):
            break
    th = t + theta0
    x = a * np.cos(th)
    y = b * np.sin(th)
    cr, sr = math.cos(rot), math.sin(rot)
    X = np.stack([cx + cr * x - sr * y, cy + sr * x + cr * y], axis=1)
    return X, L / nb, L


def _periodic_dist(p, q):
    d = np.abs(np.asarray(p) - np.asarray(q))
    d = np.minimum(d, 1.0 - d)
    return float(np.hypot(d[0], d[1]))


def config1() -> Problem:
    X, ds, _ = ellipse_points(0.5, 0.5, 0.3, 0.15, 128)
    return Problem("C1", 64, 1.0, 1.0, 1e-2, [128], [1e2], [ds], X, steps=1)


def config2(kappa: float = 1e2, N: int = 256, nb: int = 512) -> Problem:
    X, ds, _ = ellipse_points(0.5, 0.5, 0.3, 0.15, nb)
    return Problem(f"C2(kappa={kappa:g})", N, 1.0, 1.0, 1e-3, [nb], [kappa], [ds], X, steps=10)


def _random_membranes(N, count, seed, rlo, rhi, aspect, kap_lo, kap_hi):
    """Draw order per membrane: centre x, centre y, radius, [aspect, orientation],
    log10 kappa; rejection on the periodic min-separation r_i + r_j + 4h."""
    rng = np.random.default_rng(seed)
    h = 1.0 / N
    placed = []
    tries = 0
    while len(placed) < count:
        tries += 1
        if tries > 200000:
            raise RuntimeError("could not place membranes")
        c = rng.uniform(0.0, 1.0, size=2)
        r = rng.uniform(rlo, rhi)
        ar, rot = (rng.uniform(1.0, 2.0), rng.uniform(0.0, np.pi)) if aspect else (1.0, 0.0)
        lk = rng.uniform(kap_lo, kap_hi)
        if any(_periodic_dist(c, p[0]) < r + p[1] + 4 * h for p in placed):
            continue
        placed.append((c, r, ar, rot, 10.0 ** lk))
    nbs, kaps, dss, Xs = [], [], [], []
    for c, r, ar, rot, kap in placed:
        a, b = r, r / ar
        # perimeter first, then nb = round(perimeter / (h/2)) (circles: 2 pi r / (h/2))
        L = 2 * np.pi * _arclength_series(a, b)[0].real
        nb = int(round(L / (h / 2)))
        X, ds, _ = ellipse_points(c[0], c[1], a, b, nb, rot=rot)
        nbs.append(nb)
        kaps.append(kap)
        dss.append(ds)
        Xs.append(X)
    return nbs, kaps, dss, np.concatenate(Xs, axis=0)


def config3() -> Problem:
    nbs, kaps, dss, X = _random_membranes(1024, 16, 0, 0.03, 0.06, False, 3.0, 6.0)
    return Problem("C3", 1024, 1.0, 1.0, 1e-3, nbs, kaps, dss, X, steps=5)


def config4(N: int = 8192) -> Problem:
    nbs, kaps, dss, X = _random_membranes(N, 256, 1, 0.005, 0.015, True, 3.0, 6.0)
    return Problem("C4", N, 1.0, 1.0, 1e-4, nbs, kaps, dss, X, steps=1)


def config5_problem(index: int, N: int = 256, nb: int = 512) -> Problem:
    """Problem `index` of the C5 batch: seed 5 + index; draws a, b ~ U[0.1, 0.35],
    log10 kappa ~ U[1, 6]."""
    rng = np.random.default_rng(5 + index)
    a, b = rng.uniform(0.1, 0.35, size=2)
    kap = 10.0 ** rng.uniform(1.0, 6.0)
    X, ds, _ = ellipse_points(0.5, 0.5, a, b, nb)
    return Problem(f"C5[{index}]", N, 1.0, 1.0, 1e-3, [nb], [kap], [ds], X, steps=1)


def small_problem(N=32, nb=64, kappa=1e2, dt=1e-2, a=0.3, b=0.15, cx=0.5, cy=0.5, rot=0.0) -> Problem:
    X, ds, _ = ellipse_points(cx, cy, a, b, nb, rot=rot)
    return Problem(f"small(N={N})", N, 1.0, 1.0, dt, [nb], [kappa], [ds], X, steps=1)


# ---- paper-reproduction mode

#: Table 1: largest stable alpha = gamma dt of the explicit scheme.
PAPER_ALPHA_EXP = {32: 6.09, 64: 3.93, 128: 2.82, 256: 2.28}


@dataclass
class AnnulusMesh:
    """Thick fiber mesh (fiber.hpp:36-50): node (k, l) at X[k + l * m1], closed in s1."""
    N: int
    m1: int
    m2: int
    ds: float
    X: np.ndarray  # (m1 * m2, 2)


def paper_annulus(N: int, centre=(0.5, 0.5), r: float = 0.25, w: float = 1.0 / 16) -> AnnulusMesh:
    """The annulus of Eq. 21: X(s1, s2) = centre + (r + s2)(cos(s1/r), sin(s1/r)) with
    M1 = 19N/8 nodes in s1, M2 = 3N/32 + 1 rings across the thickness w and
    ds = 2 pi r / M1."""
    if (19 * N) % 8 or (3 * N) % 32:
        raise ValueError("M1 = 19N/8 and M2 = 3N/32 + 1 must be integers")
    m1, m2 = 19 * N // 8, 3 * N // 32 + 1
    ds = 2 * math.pi * r / m1
    k = np.arange(m1)
    X = np.empty((m2, m1, 2))
    for l in range(m2):
        rad = r + l * (w / (m2 - 1))
        X[l, :, 0] = centre[0] + rad * np.cos(k * ds / r)
        X[l, :, 1] = centre[1] + rad * np.sin(k * ds / r)
    return AnnulusMesh(N, m1, m2, ds, X.reshape(-1, 2))
