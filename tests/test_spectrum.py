"""Arnoldi probe of the multigrid iteration matrix (§5.2):
E x = x - V(0, A x) on the mean-zero-pressure subspace.  The GPU probe's
dominant Ritz value is checked against the dense spectrum of E built column
by column with the CPU oracle's own V-cycle and operator (SPEC: "recovers the
top moduli ... (oracle)")."""
import numpy as np
import pytest

from paper_1311_5614_b200 import configs
from paper_1311_5614_b200.ibmg import SaddleSystem
import oracle as O

pytestmark = pytest.mark.gpu


def dense_E(o, N):
    n2 = N * N
    m = 3 * n2

    def proj(x):
        x = x.copy()
        x[2 * n2:] -= x[2 * n2:].mean()
        return x

    E = np.empty((m, m))
    for k in range(m):
        e = np.zeros(m)
        e[k] = 1.0
        x = proj(e)
        E[:, k] = x - proj(o.vcycle(o.apply(x)))
    return E


@pytest.mark.parametrize("kappa", [0.0, 1e3])
def test_dominant_ritz_value_matches_dense_oracle(kappa):
    N = 16
    prob = configs.small_problem(N=N, nb=32, kappa=max(kappa, 0.0))
    g = SaddleSystem.from_problem(prob)
    o = O.Oracle(prob)
    lam = np.linalg.eigvals(dense_E(o, N))
    rho_dense = np.abs(lam).max()
    ritz, H = g.iteration_matrix_spectrum(m=30, seed=3)
    rho = abs(ritz[0])
    assert H.shape == (31, 30)
    # 30 Arnoldi steps on a 768-dim non-normal operator: Ritz convergence ~1e-5
    assert abs(rho - rho_dense) <= 1e-4 * rho_dense, (rho, rho_dense)
    assert 0.0 < rho < 1.0  # a convergent V-cycle


def splitmix_uniform(m, seed):
    """The probe's start vector (ibmg.cu ibmg_vcycle_spectrum): splitmix64 -> U[-1, 1)."""
    out = np.empty(m)
    z = seed
    M64 = (1 << 64) - 1
    for i in range(m):
        z = (z + 0x9E3779B97F4A7C15) & M64
        t = z
        t = ((t ^ (t >> 30)) * 0xBF58476D1CE4E5B9) & M64
        t = ((t ^ (t >> 27)) * 0x94D049BB133111EB) & M64
        t ^= t >> 31
        out[i] = (t >> 11) * (2.0 / 9007199254740992.0) - 1.0
    return out


def test_hessenberg_matches_oracle_arnoldi():
    """Same start vector, same CGS2 Arnoldi on the oracle's V-cycle and operator:
    the GPU Hessenberg matrix agrees entry by entry (parity of the probe)."""
    N, m = 16, 12
    prob = configs.small_problem(N=N, nb=32, kappa=1e3)
    g = SaddleSystem.from_problem(prob)
    o = O.Oracle(prob)
    n2 = N * N

    def proj(x):
        x = x.copy()
        x[2 * n2:] -= x[2 * n2:].mean()
        return x

    v = proj(splitmix_uniform(3 * n2, 5))
    V = [v / np.linalg.norm(v)]
    Ho = np.zeros((m + 1, m))
    for j in range(m):
        w = proj(V[j] - proj(o.vcycle(o.apply(V[j]))))
        B = np.array(V)
        h1 = B @ w
        w = w - B.T @ h1
        h2 = B @ w
        w = w - B.T @ h2
        Ho[: j + 1, j] = h1 + h2
        Ho[j + 1, j] = np.linalg.norm(w)
        V.append(w / Ho[j + 1, j])
    _, Hg = g.iteration_matrix_spectrum(m=m, seed=5)
    assert np.abs(Hg - Ho).max() <= 1e-9 * np.abs(Ho).max()


def test_probe_is_seed_independent_and_deterministic():
    prob = configs.small_problem(N=32, nb=64, kappa=1e2)
    g = SaddleSystem.from_problem(prob)
    r1, _ = g.iteration_matrix_spectrum(m=30, seed=1)
    r1b, _ = g.iteration_matrix_spectrum(m=30, seed=1)
    r2, _ = g.iteration_matrix_spectrum(m=30, seed=7)
    assert np.array_equal(r1, r1b)
    # clustered dominant moduli at 3072 DOFs: 30-step estimates agree to ~1%
    assert abs(abs(r1[0]) - abs(r2[0])) <= 2e-2 * abs(r1[0])


def test_rho_predicts_stationary_convergence():
    """iterations of w <- w + V(0, b - A w) to 1e-6 ~ log(1e-6)/log(rho)
    (the probe's operator is exactly that iteration's error propagation)."""
    N = 32
    prob = configs.small_problem(N=N, nb=64, kappa=1e2)
    g = SaddleSystem.from_problem(prob)
    rho = abs(g.iteration_matrix_spectrum(m=30, seed=2)[0][0])
    b = g.build_rhs(np.random.default_rng(0).uniform(-1, 1, 2 * N * N))
    w = np.zeros(3 * N * N)
    r0 = np.linalg.norm(b)
    it = 0
    while it < 200:
        r, nrm = g.residual(b, w)
        if nrm <= 1e-6 * r0:
            break
        w = w + g.v_cycle(r)
        it += 1
    pred = np.log(1e-6) / np.log(rho)
    assert 0.7 * pred - 2 <= it <= 1.3 * pred + 2, (it, pred, rho)
