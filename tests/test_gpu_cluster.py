"""The cluster-resident bottom of the V-cycle (k_cluster_cycle, levels with
n <= 128 in one 16-CTA thread-block cluster, DSMEM; cluster_kernel.cuh;
opt-in with IBMG_CLUSTER=1 at context creation, measured slower than the
default on B200) against the default launch-per-phase path
(k_sweep_df dataflow sweeps, restriction / prolongation launches,
single-CTA k_coarse_cycle) and against the CPU oracle.

The partitioned levels relax tiles and big blocks with the same arithmetic as
k_sweep_df; the replicated levels and the restrictions sum E' rows in a
different order than the old kernels, so the two paths agree to round-off.
"""
import os

import numpy as np
import pytest

from helpers import rand, rel
from paper_1311_5614_b200 import configs
from paper_1311_5614_b200.ibmg import SaddleSystem
import oracle as O

pytestmark = pytest.mark.gpu


def make(prob, cluster):
    old = os.environ.get("IBMG_CLUSTER")
    os.environ["IBMG_CLUSTER"] = "1" if cluster else "0"
    try:
        return SaddleSystem.from_problem(prob)
    finally:
        if old is None:
            del os.environ["IBMG_CLUSTER"]
        else:
            os.environ["IBMG_CLUSTER"] = old


CASES = {
    "C1": configs.config1,                       # N = 64: the whole V-cycle in the cluster
    "N128": lambda: configs.config2(1e4, N=128, nb=256),  # N = 128: ditto, two partitioned levels
    "C2k6": lambda: configs.config2(1e6),        # N = 256: level 0 outside, 128..4 inside
    "C3": configs.config3,                       # 16 membranes: dense coarse levels
}


@pytest.mark.parametrize("name", list(CASES))
def test_cluster_vcycle_matches_old_path_and_oracle(name):
    prob = CASES[name]()
    g1, g0 = make(prob, True), make(prob, False)
    n = prob.N
    b = g1.build_rhs(rand(2 * n * n, seed=3))
    z1, z0 = g1.v_cycle(b), g0.v_cycle(b)
    assert rel(z1, z0) < 1e-11, rel(z1, z0)
    if n <= 256:
        zo = O.Oracle(prob, threads=os.cpu_count() or 1).vcycle(b)
        assert rel(z1, zo) < 1e-10, rel(z1, zo)
    # bitwise repeatable
    assert np.array_equal(z1, g1.v_cycle(b))
    g1.close()
    g0.close()


@pytest.mark.parametrize("name", ["C1", "C2k6", "C3"])
def test_cluster_step_matches_old_path(name):
    prob = CASES[name]()
    n = prob.N
    out = []
    for cl in (True, False):
        g = make(prob, cl)
        u, p, X = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
        st = g.step_implicit(u, p, X)
        out.append((u, p, X, st))
        g.close()
    (u1, p1, X1, s1), (u0, p0, X0, s0) = out
    assert s1["converged"] and s0["converged"]
    assert abs(s1["iters"] - s0["iters"]) <= 1, (s1["iters"], s0["iters"])
    assert rel(u1, u0) < 1e-9 and rel(p1, p0) < 1e-9 and rel(X1, X0) < 1e-12


def test_cluster_path_is_selected():
    """IBMG_CLUSTER=1 runs the cluster kernel (fewer launches than the default
    path for N = 256); the default context does not."""
    prob = CASES["C2k6"]()
    g1, g0 = make(prob, True), make(prob, False)
    b = g1.build_rhs(rand(2 * prob.N ** 2, seed=5))
    l1, l0 = g1.kernel_launches, g0.kernel_launches
    g1.v_cycle(b)
    g0.v_cycle(b)
    assert g1.kernel_launches - l1 < g0.kernel_launches - l0
    g1.profile(True)
    g1.v_cycle(b)
    assert "k_cluster_cycle" in g1.profile_report()
    assert g1.cluster_level >= 0 and g0.cluster_level == -1
    g1.close()
    g0.close()
