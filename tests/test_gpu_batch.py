"""The lockstep batch (ibmg_batch_*, batch.cuh) against the single-context
step: every problem's result is bitwise the same (the batched launches run
each problem's arithmetic in the same order; only the interleaving of the
problems' tasks differs), with the same iteration counts, and the oracle
agrees within the north_star bar."""
import os

import numpy as np
import pytest

from helpers import rel
from paper_1311_5614_b200 import configs
from paper_1311_5614_b200.ibmg import BatchSystem, SaddleSystem
import oracle as O

pytestmark = pytest.mark.gpu


def run_single(probs):
    g = SaddleSystem(256, 1.0, 1.0, 1e-3)
    out = []
    for pr in probs:
        g.set_structures(pr.nb, pr.kappa, pr.ds, pr.X)
        n = pr.N
        u, p, X = np.zeros(2 * n * n), np.zeros(n * n), pr.X.reshape(-1).copy()
        st = g.step_implicit(u, p, X)
        out.append((u, p, X, st))
    g.close()
    return out


@pytest.mark.parametrize("count,slots", [(6, 6), (5, 8)])
def test_batch_equals_single_context(count, slots):
    probs = [configs.config5_problem(i) for i in (0, 7, 100, 250, 401, 511)[:count]]
    ref = run_single(probs)
    B = BatchSystem(256, slots, 1.0, 1.0, 1e-3)
    for k, pr in enumerate(probs):
        B.set_structures(k, pr.nb, pr.kappa, pr.ds, pr.X)
    n = 256
    us = [np.zeros(2 * n * n) for _ in probs]
    ps = [np.zeros(n * n) for _ in probs]
    Xs = [pr.X.reshape(-1).copy() for pr in probs]
    sts = B.step_implicit(us, ps, Xs)
    for k in range(count):
        u0, p0, X0, s0 = ref[k]
        assert sts[k]["converged"] and sts[k]["iters"] == s0["iters"], (k, sts[k], s0)
        assert np.array_equal(us[k], u0) and np.array_equal(ps[k], p0) and np.array_equal(Xs[k], X0), k
    # a second step of the same batch (epochs, reused tables) stays equal to the single context's second step
    sts2 = B.step_implicit(us, ps, Xs)
    g = SaddleSystem(256, 1.0, 1.0, 1e-3)
    for k, pr in enumerate(probs):
        g.set_structures(pr.nb, pr.kappa, pr.ds, pr.X)
        u, p, X = ref[k][0].copy(), ref[k][1].copy(), ref[k][2].copy()
        s = g.step_implicit(u, p, X)
        assert sts2[k]["iters"] == s["iters"]
        assert np.array_equal(us[k], u) and np.array_equal(Xs[k], X), k
    g.close()
    B.close()


def test_batch_device_arrays_match_oracle():
    import torch
    probs = [configs.config5_problem(i) for i in (3, 44, 300)]
    B = BatchSystem(256, 3, 1.0, 1.0, 1e-3)
    n = 256
    for k, pr in enumerate(probs):
        B.set_structures(k, pr.nb, pr.kappa, pr.ds, pr.X)
    us = [torch.zeros(2 * n * n, dtype=torch.float64, device="cuda") for _ in probs]
    ps = [torch.zeros(n * n, dtype=torch.float64, device="cuda") for _ in probs]
    Xs = [torch.tensor(pr.X.reshape(-1), dtype=torch.float64, device="cuda") for pr in probs]
    sts = B.step_implicit(us, ps, Xs)
    for k, pr in enumerate(probs):
        uo, po, Xo, so = O.Oracle(pr, threads=os.cpu_count() or 1).step(np.zeros(2 * n * n), pr.X)
        assert sts[k]["converged"] and abs(sts[k]["iters"] - so["iters"]) <= 2
        assert rel(us[k].cpu().numpy(), uo) < 1e-8 and rel(ps[k].cpu().numpy(), po) < 1e-8
        assert rel(Xs[k].cpu().numpy().reshape(-1, 2), Xo) < 1e-8
    B.close()
