"""Slab partition at scale: one implicit step of a config through the one-GPU
context and through a SlabGroup of P slabs (sharing GPU 0, or spread over the
visible GPUs with --spread), then the relative differences of u, p, X^{n+1}
and the iteration counts.  The contexts run one after the other (C4 needs
~115 GB for the single context, ~65 GB per slab).

  python tools/slab_check.py --config C4 --slabs 2
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1311_5614_b200 import configs  # noqa: E402
from paper_1311_5614_b200.ibmg import SaddleSystem, SlabGroup  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4", choices=["C2", "C3", "C4"])
    ap.add_argument("--slabs", type=int, default=2)
    ap.add_argument("--spread", action="store_true", help="slab r on GPU r % device_count")
    ap.add_argument("--min-cells", type=int, default=1 << 16)
    ap.add_argument("--skip-single", action="store_true")
    ap.add_argument("--single-only", action="store_true")
    a = ap.parse_args()
    prob = {"C2": lambda: configs.config2(1e6), "C3": configs.config3, "C4": configs.config4}[a.config]()
    n = prob.N
    out = {"config": a.config, "N": n, "npts": prob.npts, "slabs": a.slabs}
    res = {}
    if not a.skip_single:
        s = SaddleSystem.from_problem(prob)
        u, p, X = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
        t0 = time.perf_counter()
        st = s.step_implicit(u, p, X)
        out["single"] = dict(st, wall_s=time.perf_counter() - t0)
        res["single"] = (u, p, X)
        s.close()
        del s
    if a.single_only:
        print(json.dumps(out))
        return
    devs = None
    if a.spread:
        import torch
        nd = torch.cuda.device_count()
        devs = [r % nd for r in range(a.slabs)]
    g = SlabGroup(n, a.slabs, devices=devs, rho=prob.rho, mu=prob.mu, dt=prob.dt, min_cells=a.min_cells)
    g.set_structures(prob.nb, prob.kappa, prob.ds, prob.X)
    u, p, X = np.zeros(2 * n * n), np.zeros(n * n), prob.X.reshape(-1).copy()
    t0 = time.perf_counter()
    st = g.step_implicit(u, p, X)
    out["group"] = dict(st, wall_s=time.perf_counter() - t0, distributed_levels=g.distributed_levels,
                        exchanges=g.exchanges, launches=g.kernel_launches, devices=devs or [0] * a.slabs)
    if "single" in res:
        us, ps, Xs = res["single"]
        out["rel_u"], out["rel_p"], out["rel_X"] = rel(u, us), rel(p, ps), rel(X, Xs)
        out["iters_diff"] = out["group"]["iters"] - out["single"]["iters"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
