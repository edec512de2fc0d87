"""A/B of one implicit step between two environment settings read at context
creation (e.g. IBMG_CLUSTER=1 vs 0): device ms per step (CUDA events on the
solver stream, inputs in HBM) and the live per-kernel profile of one step.
usage: python tools/ab_step.py CONFIG VAR=a VAR=b [steps]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_5614_b200 import configs  # noqa: E402
from paper_1311_5614_b200.ibmg import SaddleSystem  # noqa: E402

cfg = sys.argv[1]
settings = [a.split("=") for a in sys.argv[2:4]]
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
prob = {"C1": configs.config1, "C2": lambda: configs.config2(1e4), "C2k6": lambda: configs.config2(1e6),
        "C3": configs.config3, "C4": configs.config4, "C5": lambda: configs.config5_problem(7)}[cfg]()
n2 = prob.N ** 2
res = {}
for var, val in settings:
    os.environ[var] = val
    g = SaddleSystem.from_problem(prob)
    st_ = torch.cuda.ExternalStream(g.stream)
    u = torch.zeros(2 * n2, dtype=torch.float64, device="cuda")
    p = torch.zeros(n2, dtype=torch.float64, device="cuda")
    X0 = torch.tensor(prob.X.reshape(-1), dtype=torch.float64, device="cuda")
    X = X0.clone()
    ms, its = [], []
    for s in range(steps + 2):
        u.zero_()
        X.copy_(X0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st_)
        st = g.step_implicit(u, p, X)
        e1.record(st_)
        e1.synchronize()
        if s >= 2:
            ms.append(e0.elapsed_time(e1))
            its.append(st["iters"])
    g.profile(True)
    u.zero_()
    X.copy_(X0)
    g.step_implicit(u, p, X)
    rep = g.profile_report()
    g.profile(False)
    top = sorted(rep.items(), key=lambda kv: -kv[1][0])[:10]
    res[f"{var}={val}"] = {"ms": float(np.median(ms)), "iters": its, "u_norm": float(u.norm()),
                          "profile": {k: [round(v[0], 3), v[1]] for k, v in top}}
    g.close()
print(json.dumps({"config": cfg, **res}, indent=1))
