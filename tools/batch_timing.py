"""Phase timing of the lockstep batch (C5 problems): prepare (per-slot
rebuild + RHS on worker threads) and solve (batched FGMRES) of one chunk,
host wall clock after synchronisation.  usage: python tools/batch_timing.py [slots] [chunks]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_5614_b200 import configs  # noqa: E402
from paper_1311_5614_b200.ibmg import BatchSystem  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
nch = int(sys.argv[2]) if len(sys.argv) > 2 else 3
probs = [configs.config5_problem(i) for i in range(S * nch)]
B = BatchSystem(256, S, 1.0, 1.0, 1e-3)
n2 = 65536
us = [torch.zeros(2 * n2, dtype=torch.float64, device="cuda") for _ in range(S)]
ps = [torch.zeros(n2, dtype=torch.float64, device="cuda") for _ in range(S)]
for rep in range(2):
    for c in range(nch):
        ch = probs[c * S:(c + 1) * S]
        Xs = []
        t0 = time.perf_counter()
        for k, pr in enumerate(ch):
            B.set_structures(k, pr.nb, pr.kappa, pr.ds, pr.X)
            us[k].zero_()
            Xs.append(torch.tensor(pr.X.reshape(-1), dtype=torch.float64, device="cuda"))
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        B.prepare(us, Xs)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        sts = B.solve(us, ps, Xs)
        t3 = time.perf_counter()
        its = [s["iters"] for s in sts]
        if rep:
            print(f"chunk {c}: structures {1e3*(t1-t0):.1f} ms, prepare {1e3*(t2-t1):.1f} ms, solve {1e3*(t3-t2):.1f} ms "
                  f"({1e3*(t3-t2)/S:.3f} ms/problem), iters min/mean/max {min(its)}/{np.mean(its):.1f}/{max(its)}",
                  flush=True)
B.close()
