"""Paper-reproduction mode on the GPU: Table 2 through the C ABI with timings and the
per-level coupling reach (pipeline skew) of the lexicographic dataflow sweep."""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_1311_5614_b200 import configs  # noqa: E402
from paper_1311_5614_b200.paper import PaperSystem  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 64
ORDER = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # 0 lexicographic (the paper), 1 multicolour
mesh = configs.paper_annulus(N)
aexp = configs.PAPER_ALPHA_EXP[N]
out = []
for box in (1, 4, 8):
    for nu in ((1, 0), (1, 1), (2, 1), (2, 2)):
        row = {"box": box, "nu": nu, "order": ORDER, "cells": []}
        for rel in (10, 100, 500):
            t0 = time.time()
            g = PaperSystem(N, box, nu[0], nu[1], rel * aexp, mesh, order=ORDER)
            t1 = time.time()
            _, st, _ = g.gmres_solve(g.build_rhs(True, rel * aexp), 1e-6, 100)
            row["cells"].append({"rel": rel, "iters": st["iters"], "converged": st["converged"],
                                 "setup_s": round(t1 - t0, 3), "solve_ms": round(st["solve_ms"], 2),
                                 "reach": [g.level_reach(l) for l in range(g.nlevels)], "launches": g.kernel_launches})
        print(json.dumps(row), flush=True)
