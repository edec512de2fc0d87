"""Setup (rebuild at X^n) breakdown: per-kernel event timing of one step's rebuild
vs its wall time (the difference is host work + synchronisation)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_5614_b200 import configs  # noqa: E402
from paper_1311_5614_b200.ibmg import SaddleSystem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
prob = {"C2": lambda: configs.config2(1e4), "C3": configs.config3, "C4": configs.config4}[cfg]()
g = SaddleSystem.from_problem(prob)
for _ in range(3):
    g.set_structures(prob.nb, prob.kappa, prob.ds, prob.X)
t0 = time.perf_counter()
for _ in range(5):
    g.set_structures(prob.nb, prob.kappa, prob.ds, prob.X)
wall = (time.perf_counter() - t0) / 5 * 1e3
g.profile(True)
g.set_structures(prob.nb, prob.kappa, prob.ds, prob.X)
rep = g.profile_report()
tot = sum(v[0] for v in rep.values())
print(f"{cfg}: rebuild wall {wall:.3f} ms, kernels (event-timed) {tot:.3f} ms")
for k, (ms, n) in sorted(rep.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:32s} {ms:8.3f} ms  x{n}")
