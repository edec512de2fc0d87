"""Per-kernel event timing of one implicit step (setup + solve) for a config,
next to its wall time.  usage: python tools/profile_step.py [C2|C3|C4] [kappa]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_5614_b200 import configs  # noqa: E402
from paper_1311_5614_b200.ibmg import SaddleSystem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
kappa = float(sys.argv[2]) if len(sys.argv) > 2 else 1e4
prob = {"C2": lambda: configs.config2(kappa), "C3": configs.config3, "C4": configs.config4}[cfg]()
g = SaddleSystem.from_problem(prob)
N = prob.N
u = np.zeros(2 * N * N)
p = np.zeros(N * N)
X = prob.X.copy()
for _ in range(3):
    st = g.step_implicit(u, p, X)
t0 = time.perf_counter()
for _ in range(3):
    st = g.step_implicit(u, p, X)
wall = (time.perf_counter() - t0) / 3 * 1e3
g.profile(True)
st = g.step_implicit(u, p, X)
rep = g.profile_report()
g.profile(False)
tot = sum(v[0] for v in rep.values())
print(f"{cfg} kappa={kappa:g}: step wall {wall:.3f} ms, kernels (event-timed) {tot:.3f} ms, stats {st}")
for k, (ms, n) in sorted(rep.items(), key=lambda kv: -kv[1][0]):
    print(f"  {k:32s} {ms:8.3f} ms  x{n}")
