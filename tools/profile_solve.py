"""Short driver for ncu captures of the solve kernels: C2 (kappa = 1e4) or C4
context, one implicit step.  usage: python tools/profile_solve.py [C2|C4]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_5614_b200 import configs  # noqa: E402
from paper_1311_5614_b200.ibmg import SaddleSystem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
prob = {"C2": lambda: configs.config2(1e4), "C3": configs.config3, "C4": configs.config4}[cfg]()
g = SaddleSystem.from_problem(prob)
N = prob.N
u = np.zeros(2 * N * N)
p = np.zeros(N * N)
X = prob.X.copy()
st = g.step_implicit(u, p, X)
print("ok", st)
