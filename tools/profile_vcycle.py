"""Short driver for ncu captures: C2 (kappa = 1e4) context, RHS, a few V-cycles.
usage: python tools/profile_vcycle.py [N] [cycles]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_5614_b200 import configs  # noqa: E402
from paper_1311_5614_b200.ibmg import SaddleSystem  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 3
prob = configs.config3() if N == 1024 else configs.config2(1e4, N=N, nb=2 * N)
g = SaddleSystem.from_problem(prob)
b = g.build_rhs(np.zeros(2 * N * N))
for _ in range(cycles):
    z = g.v_cycle(b)
print("ok", float(np.linalg.norm(z)))
