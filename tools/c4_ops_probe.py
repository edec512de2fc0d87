"""C4 fine-level operator probe: the fused apply with and without the E' part
(point forces + face gathers), event-timed per kernel by ibmg_profile."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_5614_b200 import configs  # noqa: E402
from paper_1311_5614_b200.ibmg import SaddleSystem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
prob = {"C3": configs.config3, "C4": configs.config4}[cfg]()
g = SaddleSystem.from_problem(prob)
N = prob.N
w = torch.rand(3 * N * N, dtype=torch.float64, device="cuda") - 0.5
out = torch.empty_like(w)
torch.cuda.synchronize()
for implicit in (True,):
    g.set_scheme(implicit)
    for _ in range(2):
        g.apply(w, out)
    g.profile(True)
    for _ in range(5):
        g.apply(w, out)
        z = g.v_cycle(w) if False else None
    print("implicit" if implicit else "explicit (no E')", g.profile_report(), flush=True)
    g.profile(False)
g.set_scheme(True)
b = torch.rand(3 * N * N, dtype=torch.float64, device="cuda") - 0.5
for _ in range(1):
    g.v_cycle(b)
g.profile(True)
for _ in range(3):
    g.v_cycle(b)
print("v_cycle x3", g.profile_report(), flush=True)
