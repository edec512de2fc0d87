"""ncu target: a few fine-level operator applies on a C4-sized (or given N) periodic grid
without structures (the E' part costs nothing there: tools/c4_ops_probe.py)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_5614_b200.ibmg import SaddleSystem  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
g = SaddleSystem(N, dt=1e-4)
w = torch.rand(3 * N * N, dtype=torch.float64, device="cuda") - 0.5
out = torch.empty_like(w)
for _ in range(3):
    g.apply(w, out)
torch.cuda.synchronize()
g.profile(True)
for _ in range(10):
    g.apply(w, out)
rep = g.profile_report()
for k, (ms, cnt) in rep.items():
    if "apply" in k:
        gb = 48.0 * N * N / 1e9
        print(k, "ms/launch", round(ms / cnt, 4), "GB/s", round(gb / (ms / cnt) * 1e3, 1))
