"""Phase timeline of one k_cluster_cycle launch (debug): CTA 0's stamps after
each cluster barrier.  usage: python tools/trace_cluster.py [C2|C3|C1]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_5614_b200 import configs  # noqa: E402
from paper_1311_5614_b200.ibmg import SaddleSystem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
prob = {"C1": configs.config1, "C2": lambda: configs.config2(1e4), "C3": configs.config3}[cfg]()
g = SaddleSystem.from_problem(prob)
L = g._L
lt = g.cluster_level
n = g.level_n(lt)
b = torch.tensor(np.random.default_rng(0).uniform(-1, 1, 3 * n * n), device="cuda")
w = torch.zeros_like(b)
out = np.zeros(4000, np.uint64)
for rep in range(4):
    L.ibmg_debug_cluster_trace(g._h, b.data_ptr(), w.data_ptr(), out.ctypes.data, 4000)
st = out.reshape(-1, 2).astype(np.int64)
st = st[st[:, 0] > 0]
KIND = {1: "tile colour", 2: "Q plain", 3: "big colour", 4: "P residual", 5: "Q E' dots", 6: "restrict",
        7: "prolong"}
print(f"{cfg}: cluster levels from n={n}, {len(st)} stamps, total {(st[-1, 0] - st[0, 0]) / 1e3:.1f} us")
agg = {}
for k in range(1, len(st)):
    dt = (st[k, 0] - st[k - 1, 0]) / 1e3
    tag = int(st[k, 1])
    if tag in (800, 900, 1000):
        name = {800: "entry", 900: "exit", 1000: "coarsest"}[tag]
    else:
        lg, ph, idx = tag // 10000, (tag % 10000) // 100, tag % 100
        name = f"n={1 << lg} {KIND.get(ph, ph)}" + (f" {idx}" if ph in (1, 3) else "")
    print(f"  {dt:7.2f} us  {name}")
    key = name.rsplit(" ", 1)[0] if name[-1].isdigit() and ("colour" in name) else name
    agg[key] = agg.get(key, 0.0) + dt
print("per phase kind (us):")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
    print(f"  {v:8.2f}  {k}")
