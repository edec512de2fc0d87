"""Task timeline of one dataflow sweep per level (debug): where the critical path goes.
usage: python tools/trace_sweep.py [C2|C3]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_5614_b200 import configs  # noqa: E402
from paper_1311_5614_b200.ibmg import SaddleSystem  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
prob = configs.config3() if cfg == "C3" else configs.config2(1e4)
g = SaddleSystem.from_problem(prob)
L = g._L
N = prob.N
b = torch.tensor(g.build_rhs(np.zeros(2 * N * N)), device="cuda")
w = torch.zeros_like(b)
for level in range(g.num_levels):
    n = g.level_n(level)
    if n > 512 or n < 64:
        continue
    nb = 3 * n * n
    bl, wl = b[:nb].clone(), w[:nb].clone()
    words = L.ibmg_debug_sweep_trace(g._h, level, bl.data_ptr(), wl.data_ptr(), None, 0)
    out = np.zeros(words, np.uint64)
    for rep in range(3):  # warm, then measure
        L.ibmg_debug_sweep_trace(g._h, level, bl.data_ptr(), wl.data_ptr(), out.ctypes.data, words)
    nt = (n // 16) ** 2
    tiles = out[: 6 * nt].reshape(-1, 6).astype(np.int64)
    bigs = out[6 * nt:].reshape(-1, 9).astype(np.int64)
    t0 = min(tiles[:, 0].min(), bigs[:, 0].min() if len(bigs) else 1 << 62)
    print(f"level {level} n={n}: tiles={nt} big={len(bigs)}")
    print("  tile wait / work (us): mean %.2f / %.2f, last tile done at %.2f" % (
        np.mean(tiles[:, 1] - tiles[:, 0]) / 1e3, np.mean(tiles[:, 2] - tiles[:, 1]) / 1e3, (tiles[:, 2].max() - t0) / 1e3))
    print("  tile task phases (us): stage %.2f | 8 passes %.2f | write+publish %.2f" % (
        np.mean(tiles[:, 4] - tiles[:, 1]) / 1e3, np.mean(tiles[:, 5] - tiles[:, 4]) / 1e3,
        np.mean(tiles[:, 2] - tiles[:, 5]) / 1e3))
    per = nt // 4
    for tc in range(4):
        m = slice(tc * per, (tc + 1) * per)
        print("    tile colour %d: start %.2f, deps met %.2f, done %.2f us (work mean %.2f)" % (
            tc, (tiles[m, 0].min() - t0) / 1e3, (tiles[m, 1].max() - t0) / 1e3, (tiles[m, 2].max() - t0) / 1e3,
            np.mean(tiles[m, 2] - tiles[m, 1]) / 1e3))
    if len(bigs):
        print("  big wait-deps / wait-slab / solve (us): mean %.2f / %.2f / %.2f; end at %.2f" % (
            np.mean(bigs[:, 1] - bigs[:, 0]) / 1e3, np.mean(bigs[:, 2] - bigs[:, 1]) / 1e3,
            np.mean(bigs[:, 3] - bigs[:, 2]) / 1e3, (bigs[:, 3].max() - t0) / 1e3))
        if bigs[:, 6].any():  # per-phase stamps (slab-slot variant only: IBMG_DF_ES=0)
            print("  solve phases (us): residual %.2f | sync %.2f | matvec+sync %.2f | write+publish %.2f" % (
                np.mean(bigs[:, 6] - bigs[:, 2]) / 1e3, np.mean(bigs[:, 7] - bigs[:, 6]) / 1e3,
                np.mean(bigs[:, 8] - bigs[:, 7]) / 1e3, np.mean(bigs[:, 3] - bigs[:, 8]) / 1e3))
        for col in range(int(bigs[:, 4].max()) + 1):
            m = bigs[:, 4] == col
            print(f"    colour {col}: {m.sum():3d} blocks, start {(bigs[m,0].min()-t0)/1e3:7.2f} done {(bigs[m,3].max()-t0)/1e3:7.2f} us")

# coarse kernel phases (levels n <= 32)
lc = next(l for l in range(g.num_levels) if g.level_n(l) <= 32)
nc = g.level_n(lc)
bc = torch.tensor(np.random.default_rng(0).uniform(-1, 1, 3 * nc * nc), device="cuda")
wc = torch.zeros_like(bc)
out = np.zeros(64, np.uint64)
for rep in range(3):
    L.ibmg_debug_coarse_trace(g._h, bc.data_ptr(), wc.data_ptr(), out.ctypes.data, 64)
st = out[out > 0].astype(np.int64)
print("coarse kernel phases (us):", np.round(np.diff(st) / 1e3, 2).tolist(), "total %.1f" % ((st[-1] - st[0]) / 1e3))
