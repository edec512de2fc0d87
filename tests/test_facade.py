"""The C++ facade (include/ibmg/b200.hpp): a compiled reference-style caller
runs one implicit step on the GPU; results are checked against the oracle."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_1311_5614_b200 import build
from paper_1311_5614_b200.configs import Problem
import oracle as O


def test_facade_compiles_and_links():
    exe = build.build_facade_test()
    assert os.path.exists(exe)
    assert "libibmg_b200.so" in subprocess.run(["ldd", exe], capture_output=True, text=True).stdout


@pytest.mark.gpu
def test_facade_step_matches_oracle():
    out = subprocess.run([build.build_facade_test()], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["converged"] == 1 and r["threw"] == 1
    N, nb = 64, 128
    t = 2 * np.pi * np.arange(nb) / nb
    X = np.stack([0.5 + 0.3 * np.cos(t), 0.5 + 0.15 * np.sin(t)], 1)
    prob = Problem("facade", N, 1.0, 1.0, 1e-2, [nb], [1e2], [r["ds"]], X)
    u, p, Xn, st = O.Oracle(prob).step(np.zeros(2 * N * N), X)
    assert abs(st["iters"] - r["iters"]) <= 2
    assert abs(np.sum(u * u) - r["u2"]) <= 1e-8 * np.sum(u * u)
    assert abs(np.sum(p * p) - r["p2"]) <= 1e-8 * np.sum(p * p)
    assert abs(np.sum(Xn) - r["xsum"]) <= 1e-12 * abs(np.sum(Xn))


def test_paper_facade_compiles_and_links():
    exe = build.build_paper_facade_test()
    assert "libibmg_b200.so" in subprocess.run(["ldd", exe], capture_output=True, text=True).stdout


@pytest.mark.gpu
def test_paper_facade_table2_cell():
    """include/ibmg/b200_paper.hpp from C++: Table 2's b = 4, V(1,1), relative stiffness 100
    cell (11 iterations) and the reference's size-mismatch exception."""
    out = subprocess.run([build.build_paper_facade_test()], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    f = out.stdout.split()
    assert abs(int(f[1]) - 11) <= 2 and f[3] == "1" and float(f[7]) <= 1e-6 and f[9] == "1" and int(f[11]) > 0
