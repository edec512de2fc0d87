"""Mesh / field text IO: the host-side writer reproduces the
reference's own write_fiber_mesh output byte for byte (golden file made by
tests/golden/make_mesh_golden.py through oracle/_ref), the reader parses it
exactly, and checkpoints round-trip bitwise.  CPU only."""
import io
import os

import numpy as np
import pytest

from paper_1311_5614_b200 import configs, meshio

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_mesh_c1.txt")


def test_writer_matches_reference_bytes():
    prob = configs.config1()
    f = io.StringIO()
    meshio.write_fiber_mesh(f, prob.X, prob.ds[0])
    assert f.getvalue() == open(GOLD).read()


def test_reader_parses_reference_file_exactly():
    prob = configs.config1()
    with open(GOLD) as f:
        X, ds, per, m1, m2 = meshio.read_fiber_mesh(f)
    assert (m1, m2, per) == (prob.npts, 1, True)
    assert ds == prob.ds[0]
    assert np.array_equal(X, prob.X.reshape(-1, 2))


def test_bad_input_raises_like_reference():
    with pytest.raises(RuntimeError, match="bad header"):
        meshio.read_fiber_mesh(io.StringIO("3 1 0.1\n"))
    with pytest.raises(RuntimeError, match="out of range"):
        meshio.read_fiber_mesh(io.StringIO("2 1 0.1 1\n0 0 0 0\n5 0 1 1\n"))


def test_checkpoint_round_trip(tmp_path):
    prob = configs.config3()
    N = 32
    rng = np.random.default_rng(0)
    u, p = rng.standard_normal(2 * N * N), rng.standard_normal(N * N)
    path = tmp_path / "ck.txt"
    meshio.save_checkpoint(path, u, p, prob.X, prob.nb, prob.ds, N)
    u2, p2, X2, nb2, ds2, N2 = meshio.load_checkpoint(path)
    assert N2 == N and nb2 == list(prob.nb) and ds2 == list(prob.ds)
    assert np.array_equal(u2, u) and np.array_equal(p2, p) and np.array_equal(X2, prob.X.reshape(-1, 2))


def test_checkpoint_restores_run_parameters(tmp_path):
    """kappa per membrane and rho, mu, dt survive the round trip (a trailing
    'params' section after the reference-format mesh blocks)."""
    prob = configs.config3()
    N = 16
    u, p = np.zeros(2 * N * N), np.zeros(N * N)
    path = tmp_path / "ck.txt"
    meshio.save_checkpoint(path, u, p, prob.X, prob.nb, prob.ds, N, kappa=prob.kappa, rho=prob.rho, mu=prob.mu,
                           dt=prob.dt)
    *_, nb2, ds2, N2, prm = meshio.load_checkpoint(path, with_params=True)
    assert nb2 == list(prob.nb) and ds2 == list(prob.ds)
    assert np.array_equal(prm["kappa"], np.asarray(prob.kappa, np.float64).reshape(-1))
    assert (prm["rho"], prm["mu"], prm["dt"]) == (prob.rho, prob.mu, prob.dt)
    # the mesh blocks stay byte-identical to the reference writer's
    text = open(path).read()
    f = io.StringIO()
    meshio.write_structures(f, prob.nb, prob.ds, prob.X)
    assert f.getvalue() in text


def test_cpp_facade_round_trips_reference_file(tmp_path):
    """include/ibmg/b200.hpp's reader + writer reproduce the reference's file."""
    import shutil
    import subprocess
    cxx = shutil.which("g++")
    if not cxx:
        pytest.skip("g++ unavailable")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "meshio_rt"
    # header-only IO: no CUDA library needed at link time beyond the declarations
    subprocess.check_call([cxx, "-std=c++20", "-O1", "-I", os.path.join(root, "include"), "-o", str(exe),
                           os.path.join(root, "tests", "cpp", "meshio_roundtrip.cpp")])
    out = subprocess.check_output([str(exe), GOLD]).decode()
    assert out == open(GOLD).read()
