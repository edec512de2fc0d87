"""In-tree build of the sm_100a CUDA library (libibmg_b200.so) and the oracle.

nvcc cross-compiles for sm_100a without a GPU; the .so files are git-ignored
but travel to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libibmg_b200.so")
SRCS = ["ibmg.cu", "paper_mode.cu"]
DEPS = ["ibmg.cu", "paper_mode.cu", "common.cuh", "cluster_kernel.cuh", "batch.cuh", "grid_kernels.cuh", "ib_kernels.cuh", "smoother_kernels.cuh", "coarse_kernel.cuh",
        "slab_group.cuh"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.isabs(c) and os.path.exists(c):
            return c
    return "nvcc"


def stale(target, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_cuda(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(HERE, "csrc", d) for d in DEPS] + [os.path.join(ROOT, "include", "ibmg_gpu.h"), os.path.join(ROOT, "include", "ibmg_paper.h")]
    if force or stale(LIB, deps):
        cmd = [nvcc()] + NVCC_FLAGS + ["-o", LIB] + [os.path.join(HERE, "csrc", s) for s in SRCS] + ["-ldl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    return LIB


FACADE_SRC = os.path.join(ROOT, "tests", "cpp", "facade_step.cpp")
FACADE_BIN = os.path.join(ROOT, "tests", "cpp", "facade_step")


def build_facade_test() -> str:
    """C++ caller of the ibmg::b200 facade (include/ibmg/b200.hpp) linked to the library."""
    deps = [FACADE_SRC, LIB, os.path.join(ROOT, "include", "ibmg", "b200.hpp")]
    if stale(FACADE_BIN, deps):
        cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
        subprocess.check_call([cxx, "-O2", "-std=c++20", "-I", os.path.join(ROOT, "include"), "-o", FACADE_BIN,
                               FACADE_SRC, "-L", HERE, "-libmg_b200", "-Wl,-rpath," + HERE])
    return FACADE_BIN


PAPER_FACADE_SRC = os.path.join(ROOT, "tests", "cpp", "facade_paper.cpp")
PAPER_FACADE_BIN = os.path.join(ROOT, "tests", "cpp", "facade_paper")


def build_paper_facade_test() -> str:
    """C++ caller of the paper-mode facade (include/ibmg/b200_paper.hpp)."""
    deps = [PAPER_FACADE_SRC, LIB, os.path.join(ROOT, "include", "ibmg", "b200_paper.hpp"),
            os.path.join(ROOT, "include", "ibmg_paper.h")]
    if stale(PAPER_FACADE_BIN, deps):
        cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
        subprocess.check_call([cxx, "-O2", "-std=c++20", "-I", os.path.join(ROOT, "include"), "-o", PAPER_FACADE_BIN,
                               PAPER_FACADE_SRC, "-L", HERE, "-libmg_b200", "-Wl,-rpath," + HERE])
    return PAPER_FACADE_BIN


def build_oracle() -> None:
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "oracle")])


if __name__ == "__main__":
    build_cuda(force="--force" in sys.argv, verbose=True)
    build_facade_test()
    build_paper_facade_test()
    build_oracle()
