"""The C-ABI boundary: the sm_100a library loads on a CPU host, exports every
entry point include/ibmg_gpu.h declares, and validates arguments like the
reference's constructors (std::invalid_argument -> status 1) without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1311_5614_b200 import ibmg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header="ibmg_gpu.h"):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ibmg_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = ibmg.lib()
    names = declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(ibmg.EXPORTS) == set(names)


def test_library_exports_the_paper_mode_abi():
    """include/ibmg_paper.h: every symbol exported, arguments validated
    like the reference's constructors before any CUDA call, null handles rejected."""
    from paper_1311_5614_b200 import paper
    L = paper.lib()
    names = declared("ibmg_paper.h")
    assert not [n for n in names if not hasattr(L, n)]
    assert set(paper.EXPORTS) == set(names)
    for bad in (dict(N=12), dict(N=4), dict(box=3), dict(box=32), dict(alpha=-1.0), dict(nu1=0, nu2=0),
                dict(coarsest_n=3), dict(order=2)):
        p = dict(N=32, box=4, nu1=1, nu2=1, coarsest_n=4, alpha=1.0, device=0, order=0)
        p.update(bad)
        h = C.c_void_p()
        assert L.ibmg_paper_create(C.byref(paper.PaperParams(**p)), C.byref(h)) == 1 and not h.value, bad
    x = np.zeros(4)
    assert L.ibmg_paper_num_levels(None) == -1 and L.ibmg_paper_level_n(None, 0) == -1
    assert L.ibmg_paper_apply(None, 0, x.ctypes.data, x.ctypes.data) == 1
    assert L.ibmg_paper_last_error(None) == b"null context"


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {ibmg.lib_path()} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out


@pytest.mark.parametrize("bad", [dict(N=12), dict(N=4), dict(rho=0.0), dict(dt=-1.0), dict(restart=0),
                                 dict(rtol=2.0), dict(coarsest_n=8), dict(nu1=0, nu2=0)])
def test_create_rejects_invalid_params(bad):
    p = dict(N=64, rho=1.0, mu=1.0, dt=1e-2, nu1=1, nu2=1, restart=30, max_iters=100, rtol=1e-10,
             coarsest_n=4, device=0)
    p.update(bad)
    h = C.c_void_p()
    rc = ibmg.lib().ibmg_create(C.byref(ibmg.Params(**p)), C.byref(h))
    assert rc == 1 and not h.value


def test_null_context_is_invalid():
    L = ibmg.lib()
    assert L.ibmg_num_levels(None) == -1
    x = np.zeros(4)
    assert L.ibmg_apply(None, 0, x.ctypes.data, x.ctypes.data, 0) == 1
    assert L.ibmg_last_error(None) == b"null context"


def test_product_path_never_loads_the_oracle():
    """The GPU library must not link or open the CPU oracle (test infrastructure);
    only build.py (which compiles the checker) may name it."""
    deps = os.popen(f"ldd {ibmg.lib_path()} 2>/dev/null").read()
    assert "oracle" not in deps
    pkg = os.path.join(ROOT, "paper_1311_5614_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py") and f != "build.py":
            src = open(os.path.join(pkg, f)).read()
            assert not re.search(r"import oracle|from oracle|libibmg_oracle|orc_", src), f
    for f in os.listdir(os.path.join(pkg, "csrc")):
        assert "orc_" not in open(os.path.join(pkg, "csrc", f)).read(), f


@pytest.mark.parametrize("nslabs,N,restart", [(0, 64, 30), (9, 64, 30), (3, 64, 30), (2, 12, 30), (2, 64, 64)])
def test_group_create_rejects_invalid_params(nslabs, N, restart):
    """Slab groups validate like contexts (status 1, no handle), before any CUDA call."""
    p = ibmg.Params(N, 1.0, 1.0, 1e-2, 1, 1, restart, 100, 1e-10, 4, 0)
    h = C.c_void_p()
    L = ibmg.lib()
    dev = (C.c_int * 9)(*([0] * 9))
    assert L.ibmg_group_create(C.byref(p), nslabs, dev, 64, 0, C.byref(h)) == 1 and not h.value
    assert L.ibmg_group_create_nccl(C.byref(p), 0, nslabs, b"\0" * 128, 64, 0, C.byref(h)) == 1 and not h.value


def test_group_null_handles():
    L = ibmg.lib()
    assert L.ibmg_group_distributed_levels(None) == -1
    assert L.ibmg_group_kernel_launches(None) == -1
    assert L.ibmg_group_last_error(None) == b"null group"
    x = np.zeros(4)
    assert L.ibmg_group_vcycle(None, x.ctypes.data, x.ctypes.data) == 1
    assert L.ibmg_vcycle_spectrum(None, 4, 1, x.ctypes.data, None) == 1
    assert L.ibmg_set_scheme(None, 0) == 1
