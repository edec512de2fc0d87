"""Write tests/golden/ref_mesh_c1.txt with the REFERENCE's own write_fiber_mesh
(fiber.cpp:142-150, via oracle/_ref/libibmg_ref.so) for the C1 ellipse, so the
host-side mesh IO (paper_1311_5614_b200/meshio.py) is pinned byte for byte."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1311_5614_b200 import configs  # noqa: E402


def main():
    L = C.CDLL(os.path.join(ROOT, "oracle", "_ref", "libibmg_ref.so"))
    L.ref_write_fiber_mesh.restype = C.c_long
    L.ref_write_fiber_mesh.argtypes = [C.c_int, C.c_double, C.c_void_p, C.c_char_p, C.c_long]
    prob = configs.config1()
    X = np.ascontiguousarray(prob.X, np.float64).reshape(-1)
    n = L.ref_write_fiber_mesh(prob.npts, prob.ds[0], X.ctypes.data, None, 0)
    buf = C.create_string_buffer(n + 1)
    L.ref_write_fiber_mesh(prob.npts, prob.ds[0], X.ctypes.data, buf, n + 1)
    with open(os.path.join(ROOT, "tests", "golden", "ref_mesh_c1.txt"), "wb") as f:
        f.write(buf.value)


if __name__ == "__main__":
    main()
