"""Generate tests/golden/c4_oracle.npz: one C4 implicit step (N = 8192, 256
membranes, 222k points; BASELINE configs[3]) on the CPU oracle — TEST
INFRASTRUCTURE, the checker only.  Needs a large-memory host (the oracle's
assembled level matrices and 61 Krylov vectors of 1.6 GB: ~170 GB); run on
the GPU box's host (tools/ is not on any product path):

    python tools/make_c4_oracle_fixture.py [out.npz]

Stores what tests/test_gpu_scale_parity.py compares: the iteration count, the
X^{n+1} - X^n displacement of every point, u and p at 2^16 seeded sample DOFs
each, the full-field norms, and the host's memory/core count."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def meminfo_gb():
    with open("/proc/meminfo") as f:
        for line in f:
            if line.startswith("MemTotal:"):
                return int(line.split()[1]) / 2**20
    return 0.0


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "tests", "golden", "c4_oracle.npz")
    import oracle as O
    from paper_1311_5614_b200 import configs
    mem = meminfo_gb()
    threads = os.cpu_count() or 1
    print(f"MemTotal {mem:.0f} GiB, {threads} threads", flush=True)
    if mem < 150:
        print("not enough host memory for the C4 oracle", flush=True)
        return 2
    prob = configs.config4()
    n = prob.N
    nn = n * n
    t0 = time.time()
    o = O.Oracle(prob, threads=threads)
    t1 = time.time()
    print(f"oracle built in {t1 - t0:.0f} s", flush=True)
    u, p, X, st = o.step(np.zeros(2 * nn), prob.X.copy())
    t2 = time.time()
    print(f"step {st} in {t2 - t1:.0f} s", flush=True)
    rng = np.random.default_rng(2026)
    su = np.sort(rng.choice(2 * nn, 1 << 16, replace=False)).astype(np.int64)
    sp = np.sort(rng.choice(nn, 1 << 16, replace=False)).astype(np.int64)
    np.savez_compressed(out, N=n, npts=prob.npts, iters=st["iters"], relres=st["relres"],
                        dX=(X - prob.X), sample_u=su, sample_p=sp, u_s=u[su], p_s=p[sp],
                        u_norm=np.linalg.norm(u), p_norm=np.linalg.norm(p),
                        host_mem_gib=mem, host_threads=threads, build_s=t1 - t0, step_s=t2 - t1)
    print("wrote", out, flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
