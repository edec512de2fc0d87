#!/usr/bin/env python
"""bench.py — implicit IB step solve time on B200 (BASELINE.json metric).

Workload (default "C3": BASELINE.json configs[2], the largest configuration
quoted single-GPU): periodic unit square, MAC grid N=1024, fp64, rho = mu = 1,
dt = 1e-3; 16 circular membranes (seed 0, r ~ U[0.03, 0.06], spacing h/2,
kappa 10^U[3, 6]); 5 consecutive backward-Euler steps from u = 0, each solved
by FGMRES(30) preconditioned by one V(1,1) cycle (multicolour Vanka + big
boxes, coarsening to 4x4) to relative residual 1e-10.  --config C2 runs
configs[1] (N=256, kappa {1e2, 1e4, 1e6} x 10 steps), C4 the N=8192 problem
on one GPU, C5 the batch of 512 N=256 problems.

A bench "step" is one implicit step.  The configured steps of every block
(C2: one block per kappa) are visited round-robin, each block advancing its
own trajectory and restarting from u = 0, X^0 after its last configured step,
so any --steps >= (blocks x steps per block) times every configured step
(C3: --steps 5 covers the whole 5-step trajectory; the driver's 20 cover it
four times).
  value  : device time per implicit step (ms), CUDA events on the solver's
           stream, inputs resident in HBM, L2 flushed (256 MiB write) between
           steps, max over ranks.
  e2e    : the same steps through the C ABI with HOST buffers (pinned; H2D of
           u^n, X^n and D2H of u, p, X inside the timed region), wall clock.
  roofline: live per-kernel CUDA-event timing (ibmg_profile) of the dominant
           kernel over one profiled pass of every configured step.
  cpu_baseline: the CPU oracle (oracle/, kind "port": the reference ships no
           solver) on all host threads, a bounded sample.
  secondary.C4: the N=8192 problem on this GPU (1 timed step): ms/step, the
           V-cycle roofline fraction and the dominant kernel's.
--impl reference runs that oracle port on the same schedule (rank 0 only).
Multi-GPU (torchrun): C2/C3 do not shard; every rank runs an independent
replica ("replicas only"); scaling "weak".
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "implicit IB step solve time (ms); fine-grid DOF·V-cycles/s vs HBM roofline"


def workloads():
    """name -> (list of problem blocks, steps per block, description).  A bench
    step is one implicit step; the state resets at the start of each block."""
    from paper_1311_5614_b200 import configs
    return {
        "C2": ([configs.config2(k) for k in (1e2, 1e4, 1e6)], 10,
               "C2: periodic N=256 MAC grid fp64, ellipse (0.5,0.5) a=0.3 b=0.15, Nb=512, "
               "kappa {1e2,1e4,1e6} x 10 implicit steps, dt=1e-3, FGMRES(30)+V(1,1) box relaxation, rtol 1e-10"),
        "C3": ([configs.config3()], 5,
               "C3: periodic N=1024 MAC grid fp64, 16 circles (seed 0, r~U[0.03,0.06], ds=h/2, kappa 10^U[3,6]), "
               "5 implicit steps, dt=1e-3, FGMRES(30)+V(1,1) box relaxation, rtol 1e-10"),
        "C4": ([configs.config4()], 1,
               "C4: periodic N=8192 MAC grid fp64, 256 circular/elliptic membranes (seed 1, r~U[0.005,0.015], aspect "
               "U[1,2], ds=h/2, kappa 10^U[3,6]), one implicit step, dt=1e-4, FGMRES(30)+V(1,1), rtol 1e-10, 1 GPU"),
        "C1": ([configs.config1()], 1,
               "C1: periodic N=64, ellipse Nb=128, kappa=1e2, dt=1e-2, one implicit step"),
    }


WL = {}

THROTTLE_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
                 0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
                 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def workload_config():
    """The `config` object of both arms (identical dicts: no arm-specific text)."""
    probs, per, desc = WL["blocks"], WL["per"], WL["desc"]
    N = probs[0].N
    return {
        "workload": desc, "name": WL["name"], "N": N, "Nb": [p.npts for p in probs],
        "kappas": [p.kappa if len(p.kappa) > 1 else p.kappa[0] for p in probs], "steps_per_block": per,
        "dt": probs[0].dt, "dof": 3 * N * N,
        "step_order": "blocks round-robin, each block's trajectory restarted after its last configured step",
        "l2": "flushed between timed steps (256 MiB write)",
    }


DATA = "synthetic (seeded BASELINE.json geometry, u0 = 0)"


def step_schedule(total):
    """(block, step index in block) for bench steps 0..total-1: blocks are
    visited round-robin (C2: kappa 1e2, 1e4, 1e6, 1e2, ...), each advancing
    its own trajectory; index 0 restarts it from u = 0, X^0."""
    per, nblocks = WL["per"], len(WL["blocks"])
    return [(s % nblocks, (s // nblocks) % per) for s in range(total)]


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.samples = []
        self._p = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self._p = None
        return self

    def _read(self):
        for line in self._p.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 3:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]), int(parts[2], 16)))
                except ValueError:
                    pass

    def __exit__(self, *a):
        if self._p:
            self._p.terminate()
            try:
                self._p.wait(timeout=2)
            except Exception:
                self._p.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = sorted(s[0] for s in self.samples)
        mask = 0
        for s in self.samples:
            mask |= s[2]
        reasons = [name for bit, name in THROTTLE_BITS.items() if mask & bit and name != "gpu_idle"]
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples)}


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def measured_traffic(config, kernel):
    """DRAM bytes per launch of `kernel` from a committed ncu --set full capture
    (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)[config][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


def cgs_bytes(step_iters, restart, M):
    """Compulsory bytes of the fused CGS2 sweeps of FGMRES steps with the given
    Arnoldi-step counts: at basis index j the three sweeps read V_0..V_j and w
    (j + 2 vectors) and read+write w twice more (2 (j + 3)), 8 B per DOF."""
    tot = 0
    for it in step_iters:
        j = 0
        for _ in range(it):
            tot += (3 * j + 8) * 8 * M
            j = j + 1 if j + 1 < restart else 0
    return tot


def ortho_bytes(step_iters, restart, M, which):
    """Compulsory bytes of the two-pass orthogonalisation (k_ortho_dots /
    k_ortho_update) at basis index j: the dots read V_0..V_j and w (j + 2
    vectors); the update reads them and writes V_j and w (j + 4)."""
    tot = 0
    for it in step_iters:
        j = 0
        for _ in range(it):
            tot += ((j + 2) if which == "dots" else (j + 4)) * 8 * M
            j = j + 1 if j + 1 < restart else 0
    return tot


def kernel_algorithmic_bytes(name, ctxinfo, vcycles, fgmres_iters, restarts):
    """Algorithmic (compulsory fp64) bytes of all launches of `name` in the
    profiled pass (SURVEY.md §8d per-cell figures x cells)."""
    if "k_cgs_sweep" in name:
        return cgs_bytes(ctxinfo["step_iters"], 30, 3 * ctxinfo["N"] ** 2)
    if "k_ortho_dots" in name or "k_ortho_update" in name:
        return ortho_bytes(ctxinfo["step_iters"], 30, 3 * ctxinfo["N"] ** 2,
                           "dots" if "dots" in name else "update")
    lv = ctxinfo["levels"]  # list of (n, nbig) for multi-tile levels (n >= 32)
    sweeps = 2  # V(1,1)
    N = ctxinfo["N"]
    big_bytes = 3136 * 8 + 2000 * 12 + 56 * 24  # inverse + E' slab (~2000 entries x 12 B) + block w/b traffic
    if name.startswith("k_plain_tiles") or name == "k_plain_df":  # levels n > 512: every cell once per sweep
        return sum(72 * n * n * sweeps for n, _ in lv if n > 512) * vcycles
    if name == "k_big_phase":
        return sum(big_bytes * nb * sweeps for n, nb in lv if n > 512) * vcycles
    if name == "k_sweep_df":  # levels 64 <= n <= 512: the whole sweep (plain cells + big blocks)
        return sum((72 * n * n + big_bytes * nb) * sweeps for n, nb in lv if 64 <= n <= 512) * vcycles
    if name.startswith("k_residual_restrict"):
        return sum(54 * n * n for n, _ in lv) * vcycles
    if name == "k_prolong_add":
        return sum(54 * n * n for n, _ in lv) * vcycles
    if name == "k_stokes_apply":
        return 48 * N * N * (fgmres_iters + restarts + 3)
    return None


def profile_pass(ctxs, states_reset, sched):
    """Live per-kernel CUDA-event timing (ibmg_profile) over the steps of
    `sched`; returns ({kernel: [ms, launches]}, per-step iterations, restarts)."""
    prof_tot, step_iters, prs = {}, [], 0
    for kb, si in sched:
        u, p, X = states_reset(kb, si)
        ctxs[kb].profile(True)  # per step: "(idle)" is the device gap inside a step only
        st = ctxs[kb].step_implicit(u, p, X)
        for k, (tms, cnt) in ctxs[kb].profile_report().items():
            a = prof_tot.setdefault(k, [0.0, 0])
            a[0] += tms
            a[1] += cnt
        ctxs[kb].profile(False)
        step_iters.append(st["iters"])
        prs += st["restarts"]
    return prof_tot, step_iters, prs


def roofline_of(prof_tot, ctxs, N_GRID, step_iters, restarts, wl_name):
    """The dominant kernel with a byte model: achieved GB/s on algorithmic bytes."""
    pv = sum(step_iters)
    step_prof_ms = sum(v[0] for v in prof_tot.values())
    ranked = sorted(prof_tot.items(), key=lambda kv: -kv[1][0])
    c0 = ctxs[0]
    lv_info = []
    for l in range(c0.num_levels):
        nl = c0.level_n(l)
        if nl >= 32:
            lv_info.append((nl, float(np.mean([int(c.big_blocks(l).sum()) for c in ctxs]))))
    info = {"N": N_GRID, "levels": lv_info, "step_iters": step_iters}
    peak, peak_kind = measured_peak_hbm()
    roof = None
    for name, (tms, cnt) in ranked:
        byts = kernel_algorithmic_bytes(name, info, pv, pv, restarts)
        if byts is None:
            continue
        avg_s = tms / cnt * 1e-3
        ach = byts / cnt / avg_s / 1e9
        roof = {"bound": "hbm", "kernel": name, "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "traffic": measured_traffic(wl_name, name),
                "traffic_unit": "B/launch (ncu, profiles/traffic.json)", "peak_source": peak_kind,
                "bytes_per_launch": byts / cnt, "avg_launch_us": round(avg_s * 1e6, 3),
                "share_of_step": round(tms / step_prof_ms, 4), "launches": cnt}
        break
    shares = {k: {"ms": round(v[0], 4), "launches": v[1], "share": round(v[0] / step_prof_ms, 4)}
              for k, v in ranked[:14]}
    return roof, shares


def run_ours(args, rank, world):
    import torch
    from paper_1311_5614_b200.ibmg import SaddleSystem

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    probs = WL["blocks"]
    N_GRID = probs[0].N
    ctxs = [SaddleSystem.from_problem(p, device=dev) for p in probs]
    n2 = N_GRID * N_GRID
    NBs = [p.npts for p in probs]
    D = f"cuda:{dev}"
    X0 = [torch.tensor(p.X.reshape(-1), dtype=torch.float64, device=D) for p in probs]
    # one trajectory state per block (C2: per kappa), advanced round-robin
    U = [torch.zeros(2 * n2, dtype=torch.float64, device=D) for _ in probs]
    P = [torch.zeros(n2, dtype=torch.float64, device=D) for _ in probs]
    Xs = [x.clone() for x in X0]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=D)
    streams = [torch.cuda.ExternalStream(c.stream, device=D) for c in ctxs]

    def state(kb, si):
        if si == 0:  # restart this block's trajectory
            U[kb].zero_()
            P[kb].zero_()
            Xs[kb].copy_(X0[kb])
        return U[kb], P[kb], Xs[kb]

    def run(total, timed):
        ms, iters, setup, restarts, conv = [], [], [], [], True
        for kb, si in step_schedule(total):
            u, p, X = state(kb, si)
            flush.zero_()
            torch.cuda.synchronize()
            if timed:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(streams[kb])
            st = ctxs[kb].step_implicit(u, p, X)
            if timed:
                e1.record(streams[kb])
                e1.synchronize()
                ms.append(e0.elapsed_time(e1))
            iters.append(st["iters"])
            setup.append(st["setup_ms"])
            restarts.append(st["restarts"])
            conv = conv and bool(st["converged"])
        return ms, iters, setup, restarts, conv

    run(args.warmup, False)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    launches0 = sum(c.kernel_launches for c in ctxs)
    with ClockSampler(dev) as clk:
        ms, iters, setup, restarts, conv = run(args.steps, True)
    torch.cuda.synchronize()
    launches = sum(c.kernel_launches for c in ctxs) - launches0
    if world > 1:
        torch.distributed.barrier()
    from paper_1311_5614_b200 import dist as Dd
    tmax, tsum, _ = Dd.reduce_stats([float(sum(ms)), float(sum(iters))], device=D)
    total_ms_max, vcyc_all = float(tmax[0]), float(tsum[1])

    # e2e: same steps through the C ABI with host buffers in pinned memory
    # (numpy views of page-locked torch tensors; the H2D / D2H copies run inside)
    def pinned(n):
        return torch.zeros(n, dtype=torch.float64, pin_memory=True).numpy()

    Uh = [pinned(2 * n2) for _ in probs]
    Ph = [pinned(n2) for _ in probs]
    Xh = [pinned(int(p_.X.size)) for p_ in probs]
    e2e_ms = []
    for kb, si in step_schedule(args.steps):
        if si == 0:
            Uh[kb][:] = 0.0
            Ph[kb][:] = 0.0
            Xh[kb][:] = probs[kb].X.reshape(-1)
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctxs[kb].step_implicit(Uh[kb], Ph[kb], Xh[kb])
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    h2d = 8 * (2 * n2 + 2 * int(np.mean(NBs)))
    d2h = 8 * (2 * n2 + n2 + 2 * int(np.mean(NBs)))

    # auxiliary: each block's whole configured trajectory through ibmg_run_simulation (the state stays on
    # the device between the steps, host arrays cross PCIe once each way); wall clock per step
    traj_ms = []
    for kb in range(len(probs)):
        Uh[kb][:] = 0.0
        Ph[kb][:] = 0.0
        Xh[kb][:] = probs[kb].X.reshape(-1)
        ctxs[kb].run_simulation(0, Uh[kb], Ph[kb], Xh[kb])  # (the device state buffer is allocated on first use)
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sts = ctxs[kb].run_simulation(WL["per"], Uh[kb], Ph[kb], Xh[kb])
        traj_ms.append((time.perf_counter() - t0) * 1e3 / max(len(sts), 1))

    result = None
    if rank == 0:
        # profiled pass (live CUDA-event timing per kernel) over every configured step
        sched = [(kb, si) for si in range(WL["per"]) for kb in range(len(probs))]
        prof_tot, step_iters, prs = profile_pass(ctxs, state, sched)
        roof, kernel_shares = roofline_of(prof_tot, ctxs, N_GRID, step_iters, prs, WL["name"])
        result = {
            "total_ms_max": total_ms_max, "vcyc_all": vcyc_all, "ms": ms, "iters": iters, "setup": setup,
            "launches": launches, "clocks": clk.summary(), "e2e_ms": e2e_ms, "h2d": h2d, "d2h": d2h, "traj_ms": traj_ms,
            "roofline": roof, "kernels": kernel_shares, "converged": conv,
        }
    for c in ctxs:
        c.close()
    return result


def run_secondary_c4(dev, steps=1, warmup=1):
    """The N=8192 configuration (BASELINE configs[3]) on this one GPU: device
    time per implicit step (CUDA events, inputs in HBM), its DOF.V-cycles/s
    roofline fraction and the dominant kernel's roofline from a profiled step."""
    import torch
    from paper_1311_5614_b200 import configs
    from paper_1311_5614_b200.ibmg import SaddleSystem
    free, _ = torch.cuda.mem_get_info(dev)
    if free < 130 * 2**30:
        return {"skipped": f"needs ~130 GiB free device memory, {free / 2**30:.0f} GiB free"}
    prob = configs.config4()
    D = f"cuda:{dev}"
    ctx = SaddleSystem.from_problem(prob, device=dev)
    n2 = prob.N ** 2
    u = torch.zeros(2 * n2, dtype=torch.float64, device=D)
    p = torch.zeros(n2, dtype=torch.float64, device=D)
    X0 = torch.tensor(prob.X.reshape(-1), dtype=torch.float64, device=D)
    X = X0.clone()
    stream = torch.cuda.ExternalStream(ctx.stream, device=D)

    def one():
        u.zero_()
        X.copy_(X0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        st = ctx.step_implicit(u, p, X)
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1), st

    for _ in range(warmup):
        one()
    ms, its = [], []
    for _ in range(steps):
        t, st = one()
        ms.append(t)
        its.append(st["iters"])
    v = float(np.mean(ms))
    peak, _ = measured_peak_hbm()
    dofv = 3 * n2 * float(np.mean(its)) / (v * 1e-3)

    def reset(kb, si):
        u.zero_()
        X.copy_(X0)
        return u, p, X

    prof_tot, step_iters, prs = profile_pass([ctx], reset, [(0, 0)])
    roof, shares = roofline_of(prof_tot, [ctx], prob.N, step_iters, prs, "C4")
    ctx.close()
    return {"config": "C4: periodic N=8192 fp64, 256 membranes (seed 1), dt=1e-4, one implicit step, 1 GPU",
            "ms_per_step": round(v, 3), "steps": steps, "warmup": warmup, "vcycles_per_step": float(np.mean(its)),
            "dof_vcycles_per_s": dofv, "vcycle_roofline_frac": round(dofv * 112 / (peak * 1e9), 4),
            "roofline": roof, "kernels": {k: v_ for k, v_ in list(shares.items())[:8]}}


def run_batch(args, rank, world):
    """C5: a batch of independent N=256 problems (seed 5 + index), one implicit
    step each, sharded across ranks (replicas, no collective).  On one GPU the
    problems of this rank are spread over `workers` host threads, each owning a
    solver context on its own CUDA stream, so the latency-bound problems overlap
    on the device.  Returns per-rank wall/device time and counts."""
    import threading as th

    import torch
    from paper_1311_5614_b200 import configs
    from paper_1311_5614_b200.ibmg import SaddleSystem

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    from paper_1311_5614_b200 import dist as D
    mine = D.shard(args.batch, rank, world)
    probs = {i: configs.config5_problem(i) for i in mine}
    W = min(args.workers, len(mine))
    ctxs = [SaddleSystem(256, 1.0, 1.0, 1e-3, device=dev) for _ in range(W)]
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    glim = args.ctx_grid if args.ctx_grid > 0 else max(8, (2 * sms) // W)
    for c in ctxs:  # share the SMs among the concurrent contexts
        c.set_grid_limit(glim)
    n2 = 256 * 256

    def work(w, host, out):
        c = ctxs[w]
        if host:
            u, p = np.zeros(2 * n2), np.zeros(n2)
        else:
            u = torch.zeros(2 * n2, dtype=torch.float64, device=f"cuda:{dev}")
            p = torch.zeros(n2, dtype=torch.float64, device=f"cuda:{dev}")
        for i in mine[w::W]:
            pr = probs[i]
            X = pr.X.reshape(-1).copy() if host else torch.tensor(pr.X.reshape(-1), device=f"cuda:{dev}")
            c.set_structures(pr.nb, pr.kappa, pr.ds, X)
            if host:
                u[:] = 0.0
            else:
                u.zero_()
            st = c.step_implicit(u, p, X)
            out.append((i, st["iters"], bool(st["converged"])))

    def run(host):
        outs = [[] for _ in range(W)]
        ts = [th.Thread(target=work, args=(w, host, outs[w])) for w in range(W)]
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        return max(e0.elapsed_time(e1), wall), [r for o in outs for r in o]

    # warm-up: one pass over this rank's whole shard (every worker context
    # grows its buffers to its problems' sizes), untimed
    run(False)
    launches0 = sum(c.kernel_launches for c in ctxs)
    with ClockSampler(dev) as clk:
        ms, res = run(False)
    launches = sum(c.kernel_launches for c in ctxs) - launches0
    e2e_ms, _ = run(True)
    tmax, tsum, tmin = D.reduce_stats([ms, e2e_ms, len(res), sum(r[1] for r in res), all(r[2] for r in res)],
                                      device=f"cuda:{dev}")
    ms, e2e_ms, nprob, vcyc, conv = float(tmax[0]), float(tmax[1]), float(tsum[2]), float(tsum[3]), bool(tmin[4])
    for c in ctxs:
        c.close()
    return {"ms": ms, "e2e_ms": e2e_ms, "nprob": nprob, "vcyc": vcyc, "conv": conv, "launches": launches,
            "clocks": clk.summary(), "workers": W, "warmup_problems": len(mine)}


def run_batch_lockstep(args, rank, world):
    """C5 through the lockstep batch (ibmg_batch_*): this rank's
    problems in chunks of `slots`, sorted by kappa (similar iteration counts
    keep the lockstep rounds full).  Two batch objects alternate: while one
    solves chunk i (the batched FGMRES), a second host thread sets the
    structures of chunk i+1 on the other and prepares it (upload, rebuild at
    X^n with the host colouring, RHS), so the setup overlaps the solves.
    Device arrays for the value, host arrays for e2e; wall clock around the
    whole host-synchronous pipeline (every solve returns after its results are
    back), max over ranks."""
    import threading as th

    import torch
    from paper_1311_5614_b200 import configs
    from paper_1311_5614_b200 import dist as D
    from paper_1311_5614_b200.ibmg import BatchSystem

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    mine = D.shard(args.batch, rank, world)
    probs = {i: configs.config5_problem(i) for i in mine}
    order = sorted(mine, key=lambda i: probs[i].kappa[0])
    S = max(1, min(args.slots, len(order)))
    Bs = [BatchSystem(256, S, 1.0, 1.0, 1e-3, device=dev) for _ in range(2)]
    n2 = 256 * 256
    Dv = f"cuda:{dev}"

    def pinned(n):  # page-locked host buffers (numpy views): truly asynchronous copies
        return torch.zeros(n, dtype=torch.float64, pin_memory=True).numpy()

    def arrays(host):
        if host:
            return ([pinned(2 * n2) for _ in range(S)], [pinned(n2) for _ in range(S)],
                    [pinned(2 * 512) for _ in range(S)])
        return ([torch.zeros(2 * n2, dtype=torch.float64, device=Dv) for _ in range(S)],
                [torch.zeros(n2, dtype=torch.float64, device=Dv) for _ in range(S)],
                [torch.zeros(2 * 512, dtype=torch.float64, device=Dv) for _ in range(S)])

    def run(host, sub):
        chunks = [sub[c0:c0 + S] for c0 in range(0, len(sub), S)]
        bufs = [arrays(host), arrays(host)]
        views = [None, None]
        res = []

        def prepare(i):
            B, (us, ps, Xs) = Bs[i % 2], bufs[i % 2]
            ch = chunks[i]
            xv = []
            for k, pi in enumerate(ch):
                pr = probs[pi]
                B.set_structures(k, pr.nb, pr.kappa, pr.ds, pr.X)
                m = pr.X.size
                if host:
                    us[k][:] = 0.0
                    Xs[k][:m] = pr.X.reshape(-1)
                else:
                    us[k].zero_()
                    Xs[k][:m].copy_(torch.from_numpy(pr.X.reshape(-1)))
                xv.append(Xs[k][:m])
            views[i % 2] = (us[:len(ch)], ps[:len(ch)], xv)
            B.prepare(views[i % 2][0], xv)

        torch.cuda.synchronize()
        t0 = time.perf_counter()
        prepare(0)
        for i in range(len(chunks)):
            nxt = th.Thread(target=prepare, args=(i + 1,)) if i + 1 < len(chunks) else None
            if nxt:
                nxt.start()
            us, ps, xv = views[i % 2]
            sts = Bs[i % 2].solve(us, ps, xv)
            res += [(pi, st["iters"], bool(st["converged"])) for pi, st in zip(chunks[i], sts)]
            if nxt:
                nxt.join()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3, res

    run(False, order)  # warm-up: one pass over the shard (every slot's buffers grown to its problems' sizes)
    if world > 1:
        torch.distributed.barrier()
    launches0 = sum(B.kernel_launches for B in Bs)
    with ClockSampler(dev) as clk:
        ms, res = run(False, order)
    launches = sum(B.kernel_launches for B in Bs) - launches0
    e2e_ms, _ = run(True, order)
    tmax, tsum, tmin = D.reduce_stats([ms, e2e_ms, len(res), sum(r[1] for r in res), all(r[2] for r in res)],
                                      device=Dv)
    for B in Bs:
        B.close()
    return {"ms": float(tmax[0]), "e2e_ms": float(tmax[1]), "nprob": float(tsum[2]), "vcyc": float(tsum[3]),
            "conv": bool(tmin[4]), "launches": launches, "clocks": clk.summary(), "workers": S,
            "warmup_problems": len(order)}


def cpu_oracle_steps(steps_sched, threads):
    """The oracle on a schedule of (block, step index in block), one trajectory
    state per block (as the GPU arm)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    probs = WL["blocks"]
    N_GRID = probs[0].N
    ctxs = [O.Oracle(pr, threads=threads) for pr in probs]
    ms, iters = [], []
    st_u = [None] * len(probs)
    st_X = [None] * len(probs)
    for kb, si in steps_sched:
        if si == 0 or st_u[kb] is None:
            st_u[kb] = np.zeros(2 * N_GRID * N_GRID)
            st_X[kb] = probs[kb].X.copy()
        t0 = time.perf_counter()
        st_u[kb], p, st_X[kb], st = ctxs[kb].step(st_u[kb], st_X[kb])
        ms.append((time.perf_counter() - t0) * 1e3)
        iters.append(st["iters"])
    return ms, iters


def cpu_baseline(threads):
    """Bounded sample (10-30 s of CPU work): C2 the first 2 steps of each kappa,
    C3 the first configured step, C1 all."""
    per = {"C2": 2, "C3": 1}.get(WL["name"], 1)
    sched = [(kb, si) for kb in range(len(WL["blocks"])) for si in range(per)]
    ms, iters = cpu_oracle_steps(sched, threads)
    return {"value": round(float(np.mean(ms)), 3), "unit": "ms", "cores": threads, "kind": "port",
            "sample": f"first {per} implicit {WL['name']} step(s) of each block ({len(sched)} steps, {sum(iters)} "
                      f"V-cycles) on the CPU oracle (oracle/ibmg_oracle.cpp, OpenMP {threads} threads); ms per step"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--no-secondary", action="store_true", help="skip the C4 one-GPU secondary measurement")
    ap.add_argument("--batch", type=int, default=512, help="C5: number of independent N=256 problems")
    ap.add_argument("--ctx-grid", type=int, default=0, help="C5: CTA cap per context (0: 2 x SMs / workers)")
    ap.add_argument("--workers", type=int, default=10, help="C5 --c5-mode contexts: concurrent solver contexts per GPU (8-12 measured best on B200, 16 host cores)")
    ap.add_argument("--c5-mode", default="batch", choices=["batch", "contexts"],
                    help="C5: lockstep batch (ibmg_batch_*) or concurrent single-problem contexts")
    ap.add_argument("--slots", type=int, default=64, help="C5 --c5-mode batch: problems per lockstep batch (32-64 measured best)")
    ap.add_argument("--slabs", type=int, default=0,
                    help="C3/C4: slab-partition the problem (DESIGN.md §7): P slabs over the visible GPUs in this "
                         "process (P2P-fused exchange), or under torchrun one slab per rank over NCCL")
    args = ap.parse_args()
    if args.config == "C5":
        return main_batch(args)
    blocks, per, desc = workloads()[args.config]
    WL.update(name=args.config, blocks=blocks, per=per, desc=desc)
    N_GRID = blocks[0].N
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    threads = os.cpu_count() or 1

    if args.impl == "reference":
        if rank != 0:
            return
        # bounded sample: every configured step once (the schedule repeats after blocks x steps per
        # block, so its mean is the mean of any --steps that covers them) after one warm-up step;
        # C3's 5 steps take ~45 s on 16 host threads, where 20 + 3 would take 3.5 minutes
        distinct = len(WL["blocks"]) * WL["per"]
        nrun = min(args.steps, distinct)
        cpu_oracle_steps(step_schedule(min(args.warmup, 1)), threads)
        ms, iters = cpu_oracle_steps(step_schedule(nrun), threads)
        v = float(np.mean(ms))
        line = {"metric": METRIC, "value": round(v, 3), "unit": "ms", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(v, 3), "higher_is_better": False, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": DATA, "impl": "reference",
                "config": workload_config(),
                "parallelism": f"CPU oracle port, OpenMP over independent boxes ({threads} threads)",
                "dof_vcycles_per_s": 3 * WL["blocks"][0].N ** 2 * sum(iters) / (sum(ms) * 1e-3),
                "vcycles_per_step": round(sum(iters) / len(iters), 2),
                "cpu_baseline": {"value": round(v, 3), "unit": "ms", "cores": threads, "kind": "port",
                                 "sample": f"the first {nrun} steps of the GPU arm's {WL['name']} step schedule "
                                           f"({distinct} distinct configured steps; {sum(iters)} V-cycles) on the CPU "
                                           "oracle after 1 warm-up step (the reference ships no solver; SURVEY.md §0)"},
                "e2e": {"value": round(v, 3), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    if args.slabs:
        return run_slabs(args, rank, world)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
    res = run_ours(args, rank, world)
    if rank == 0:
        ms_step = res["total_ms_max"] / args.steps
        dofv = 3 * N_GRID ** 2 * res["vcyc_all"] / (res["total_ms_max"] * 1e-3)
        peak, _ = measured_peak_hbm()
        line = {
            "metric": METRIC, "value": round(ms_step, 4), "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": workload_config(),
            "parallelism": f"replicas x{world} ({args.config} runs one problem per GPU)",
            "dof_vcycles_per_s": dofv,
            "dof_vcycles_roofline_frac": dofv * 112 / (peak * 1e9 * world),
            "vcycles_per_step": round(res["vcyc_all"] / world / args.steps, 2),
            "setup_ms_mean": round(float(np.mean(res["setup"])), 4),
            "converged": res["converged"],
            "gpu_launches": res["launches"],
            "clocks": res["clocks"],
            "e2e": {"value": round(float(np.mean(res["e2e_ms"])), 4), "unit": "ms",
                    "h2d_bytes_per_step": res["h2d"], "d2h_bytes_per_step": res["d2h"]},
            "trajectory": {"api": "ibmg_run_simulation (state resident on the device between the steps; host "
                                  "arrays cross PCIe once per trajectory)",
                           "steps": WL["per"], "ms_per_step": round(float(np.mean(res["traj_ms"])), 4)},
            "roofline": res["roofline"],
            "kernels": res["kernels"],
        }
        if world == 1 and not args.no_secondary and args.config != "C4":
            try:
                line["secondary"] = {"C4": run_secondary_c4(int(os.environ.get("LOCAL_RANK", "0")))}
            except Exception as e:  # reported, never fatal for the headline
                line["secondary"] = {"C4": {"error": str(e)[:200]}}
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(os.cpu_count() or 1)
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_slabs(args, rank, world):
    """One problem slab-partitioned.  world == 1: `--slabs` slabs
    in this process, slab r on GPU r mod device_count (exchanges fused into the
    smoother kernels as peer stores); torchrun: one slab per rank over NCCL.
    Each step goes through the group's public call with host arrays, so the
    value is end to end (H2D of u^n, X^n, D2H of u, p, X inside), wall clock
    after the group's device synchronisation, max over ranks."""
    import torch
    from paper_1311_5614_b200.ibmg import SlabGroup
    from paper_1311_5614_b200 import dist as D
    prob = WL["blocks"][0]
    N = prob.N
    kw = dict(rho=prob.rho, mu=prob.mu, dt=prob.dt)
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("gloo")
        g = SlabGroup.nccl_group(N, **kw)
        nslab, devs, mode = world, world, "NCCL, one slab per rank"
    else:
        nd = max(1, torch.cuda.device_count())
        devices = [r % nd for r in range(args.slabs)]
        g = SlabGroup(N, args.slabs, devices=devices, **kw)
        nslab, devs, mode = args.slabs, len(set(devices)), "in-process, P2P-fused exchange"
    g.set_structures(prob.nb, prob.kappa, prob.ds, prob.X)
    u, p, X = np.zeros(2 * N * N), np.zeros(N * N), prob.X.reshape(-1).copy()
    for _ in range(args.warmup):
        u[:] = 0.0
        X[:] = prob.X.reshape(-1)
        g.step_implicit(u, p, X)
    wall, stats = [], []
    l0 = g.kernel_launches
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        for s in range(args.steps):
            if s % WL["per"] == 0:
                u[:] = 0.0
                X[:] = prob.X.reshape(-1)
            t0 = time.perf_counter()
            st = g.step_implicit(u, p, X)
            wall.append((time.perf_counter() - t0) * 1e3)
            stats.append(st)
    tmax, _, _ = D.reduce_stats([float(sum(wall))])
    if rank == 0:
        v = float(tmax[0]) / args.steps
        vc = sum(st["iters"] for st in stats)
        line = {
            "metric": METRIC, "value": round(v, 3), "unit": "ms", "n_gpus": devs, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(v, 3), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded geometry, u0 = 0)",
            "config": dict(workload_config(), parallelism=f"slab partition x{nslab} on {devs} GPU(s), {mode}",
                           distributed_levels=g.distributed_levels,
                           timing="end to end through ibmg_group_step (host arrays), wall clock, max over ranks"),
            "dof_vcycles_per_s": 3 * N * N * vc / (sum(wall) * 1e-3),
            "vcycles_per_step": vc / args.steps,
            "setup_ms_mean": round(float(np.mean([st["setup_ms"] for st in stats])), 3),
            "solve_ms_mean": round(float(np.mean([st["solve_ms"] for st in stats])), 3),
            "converged": all(st["converged"] for st in stats),
            "gpu_launches": g.kernel_launches - l0,
            "exchanges": g.exchanges,
            "clocks": clk.summary(),
            "e2e": {"value": round(v, 3), "unit": "ms", "h2d_bytes_per_step": 8 * (2 * N * N + X.size) * nslab,
                    "d2h_bytes_per_step": 8 * (3 * N * N + X.size)},
        }
        print(json.dumps(line), flush=True)
    g.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main_batch(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    threads = os.cpu_count() or 1
    desc = (f"C5: batch of {args.batch} independent problems, periodic N=256 fp64, one ellipse each (seed 5+i, "
            "semi-axes U[0.1,0.35], Nb=512, kappa 10^U[1,6]), dt=1e-3, one implicit step each, FGMRES(30)+V(1,1)")
    cfg = {"workload": desc, "name": "C5", "N": 256, "batch": args.batch, "dof": 3 * 256 * 256}
    par = (f"batch sharded over {world} GPU(s) (replicas), " +
           (f"lockstep batches of {args.slots} problems/GPU (ibmg_batch)" if args.c5_mode == "batch"
            else f"{args.workers} concurrent contexts/GPU"))
    if args.impl == "reference":
        if rank != 0:
            return
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        from paper_1311_5614_b200 import configs
        sample = max(1, min(args.steps, 8))
        ms = []
        for i in range(sample):
            pr = configs.config5_problem(i)
            t0 = time.perf_counter()
            O.Oracle(pr, threads=threads).step(np.zeros(2 * 256 * 256), pr.X)
            ms.append((time.perf_counter() - t0) * 1e3)
        v = float(np.mean(ms))
        print(json.dumps({"metric": METRIC, "value": round(v, 3), "unit": "ms", "n_gpus": args.gpus,
                          "steps": sample, "warmup": 0, "ms_per_step": round(v, 3), "higher_is_better": False,
                          "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                          "impl": "reference", "config": cfg, "parallelism": f"CPU oracle port ({threads} threads)",
                          "problems_per_s": 1e3 / v,
                          "cpu_baseline": {"value": round(v, 3), "unit": "ms", "cores": threads, "kind": "port",
                                           "sample": f"{sample} C5 problems (oracle port, ms per problem)"},
                          "e2e": {"value": round(v, 3), "unit": "ms", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dist.init_process_group("nccl")
    r = run_batch_lockstep(args, rank, world) if args.c5_mode == "batch" else run_batch(args, rank, world)
    if rank == 0:
        ms_per = r["ms"] / r["nprob"]
        line = {"metric": METRIC, "value": round(ms_per, 4), "unit": "ms", "n_gpus": world,
                "steps": int(r["nprob"]), "warmup": r["warmup_problems"], "ms_per_step": round(ms_per, 4),
                "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded C5 geometry)", "config": cfg, "parallelism": par,
                "problems_per_s": r["nprob"] / (r["ms"] * 1e-3),
                "dof_vcycles_per_s": 3 * 256 * 256 * r["vcyc"] / (r["ms"] * 1e-3),
                "vcycles_per_problem": r["vcyc"] / r["nprob"], "converged": r["conv"],
                "gpu_launches": r["launches"], "clocks": r["clocks"],
                "e2e": {"value": round(r["e2e_ms"] / r["nprob"], 4), "unit": "ms",
                        "h2d_bytes_per_step": 8 * (2 * 256 * 256 + 2 * 512),
                        "d2h_bytes_per_step": 8 * (3 * 256 * 256 + 2 * 512)}}
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
