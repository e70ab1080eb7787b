#!/usr/bin/env python
"""bench.py — active-cell Newton iterations/s of the localized FIM solver.

Contract:
  python bench.py --gpus N --steps K --warmup W [--impl reference]
One JSON line on rank 0.

Workload (config.workload): BASELINE.json configs[1] — 2D two-phase
oil-water, 256x256, 40-line DFN, 30 backward-Euler timesteps, solved with the
adaptive-localized Newton (Algorithm 1).  One bench "step" = one full run of
that case (all 30 timesteps, Newton + Krylov + set estimation) from the same
seeded initial state.  metric = Σ n_A over all Newton iterations / time.

  value : device-resident run (state already in HBM), CUDA events on the
          context stream, L2 flushed (512 MB write) before every step.
  e2e   : the same run through the public C-ABI entry point rsim_run_case
          with pinned host buffers (H2D of the initial state + D2H of the
          final state inside the timed region).
  roofline : dominant kernel of the workload (per-phase CUDA-event time).
  c5_sweep : config 5 (1024x1024x32) kernel throughput at several active
          fractions — compaction (K7), assembly (K1), 50 BiCGSTAB iterations.
  cpu_baseline : the CPU oracle (oracle/, C++ restatement) on this box's
          host cores, same workload, bounded sample.
Multi-GPU: the path does not shard across GPUs in this tier (one GPU per
case) => N independent replicas, max time over ranks.
"""
from __future__ import annotations

import argparse
import json
from pathlib import Path
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK = 6650.0


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, dev: int):
        self.dev = dev
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        for line in (self.out or "").strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        busy = [s for s in sm if s > 0.5 * mx] or sm
        return {"sm_mhz": float(np.median(busy)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def init_dist(ws, lr, backend="nccl"):
    if ws <= 1:
        return None
    import torch
    import torch.distributed as dist
    if backend == "nccl":
        torch.cuda.set_device(lr)
    dist.init_process_group(backend, init_method="env://")
    return dist


def _dev(dist):
    return "cuda" if dist.get_backend() == "nccl" else "cpu"


def dist_max(dist, v: float) -> float:
    """Max over ranks (replica timing: the job takes as long as its slowest rank)."""
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=_dev(dist))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_sum(dist, v: float) -> float:
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=_dev(dist))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier(dist):
    if dist is not None:
        dist.barrier()


# --------------------------------------------------------------------------
# algorithmic bytes: b unknowns/cell, s Cartesian slots
def bytes_krylov_row_iter(b, s):
    # 2 SpMVs (s column indices + s blocks + x_l + y write) + 14 vector passes:
    # (r0,v),(r,r) 2, s update 3, (r0,s),(r0,t) 1, x/r/next-p update 8 (x, p,
    # s, t, v read; x, r, p written -- the next p is formed in the x/r pass)
    spmv = s * (8 * b * b + 4) + 16 * b
    return 2 * spmv + 112 * b


def bytes_krylov_row_init(b):
    return 8 * b * 4  # read rhs, write r, r0, x


def bytes_assembly_row(b, D, s, nnc_per_row=0.0):
    # 24b + 8 + 8D + 12·NNC + 4 + (1+s)·8b²
    return 24 * b + 8 + 8 * D + 12 * nnc_per_row + 4 + (1 + s) * 8 * b * b


def bytes_k7(n, nA, m):
    return (19 + 2 * m) * n + 4 * nA


WORKLOAD = {"config": 2, "solver": 1, "name": "c2_oilwater_256x256_dfn40_localized_newton_30steps"}


def run_reference(args, rank, ws):  # noqa: C901
    """--impl reference: the CPU oracle (port of SPEC + Algorithms 1-2) on all host threads."""
    if rank != 0:
        return
    import paper_2008_01539_b200 as pkg
    import oracle
    from oracle import Oracle
    cores = len(os.sched_getaffinity(0))
    oracle.set_threads(cores)
    case = pkg.Case(WORKLOAD["config"])
    s0 = case.init_state()
    dts = case.schedule()
    opts = case.solver_opts()
    if args.precond is not None:
        opts.precond = args.precond
    orc = Oracle(case)
    for _ in range(args.warmup):
        orc.run_case(WORKLOAD["solver"], s0, dts, opts)
    tot_na, tot_t = 0, 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = orc.run_case(WORKLOAD["solver"], s0, dts, opts)
        tot_t += time.perf_counter() - t0
        tot_na += r["sum_na"]
    v = tot_na / tot_t
    line = {
        "metric": "active-cell Newton iters/s", "value": v, "unit": "active-cell iters/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": WORKLOAD["name"], "n_cells": case.n, "timesteps": len(dts), "parallelism": "replicas"},
        "cpu_baseline": {"value": v, "unit": "active-cell iters/s", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} full runs of the workload (oracle/, OpenMP {cores} threads)"},
        "e2e": {"value": v, "unit": "active-cell iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(case, s0, dts, opts):
    import oracle
    from oracle import Oracle
    cores = len(os.sched_getaffinity(0))
    oracle.set_threads(cores)
    orc = Oracle(case)
    tot_na, tot_t, runs = 0, 0.0, 0
    while tot_t < 10.0 and runs < 30:
        t0 = time.perf_counter()
        r = orc.run_case(WORKLOAD["solver"], s0, dts, opts)
        tot_t += time.perf_counter() - t0
        tot_na += r["sum_na"]
        runs += 1
    return {"value": tot_na / tot_t, "unit": "active-cell iters/s", "cores": cores, "kind": "port",
            "sample": f"{runs} full runs of the workload ({tot_t:.1f} s, oracle/ OpenMP {cores} threads)",
            "model": _cpu_model()}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def c5_sweep(pkg, fractions, reps, hbm, ilu_fracs=()):
    """Config 5: K7 compaction, K1 assembly, 50 BiCGSTAB iterations per active fraction
    (block-Jacobi); the ILU(0) second row at the fractions in ilu_fracs
    (level-scheduled factorisation + 50 iterations, one timed run)."""
    import ctypes as C
    case = pkg.Case(5)
    sim = pkg.GpuSimulator(case)
    L, ctx = sim.L, sim._ctx
    n, b, s = case.n, 1, 6
    opts = case.solver_opts(fixed_lin_iters=50, lin_maxit=50, precond=pkg.PREC_BJACOBI)  # Jacobi
    out = []
    s0 = case.init_state()
    sim.set_state(s0, 86400.0)
    for frac in fractions:
        dp, f_ach, R = case.c5_field(frac, 2, 1e-3)
        sim.upload_dp(dp)
        L.rsim_gpu_state_from_dp(ctx, 30e6, 20e6)
        ms = {"k7": [], "k1": [], "krylov": []}
        for r in range(reps + 1):
            L.rsim_gpu_flush_l2(ctx)
            L.rsim_gpu_mark(ctx, 10)
            stt = pkg.GpuStats()
            L.rsim_gpu_support_active(ctx, 1e-3, 2, None)
            L.rsim_gpu_mark(ctx, 11)
            L.rsim_gpu_stats_get(ctx, C.byref(stt))
            nA = stt.n_active
            L.rsim_gpu_flush_l2(ctx)
            L.rsim_gpu_mark(ctx, 12)
            L.rsim_gpu_assemble(ctx)
            L.rsim_gpu_mark(ctx, 13)
            L.rsim_gpu_flush_l2(ctx)
            L.rsim_gpu_mark(ctx, 14)
            L.rsim_gpu_linear_solve(ctx, C.byref(opts))
            L.rsim_gpu_mark(ctx, 15)
            L.rsim_gpu_stats_get(ctx, C.byref(stt))
            if r == 0:
                continue  # warm-up
            for key, a, bb in (("k7", 10, 11), ("k1", 12, 13), ("krylov", 14, 15)):
                v = C.c_double()
                L.rsim_gpu_elapsed(ctx, a, bb, C.byref(v))
                ms[key].append(v.value)
        m = {k: float(np.median(v)) for k, v in ms.items()}
        ilu = None
        if any(abs(frac - f) < 1e-9 for f in ilu_fracs):
            oi = case.solver_opts(fixed_lin_iters=50, lin_maxit=50, precond=pkg.PREC_ILU0)
            for r in range(2):
                L.rsim_gpu_mark(ctx, 14)
                L.rsim_gpu_linear_solve(ctx, C.byref(oi))
                L.rsim_gpu_mark(ctx, 15)
            v = C.c_double()
            L.rsim_gpu_elapsed(ctx, 14, 15, C.byref(v))
            ilu = v.value
        by7 = bytes_k7(n, nA, 2)
        by1 = nA * bytes_assembly_row(b, 3, s)
        byk = nA * (50 * bytes_krylov_row_iter(b, s) + bytes_krylov_row_init(b))
        out.append({
            "target_fraction": frac, "active_fraction": nA / n, "n_active": nA, "lin_iters": stt.lin_iters,
            "k7_ms": m["k7"], "k7_gbs": by7 / m["k7"] / 1e6,
            "k1_ms": m["k1"], "k1_gbs": by1 / m["k1"] / 1e6,
            "krylov50_ms": m["krylov"], "krylov_gbs": byk / m["krylov"] / 1e6,
            "k1_frac": by1 / m["k1"] / 1e6 / hbm, "krylov_frac": byk / m["krylov"] / 1e6 / hbm,
            "k7_frac": by7 / m["k7"] / 1e6 / hbm,
            "active_cell_iters_per_s": nA / ((m["k7"] + m["k1"] + m["krylov"]) / 1e3),
        })
        if ilu is not None:
            out[-1]["krylov50_ilu0_ms"] = ilu  # includes the per-assembly level schedule + factorisation
    sim.close()
    return out


def direct_line(pkg, no_cpu, reps=3):
    """Exact dense-LU solve (lin_method = LIN_DIRECT): config 5
    full sets of 2048 and 4096 (the maximum) unknowns; GPU time per solve (build +
    factorisation + triangular solves) and, at 2048, the oracle's on one host core."""
    import ctypes as C
    from oracle import Oracle
    out = []
    for nx, ny in ((32, 64), (64, 64)):
        case = pkg.Case(5, nx=nx, ny=ny, nz=1)
        sim = pkg.GpuSimulator(case)
        L, ctx = sim.L, sim._ctx
        s0 = case.init_state()
        s0.u[::case.b] -= np.random.default_rng(7).uniform(0, 3e6, case.n)
        sim.set_state(s0, 86400.0)
        sim.set_active(None)
        sim.assemble()
        opts = case.solver_opts(lin_method=pkg.LIN_DIRECT)
        ms = []
        for r in range(reps + 1):
            L.rsim_gpu_mark(ctx, 16)
            L.rsim_gpu_linear_solve(ctx, C.byref(opts))
            L.rsim_gpu_mark(ctx, 17)
            v = C.c_double()
            L.rsim_gpu_elapsed(ctx, 16, 17, C.byref(v))
            if r:
                ms.append(v.value)
        st = sim.stats()
        xg = sim.solution(case.n)
        sim.close()
        row = {"n_unknowns": case.n * case.b, "ms": float(np.median(ms)), "status": st.status,
               "gpu_launches_per_solve": 3}
        if not no_cpu and case.n <= 2048:
            o = Oracle(case)
            o.set_state(s0, 86400.0)
            o.assemble(np.arange(case.n, dtype=np.int32))
            t0 = time.perf_counter()
            rc, xo, _, _ = o.linear_solve(case.n, opts)
            row["cpu_oracle_ms"] = (time.perf_counter() - t0) * 1e3
            row["cpu_oracle_cores"] = 1
            row["bit_exact_vs_oracle"] = bool(rc == st.status and np.array_equal(xg, xo))
        out.append(row)
    return out


def flash_field(n):
    """Cells of a square 2D grid in natural order: a smooth depletion field (pressure
    drawn down from 3500 psi towards 14.7 psi around 64 seeded producers, the C1
    fraction varying smoothly 0.2-0.8), as a simulator hands cells to the flash.
    Returns p [Pa], z [n*2] and the generator."""
    rng = np.random.default_rng(2008015393)
    side = int(np.sqrt(n))
    n = side * side
    yy, xx = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
    sx, sy = rng.uniform(0, side, 64), rng.uniform(0, side, 64)
    d2 = np.minimum.reduce([(xx.ravel() - a) ** 2.0 + (yy.ravel() - b) ** 2.0 for a, b in zip(sx, sy)])
    rr = 0.08 * side
    p = (14.7 + (3500.0 - 14.7) * (1.0 - np.exp(-d2 / (2 * rr * rr)))) * 6894.757293168361
    z1 = 0.5 + 0.3 * np.sin(2 * np.pi * xx.ravel() / side) * np.cos(2 * np.pi * yy.ravel() / side)
    return p, np.stack([z1, 1.0 - z1], axis=1).reshape(-1), rng


def eos_flash_line(pkg, n, reps, no_cpu):
    """Peng-Robinson flash throughput (paper Case 3 fluid C1/C10
    at 340 K): n cells with seeded pressures 14.7-3500 psi and overall compositions,
    device-resident (rsim_eos_flash_dev on the torch stream, CUDA events), plus the
    oracle on the host cores over a bounded sample.  Compute-bound (rlog / rexp per
    stability and successive-substitution step), so no HBM roofline."""
    import ctypes as C
    import torch
    e = pkg.eos_case3()
    p, z, rng = flash_field(n)
    n = len(p)
    dev = torch.device("cuda")
    tp, tz = torch.from_numpy(p).to(dev), torch.from_numpy(z).to(dev)
    st = torch.empty(n, dtype=torch.uint8, device=dev)
    nu = torch.empty(n, dtype=torch.float64, device=dev)
    tx, ty = torch.empty(2 * n, dtype=torch.float64, device=dev), torch.empty(2 * n, dtype=torch.float64, device=dev)
    zf = torch.empty(2 * n, dtype=torch.float64, device=dev)
    it = torch.empty(n, dtype=torch.int32, device=dev)
    L = pkg._abi.lib()
    stream = torch.cuda.current_stream()

    def run():
        rc = L.rsim_eos_flash_dev(C.byref(e), 340.0, n, tp.data_ptr(), tz.data_ptr(), st.data_ptr(), nu.data_ptr(),
                                  tx.data_ptr(), ty.data_ptr(), zf.data_ptr(), it.data_ptr(), stream.cuda_stream)
        assert rc == 0, rc

    def timed():
        for _ in range(3):
            run()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(reps):
            run()
        ev1.record(stream)
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / reps

    ms = timed()
    stc = st.cpu().numpy()
    out = {"cells": n, "ms": ms, "cells_per_s": n / (ms / 1e3), "two_phase_fraction": float((stc == 2).mean()),
           "mean_iters": float(it.double().mean().item()), "gpu_launches_per_flash": 1,
           "fluid": "C1/C10 (paper Case 3), 340 K",
           "field": "2D grid order, smooth depletion field 14.7-3500 psi around 64 seeded producers, z_C1 0.2-0.8"}
    perm = torch.from_numpy(rng.permutation(n)).to(dev)  # same cells, random order: worst-case warp divergence
    tp.copy_(tp[perm])
    tz.copy_(tz.view(n, 2)[perm].reshape(-1))
    ms_s = timed()
    out["cells_per_s_shuffled"] = n / (ms_s / 1e3)
    tp.copy_(torch.from_numpy(p).to(dev))
    tz.copy_(torch.from_numpy(z).to(dev))
    run()
    if not no_cpu:
        import oracle
        cores = len(os.sched_getaffinity(0))
        oracle.set_threads(cores)
        m = min(n, 1 << 17)
        t0 = time.perf_counter()
        o = oracle.eos_flash(e, 340.0, p[:m], z[:2 * m])
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": m / dt, "unit": "cells/s", "cores": cores, "kind": "port",
                               "sample": f"first {m} cells ({dt:.2f} s, oracle/ OpenMP {cores} threads)"}
        out["bit_exact_vs_oracle_sample"] = bool(np.array_equal(o["nu_g"], nu[:m].cpu().numpy()))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--c5", default="0.01,0.05,0.2,0.5,1.0", help="config-5 active fractions ('' to skip)")
    ap.add_argument("--c5-ilu", default="0.05", help="fractions that also get the ILU(0) row ('' to skip)")
    ap.add_argument("--c5-reps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--direct", type=int, default=1, help="time the exact dense-LU solve at N = 2048 / 4096 (0 to skip)")
    ap.add_argument("--flash-cells", type=int, default=1 << 22, help="PR flash bench cells (0 to skip)")
    ap.add_argument("--precond", type=int, default=None,
                    help="0 block-Jacobi, 2 block-Jacobi + first-order Neumann polynomial (default: case default)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, ws, lr = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, ws)

    dist = init_dist(ws, lr)
    import paper_2008_01539_b200 as pkg
    import ctypes as C
    from paper_2008_01539_b200 import _abi as A
    pkg._abi.lib().rsim_gpu_set_device(lr)
    hbm, peak_kind = peaks()

    case = pkg.Case(WORKLOAD["config"])
    s0 = case.init_state()
    dts = case.schedule()
    opts = case.solver_opts()
    if args.precond is not None:
        opts.precond = args.precond
    sim = pkg.GpuSimulator(case)
    L, ctx = sim.L, sim._ctx
    b, D = case.b, (3 if case.nz > 1 else 2)
    s = 2 * D
    sim.set_state(s0, float(dts[0]))
    L.rsim_gpu_checkpoint(ctx, 0)
    d = np.ascontiguousarray(dts, np.float64)
    it, lin, cuts = C.c_int32(), C.c_int32(), C.c_int32()
    ma, na = C.c_double(), C.c_int64()

    def run_dev():
        rc = L.rsim_run_case_dev(ctx, WORKLOAD["solver"], A.ptr(d, C.c_double), len(d), C.byref(opts), C.byref(it),
                                 C.byref(ma), C.byref(na), C.byref(lin), C.byref(cuts))
        if rc != 0:
            raise RuntimeError(f"run_case_dev failed rc={rc}: {L.rsim_gpu_last_error()}")
        return na.value

    for _ in range(args.warmup):
        L.rsim_gpu_checkpoint(ctx, 1)
        run_dev()
    # ---- device-resident timed region (phase timers OFF: no extra events)
    L.rsim_gpu_timers(ctx, 0, None, None)
    cnt = np.zeros(5, np.int64)
    L.rsim_gpu_counters(ctx, A.ptr(cnt, C.c_int64), 1)
    launches0 = C.c_int32()
    barrier(dist)
    L.rsim_gpu_stats_get(ctx, C.byref(pkg.GpuStats()))
    tot_ms, tot_na = 0.0, 0
    with Clocks(lr) as clk:
        L.rsim_gpu_timers(ctx, -1, None, C.byref(launches0))
        for _ in range(args.steps):
            L.rsim_gpu_checkpoint(ctx, 1)
            L.rsim_gpu_flush_l2(ctx)
            L.rsim_gpu_mark(ctx, 0)
            tot_na += run_dev()
            L.rsim_gpu_mark(ctx, 1)
            v = C.c_double()
            L.rsim_gpu_elapsed(ctx, 0, 1, C.byref(v))
            tot_ms += v.value
        launches1 = C.c_int32()
        L.rsim_gpu_timers(ctx, -1, None, C.byref(launches1))
    barrier(dist)
    L.rsim_gpu_counters(ctx, A.ptr(cnt, C.c_int64), 1)
    n_iters, n_lin, iters_per_run = it.value, lin.value, it.value
    t_max = dist_max(dist, tot_ms)
    na_all = dist_sum(dist, float(tot_na))
    value = na_all / (t_max / 1e3)
    n_launch = int(launches1.value - launches0.value)
    # ---- phase breakdown (separate pass with per-phase CUDA events; not part of `value`)
    L.rsim_gpu_timers(ctx, 1, None, None)
    L.rsim_gpu_checkpoint(ctx, 1)
    L.rsim_gpu_flush_l2(ctx)
    run_dev()
    phase_ms = np.zeros(4)
    L.rsim_gpu_timers(ctx, 0, A.ptr(phase_ms, C.c_double), None)
    phase_ms *= args.steps  # per-run breakdown scaled to the timed steps

    # ---- e2e through the public C-ABI entry point with pinned host buffers
    import torch
    u_pin = torch.empty(len(s0.u), dtype=torch.float64, pin_memory=True).numpy()
    st_pin = torch.empty(len(s0.status), dtype=torch.uint8, pin_memory=True).numpy()
    e2e_t, e2e_na = 0.0, 0
    for k in range(args.steps + 1):
        u_pin[:] = s0.u
        st_pin[:] = s0.status
        L.rsim_gpu_flush_l2(ctx)
        L.rsim_gpu_stats_get(ctx, C.byref(pkg.GpuStats()))
        t0 = time.perf_counter()
        rc = L.rsim_run_case(ctx, WORKLOAD["solver"], A.ptr(u_pin, C.c_double), A.ptr(st_pin, C.c_uint8),
                             A.ptr(d, C.c_double), len(d), C.byref(opts), C.byref(it), C.byref(ma), C.byref(na),
                             C.byref(lin), C.byref(cuts))
        dt_ = time.perf_counter() - t0
        if rc != 0:
            raise RuntimeError("rsim_run_case failed")
        if k > 0:
            e2e_t += dt_
            e2e_na += na.value
    e2e_t = dist_max(dist, e2e_t)
    e2e_v = dist_sum(dist, float(e2e_na)) / e2e_t
    h2d = s0.u.nbytes + s0.status.nbytes + d.nbytes
    d2h = s0.u.nbytes + s0.status.nbytes

    # ---- roofline of the dominant kernel (per-phase CUDA-event time)
    names = ["set_estimation_K7", "assembly_K1", "krylov_bicgstab_K3K5", "update_K6"]
    dom = int(np.argmax(phase_ms))
    row_iters, solves, krylov_rows, asm_rows = int(cnt[1]), int(cnt[2]), int(cnt[3]), int(cnt[0])
    nnc_per_row = case.n_nnc / case.n
    if dom == 2:
        alg = row_iters * bytes_krylov_row_iter(b, s) + krylov_rows * bytes_krylov_row_init(b)
        per_launch_units = f"{bytes_krylov_row_iter(b, s)} B per row-iteration + {bytes_krylov_row_init(b)} B per row init"
    elif dom == 1:
        alg = asm_rows * bytes_assembly_row(b, D, s, nnc_per_row)
        per_launch_units = f"{bytes_assembly_row(b, D, s, nnc_per_row):.1f} B per active row"
    else:
        alg = int(cnt[4]) * bytes_k7(case.n, 0, 2)
        per_launch_units = f"{bytes_k7(case.n, 0, 2)} B per full-grid set update"
    achieved = alg / (phase_ms[dom] / 1e3) / 1e9
    # measured DRAM traffic per launch of that kernel (ncu --set full, committed
    # under profiles/): compare with the algorithmic bytes per launch
    kern = {0: "k_scatter_rg", 1: "k_assemble", 2: "k_krylov_dsm", 3: "k_update"}[dom]
    traffic = None
    try:
        tj = json.load(open(Path(__file__).resolve().parent / "profiles" / "r01_traffic.json"))
        traffic = tj["dram_bytes_per_launch"].get(kern)
    except (OSError, ValueError, KeyError):
        pass
    launches_dom = solves if dom == 2 else max(1, iters_per_run * args.steps)
    roof = {"kernel": names[dom], "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "peak_kind": peak_kind, "traffic": traffic,
            "traffic_unit": "DRAM bytes per launch (ncu --set full, profiles/r01_ncu_summary.md)",
            "algorithmic_bytes_per_launch": alg / launches_dom,
            "algorithmic_bytes": per_launch_units,
            "phase_ms_per_step": {k: float(v) / args.steps for k, v in zip(names, phase_ms)},
            "krylov_solves_per_step": solves / args.steps, "krylov_row_iters_per_step": row_iters / args.steps}

    line = {
        "metric": "active-cell Newton iters/s", "value": value, "unit": "active-cell iters/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY.md App. A)",
        "config": {"workload": WORKLOAD["name"], "n_cells": case.n, "timesteps": len(dts),
                   "newton_iters_per_run": iters_per_run, "krylov_iters_per_run": n_lin,
                   "sum_nA_per_run": tot_na // args.steps, "l2": "flushed (512 MB write) before every step",
                   "parallelism": f"replicas x{ws}"},
        "e2e": {"value": e2e_v, "unit": "active-cell iters/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "api": "rsim_run_case (C-ABI), pinned host buffers"},
        "gpu_launches": n_launch,
        "roofline": roof,
        "clocks": clk.summary(),
    }
    if rank == 0:  # the paper's comparison on the same workload (one timed run each, after the timed region)
        cmp = {}
        for sv, nm in ((0, "standard"), (1, "localized"), (2, "adaptive_dd")):
            sim.run_case(sv, s0, dts, opts)
            sim.L.rsim_gpu_mark(sim._ctx, 20)
            r = sim.run_case(sv, s0, dts, opts)
            sim.L.rsim_gpu_mark(sim._ctx, 21)
            ms = C.c_double()
            sim.L.rsim_gpu_elapsed(sim._ctx, 20, 21, C.byref(ms))
            cmp[nm] = {"ms_per_run": ms.value, "newton_iters": r["iterations"], "krylov_iters": r["lin_iters"],
                       "sum_nA": r["sum_na"], "total_MA": r["total_ma"], "status": r["status"]}
        line["solver_comparison"] = cmp
    sim.close()
    if rank == 0 and args.c5:
        fr = [float(x) for x in args.c5.split(",") if x]
        ilu_fr = [float(x) for x in args.c5_ilu.split(",") if x.strip()]
        line["c5_sweep"] = c5_sweep(pkg, fr, args.c5_reps, hbm, ilu_fr)
    if rank == 0 and args.flash_cells > 0:
        line["eos_flash"] = eos_flash_line(pkg, args.flash_cells, 5, args.no_cpu)
    if rank == 0 and args.direct:
        line["direct_solve"] = direct_line(pkg, args.no_cpu)
    if rank == 0 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(case, s0, dts, opts)
    barrier(dist)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
