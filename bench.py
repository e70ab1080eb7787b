#!/usr/bin/env python
"""bench.py — active-cell Newton iterations/s of the localized FIM solver on one B200.

Contract:
  python bench.py --gpus N --steps K --warmup W [--impl reference]
One JSON line on rank 0.

Headline workload (config.workload): BASELINE.json configs[3] — config 4, the
3D three-phase black-oil model with gas liberation, 512x512x16 = 4.2 M cells,
400 DFN planes + 20 stage fractures, the whole 20-step schedule, adaptive-
localized Newton (Algorithm 1).  It is the largest full-Newton config that fits
one GPU (config 5 is a kernel sweep).  One bench "step" = one whole run from the
seeded initial state.  metric = Σ n_A over every Newton iteration / time.

  value : device-resident runs (state already in HBM), CUDA events on the
          context stream, L2 flushed (512 MB write) before every step.
  e2e   : the same run through the public C-ABI entry point rsim_run_case
          with pinned host buffers (H2D of the initial state + D2H of the
          final state inside the timed region).
  roofline : dominant phase of the workload (per-phase CUDA events).
  parity_vs_oracle : the timed run's totals and final-state sha256 against the
          oracle fixture of the same run (tests/golden/, make_golden.py), plus a
          live bit-exact check against the oracle's CPU sample in this run.
  cpu_baseline : the CPU oracle (oracle/, C++ restatement, OpenMP on every
          host core) on a bounded sample of the same workload, with the GPU's
          rate on exactly that sample beside it.
  per_config : configs 1-3 with the same fields (c3 logs the active fraction
          of every Newton iteration); c5_sweep : config 5 kernel throughput
          (K7 / K1 / 50 BiCGSTAB) at 1-100 % active; eos_flash; direct_solve.
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
# algorithmic bytes: b unknowns/cell, s Cartesian slots, nnc NNC entries per row
def bytes_spmv_row(b, s, nnc=0.0, cols=True):
    # per row: (s + NNC) column indices (4 B, absent when the columns are structural)
    # and b×b blocks, own x read + y write (unit diagonal implicit)
    return (s + nnc) * (8 * b * b + (4 if cols else 0)) + 16 * b


def bytes_krylov_row_iter(b, s, nnc=0.0, neumann=False, cols=True):
    # one BiCGSTAB iteration: 2 SpMVs (4 with the first-order Neumann polynomial:
    # M⁻¹z = 2z − Âz before each product) + 14 vector passes: (r0,v),(r,r) 2,
    # s update 3, (r0,s),(r0,t) 1, x/r/next-p update 8 (x, p, s, t, v read; x, r, p written)
    return (4 if neumann else 2) * bytes_spmv_row(b, s, nnc, cols) + 112 * b


def bytes_krylov_counted(b, s, rows_its, blk_its, neumann=False):
    # b > 1, partial sets, from the work counters (rsim_gpu_block_counters): per row and
    # SpMV the s column indices + own x read + y write; per STORED block (active Cartesian
    # neighbour; frozen neighbours have no block and their value slots are not read) its b²
    # values — pressure-only blocks included: the kernels load them whole;
    # + the 14 vector passes.  NNC blocks (rare) are left out.
    k = 4 if neumann else 2
    return k * (rows_its * (4 * s + 16 * b) + 8 * b * b * blk_its) + 112 * b * rows_its


def bytes_krylov_row_init(b):
    return 8 * b * 4  # read rhs, write r, r0, x


def bytes_assembly_row(b, D, s, nnc_per_row=0.0):
    # 24b + 8 + 8D + 12·NNC + 4 + (1+s)·8b²
    return 24 * b + 8 + 8 * D + 12 * nnc_per_row + 4 + (1 + s) * 8 * b * b


def bytes_k7(n, nA, m):
    return (19 + 2 * m) * n + 4 * nA


# The named synthetic grids (BASELINE.json configs[0..3]).  The
# first solver is the config's measured line; the others are the paper's comparison.
# Fixtures: tests/golden/<name>.npz, made by tests/golden/make_golden.py from the CPU
# oracle on exactly these runs (whole schedule, seeded initial state).
CONFIGS = {
    1: dict(key="c1", workload="c1_singlephase_100x100_fracture_20steps", solvers=("localized", "standard"),
            fixtures={"localized": "c1_localized", "standard": "c1_bench_standard"}, cpu="full"),
    2: dict(key="c2", workload="c2_oilwater_256x256_dfn40_30steps", solvers=("localized", "adaptive_dd", "standard"),
            fixtures={"localized": "c2_bench_localized", "adaptive_dd": "c2_bench_dd"}, cpu="full"),
    3: dict(key="c3", workload="c3_hydrofrac_256x256x32_12stages_20steps",
            solvers=("localized", "adaptive_dd", "standard"),
            fixtures={"localized": "c3_full_localized", "adaptive_dd": "c3_full_dd"}, cpu="step1"),
    4: dict(key="c4", workload="c4_blackoil_512x512x16_dfn400_20stages_20steps", solvers=("localized", "adaptive_dd"),
            fixtures={"localized": "c4_full_localized", "adaptive_dd": "c4_full_dd"}, cpu="newton1"),
}
HEADLINE = 4  # the largest full-Newton config that fits one GPU (c5 is a kernel sweep)
SOLVER_ID = {"standard": 0, "localized": 1, "adaptive_dd": 2}
GOLDEN = Path(ROOT) / "tests" / "golden"
CPU_SAMPLES = {
    "full": "whole runs of the workload (every timestep)",
    "step1": "the first timestep of the workload (run_case over dts[:1])",
    "newton1": "the first Newton iteration of the first timestep (newton_localized, max_newton = 1, "
               "from the seeded state and V_A^init)",
}


def opts_for(case, solver: str, precond=None):
    """Solver options of a config (tests/golden/make_golden.py opts_for: m = 4 for DD, App. A)."""
    o = case.solver_opts()
    if precond is not None:
        o.precond = precond
    if solver == "adaptive_dd":
        o.m = 4
    return o


def state_digest(u, st) -> dict:
    import hashlib
    return {"u_sha256": hashlib.sha256(np.ascontiguousarray(u, np.float64).tobytes()).hexdigest(),
            "st_sha256": hashlib.sha256(np.ascontiguousarray(st, np.uint8).tobytes()).hexdigest()}


def fixture_check(name: str, r: dict, u, st) -> dict:
    """GPU run totals + final-state digest against the oracle fixture of the same run."""
    p = GOLDEN / f"{name}.npz"
    if not p.exists():
        return {"fixture": name, "match": None, "why": "fixture missing"}
    g = np.load(p)
    dg = state_digest(u, st)
    ref = ({"u_sha256": str(g["u_sha256"]), "st_sha256": str(g["st_sha256"])} if "u_sha256" in g
           else state_digest(g["u"], g["st"]))
    bad = [k for k in ("status", "iterations", "sum_na", "lin_iters", "cuts") if int(r[k]) != int(g[k])]
    if float(r["total_ma"]) != float(g["total_ma"]):
        bad.append("total_ma")
    bad += [k for k in ("u_sha256", "st_sha256") if dg[k] != ref[k]]
    return {"fixture": name, "match": not bad, "mismatch": bad,
            "checked": "status, Newton/Krylov iterations, Σn_A, cuts, M_A, sha256 of final u and status"}


class GpuRun:
    """One config on one GPU context: device-resident run_case with checkpoint restore."""

    def __init__(self, pkg, cfg: int, solver: str, precond=None):
        import ctypes as C
        self.C, self.pkg = C, pkg
        self.case = pkg.Case(cfg)
        self.s0 = self.case.init_state()
        self.dts = np.ascontiguousarray(self.case.schedule(), np.float64)
        self.solver = solver
        self.opts = opts_for(self.case, solver, precond)
        self.sim = pkg.GpuSimulator(self.case)
        self.L, self.ctx = self.sim.L, self.sim._ctx
        self.sim.set_state(self.s0, float(self.dts[0]))
        self.L.rsim_gpu_checkpoint(self.ctx, 0)
        self.it, self.lin, self.cuts = C.c_int32(), C.c_int32(), C.c_int32()
        self.ma, self.na = C.c_double(), C.c_int64()

    def totals(self, rc):
        return {"status": rc, "iterations": self.it.value, "sum_na": self.na.value, "lin_iters": self.lin.value,
                "cuts": self.cuts.value, "total_ma": self.ma.value}

    def run_dev(self, solver=None, restore=True):
        from paper_2008_01539_b200 import _abi as A
        C = self.C
        sid = SOLVER_ID[solver or self.solver]
        opts = self.opts if solver in (None, self.solver) else opts_for(self.case, solver)
        if restore:
            self.L.rsim_gpu_checkpoint(self.ctx, 1)
        rc = self.L.rsim_run_case_dev(self.ctx, sid, A.ptr(self.dts, C.c_double), len(self.dts), C.byref(opts),
                                      C.byref(self.it), C.byref(self.ma), C.byref(self.na), C.byref(self.lin),
                                      C.byref(self.cuts))
        if rc != 0:
            raise RuntimeError(f"run_case_dev failed rc={rc}: {self.L.rsim_gpu_last_error()}")
        return self.totals(rc)

    def timed_dev(self, solver=None):
        """One device-resident run, L2 flushed first, CUDA events on the context stream."""
        C = self.C
        self.L.rsim_gpu_checkpoint(self.ctx, 1)  # seeded initial state (outside the timed region)
        self.L.rsim_gpu_flush_l2(self.ctx)
        self.L.rsim_gpu_mark(self.ctx, 0)
        r = self.run_dev(solver, restore=False)
        self.L.rsim_gpu_mark(self.ctx, 1)
        v = C.c_double()
        self.L.rsim_gpu_elapsed(self.ctx, 0, 1, C.byref(v))
        return v.value, r

    def state(self):
        s = self.sim.get_state()
        return s.u, s.status

    def close(self):
        self.sim.close()


def measure_config(pkg, cfg: int, steps: int, warmup: int, hbm: float, peak_kind: str, dist=None, lr=0,
                   e2e_runs: int | None = None, compare: bool = True) -> dict:
    """value / e2e / roofline / launches / clocks / parity of one config's main solver;
    the paper's solver comparison on the same workload."""
    from paper_2008_01539_b200 import _abi as A
    import ctypes as C
    spec = CONFIGS[cfg]
    main = spec["solvers"][0]
    R = GpuRun(pkg, cfg, main)
    L, ctx, case = R.L, R.ctx, R.case
    b, D = case.b, (3 if case.nz > 1 else 2)
    s = 2 * D
    for _ in range(warmup):
        R.run_dev()
    # ---- device-resident timed region (phase timers off: no extra events)
    L.rsim_gpu_timers(ctx, 0, None, None)
    cnt = np.zeros(5, np.int64)
    barrier(dist)
    tot_ms, tot_na = 0.0, 0
    l0, l1 = C.c_int32(), C.c_int32()
    with Clocks(lr) as clk:
        L.rsim_gpu_timers(ctx, -1, None, C.byref(l0))
        for _ in range(steps):
            ms, r = R.timed_dev()
            tot_ms += ms
            tot_na += r["sum_na"]
        L.rsim_gpu_timers(ctx, -1, None, C.byref(l1))
    barrier(dist)
    u_end, st_end = R.state()
    t_max = dist_max(dist, tot_ms)
    value = dist_sum(dist, float(tot_na)) / (t_max / 1e3)
    out = {"workload": spec["workload"], "solver": main, "n_cells": case.n, "b": b, "timesteps": len(R.dts),
           "value": value, "unit": "active-cell iters/s", "ms_per_step": t_max / steps, "steps": steps,
           "warmup": warmup, "gpu_launches": int(l1.value - l0.value), "clocks": clk.summary(),
           "run": dict(r),
           "active_fraction_mean": r["total_ma"] / max(1, r["iterations"])}
    parity = {main: fixture_check(spec["fixtures"][main], r, u_end, st_end)}
    # ---- phase breakdown (separate run with per-phase CUDA events; not part of `value`)
    L.rsim_gpu_timers(ctx, 1, None, None)
    L.rsim_gpu_checkpoint(ctx, 1)
    L.rsim_gpu_flush_l2(ctx)
    L.rsim_gpu_counters(ctx, None, 1)
    L.rsim_gpu_block_counters(ctx, None, 1)
    R.run_dev(restore=False)
    phase_ms = np.zeros(4)
    L.rsim_gpu_timers(ctx, 0, A.ptr(phase_ms, C.c_double), None)
    L.rsim_gpu_counters(ctx, A.ptr(cnt, C.c_int64), 1)  # work counters of this one run
    bcnt = np.zeros(2, dtype=np.int64)
    L.rsim_gpu_block_counters(ctx, A.ptr(bcnt, C.c_int64), 1)
    # ---- e2e through the public C-ABI entry point with pinned host buffers
    import torch
    u_pin = torch.empty(len(R.s0.u), dtype=torch.float64, pin_memory=True).numpy()
    st_pin = torch.empty(len(R.s0.status), dtype=torch.uint8, pin_memory=True).numpy()
    ne = steps if e2e_runs is None else max(1, min(steps, e2e_runs))
    e2e_t, e2e_na = 0.0, 0
    for k in range(ne + 1):
        u_pin[:] = R.s0.u
        st_pin[:] = R.s0.status
        L.rsim_gpu_flush_l2(ctx)
        L.rsim_gpu_stats_get(ctx, C.byref(pkg.GpuStats()))
        t0 = time.perf_counter()
        rc = L.rsim_run_case(ctx, SOLVER_ID[main], A.ptr(u_pin, C.c_double), A.ptr(st_pin, C.c_uint8),
                             A.ptr(R.dts, C.c_double), len(R.dts), C.byref(R.opts), C.byref(R.it), C.byref(R.ma),
                             C.byref(R.na), C.byref(R.lin), C.byref(R.cuts))
        dt_ = time.perf_counter() - t0
        if rc != 0:
            raise RuntimeError("rsim_run_case failed")
        if k > 0:
            e2e_t += dt_
            e2e_na += R.na.value
    e2e_t = dist_max(dist, e2e_t)
    out["e2e"] = {"value": dist_sum(dist, float(e2e_na)) / e2e_t, "unit": "active-cell iters/s",
                  "h2d_bytes_per_step": int(R.s0.u.nbytes + R.s0.status.nbytes + R.dts.nbytes),
                  "d2h_bytes_per_step": int(R.s0.u.nbytes + R.s0.status.nbytes), "runs": ne,
                  "api": "rsim_run_case (C-ABI), pinned host buffers"}
    parity[main]["e2e_state_match"] = state_digest(u_pin, st_pin) == state_digest(u_end, st_end)
    # ---- roofline of the dominant phase (per-phase CUDA-event time, algorithmic bytes)
    names = ["set_estimation_K7", "assembly_K1", "krylov_bicgstab_K3K5", "update_K6"]
    dom = int(np.argmax(phase_ms))
    asm_rows, row_iters, solves, krylov_rows, k7_updates = (int(x) for x in cnt)
    nnc = case.n_nnc * 2 / case.n  # NNC entries per row (each NNC is stored in both rows)
    neu = R.opts.precond == pkg.PREC_NEUMANN1
    if dom == 2:
        if b > 1:  # counted: the blocks actually stored (frozen neighbours have none)
            blk_its, po_its = int(bcnt[0]), int(bcnt[1])
            alg_it = bytes_krylov_counted(b, s, row_iters, blk_its, neu)
            per = alg_it / max(1, row_iters)
            extra = f"; {blk_its / max(1, row_iters):.2f} stored blocks per row, " \
                    f"{po_its / max(1, blk_its):.3f} of them pressure-only (loaded whole); all {s} slots filled: " \
                    f"{bytes_krylov_row_iter(b, s, nnc, neu):.1f} B"
        else:
            per = bytes_krylov_row_iter(b, s, nnc, neu)
            alg_it, extra = row_iters * per, ""
        alg = alg_it + krylov_rows * bytes_krylov_row_init(b)
        units = f"{per:.1f} B per row-iteration ({'Neumann-1: 4' if neu else '2'} SpMVs) + " \
                f"{bytes_krylov_row_init(b)} B per row init" + extra
        launches_dom = solves
    elif dom == 1:
        per = bytes_assembly_row(b, D, s, nnc)
        alg, units, launches_dom = asm_rows * per, f"{per:.1f} B per active row", max(1, r["iterations"])
    else:
        alg = k7_updates * bytes_k7(case.n, 0, R.opts.m)
        units, launches_dom = f"{bytes_k7(case.n, 0, R.opts.m)} B per full-grid set update", max(1, k7_updates)
    achieved = alg / (phase_ms[dom] / 1e3) / 1e9
    out["roofline"] = {"kernel": names[dom], "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                       "frac": achieved / hbm, "peak_kind": peak_kind, "traffic": None,
                       "traffic_note": "ncu DRAM bytes of this kernel: profiles/ (not measurable inside this run)",
                       "algorithmic_bytes_per_launch": alg / max(1, launches_dom), "algorithmic_bytes": units,
                       "phase_ms_per_run": {k: float(v) for k, v in zip(names, phase_ms)},
                       "krylov_solves_per_run": solves, "krylov_row_iters_per_run": row_iters}
    # ---- the paper's comparison on the same workload (one timed device-resident run each)
    if compare:
        cmp = {main: {"ms_per_run": t_max / steps, **out["run"]}}
        for sv in spec["solvers"][1:]:
            if case.n <= 1 << 20:
                R.run_dev(sv)  # warm (small configs; the big ones are warm from the main solver)
            ms, rr = R.timed_dev(sv)
            cmp[sv] = {"ms_per_run": ms, **rr}
            if sv in spec["fixtures"]:
                u2, st2 = R.state()
                parity[sv] = fixture_check(spec["fixtures"][sv], rr, u2, st2)
        out["solver_comparison"] = cmp
    out["parity_vs_oracle"] = parity
    out["_R"] = R
    out["_final"] = (u_end, st_end)
    return out


def cpu_sample(cfg: int, threads: int, budget_s: float = 10.0, max_runs: int = 30) -> dict:
    """The CPU oracle (oracle/, OpenMP) on a bounded sample of config cfg's workload.
    Returns the rate and the sample's result (for the live GPU-vs-oracle check)."""
    import oracle
    from oracle import Oracle
    oracle.set_threads(threads)
    spec = CONFIGS[cfg]
    main = spec["solvers"][0]
    case = oracle.Case(cfg)
    s0, dts = case.init_state(), case.schedule()
    opts = opts_for(case, main)
    orc = Oracle(case)
    kind = spec["cpu"]
    tot_na, tot_t, runs, last = 0, 0.0, 0, None
    while runs < 1 or (tot_t < budget_s and runs < max_runs):
        if kind == "newton1":
            opts.max_newton = 1
            va = orc.initial_active(None, opts.eps_set, opts.m)
            t0 = time.perf_counter()
            _, rep, rc = orc.newton_localized(s0, float(dts[0]), va, opts.m, opts.eps_set, opts)
            dt = time.perf_counter() - t0
            na = rep.sum_na
            last = {"records": rep.records(), "rc": rc}
        else:
            d = dts if kind == "full" else dts[:1]
            t0 = time.perf_counter()
            r = orc.run_case(SOLVER_ID[main], s0, d, opts)
            dt = time.perf_counter() - t0
            na = r["sum_na"]
            last = r
        tot_na, tot_t, runs = tot_na + na, tot_t + dt, runs + 1
        if kind != "full":
            break
    return {"value": tot_na / tot_t, "unit": "active-cell iters/s", "cores": threads, "kind": "port",
            "sample": f"{runs} x {CPU_SAMPLES[kind]} ({tot_t:.1f} s, oracle/ OpenMP {threads} threads)",
            "model": _cpu_model(), "_last": last, "_kind": kind, "_seconds": tot_t}


def gpu_same_sample(R: GpuRun, kind: str, cpu_last, final=None) -> dict:
    """The GPU on exactly the CPU sample (rate like for like) + live bit-exact check."""
    C = R.C
    if kind == "full":
        u, st = final  # final state of the timed runs (the whole workload)
        ok = state_digest(u, st) == state_digest(cpu_last["states"].u, cpu_last["states"].status)
        return {"live_oracle_match": bool(ok), "checked": "sha256 of the final u / status after the whole run"}
    if kind == "step1":
        R.L.rsim_gpu_checkpoint(R.ctx, 1)
        s0 = R.s0
        R.L.rsim_gpu_mark(R.ctx, 2)
        r = R.sim.run_case(SOLVER_ID[R.solver], s0, R.dts[:1], R.opts)
        R.L.rsim_gpu_mark(R.ctx, 3)
        v = C.c_double()
        R.L.rsim_gpu_elapsed(R.ctx, 2, 3, C.byref(v))
        ok = all(r[k] == cpu_last[k] for k in ("status", "iterations", "sum_na", "lin_iters", "cuts")) and \
            np.array_equal(r["states"].u, cpu_last["states"].u)
        return {"value": r["sum_na"] / (v.value / 1e3), "ms": v.value, "live_oracle_match": bool(ok),
                "checked": "totals and final u of the first timestep, bit for bit"}
    # newton1: the first Newton iteration from the seeded state
    opts = opts_for(R.case, R.solver)
    opts.max_newton = 1
    R.sim.set_state(R.s0, float(R.dts[0]))
    R.sim.initial_active(True, opts.eps_set, opts.m)
    va = R.sim.active()
    R.L.rsim_gpu_mark(R.ctx, 2)
    _, rep = R.sim.newton_localized(R.s0, float(R.dts[0]), va, opts.m, opts.eps_set, opts)
    R.L.rsim_gpu_mark(R.ctx, 3)
    v = C.c_double()
    R.L.rsim_gpu_elapsed(R.ctx, 2, 3, C.byref(v))
    g, o = rep.records(), cpu_last["records"]
    ok = len(g) == len(o) and all(a == b for a, b in zip(g, o))
    return {"value": rep.sum_na / (v.value / 1e3), "ms": v.value, "live_oracle_match": bool(ok),
            "checked": "per-iteration records (n_A, Krylov iterations, ‖δp‖∞, ‖F‖₂, ‖F‖∞, Krylov residual), bit for bit"}


def cpu_serial(cfg: int) -> dict | None:
    """One thread (the SPEC's serial oracle) on one whole run: c1, c2 only."""
    if CONFIGS[cfg]["cpu"] != "full":
        return None
    r = cpu_sample(cfg, 1, budget_s=0.0, max_runs=1)
    return {"value": r["value"], "unit": r["unit"], "cores": 1, "sample": r["sample"]}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def strip(d: dict) -> dict:
    return {k: v for k, v in d.items() if not k.startswith("_")}


def run_reference(args, rank, ws):
    """--impl reference: the CPU oracle (port of SPEC + Algorithms 1-2, oracle/) on all host
    threads, on the headline config's bounded sample; never loads the product library."""
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    spec = CONFIGS[HEADLINE]
    vals, secs, sample = [], 0.0, ""
    for k in range(args.warmup + args.steps):
        r = cpu_sample(HEADLINE, cores, budget_s=0.0, max_runs=1)
        if k >= args.warmup:
            vals.append(r["value"])
            secs += r["_seconds"]
            sample = r["sample"]
    v = len(vals) / sum(1.0 / x for x in vals)  # Σ n_A / Σ t over the timed samples (equal n_A per sample)
    loaded = sorted({ln.split()[-1] for ln in open("/proc/self/maps") if "rsim" in ln and ".so" in ln})
    c = cpu_case(HEADLINE)
    line = {
        "metric": "active-cell Newton iters/s", "value": v, "unit": "active-cell iters/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, SURVEY.md App. A)", "impl": "reference",
        "config": config_key(HEADLINE, c.n, len(c.schedule()), ws),
        "cpu_baseline": {"value": v, "unit": "active-cell iters/s", "cores": cores, "kind": "port",
                         "sample": f"each step: {sample}"},
        "e2e": {"value": v, "unit": "active-cell iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "native_libs_loaded": loaded,
    }
    print(json.dumps(line), flush=True)


def cpu_case(cfg: int):
    import oracle  # the oracle library's own linked case generator (no product library)
    return oracle.Case(cfg)


def config_key(cfg: int, n: int, nsteps: int, ws: int) -> dict:
    """The `config` object: identical in both arms (workload identity only)."""
    return {"workload": CONFIGS[cfg]["workload"], "n_cells": n, "timesteps": nsteps,
            "solver": CONFIGS[cfg]["solvers"][0], "parallelism": f"replicas x{ws}"}


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
        # full set: the ELL columns are structural (computed from the cell coordinates, not loaded)
        byk = nA * (50 * bytes_krylov_row_iter(b, s, cols=nA < n) + bytes_krylov_row_init(b))
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
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--configs", default="1,2,3", help="per-config lines besides the headline ('' to skip)")
    ap.add_argument("--paper", type=int, default=1, help="paper Tables 2/3/5/6 on the EDFM case files (0 to skip)")
    ap.add_argument("--c5", default="0.01,0.05,0.2,0.5,1.0", help="config-5 active fractions ('' to skip)")
    ap.add_argument("--c5-ilu", default="0.05", help="fractions that also get the ILU(0) row ('' to skip)")
    ap.add_argument("--c5-reps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--direct", type=int, default=1, help="time the exact dense-LU solve at N = 2048 / 4096 (0 to skip)")
    ap.add_argument("--flash-cells", type=int, default=1 << 22, help="PR flash bench cells (0 to skip)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank, ws, lr = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, ws)

    dist = init_dist(ws, lr)
    import paper_2008_01539_b200 as pkg
    pkg._abi.lib().rsim_gpu_set_device(lr)
    hbm, peak_kind = peaks()
    cores = len(os.sched_getaffinity(0))

    # ---- headline: the largest full-Newton config (c4), whole 20-step schedule, localized Newton
    h = measure_config(pkg, HEADLINE, args.steps, args.warmup, hbm, peak_kind, dist, lr, e2e_runs=2,
                       compare=(rank == 0 and ws == 1))
    R = h.pop("_R")
    line = {
        "metric": "active-cell Newton iters/s", "value": h["value"], "unit": "active-cell iters/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": h["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY.md App. A)",
        "config": config_key(HEADLINE, R.case.n, len(R.dts), ws),
        "e2e": h["e2e"], "gpu_launches": h["gpu_launches"], "roofline": h["roofline"], "clocks": h["clocks"],
        "workload_detail": {"b": h["b"], "run": h["run"], "active_fraction_mean": h["active_fraction_mean"],
                            "step": "one whole run of the schedule from the seeded initial state",
                            "l2": "flushed (512 MB write) before every step"},
        "parity_vs_oracle": h["parity_vs_oracle"],
    }
    if "solver_comparison" in h:
        line["solver_comparison"] = h["solver_comparison"]
    final = h.pop("_final")
    if rank == 0 and ws == 1 and not args.no_cpu:
        cb = cpu_sample(HEADLINE, cores)
        same = gpu_same_sample(R, cb["_kind"], cb["_last"], final)
        line["cpu_baseline"] = strip(cb)
        line["cpu_baseline"]["gpu_same_sample"] = same
        line["parity_vs_oracle"]["live_sample"] = same.get("live_oracle_match")
    R.close()

    # ---- the other named grids (c1..c3), each with its own value / e2e / roofline / CPU baseline
    if rank == 0 and ws == 1 and args.configs:
        per = {}
        for cfg in (int(x) for x in args.configs.split(",") if x.strip()):
            small = cfg in (1, 2)
            m = measure_config(pkg, cfg, args.steps if not small else max(args.steps, 5), 3 if small else 1,
                               hbm, peak_kind, None, lr, e2e_runs=None if small else 2)
            Rc = m.pop("_R")
            if not args.no_cpu:
                cb = cpu_sample(cfg, cores)
                same = gpu_same_sample(Rc, cb["_kind"], cb["_last"], m["_final"])
                m["cpu_baseline"] = strip(cb)
                m["cpu_baseline"]["gpu_same_sample"] = same
                m["parity_vs_oracle"]["live_sample"] = same.get("live_oracle_match")
                ser = cpu_serial(cfg)
                if ser:
                    m["cpu_baseline"]["serial"] = ser
            if cfg == 3:  # BASELINE configs[2]: active fraction per Newton iteration, logged
                m["active_fraction_per_iteration"] = active_fraction_log(pkg, cfg)
            Rc.close()
            m.pop("_final")
            per[CONFIGS[cfg]["key"]] = m
        line["per_config"] = per
    if rank == 0 and ws == 1 and args.paper:
        line["paper_tables"] = paper_tables(pkg)
    if rank == 0 and ws == 1 and args.c5:
        fr = [float(x) for x in args.c5.split(",") if x]
        ilu_fr = [float(x) for x in args.c5_ilu.split(",") if x.strip()]
        line["c5_sweep"] = c5_sweep(pkg, fr, args.c5_reps, hbm, ilu_fr)
    if rank == 0 and ws == 1 and args.flash_cells > 0:
        line["eos_flash"] = eos_flash_line(pkg, args.flash_cells, 5, args.no_cpu)
    if rank == 0 and ws == 1 and args.direct:
        line["direct_solve"] = direct_line(pkg, args.no_cpu)
    barrier(dist)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


# Paper Tables 2 / 3 / 5 / 6 (§5) with the SPEC acceptance bands 2, 3, 5, 6
# on the EDFM case files (cases/*.case; geometry is a [choice]).
PAPER = {"paper_case1": {"table": 2, "localized": (159, 11.4, 0.072), "standard": (156, 156, 1.0),
                         "dd_table": 5, "adaptive_dd": (804, 20.8, 0.026)},
         "paper_case2": {"table": 3, "localized": (155, 10.1, 0.065), "standard": (153, 153, 1.0),
                         "dd_table": 6, "adaptive_dd": (255, 13.6, 0.053)}}


def paper_tables(pkg) -> dict:
    out = {}
    for name, ref in PAPER.items():
        path = os.path.join(ROOT, "cases", name + ".case")
        r = {}
        for sv in ("standard", "localized", "adaptive_dd"):
            m = pkg.simulate_file(path, sv, None, write_fields=False)
            r[sv] = {"timesteps": m["timesteps"], "iterations": m["total_iters"], "total_MA": m["total_ma"],
                     "avg_MA": m["avg_ma"], "outer_iterations": m["total_outer"], "krylov_iters": m["total_lin"],
                     "cuts": m["cuts"], "solver_wall_s": m["wall_s"], "status": m["status"],
                     "paper_iterations_totalMA_avgMA": ref[sv]}
        std, loc, dd = r["standard"], r["localized"], r["adaptive_dd"]
        bands = {"localized_total_MA <= standard/6": loc["total_MA"] <= std["total_MA"] / 6,
                 "localized_avg_MA <= 0.15": loc["avg_MA"] <= 0.15}
        if name == "paper_case1":
            bands["localized_iterations <= 1.25 x standard"] = loc["iterations"] <= 1.25 * std["iterations"]
            bands["dd_total_MA <= standard/5"] = dd["total_MA"] <= std["total_MA"] / 5
            bands["dd_inner <= 8 x standard"] = dd["iterations"] <= 8 * std["iterations"]
            bands["dd_outer_per_step <= 2 x standard_per_step"] = \
                dd["outer_iterations"] / dd["timesteps"] <= 2 * std["iterations"] / std["timesteps"]
        else:
            bands["dd_total_MA <= standard/6"] = dd["total_MA"] <= std["total_MA"] / 6
            bands["dd_inner <= 3 x standard"] = dd["iterations"] <= 3 * std["iterations"]
        r["spec_acceptance"] = {"tables": (ref["table"], ref["dd_table"]), "bands": bands}
        out[name] = r
    return out


def active_fraction_log(pkg, cfg: int) -> dict:
    """Per-iteration active fraction n_A/n of the config's whole run (the case runner's
    iterations.csv, one row per Newton iteration of every committed timestep)."""
    import tempfile
    spec = CONFIGS[cfg]
    with tempfile.TemporaryDirectory() as d:
        pkg.simulate(cfg, spec["solvers"][0], d, write_fields=False)
        rows = [ln.split(",") for ln in open(os.path.join(d, "iterations.csv")).read().splitlines()[1:]]
    rows = [r for r in rows if r[2] == "1"]  # committed attempts
    frac = [float(r[6]) for r in rows]
    per_step = {}
    for r in rows:
        per_step.setdefault(int(r[0]), []).append(round(float(r[6]), 5))
    return {"iterations": len(frac), "min": min(frac), "max": max(frac), "mean": float(np.mean(frac)),
            "per_timestep": per_step, "source": "rsim_simulate iterations.csv (column n_active/n)"}


if __name__ == "__main__":
    main()
