"""Per-phase device time (K7 set update, K1 assembly, Krylov, K6 update) of a whole
run_case on the GPU, with the work counters.  Usage: phase_profile.py CONFIG SOLVER [precond]"""
import ctypes as C, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2008_01539_b200 as pkg
from paper_2008_01539_b200 import _abi as A

cfg, solver = int(sys.argv[1]), sys.argv[2]
case = pkg.Case(cfg)
opts = case.solver_opts()
if len(sys.argv) > 3:
    opts.precond = int(sys.argv[3])
if solver == "adaptive_dd":
    opts.m = 4
sim = pkg.GpuSimulator(case)
L, ctx = sim.L, sim._ctx
s0, dts = case.init_state(), case.schedule()
sim.run_case(pkg.SOLVERS[solver], s0, dts, opts)  # warm
cnt = np.zeros(5, np.int64)
L.rsim_gpu_counters(ctx, A.ptr(cnt, C.c_int64), 1)
L.rsim_gpu_timers(ctx, 1, None, None)
t0 = time.time()
r = sim.run_case(pkg.SOLVERS[solver], s0, dts, opts)
wall = time.time() - t0
ms = np.zeros(4)
nl = C.c_int32()
L.rsim_gpu_timers(ctx, 0, A.ptr(ms, C.c_double), C.byref(nl))
L.rsim_gpu_counters(ctx, A.ptr(cnt, C.c_int64), 1)
L.rsim_gpu_timers(ctx, 0, None, None)
L.rsim_gpu_mark(ctx, 0)
r2 = sim.run_case(pkg.SOLVERS[solver], s0, dts, opts)
L.rsim_gpu_mark(ctx, 1)
v = C.c_double()
L.rsim_gpu_elapsed(ctx, 0, 1, C.byref(v))
out = dict(config=cfg, solver=solver, precond=opts.precond, wall_s=wall, run_ms_no_timers=v.value,
           phase_ms=dict(zip(["K7", "K1", "krylov", "K6"], ms.tolist())), launches=nl.value,
           counters=dict(zip(["asm_rows", "row_iters", "solves", "krylov_rows", "k7"], cnt.tolist())),
           **{k: r[k] for k in ("iterations", "lin_iters", "sum_na", "cuts", "status")})
out["active_cell_iters_per_s"] = r["sum_na"] / (v.value / 1e3)
print(json.dumps(out), flush=True)
