"""Krylov micro-benchmark on config 4's first Newton system (776 k active rows, b = 3):
assemble once, then time the grid BiCGSTAB with a fixed iteration count (default 100,
Neumann-1 as in the run).  Usage: python scripts/krylov_c4.py [iters] [reps] [precond]
Prints ms per solve, µs per iteration and the algorithmic GB/s of bench.py's formula."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2008_01539_b200 as pkg  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
precond = int(sys.argv[3]) if len(sys.argv) > 3 else None
cfg = int(os.environ.get("KC4_CONFIG", "4"))
case = pkg.Case(cfg)
s0, dts = case.init_state(), case.schedule()
opts = case.solver_opts()
sim = pkg.GpuSimulator(case)
if cfg == 5:  # the bench's config-5 set: Gaussian-decay field at KC4_FRAC active (block-Jacobi, as c5_sweep)
    sim.set_state(s0, 86400.0)
    dp, _, _ = case.c5_field(float(os.environ.get("KC4_FRAC", "0.2")), 2, 1e-3)
    sim.upload_dp(dp)
    sim.L.rsim_gpu_state_from_dp(sim._ctx, 30e6, 20e6)
    sim.L.rsim_gpu_support_active(sim._ctx, 1e-3, 2, None)
    sim.stats()  # syncs n_A to the host before the assembly (as bench.c5_sweep does)
    precond = pkg.PREC_BJACOBI if precond is None else precond
else:
    sim.set_state(s0, float(dts[0]))
    sim.initial_active(True, opts.eps_set, opts.m)
sim.assemble()
nA = sim.stats().n_active
o = case.solver_opts(fixed_lin_iters=iters, lin_maxit=iters)
if precond is not None:
    o.precond = precond
L, ctx = sim.L, sim._ctx
ms = []
for r in range(reps + 1):
    L.rsim_gpu_flush_l2(ctx)
    L.rsim_gpu_mark(ctx, 14)
    L.rsim_gpu_linear_solve(ctx, C.byref(o))
    L.rsim_gpu_mark(ctx, 15)
    v = C.c_double()
    L.rsim_gpu_elapsed(ctx, 14, 15, C.byref(v))
    if r:
        ms.append(v.value)
x = sim.solution(nA)
import hashlib  # noqa: E402
x_sha = hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()[:16]
b = case.b
nnc = case.n_nnc * 2 / case.n
per = bench.bytes_krylov_row_iter(b, 6 if case.nz > 1 else 4, nnc, o.precond == pkg.PREC_NEUMANN1, cols=nA < case.n)
m = float(np.median(ms))
print(json.dumps({"config": cfg, "frac": os.environ.get("KC4_FRAC"), "n_active": nA, "iters": iters, "ms": m, "us_per_iter": 1e3 * m / iters,
                  "alg_GBs": nA * (iters * per + bench.bytes_krylov_row_init(b)) / (m / 1e3) / 1e9,
                  "x_sum": float(np.sum(x)), "x_sha": x_sha, "env": {k: v for k, v in os.environ.items() if k.startswith("RSIM_")}}))
