"""Microbenchmark: Krylov kernel time vs fixed iteration count (slope = time
per BiCGSTAB iteration, intercept = per-solve overhead) for active sets of
several sizes on config 2 (b=2) and config 1 (b=1)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2008_01539_b200 as pkg

out = []
for cfg, sizes in ((2, (256, 1000, 2000, 4000, 8000, 16000, 30000, 65536)), (1, (200, 2000, 10000))):
    case = pkg.Case(cfg)
    sim = pkg.GpuSimulator(case)
    rng = np.random.default_rng(0)
    s = case.init_state()
    s.u[::case.b] -= rng.uniform(0, 1e6, case.n)
    sim.set_state(s, 86400.0)
    for nA in sizes:
        act = np.sort(rng.choice(case.n, min(nA, case.n), replace=False)).astype(np.int32) if nA < case.n else None
        st = sim.set_active(act)
        sim.assemble()
        L, ctx = sim.L, sim._ctx
        res = {}
        for its in (1, 2, 10, 50):
            o = case.solver_opts(fixed_lin_iters=its, lin_maxit=its)
            ts = []
            for rep in range(5):
                L.rsim_gpu_mark(ctx, 0)
                sim.linear_solve(o)
                L.rsim_gpu_mark(ctx, 1)
                v = C.c_double()
                L.rsim_gpu_elapsed(ctx, 0, 1, C.byref(v))
                ts.append(v.value * 1e3)
            res[its] = float(np.median(ts[1:]))
        slope = (res[50] - res[10]) / 40
        out.append({"config": cfg, "nA": int(st.n_active), "us": res, "us_per_iter": slope,
                    "overhead_us": res[1] - slope})
        print(json.dumps(out[-1]), flush=True)
    sim.close()
