import ctypes as C, os, sys
os.environ["RSIM_KTRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2008_01539_b200 as pkg
for cfg, nA in ((1, 250), (2, 1400), (2, 3000), (2, 6000)):
    case = pkg.Case(cfg)
    sim = pkg.GpuSimulator(case)
    rng = np.random.default_rng(0)
    s = case.init_state(); s.u[::case.b] -= rng.uniform(0, 1e6, case.n)
    sim.set_state(s, 86400.0)
    act = np.sort(rng.choice(case.n, nA, replace=False)).astype(np.int32)
    sim.set_active(act); sim.assemble()
    buf = (C.c_ulonglong * 8)()
    sim.L.rsim_gpu_ktrace(sim._ctx, buf)
    o = case.solver_opts(fixed_lin_iters=100, lin_maxit=100)
    sim.linear_solve(o); sim.stats()
    sim.L.rsim_gpu_ktrace(sim._ctx, buf)
    v = [buf[k] / 100 for k in range(8)]
    names = ["spmvV", "redV", "spmvT", "redT", "xr", "redXR", "in_csync", "loophead"]
    print(cfg, nA, {n: round(x) for n, x in zip(names, v)}, "total/iter cycles", round(sum(v)))
