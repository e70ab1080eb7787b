"""Cycle breakdown of the cluster Krylov kernel over the real bench workload
(config 2, localized Newton): RSIM_KTRACE=1 makes the kernel accumulate
clock64() deltas per phase (CTA 0 / thread 0) and per CTA (warp 0 / last warp)."""
import ctypes as C, os, sys
os.environ["RSIM_KTRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2008_01539_b200 as pkg
NK = 136
case = pkg.Case(2)
sim = pkg.GpuSimulator(case)
buf = (C.c_ulonglong * NK)()
sim.L.rsim_gpu_ktrace(sim._ctx, buf)
sched = case.schedule()[:30]
r = sim.run_case(1, case.init_state(), sched, case.solver_opts())
sim.L.rsim_gpu_ktrace(sim._ctx, buf)
n = r["lin_iters"]
names = ["spmvV", "redV", "spmvT", "redT", "xr", "redXR", "in_csync", "loophead"]
v = [buf[k] / n for k in range(8)]
print("c2 run", {k: r[k] for k in ("iterations", "lin_iters", "sum_na")})
print({a: round(x) for a, x in zip(names, v)}, "cycles/iter (excl. in_csync)", round(sum(v) - v[6]))
print("rank: csync_w0 csync_wl spmv_w0 spmv_wl redtail_w0 (cycles per Krylov iteration of the run) | remote_slots rows (summed over launches)")
for g in range(16):
    e = [buf[8 + g * 8 + k] for k in range(8)]
    if e[6] == 0:
        continue
    print(g, " ".join(f"{x / n:8.0f}" for x in e[:5]), "|", e[5], e[6])
