"""Short, profiler-friendly run of a bench workload (no timing logic):
  python scripts/prof_workload.py c2      # 8 timesteps of config 2, localized Newton
  python scripts/prof_workload.py c5 1.0  # config-5 kernels at an active fraction
Used under `ncu` for the launch lists / full captures kept in profiles/."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2008_01539_b200 as pkg

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
if which == "c2dd":  # adaptive nonlinear DD on the bench workload
    case = pkg.Case(2)
    sim = pkg.GpuSimulator(case)
    dts = case.schedule()[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]
    r = sim.run_case(2, case.init_state(), dts, case.solver_opts())
    print("c2dd", {k: v for k, v in r.items() if k != "states"})
elif which == "c2":
    case = pkg.Case(2)
    sim = pkg.GpuSimulator(case)
    dts = case.schedule()[:int(sys.argv[2]) if len(sys.argv) > 2 else 8]
    r = sim.run_case(1, case.init_state(), dts, case.solver_opts())
    print("c2", {k: v for k, v in r.items() if k != "states"})
else:
    frac = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    case = pkg.Case(5)
    sim = pkg.GpuSimulator(case)
    sim.set_state(case.init_state(), 86400.0)
    dp, f, R = case.c5_field(frac, 2, 1e-3)
    sim.upload_dp(dp)
    sim.L.rsim_gpu_state_from_dp(sim._ctx, 30e6, 20e6)
    import ctypes as C
    st = pkg.GpuStats()
    for k in range(2):
        sim.L.rsim_gpu_support_active(sim._ctx, 1e-3, 2, C.byref(st))
        sim.assemble()
        sim.linear_solve(case.solver_opts(fixed_lin_iters=50, lin_maxit=50, precond=0))
        s2 = sim.stats()
    print("c5", frac, st.n_active, s2.lin_iters)
