import time, sys
sys.path.insert(0, '/root/repo')
import paper_2008_01539_b200 as pkg
case = pkg.Case(2)
sim = pkg.GpuSimulator(case)
opts = case.solver_opts()
dts = case.schedule()[:30]
for solver, name in ((1, 'localized'), (2, 'dd'), (0, 'standard')):
    r = sim.run_case(solver, case.init_state(), dts, opts)
    t0 = time.perf_counter()
    r = sim.run_case(solver, case.init_state(), dts, opts)
    t = time.perf_counter() - t0
    print(name, {k: r[k] for k in ('status', 'iterations', 'lin_iters', 'sum_na', 'cuts')}, f"{t*1e3:.1f} ms", f"{r['sum_na']/t/1e6:.2f} M active-cell iters/s")
