import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import paper_2008_01539_b200 as pkg
from oracle import Oracle
from test_gpu_parity import perturbed_state, random_active, CASES
case = pkg.Case(**CASES['c4s'])
s = perturbed_state(case, 7); act = random_active(case, 3)
orc = Oracle(case); orc.set_state(s, 86400.0); orc.assemble(act)
sim = pkg.GpuSimulator(case); sim.set_state(s, 86400.0); sim.set_active(act); sim.assemble()
for pc in (0, 2):
    for its in (1, 2, 5, 20, 100, 168, 169, 170):
        opts = case.solver_opts(precond=pc, fixed_lin_iters=its, lin_maxit=its)
        rc, xo, it, rr = orc.linear_solve(len(act), opts)
        sim.linear_solve(opts); g = sim.stats(); xg = sim.solution(len(act))
        print(pc, its, "orc", rc, it, rr, "gpu", g.status, g.lin_iters, g.lin_relres, "equal", np.array_equal(xo, xg), np.abs(xo-xg).max())
    opts = case.solver_opts(precond=pc)
    rc, xo, it, rr = orc.linear_solve(len(act), opts)
    sim.linear_solve(opts); g = sim.stats(); xg = sim.solution(len(act))
    print(pc, "full", "orc", rc, it, rr, "gpu", g.status, g.lin_iters, g.lin_relres, np.array_equal(xo, xg))
