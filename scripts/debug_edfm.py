import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle, paper_2008_01539_b200 as pkg
from oracle import Oracle
name = sys.argv[1] if len(sys.argv) > 1 else "paper_case1_grid20"
path = f"cases/{name}.case"
co = oracle.case_from_file(path); cg = pkg.Case.from_file(path)
o = Oracle(co); sim = pkg.GpuSimulator(cg)
opts = co.solver_opts()
s = co.init_state(); dts = co.schedule()
p_prev = None
for k, dt in enumerate(dts[:48]):
    va_o = o.initial_active(p_prev, opts.eps_set, opts.m)
    sim.set_state(s, float(dt))
    if p_prev is None:
        sim.initial_active(True, opts.eps_set, opts.m)
    else:
        sim.initial_active(False, opts.eps_set, opts.m)  # uses the device p_prev? (may differ)
    va_g = sim.active()
    so, ro, rc = o.newton_localized(s, float(dt), va_o, opts.m, opts.eps_set, opts)
    sg, rg = sim.newton_localized(s, float(dt), va_o, opts.m, opts.eps_set, opts)
    no = [r["n_active"] for r in ro.records()]; ng = [r["n_active"] for r in rg.records()]
    same = no == ng and np.array_equal(so.u, sg.u)
    print(k, "va", len(va_o), len(va_g), "n_A", no, ng, "OK" if same else "DIFF", flush=True)
    if not same:
        # which iteration's set differs: recompute via estimate_active from the oracle's state
        break
    p_prev = s.u[::co.b].copy()
    s = so
