"""Full-size config runs on the GPU (c3, c4): run_case over the whole schedule,
optionally with Newton-update-limiter variants (fluid.dp_max_rel / ds_max).
Usage: python scripts/full_runs.py CONFIG SOLVER [dp_rel ds_max ...pairs] [--steps K]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2008_01539_b200 as pkg

args = sys.argv[1:]
steps = -1
if "--steps" in args:
    k = args.index("--steps"); steps = int(args[k + 1]); del args[k:k + 2]
cfg, solver = int(args[0]), args[1]
pairs = [(float(args[i]), float(args[i + 1])) for i in range(2, len(args), 2)] or [(None, None)]
case = pkg.Case(cfg, n_steps=steps)
print(f"config {cfg} n {case.n} nnc {case.n_nnc} pinned {int(case.pinned().sum())}", flush=True)
out = []
for dpr, dsm in pairs:
    fl = pkg.FluidParams.from_buffer_copy(case.fluid)
    if dpr is not None:
        fl.dp_max_rel, fl.ds_max = dpr, dsm
    sim = pkg.GpuSimulator(case, fluid=fl)
    opts = case.solver_opts()
    if solver == "adaptive_dd":
        opts.m = 4
    t0 = time.time()
    r = sim.run_case(pkg.SOLVERS[solver], case.init_state(), case.schedule(), opts)
    dt = time.time() - t0
    rec = dict(config=cfg, solver=solver, dp_max_rel=fl.dp_max_rel, ds_max=fl.ds_max, wall_s=round(dt, 3),
               **{k: v for k, v in r.items() if k != "states"})
    p = r["states"].u[:: case.b]
    rec["p_min"], rec["p_max"] = float(p.min()), float(p.max())
    if case.b == 3:
        rec["sat_cells"] = int((r["states"].status == 1).sum())
    print(json.dumps(rec), flush=True)
    out.append(rec)
    sim.close()
os.makedirs("gpurun_out", exist_ok=True)
with open(f"gpurun_out/full_c{cfg}_{solver}.json", "w") as f:
    json.dump(out, f, indent=1)
