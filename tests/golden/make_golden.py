"""Generate the committed golden fixtures under tests/golden/ from the CPU oracle.

The reference (arXiv 2008.01539, /root/reference) ships no code, case files or
golden vectors, so these fixtures are produced by the oracle
(`oracle/oracle.cpp`, itself pinned by the SPEC known-answer tests in
tests/test_oracle_kat.py) on seeded small cases.  They freeze the oracle's
bits: `tests/test_golden.py` checks that the oracle still reproduces them
(CPU) and that the sm_100a path through the C-ABI reproduces them (GPU) —
without re-running the oracle on the GPU box.

    python tests/golden/make_golden.py      # rewrites tests/golden/*.npz
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (oracle.Case: the oracle library's own case generator)
from oracle import Oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# name -> (Case kwargs, solver (0 standard, 1 localized, 2 DD), number of timesteps, precond or None)
GOLDEN = {
    "c1_standard": (dict(config=1), 0, 6, None),
    "c1_localized": (dict(config=1), 1, 20, None),
    "c1_dd": (dict(config=1), 2, 8, None),
    "c2s_localized": (dict(config=2, nx=48, ny=48, n_dfn=12), 1, 10, None),
    "c2s_dd": (dict(config=2, nx=48, ny=48, n_dfn=12), 2, 6, None),
    "c3s_localized": (dict(config=3, nx=24, ny=24, nz=4), 1, 5, None),
    "c4s_localized": (dict(config=4, nx=24, ny=24, nz=4, n_dfn=8), 1, 5, None),
    "c2s_localized_bj": (dict(config=2, nx=48, ny=48, n_dfn=12), 1, 6, 0),
}

# Full-size BASELINE configs (the bench workloads: whole schedules of configs 1-4):
# the final state is stored as a digest (sha256 of the u / status bytes) plus every
# SUBSAMPLE-th cell's unknowns, so the fixture stays small.  Generation takes minutes
# (config 4: ~20-40 min per solver on 8 host threads), so only c1 / c2 are re-checked on the CPU suite.
FULL = {
    "c2_bench_localized": (dict(config=2), 1, 30, None),
    "c2_bench_dd": (dict(config=2), 2, 30, None),
    "c3_full_localized": (dict(config=3), 1, 20, None),
    "c4_full_localized": (dict(config=4), 1, 20, None),
    "c4_full_dd": (dict(config=4), 2, 20, None),
    "c3_full_dd": (dict(config=3), 2, 20, None),
    "c1_bench_standard": (dict(config=1), 0, 20, None),
}
SUBSAMPLE = 101
CPU_RECHECK = ("c2_bench_localized", "c2_bench_dd", "c1_bench_standard")

REC_FIELDS = ["n_active", "lin_iters", "subdomain", "mode_expand", "dp_inf_A", "dp_inf_B", "f_norm2",
              "f_norminf", "lin_res"]


def opts_for(case, solver, precond):
    opts = case.solver_opts() if precond is None else case.solver_opts(precond=precond)
    if solver == 2:
        opts.m = 4
    return opts


def first_step_report(orc, case, solver, opts):
    """Newton report of the first timestep through the SPEC entry point of `solver`."""
    s0 = case.init_state()
    dt = float(case.schedule()[0])
    if solver == 0:
        _, rep, rc = orc.newton_standard(s0, dt, opts)
        labels = va = None
    else:
        va = orc.initial_active(None, opts.eps_set, opts.m)
        labels = None
        if solver == 1:
            _, rep, rc = orc.newton_localized(s0, dt, va, opts.m, opts.eps_set, opts)
        else:
            _, rep, rc, labels = orc.adaptive_nonlinear_dd(s0, dt, va, opts.m, opts.eps_set, opts)
    recs = rep.records()
    out = {f"rec_{f}": np.array([r[f] for r in recs]) for f in REC_FIELDS}
    out.update(step0_rc=rc, step0_iterations=rep.iterations, step0_outer=rep.outer_iterations,
               step0_nsub=rep.n_subdomains, step0_lin_total=rep.lin_iters_total, step0_sum_na=rep.sum_na)
    if solver != 0:
        out["step0_va"] = va
    if labels is not None:
        out["step0_labels"] = labels
    return out


def digest(u: np.ndarray, st: np.ndarray) -> dict:
    import hashlib
    b = u.size // st.size
    idx = np.arange(0, st.size, SUBSAMPLE)
    return dict(u_sha256=hashlib.sha256(np.ascontiguousarray(u, np.float64).tobytes()).hexdigest(),
                st_sha256=hashlib.sha256(np.ascontiguousarray(st, np.uint8).tobytes()).hexdigest(),
                sub_idx=idx, u_sub=u.reshape(-1, b)[idx].copy(), st_sub=st[idx].copy(),
                p_sum=float(np.sum(u[::b])), n_sat=int(np.sum(st == 1)))


def make(name):
    full = name in FULL
    kw, solver, nsteps, precond = (FULL if full else GOLDEN)[name]
    case = oracle.Case(**kw)
    opts = opts_for(case, solver, precond)
    orc = Oracle(case)
    d = first_step_report(orc, case, solver, opts)
    dts = case.schedule()[:nsteps]
    r = orc.run_case(solver, case.init_state(), dts, opts)
    d.update(solver=solver, dts=np.asarray(dts, np.float64), status=r["status"], iterations=r["iterations"],
             sum_na=r["sum_na"], lin_iters=r["lin_iters"], cuts=r["cuts"], total_ma=r["total_ma"])
    if full:
        d.update(digest(r["states"].u, r["states"].status))
        if "step0_va" in d:  # the initial active set is re-derived from the case on the GPU side
            d["step0_va_sha256"] = __import__("hashlib").sha256(d.pop("step0_va").astype(np.int32).tobytes()).hexdigest()
    else:
        d.update(u=r["states"].u, st=r["states"].status)
    return d


if __name__ == "__main__":
    oracle.set_threads(len(os.sched_getaffinity(0)))
    for name in (sys.argv[1:] or GOLDEN):
        d = make(name)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **d)
        print(name, "iters", int(d["iterations"]), "lin", int(d["lin_iters"]), "sum_na", int(d["sum_na"]),
              "status", int(d["status"]))
