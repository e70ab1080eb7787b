"""Committed golden fixtures (tests/golden/*.npz, made by tests/golden/make_golden.py).

The reference ships no golden vectors; these freeze the
SPEC-pinned oracle's results on seeded small cases of configs 1–4:
per-iteration Newton records of the first timestep (n_A, Krylov iterations,
mode, ‖δp‖∞, ‖F‖₂, ‖F‖∞, Krylov residual), DD partition labels, whole-run
totals and the final pressures / saturations / phase status.

- CPU: the oracle still reproduces every fixture bit for bit (regression pin).
- GPU: the sm_100a path through the C-ABI entry points (rsim_newton_*,
  rsim_adaptive_nonlinear_dd, rsim_run_case) reproduces every fixture bit for
  bit.  The north-star bar is looser — identical iteration
  counts, norms within 1e-10 relative, p/S within 1e-8 relative — the
  asserts below check that bar explicitly and then bit equality.
"""
import glob
import os

import numpy as np
import pytest

import paper_2008_01539_b200 as pkg

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
import importlib.util as _ilu

_spec = _ilu.spec_from_file_location("make_golden", os.path.join(HERE, "make_golden.py"))
mg = _ilu.module_from_spec(_spec)
_spec.loader.exec_module(mg)

NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(HERE, "*.npz")))
NORM_RTOL = 1e-10   # per-iteration residual norms (north star)
STATE_RTOL = 1e-8   # final pressures and saturations (north star)


def test_fixture_set_complete():
    assert sorted(mg.GOLDEN) == NAMES


def _check_records(got: dict, g) -> None:
    for f in ("n_active", "lin_iters", "subdomain", "mode_expand"):
        assert np.array_equal(got[f"rec_{f}"], g[f"rec_{f}"]), f
    for f in ("f_norm2", "f_norminf", "dp_inf_A", "lin_res"):
        a, b = got[f"rec_{f}"], g[f"rec_{f}"]
        np.testing.assert_allclose(a, b, rtol=NORM_RTOL, atol=0, err_msg=f)
        assert np.array_equal(a, b), f  # bit-exact by construction
    for k in ("step0_rc", "step0_iterations", "step0_outer", "step0_nsub", "step0_lin_total", "step0_sum_na"):
        assert int(got[k]) == int(g[k]), k
    if "step0_labels" in g:
        assert np.array_equal(got["step0_labels"], g["step0_labels"])


def _check_run(r: dict, g) -> None:
    assert r["status"] == int(g["status"]) == 0
    for k in ("iterations", "sum_na", "lin_iters", "cuts"):
        assert r[k] == int(g[k]), k
    assert r["total_ma"] == float(g["total_ma"])
    b = r["states"].u.size // r["states"].status.size
    np.testing.assert_allclose(r["states"].u[::b], g["u"][::b], rtol=STATE_RTOL, atol=0)
    assert np.array_equal(r["states"].status, g["st"])
    assert np.array_equal(r["states"].u, g["u"])


@pytest.mark.parametrize("name", NAMES)
def test_oracle_reproduces_golden(name):
    g = np.load(os.path.join(HERE, name + ".npz"))
    d = mg.make(name)
    _check_records(d, g)
    _check_run({"status": int(d["status"]), "iterations": int(d["iterations"]), "sum_na": int(d["sum_na"]),
                "lin_iters": int(d["lin_iters"]), "cuts": int(d["cuts"]), "total_ma": float(d["total_ma"]),
                "states": pkg.CellStates(d["u"], d["st"])}, g)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_reproduces_golden(name):
    g = np.load(os.path.join(HERE, name + ".npz"))
    kw, solver, nsteps, precond = mg.GOLDEN[name]
    case = pkg.Case(**kw)
    opts = mg.opts_for(case, solver, precond)
    sim = pkg.GpuSimulator(case)
    s0 = case.init_state()
    dt = float(g["dts"][0])
    if solver == 0:
        _, rep = sim.newton_standard(s0, dt, opts)
    elif solver == 1:
        _, rep = sim.newton_localized(s0, dt, g["step0_va"], opts.m, opts.eps_set, opts)
    else:
        _, rep = sim.adaptive_nonlinear_dd(s0, dt, g["step0_va"], opts.m, opts.eps_set, opts)
    recs = rep.records()
    got = {f"rec_{f}": np.array([r[f] for r in recs]) for f in mg.REC_FIELDS}
    got.update(step0_rc=rep.status, step0_iterations=rep.iterations, step0_outer=rep.outer_iterations,
               step0_nsub=rep.n_subdomains, step0_lin_total=rep.lin_iters_total, step0_sum_na=rep.sum_na)
    if solver == 2:
        got["step0_labels"] = sim.labels()
    _check_records(got, g)
    r = sim.run_case(solver, s0, g["dts"], opts)
    _check_run(r, g)
    sim.close()
