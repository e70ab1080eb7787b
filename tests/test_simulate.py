"""Case runner (SURVEY.md §8f row 1; SPEC.md sim_driver_cli, :460-531):
rsim_simulate / the `simulate` CLI / rsim_well_rates.

CPU: CLI argument errors (exit 2), no-GPU failure (exit 3), well rates
against a numpy restatement of well_term.
GPU: output files and their consistency invariants, parity of the runner's
totals and final fields with the oracle's run_case, and the SPEC acceptance
criteria 1 (solution equivalence / rate agreement with standard Newton) and
2 (locality magnitude bands) on config 1.
"""
import csv
import os
import subprocess

import numpy as np
import pytest

import paper_2008_01539_b200 as pkg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2008_01539_b200", "lib", "simulate")
PSI = 6894.757293168361
DAY = 86400.0


def _cli(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=600)


@pytest.mark.parametrize("args", [["--config", "9"], ["--config", "1", "--bogus", "1"], ["--config", "x1"],
                                  ["--config", "1", "--solver", "newtonian"], ["--config"],
                                  ["--config", "1", "--eps-p", "-1"]])
def test_cli_config_errors_exit_2(args):
    r = _cli(*args)
    assert r.returncode == 2, (r.returncode, r.stderr)
    assert "usage" in r.stderr


def test_cli_without_gpu_exits_3(tmp_path):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except Exception:
        pass
    r = _cli("--config", "1", "--out", str(tmp_path / "o"))
    assert r.returncode == 3, (r.returncode, r.stderr)


def _rates_np(case, s):
    """Σ_perf WI·L_e·(p − bhp)⁺ per equation → surface m^3/s."""
    f = case.fluid
    b = case.b
    p = s.u[::b]
    wi = case.well_wi
    dpw = np.where((wi > 0) & (p > case.graph.bhp), p - case.graph.bhp, 0.0)
    if b == 1:
        rho = f.rho_ref[1] * np.exp(f.c_f[1] * (p - f.p_ref))
        return np.array([0.0, np.sum(wi * rho / f.mu[1] * dpw) / f.rho_ref[1], 0.0])
    sw = s.u[1::b]
    rw = f.rho_ref[0] * np.exp(f.c_f[0] * (p - f.p_ref))
    ro = f.rho_ref[1] * np.exp(f.c_f[1] * (p - f.p_ref))
    den = 1.0 - f.swc - f.sor
    krw = np.clip((sw - f.swc) / den, 0, 1) ** 2
    kro = np.clip((1 - sw - f.sor) / den, 0, 1) ** 2
    return np.array([np.sum(wi * rw * krw / f.mu[0] * dpw) / f.rho_ref[0],
                     np.sum(wi * ro * kro / f.mu[1] * dpw) / f.rho_ref[1], 0.0])


@pytest.mark.parametrize("cfg", [dict(config=1), dict(config=2, nx=32, ny=32, n_dfn=6)])
def test_well_rates_match_restatement(cfg):
    case = pkg.Case(**cfg)
    rng = np.random.default_rng(3)
    s = case.init_state()
    s.u[::case.b] -= rng.uniform(0, 25e6, case.n)  # some perforations below BHP: clamped to zero
    if case.b == 2:
        s.u[1::case.b] = rng.uniform(0.1, 0.9, case.n)
    np.testing.assert_allclose(case.well_rates(s), _rates_np(case, s), rtol=1e-13, atol=0)
    s.u[::case.b] = case.graph.bhp  # p = bhp -> zero rate
    assert np.all(case.well_rates(s) == 0.0)


def _read_csv(path):
    with open(path) as f:
        return [{k: float(v) for k, v in row.items()} for row in csv.DictReader(f)]


def _summary(path):
    out = {}
    for line in open(path):
        k, _, v = line.strip().partition(" ")
        if k and v and k not in ("config", "case"):  # the first line describes the case
            out[k] = float(v)
    return out


@pytest.mark.gpu
def test_simulate_c1_outputs_parity_and_acceptance(tmp_path):
    from oracle import Oracle
    case = pkg.Case(1)
    res, rates, final_p = {}, {}, {}
    for solver in ("standard", "localized", "adaptive_dd"):
        d = tmp_path / solver
        if solver == "localized":  # through the CLI
            r = _cli("--config", "1", "--solver", solver, "--out", str(d), "--report-every", "20")
            assert r.returncode == 0, r.stderr
        else:
            pkg.simulate(1, solver, str(d), report_every_days=20.0)
        summ = _summary(d / "summary.txt")
        met = _read_csv(d / "metrics.csv")
        rt = _read_csv(d / "rates.csv")
        assert summ["status"] == 0 and summ["timesteps"] == len(met) == len(rt) == 20
        # metrics consistency: totals are the sums of the per-timestep entries (no cuts here)
        assert summ["cuts"] == 0
        assert sum(m["iterations"] for m in met) == summ["total_iterations"]
        assert sum(m["sum_nA"] for m in met) == summ["sum_nA"]
        assert abs(sum(m["sum_nA_over_n"] for m in met) - summ["total_ratio_MA"]) < 1e-9
        assert abs(rt[-1]["time_days"] - summ["simulated_days"]) < 1e-9
        res[solver], rates[solver] = summ, np.array([x["oil_rate"] for x in rt])
        dumps = sorted(p.name for p in d.glob("pressure_t*.txt"))
        assert len(dumps) == 3, dumps  # first steps past 20 and 40 days (29.5, 44.3 d) + final (66.485 d)
        final_p[solver] = np.loadtxt(d / f"pressure_t{summ['simulated_days']:.6g}.txt").ravel()
        assert final_p[solver].size == case.n
        # parity of the runner with the oracle's run_case on the same schedule
        opts = case.solver_opts()
        sv = pkg.SOLVERS[solver]
        if sv == 2:
            opts.m = 4
        ro = Oracle(case).run_case(sv, case.init_state(), case.schedule(), opts)
        assert ro["iterations"] == summ["total_iterations"] and ro["sum_na"] == summ["sum_nA"]
        assert ro["lin_iters"] == summ["total_linear_iterations"]
        assert np.array_equal(final_p[solver], ro["states"].u / PSI)  # %.17g round-trips exactly
    std = res["standard"]
    assert std["total_ratio_MA"] == std["total_iterations"]  # M_A(standard) = iteration count
    eps_psi = case.solver_opts().eps_p / PSI
    for solver in ("localized", "adaptive_dd"):
        # acceptance 1: pressure within 2 eps_p of standard Newton, oil rates within 0.5 %
        assert np.abs(final_p[solver] - final_p["standard"]).max() <= 2 * eps_psi
        np.testing.assert_allclose(rates[solver], rates["standard"], rtol=5e-3, atol=0)
        # acceptance 2 (bands of SPEC.md:537): total M_A <= standard / 6, average <= 0.15
        assert res[solver]["total_ratio_MA"] <= std["total_ratio_MA"] / 6
        assert res[solver]["average_ratio_MA_per_iteration"] <= 0.15
    assert res["localized"]["total_iterations"] <= 1.25 * std["total_iterations"]


@pytest.mark.gpu
def test_simulate_direct_solve_cli_matches_oracle(tmp_path):
    # the case runner with the exact dense-LU solve (--lin direct, SURVEY.md §8f
    # row 4) on a config-1 grid small enough for every active set (n·b = 900)
    from oracle import Oracle
    case = pkg.Case(1, nx=30, ny=30)
    d = tmp_path / "direct"
    r = _cli("--config", "1", "--nx", "30", "--ny", "30", "--solver", "localized", "--lin", "direct",
             "--out", str(d))
    assert r.returncode == 0, r.stderr
    summ = _summary(d / "summary.txt")
    assert summ["status"] == 0 and summ["cuts"] == 0
    opts = case.solver_opts(lin_method=pkg.LIN_DIRECT)
    ro = Oracle(case).run_case(1, case.init_state(), case.schedule(), opts)
    assert ro["iterations"] == summ["total_iterations"] and ro["sum_na"] == summ["sum_nA"]
    assert ro["lin_iters"] == summ["total_linear_iterations"] == summ["total_iterations"]
    final_p = np.loadtxt(d / f"pressure_t{summ['simulated_days']:.6g}.txt").ravel()
    assert np.array_equal(final_p, ro["states"].u / PSI)
    # and against the default Krylov run: the same states within the Newton tolerance
    rk = Oracle(case).run_case(1, case.init_state(), case.schedule(), case.solver_opts())
    assert np.abs(final_p - rk["states"].u / PSI).max() <= 2 * case.solver_opts().eps_p / PSI


def test_cli_rejects_unknown_linear_solver():
    r = _cli("--config", "1", "--lin", "cholesky")
    assert r.returncode == 2 and "unknown linear solver" in r.stderr
