"""GMRES(30) and level-scheduled ILU(0) (north star alternatives to BiCGSTAB /
block-Jacobi): GPU kernels vs oracle, bit-exact — solution,
iteration count, residual — on every Krylov layout (small / grid / full-set
implicit columns, b = 1, 2, 3, NNC), with block-Jacobi, Neumann-1 and ILU(0),
and whole localized runs."""
import numpy as np
import pytest

import paper_2008_01539_b200 as pkg
from oracle import Oracle

pytestmark = pytest.mark.gpu


def _state(case, seed):
    rng = np.random.default_rng(seed)
    s = case.init_state()
    s.u[::case.b] -= rng.uniform(0, 3e6, case.n)
    if case.b >= 2:
        s.u[1::case.b] = np.clip(s.u[1::case.b] + rng.uniform(-0.05, 0.1, case.n), 0, 1)
    return s


def _check(case, act, precond, its=None, seed=3, method=None):
    if act is not None:
        act = np.union1d(act, np.flatnonzero(case.pinned())).astype(np.int32)
    s = _state(case, seed)
    orc = Oracle(case)
    orc.set_state(s, 86400.0)
    orc.assemble(np.arange(case.n, dtype=np.int32) if act is None else act)
    sim = pkg.GpuSimulator(case)
    sim.set_state(s, 86400.0)
    st = sim.set_active(act)
    sim.assemble()
    opts = case.solver_opts(precond=precond, lin_method=pkg.LIN_GMRES if method is None else method)
    if its:
        opts.fixed_lin_iters = its
        opts.lin_maxit = its
    rc_o, xo, it_o, rr_o = orc.linear_solve(st.n_active, opts)
    sim.linear_solve(opts)
    g = sim.stats()
    xg = sim.solution(st.n_active)
    assert g.status == rc_o
    assert g.lin_iters == it_o
    assert np.array_equal(xg, xo), np.abs(xg - xo).max()
    assert g.lin_relres == rr_o
    sim.close()
    return it_o


PRECS = [pkg.PREC_BJACOBI, pkg.PREC_NEUMANN1, pkg.PREC_ILU0]


@pytest.mark.parametrize("precond", PRECS)
@pytest.mark.parametrize("cfg,nA", [(dict(config=1), 400), (dict(config=2, nx=96, ny=96, n_dfn=20), 2500),
                                    (dict(config=4, nx=40, ny=40, nz=4, n_dfn=6), 3000),
                                    (dict(config=5, nx=160, ny=160, nz=1), 20000)])
def test_gmres_partial_sets(cfg, nA, precond):
    case = pkg.Case(**cfg)
    rng = np.random.default_rng(nA)
    act = np.sort(rng.choice(case.n, min(nA, case.n), replace=False)).astype(np.int32)
    _check(case, act, precond)


@pytest.mark.parametrize("precond", PRECS)
def test_gmres_full_set_grid(precond):
    case = pkg.Case(2, nx=200, ny=200, n_dfn=40)
    _check(case, None, precond)


@pytest.mark.parametrize("precond", PRECS)
def test_gmres_full_set_implicit_columns_restart(precond):
    # 1.2 M rows, V_A = all cells (structural columns), 45 iterations = one restart
    case = pkg.Case(3, nx=160, ny=128, nz=60)
    assert case.n > 148 * 2048
    _check(case, None, precond, its=45)


@pytest.mark.parametrize("method,precond", [(pkg.LIN_GMRES, pkg.PREC_NEUMANN1), (pkg.LIN_GMRES, pkg.PREC_ILU0),
                                            (pkg.LIN_BICGSTAB, pkg.PREC_ILU0)])
@pytest.mark.parametrize("name,kw", [("c1", dict(config=1)), ("c2s", dict(config=2, nx=64, ny=64, n_dfn=20)),
                                     ("c4s", dict(config=4, nx=32, ny=32, nz=4, n_dfn=10))])
def test_localized_run_bit_exact(name, kw, method, precond):
    case = pkg.Case(**kw)
    opts = case.solver_opts(lin_method=method, precond=precond)
    dts = case.schedule()[:8]
    ro = Oracle(case).run_case(1, case.init_state(), dts, opts)
    sim = pkg.GpuSimulator(case)
    rg = sim.run_case(1, case.init_state(), dts, opts)
    for k in ("status", "iterations", "lin_iters", "sum_na", "cuts"):
        assert rg[k] == ro[k], (k, rg[k], ro[k])
    assert np.array_equal(rg["states"].u, ro["states"].u)
    sim.close()


# ---- BiCGSTAB with ILU(0): level-scheduled triangular solves inside the grid kernel
@pytest.mark.parametrize("cfg,nA", [(dict(config=1), 400), (dict(config=2, nx=96, ny=96, n_dfn=20), 2500),
                                    (dict(config=4, nx=40, ny=40, nz=4, n_dfn=6), 3000),
                                    (dict(config=3, nx=48, ny=48, nz=8), 9000)])
def test_bicgstab_ilu0_partial_sets(cfg, nA):
    case = pkg.Case(**cfg)
    rng = np.random.default_rng(nA)
    act = np.sort(rng.choice(case.n, min(nA, case.n), replace=False)).astype(np.int32)
    _check(case, act, pkg.PREC_ILU0, method=pkg.LIN_BICGSTAB)


def test_bicgstab_ilu0_full_set():
    case = pkg.Case(2, nx=200, ny=200, n_dfn=40)
    _check(case, None, pkg.PREC_ILU0, method=pkg.LIN_BICGSTAB)
