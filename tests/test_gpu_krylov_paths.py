"""Bit-exact parity of every Krylov code path against the oracle.

Paths: the cluster/DSMEM kernel for n_A <= 16384 rows with
64..1024 rows per CTA (G = 1..16 CTAs), and the cooperative-grid kernel for
larger systems, including the distributed level-2 reduction (> 4.2 M rows).
Sizes are chosen to hit partial warps, partial chunks and every layout."""
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


def _check(case, act, its=None, seed=1, precond=0):
    if act is not None:
        act = np.union1d(act, np.flatnonzero(case.pinned())).astype(np.int32)
    s = _state(case, seed)
    dt = 86400.0
    orc = Oracle(case)
    orc.set_state(s, dt)
    Fo, ro, rpo, co, vo = orc.assemble(np.arange(case.n, dtype=np.int32) if act is None else act)
    sim = pkg.GpuSimulator(case)
    sim.set_state(s, dt)
    st = sim.set_active(act)
    assert st.n_active == (case.n if act is None else len(act))
    sim.assemble()
    opts = case.solver_opts(precond=precond)
    if its:
        opts.fixed_lin_iters = its
        opts.lin_maxit = its
    nA = st.n_active
    rc_o, xo, it_o, rr_o = orc.linear_solve(nA, opts)
    sim.linear_solve(opts)
    g = sim.stats()
    xg = sim.solution(nA)
    assert g.status == rc_o
    assert g.lin_iters == it_o
    assert g.f_norm2 == pytest.approx(np.sqrt(np.sum(Fo.reshape(-1, case.b) ** 2)), rel=1e-12)
    assert np.array_equal(xg, xo), np.abs(xg - xo).max()
    assert g.lin_relres == rr_o
    sim.close()


@pytest.mark.parametrize("precond", [pkg.PREC_BJACOBI, pkg.PREC_NEUMANN1])
@pytest.mark.parametrize("nA", [1, 17, 63, 64, 65, 200, 257, 1000, 2049, 4095, 8191, 12000, 16384])
def test_cluster_path_exact_sizes(nA, precond):
    # config 5 has no pinned (fracture/well) cells, so |V_A| is exactly nA
    case = pkg.Case(5, nx=160, ny=160, nz=1)
    rng = np.random.default_rng(nA)
    act = np.sort(rng.choice(case.n, nA, replace=False)).astype(np.int32)
    _check(case, act, precond=precond)


@pytest.mark.parametrize("precond", [pkg.PREC_BJACOBI, pkg.PREC_NEUMANN1])
@pytest.mark.parametrize("nA", [100, 1500, 5000, 15000])
def test_cluster_path_b2_with_nnc(nA, precond):
    case = pkg.Case(2, nx=160, ny=160, n_dfn=30)
    assert case.n_nnc > 0
    rng = np.random.default_rng(nA)
    act = np.union1d(rng.choice(case.n, nA, replace=False), np.flatnonzero(case.pinned())).astype(np.int32)
    _check(case, act, precond=precond)


@pytest.mark.parametrize("precond", [pkg.PREC_BJACOBI, pkg.PREC_NEUMANN1])
@pytest.mark.parametrize("cfg,nA", [(dict(config=1), 300), (dict(config=3, nx=48, ny=48, nz=8), 5000),
                                    (dict(config=4, nx=40, ny=40, nz=4, n_dfn=6), 3000)])
def test_cluster_path_b1_b3_3d(cfg, nA, precond):
    case = pkg.Case(**cfg)
    rng = np.random.default_rng(nA)
    act = np.sort(rng.choice(case.n, min(nA, case.n), replace=False)).astype(np.int32)
    _check(case, act, precond=precond)


@pytest.mark.parametrize("precond", [pkg.PREC_BJACOBI, pkg.PREC_NEUMANN1])
@pytest.mark.parametrize("cfg", [dict(config=2, nx=200, ny=200, n_dfn=40), dict(config=4, nx=48, ny=48, nz=8, n_dfn=8)])
def test_grid_path_full_set(cfg, precond):
    case = pkg.Case(**cfg)
    _check(case, None, precond=precond)


@pytest.mark.parametrize("precond", [pkg.PREC_BJACOBI, pkg.PREC_NEUMANN1])
@pytest.mark.parametrize("cfg,nA", [(dict(config=4, nx=64, ny=64, nz=8, n_dfn=12), 20000),
                                    (dict(config=2, nx=200, ny=200, n_dfn=40), 24000),
                                    (dict(config=5, nx=128, ny=128, nz=4), 40000)])
def test_grid_path_partial_set(cfg, nA, precond):
    # partial sets on the cooperative-grid kernel (> 16384 rows): stored columns, the per-row
    # NNC flag of the assembly (b = 2 / 3 cases have DFN NNCs), row-major (b = 3) and
    # warp-tiled (b <= 2) block values, b = 1 next-round row preload and L2 prefetch
    case = pkg.Case(**cfg)
    rng = np.random.default_rng(nA)
    act = np.sort(rng.choice(case.n, nA, replace=False)).astype(np.int32)
    _check(case, act, precond=precond)


@pytest.mark.parametrize("precond", [pkg.PREC_BJACOBI, pkg.PREC_NEUMANN1])
def test_grid_path_distributed_level2_reduction(precond):
    # > 64*256*256 rows => level-2 partials reduced across CTAs (extra barrier);
    # > 2^20 rows => the unfused (store, barrier, gather) Krylov variant
    case = pkg.Case(5, nx=256, ny=128, nz=140)
    assert case.n > 64 * 256 * 256
    _check(case, None, its=3, precond=precond)


@pytest.mark.parametrize("precond", [pkg.PREC_BJACOBI, pkg.PREC_NEUMANN1])
def test_grid_path_unfused_converged(precond):
    # 1.3 M rows, b = 2, run to convergence (early-exit branch); b >= 2 uses the recompute-fused
    # variant at every size since round 2 (b = 1 above 2^20 rows is the unfused one, see above)
    case = pkg.Case(3, nx=160, ny=128, nz=64)
    assert case.n > (1 << 20)
    _check(case, None, precond=precond)
