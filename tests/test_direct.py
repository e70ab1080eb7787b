"""Exact (direct) solve of small active systems (
SPEC.md:311-325): dense LU with partial pivoting, opts.lin_method = LIN_DIRECT.

CPU: the oracle restatement (oracle.cpp direct_solve) against an independent
numpy LU with the same pivot rule (bit-equal: same operation order), against
numpy.linalg.solve and BiCGSTAB (tolerances), singular / oversize handling.
GPU: direct.cu equals the oracle bit for bit (solution, status, ‖F‖₂) on
partial and full sets with b = 1, 2, 3 and NNCs, and whole localized Newton
steps with the direct solve reproduce the oracle's reports."""
import numpy as np
import pytest

import paper_2008_01539_b200 as pkg
from oracle import Oracle

DAY = 86400.0


def _state(case, seed):
    rng = np.random.default_rng(seed)
    s = case.init_state()
    s.u[::case.b] -= rng.uniform(0, 3e6, case.n)
    if case.b >= 2:
        s.u[1::case.b] = np.clip(s.u[1::case.b] + rng.uniform(-0.05, 0.1, case.n), 0, 1)
    return s


def _dense(b, nA, rp, col, val):
    # entries of a row block added in CSR order onto the unit diagonal (as the oracle)
    N = nA * b
    W = np.zeros((N, N))
    W[np.arange(N), np.arange(N)] = 1.0
    V = val.reshape(-1, b, b)
    for l in range(nA):
        for q in range(rp[l], rp[l + 1]):
            for r in range(b):
                for c in range(b):
                    W[l * b + r, col[q] * b + c] = W[l * b + r, col[q] * b + c] + V[q][r, c]
    return W


def _lu_solve_np(W, rhs):
    """Independent restatement: right-looking LU, first-max pivot, the oracle's
    operation order, vectorised over rows (elementwise numpy ops round like the
    scalar ones: one product, one subtraction)."""
    W = W.copy()
    N = W.shape[0]
    piv = np.zeros(N, np.int64)
    for k in range(N):
        col = W[k:, k]
        assert np.all(np.isfinite(col))
        p = k + int(np.argmax(np.abs(col)))  # argmax returns the first maximum
        assert W[p, k] != 0.0
        piv[k] = p
        if p != k:
            W[[k, p], :] = W[[p, k], :]
        W[k + 1:, k] = W[k + 1:, k] / W[k, k]
        W[k + 1:, k + 1:] = W[k + 1:, k + 1:] - np.outer(W[k + 1:, k], W[k, k + 1:])
    x = rhs.copy()
    for k in range(N):
        if piv[k] != k:
            x[[k, piv[k]]] = x[[piv[k], k]]
    for k in range(N):
        x[k + 1:] = x[k + 1:] - W[k + 1:, k] * x[k]
    for k in range(N - 1, -1, -1):
        x[k] = x[k] / W[k, k]
        x[:k] = x[:k] - W[:k, k] * x[k]
    return x


CFGS = [dict(config=1, nx=10, ny=5), dict(config=2, nx=8, ny=8, n_dfn=4), dict(config=4, nx=4, ny=4, nz=2, n_dfn=2)]


@pytest.mark.parametrize("cfg", CFGS)
def test_oracle_direct_matches_numpy_lu_bit_exact(cfg):
    c = pkg.Case(**cfg)
    o = Oracle(c)
    o.set_state(_state(c, 1), DAY)
    o.set_u(_state(c, 2))
    act = np.arange(min(c.n, 50), dtype=np.int32)
    F, rhs, rp, col, val = o.assemble(act)
    rc, x, it, rr = o.linear_solve(len(act), c.solver_opts(lin_method=pkg.LIN_DIRECT))
    assert rc == 0 and it == 1 and rr == 0.0
    W = _dense(c.b, len(act), rp, col, val)
    assert np.array_equal(x, _lu_solve_np(W, rhs))
    x_ref = np.linalg.solve(W, rhs)
    assert np.abs(x - x_ref).max() <= 1e-10 * np.abs(x_ref).max()  # LAPACK: different order, κ(Â) up to ~1e3
    # Krylov cross-check: BiCGSTAB to 1e-14 agrees to 1e-10
    rc2, xk, _, _ = o.linear_solve(len(act), c.solver_opts(lin_rtol=1e-14, lin_maxit=2000))
    assert rc2 == 0
    assert np.abs(xk - x).max() <= 1e-10 * np.abs(x).max()


def test_oracle_direct_isolated_cells_elementwise():
    # block-diagonal system: Â = I, so x = rhs exactly
    c = pkg.Case(5, nx=9, ny=1, nz=1)
    o = Oracle(c)
    o.set_state(_state(c, 1), DAY)
    o.set_u(_state(c, 2))
    act = np.array([0, 2, 4, 6, 8], np.int32)
    F, rhs, rp, col, val = o.assemble(act)
    assert rp[-1] == 0
    rc, x, it, _ = o.linear_solve(len(act), c.solver_opts(lin_method=pkg.LIN_DIRECT))
    assert rc == 0 and np.array_equal(x, rhs)


def test_oracle_direct_oversize_falls_back_to_bicgstab():
    # n_A·b > DIRECT_MAX: the exact solve does not apply, BiCGSTAB runs instead (same
    # rule on the GPU, krylov.cu launch_krylov), so a growing active set never aborts a run
    c = pkg.Case(5, nx=64, ny=66, nz=1)
    assert c.n > pkg.DIRECT_MAX
    o = Oracle(c)
    o.set_state(_state(c, 1), DAY)
    o.assemble(np.arange(c.n, dtype=np.int32))
    rc, x, it, rr = o.linear_solve(c.n, c.solver_opts(lin_method=pkg.LIN_DIRECT))
    rc2, x2, it2, rr2 = o.linear_solve(c.n, c.solver_opts(lin_method=pkg.LIN_BICGSTAB))
    assert rc == rc2 == 0 and it == it2 > 1 and rr == rr2
    assert np.array_equal(x, x2)


def test_runner_rejects_out_of_range_solver_options():
    # lin_method / precond are range-checked before any GPU work (RSIM_EARG)
    for kw in (dict(lin_method=3), dict(precond=7)):
        with pytest.raises(pkg.RsimError) as e:
            pkg.simulate(1, "localized", nx=20, ny=20, n_steps=1, **kw)
        assert e.value.code == pkg.RSIM_EARG


def test_oracle_localized_newton_with_direct_solve():
    # Newton with the exact solve converges to the Krylov run's state within the
    # Newton tolerance (the Krylov residual 1e-9 vs exact)
    c = pkg.Case(1, nx=30, ny=30)
    s0 = c.init_state()
    dt = float(c.schedule()[3])
    res = {}
    for lm in (pkg.LIN_BICGSTAB, pkg.LIN_DIRECT):
        o = Oracle(c)
        opts = c.solver_opts(lin_method=lm)
        va = o.initial_active(None, opts.eps_set, 2)
        s, rep, rc = o.newton_localized(s0, dt, va, 2, opts.eps_set, opts)
        assert rc == 0
        res[lm] = s.u[::c.b].copy()
    assert np.abs(res[0] - res[2]).max() <= 2 * c.solver_opts().eps_p


# ------------------------------------------------------------------ GPU parity
def _gpu_check(case, act, seed=3):
    if act is not None:
        act = np.union1d(act, np.flatnonzero(case.pinned())).astype(np.int32)
    s = _state(case, seed)
    orc = Oracle(case)
    orc.set_state(s, DAY)
    Fo, *_ = orc.assemble(np.arange(case.n, dtype=np.int32) if act is None else act)
    sim = pkg.GpuSimulator(case)
    sim.set_state(s, DAY)
    st = sim.set_active(act)
    sim.assemble()
    opts = case.solver_opts(lin_method=pkg.LIN_DIRECT)
    rc_o, xo, it_o, rr_o = orc.linear_solve(st.n_active, opts)
    sim.linear_solve(opts)
    g = sim.stats()
    xg = sim.solution(st.n_active)
    assert rc_o == 0
    assert g.status == rc_o and g.lin_iters == it_o == 1
    assert g.f_norm2 == pytest.approx(np.sqrt(np.sum(Fo.reshape(-1, case.b) ** 2)), rel=1e-12)
    assert np.array_equal(xg, xo), np.abs(xg - xo).max()
    sim.close()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,nA", [(dict(config=1), 400), (dict(config=2, nx=64, ny=64, n_dfn=12), 1500),
                                    (dict(config=4, nx=24, ny=24, nz=4, n_dfn=6), 1000),
                                    (dict(config=5, nx=64, ny=64, nz=2), 4000)])
def test_gpu_direct_partial_sets(cfg, nA):
    case = pkg.Case(**cfg)
    rng = np.random.default_rng(nA)
    act = np.sort(rng.choice(case.n, min(nA, case.n), replace=False)).astype(np.int32)
    _gpu_check(case, act)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [dict(config=1, nx=40, ny=40), dict(config=5, nx=32, ny=32, nz=4),  # N = DIRECT_MAX
                                 dict(config=2, nx=40, ny=40, n_dfn=6)])
def test_gpu_direct_full_sets(cfg):
    _gpu_check(pkg.Case(**cfg), None)


@pytest.mark.gpu
def test_gpu_direct_oversize_falls_back_like_the_oracle():
    case = pkg.Case(5, nx=64, ny=66, nz=1)  # N = 4224 > DIRECT_MAX
    s = _state(case, 4)
    orc = Oracle(case)
    orc.set_state(s, DAY)
    orc.assemble(np.arange(case.n, dtype=np.int32))
    opts = case.solver_opts(lin_method=pkg.LIN_DIRECT)
    rc_o, xo, it_o, _ = orc.linear_solve(case.n, opts)
    sim = pkg.GpuSimulator(case)
    sim.set_state(s, DAY)
    sim.set_active(None)
    sim.assemble()
    sim.linear_solve(opts)
    g = sim.stats()
    assert rc_o == g.status == 0 and g.lin_iters == it_o > 1
    assert np.array_equal(sim.solution(case.n), xo)
    sim.close()


@pytest.mark.gpu
def test_gpu_localized_newton_with_direct_solve_matches_oracle():
    case = pkg.Case(2, nx=32, ny=32, n_dfn=6)  # n·b = 2048: every V_A fits the dense solve
    s0 = case.init_state()
    dt = float(case.schedule()[2])
    opts = case.solver_opts(lin_method=pkg.LIN_DIRECT)
    orc = Oracle(case)
    va = orc.initial_active(None, opts.eps_set, 2)
    so, rep_o, rc_o = orc.newton_localized(s0, dt, va, 2, opts.eps_set, opts)
    sim = pkg.GpuSimulator(case)
    sg, rep_g = sim.newton_localized(s0, dt, va, 2, opts.eps_set, opts)
    assert rc_o == 0 and rep_g.converged == 1
    assert rep_g.iterations == rep_o.iterations
    assert rep_g.records() == rep_o.records()
    assert np.array_equal(sg.u, so.u)
    sim.close()
