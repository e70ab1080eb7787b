"""CPU oracle pinned against the reference's own known-answer examples and
invariants (SPEC.md examples, "Invariants & Properties", AC10).  The
reference ships no code or golden vectors, so these KATs are
the pin; each test cites the SPEC line it checks."""
import math
from collections import deque

import numpy as np
import pytest

import oracle
import paper_2008_01539_b200 as pkg
from oracle import Oracle

DAY = 86400.0


def bfs(case, src, m, nnc=True):
    """Independent BFS oracle on the connection graph."""
    nx, ny, nz = case.nx, case.ny, case.nz
    nn = case.nnc() if nnc else None

    def nbrs(i):
        ix, iy, iz = i % nx, (i // nx) % ny, i // (nx * ny)
        if iz > 0: yield i - nx * ny
        if iy > 0: yield i - nx
        if ix > 0: yield i - 1
        if ix < nx - 1: yield i + 1
        if iy < ny - 1: yield i + nx
        if iz < nz - 1: yield i + nx * ny
        if nn is not None:
            ptr_, nbr, _ = nn
            yield from (int(j) for j in nbr[ptr_[i]:ptr_[i + 1]])
    dist = {s: 0 for s in src}
    q = deque(src)
    while q:
        i = q.popleft()
        if dist[i] == m:
            continue
        for j in nbrs(i):
            if j not in dist:
                dist[j] = dist[i] + 1
                q.append(j)
    return np.array(sorted(dist), np.int32)


# ---------------------------------------------------------------- grid_edfm
def test_tpfa_equal_cells_kat():
    # k=1e-19, A=0.5, d=0.25 -> Υ_half=2e-19, Υ=1e-19
    k = np.full(2, 1e-19)
    tx, ty, tz = oracle.build_matrix_grid(2, 1, 1, 0.5, 0.5, 1.0, k, k, k)
    assert tx[0] == pytest.approx(1e-19, rel=1e-15)
    assert tx[1] == 0.0 and not ty.any() and not tz.any()


def test_tpfa_connection_counts():
    k = np.ones(9) * 1e-15
    tx, ty, tz = oracle.build_matrix_grid(1, 1, 1, 1, 1, 1, k[:1], k[:1], k[:1])
    assert not (tx.any() or ty.any() or tz.any())
    tx, ty, tz = oracle.build_matrix_grid(3, 3, 1, 1, 1, 1, k, k, k)
    assert np.count_nonzero(tx) + np.count_nonzero(ty) == 12


@pytest.mark.parametrize("cfg", [dict(config=1, nx=30, ny=20), dict(config=3, nx=16, ny=16, nz=4),
                                 dict(config=5, nx=20, ny=16, nz=6)])
def test_product_tpfa_matches_oracle_bit_exact(cfg):
    c = pkg.Case(**cfg)
    tx, ty, tz = oracle.build_matrix_grid(c.nx, c.ny, c.nz, c.dx, c.dy, c.dz, c.perm(0), c.perm(1), c.perm(2))
    assert np.array_equal(tx, c.tx) and np.array_equal(ty, c.ty) and np.array_equal(tz, c.tz)
    assert (c.tx[:-1].reshape(-1)[(np.arange(c.n - 1) % c.nx) != c.nx - 1] > 0).all()  # positivity


@pytest.mark.parametrize("i,m,expect", [(12, 1, 5), (12, 2, 13), (0, 1, 3)])
def test_neighbor_set_kat(i, m, expect):
    c = pkg.Case(5, nx=5, ny=5, nz=1)  # plain 5x5 grid, no fractures
    o = Oracle(c)
    assert len(o.neighbor_set(i, m)) == expect


def test_neighbor_set_matches_bfs_with_fracture():
    c = pkg.Case(2, nx=48, ny=48, n_dfn=20)  # DFN => NNCs present
    assert c.n_nnc > 0
    o = Oracle(c)
    rng = np.random.default_rng(0)
    for i in rng.choice(c.n, 40, replace=False):
        for m in (1, 2, 3):
            got = o.neighbor_set(int(i), m)
            assert np.array_equal(got, bfs(c, [int(i)], m)), (i, m)
            if m > 1:
                assert np.isin(o.neighbor_set(int(i), m - 1), got).all()  # monotone


# ---------------------------------------------------------------- fluid_props
def test_rexp_accuracy():
    xs = np.concatenate([np.linspace(-30, 30, 4001), np.linspace(-1e-3, 1e-3, 101), [0.0, 1e-300, -700, 700]])
    for x in xs:
        ref = math.exp(x)
        assert abs(oracle.rexp(x) - ref) <= 4e-16 * ref + 1e-300, x


def test_density_kat():
    c = pkg.Case(1, nx=4, ny=4)
    f = c.fluid
    A, dA, L, dL = oracle.props(f, [f.p_ref])
    assert A[0] == f.rho_ref[1]  # p = p_ref -> ρ_ref
    A, *_ = oracle.props(f, [f.p_ref + 1e6])  # c = 1e-9, Δp = 1e6 -> ρ_ref e^{0.001}
    assert A[0] == pytest.approx(f.rho_ref[1] * math.exp(1e-3), rel=1e-15)
    f2 = pkg.FluidParams.from_buffer_copy(f)
    f2.c_f[1] = 0.0
    for p in (1e6, 3e7, 5e7):  # c_f = 0 -> constant
        assert oracle.props(f2, [p])[0][0] == f.rho_ref[1]


def test_relperm_kat():
    swc, sor = 0.2, 0.2
    den = 1 - swc - sor
    assert oracle.corey(swc, swc, den)[0] == 0.0  # s = s_r
    assert oracle.corey(1 - sor, swc, den)[0] == 1.0  # s = 1 - other residual
    assert oracle.corey(swc + 0.5 * den, swc, den)[0] == pytest.approx(0.25, rel=1e-15)  # midpoint


def _fd_props(f, u, st, h):
    A0, dA, L0, dL = oracle.props(f, u, st)
    b = len(u)
    for v in range(b):
        up, um = np.array(u, float), np.array(u, float)
        up[v] += h[v]
        um[v] -= h[v]
        Ap, _, Lp, _ = oracle.props(f, up, st)
        Am, _, Lm, _ = oracle.props(f, um, st)
        for e in range(b):
            fa = (Ap[e] - Am[e]) / (2 * h[v])
            fl = (Lp[e] - Lm[e]) / (2 * h[v])
            assert dA[e, v] == pytest.approx(fa, rel=1e-5, abs=1e-9 * (abs(A0[e]) + 1) / max(abs(u[v]), 1)), (e, v)
            assert dL[e, v] == pytest.approx(fl, rel=1e-5, abs=1e-9 * (abs(L0[e]) + 1) / max(abs(u[v]), 1)), (e, v)


@pytest.mark.parametrize("config", [1, 2, 4])
def test_property_derivatives_fd(config):
    # analytic derivatives vs central FD, 100 random states
    c = pkg.Case(config, nx=4, ny=4, nz=2 if config == 4 else 1)
    f = c.fluid
    rng = np.random.default_rng(config)
    for k in range(100):
        p = rng.uniform(9e6, 31e6)
        if c.b == 1:
            _fd_props(f, [p], 0, [1e-7 * p])
        elif c.b == 2:
            sw = rng.uniform(0.22, 0.78)
            _fd_props(f, [p, sw], 0, [1e-7 * p, 1e-7])
        else:
            sw = rng.uniform(0.21, 0.4)
            if k % 2:
                sg = rng.uniform(0.06, 0.3)
                _fd_props(f, [p, sw, sg], 1, [1e-7 * p, 1e-7, 1e-7])
            else:
                rs = rng.uniform(10, 100)
                _fd_props(f, [p, sw, rs], 0, [1e-7 * p, 1e-7, 1e-7 * rs])


# ---------------------------------------------------------------- fim_assembly
def _state(c, seed, dp=2e6):
    rng = np.random.default_rng(seed)
    s = c.init_state()
    b = c.b
    s.u[::b] -= rng.uniform(0, dp, c.n)
    if b >= 2:
        s.u[1::b] = rng.uniform(0.25, 0.7, c.n)
    if b == 3:
        sat = rng.random(c.n) < 0.5
        s.status[:] = sat.astype(np.uint8)
        s.u[2::b] = np.where(sat, rng.uniform(0.08, 0.25, c.n), rng.uniform(20, 90, c.n))
    return s


@pytest.mark.parametrize("cfg", [dict(config=1, nx=6, ny=5), dict(config=2, nx=8, ny=8, n_dfn=6),
                                 dict(config=4, nx=5, ny=5, nz=2, n_dfn=3)])
def test_jacobian_vs_finite_differences(cfg):
    # every block matches FD of the residual (rel 1e-5)
    c = pkg.Case(**cfg)
    o = Oracle(c)
    old = _state(c, 1)
    o.set_state(old, DAY)
    cur = _state(c, 2)
    o.set_u(cur)
    act = np.arange(c.n, dtype=np.int32)
    F0, D, rp, col, val = o.assemble_raw(act)
    b = c.b
    J = np.zeros((c.n * b, c.n * b))
    for l in range(c.n):
        J[l * b:(l + 1) * b, l * b:(l + 1) * b] = D[l]
        for q in range(rp[l], rp[l + 1]):
            J[l * b:(l + 1) * b, col[q] * b:(col[q] + 1) * b] = val[q]
    rng = np.random.default_rng(3)
    for j in rng.choice(c.n, 6, replace=False):
        for v in range(b):
            scale = abs(cur.u[j * b + v]) if v == 0 else (1.0 if cur.status[j] or v == 1 else abs(cur.u[j * b + v]))
            h = 1e-7 * scale
            up, um = cur.copy(), cur.copy()
            up.u[j * b + v] += h
            um.u[j * b + v] -= h
            o.set_u(up)
            Fp = o.assemble_raw(act)[0]
            o.set_u(um)
            Fm = o.assemble_raw(act)[0]
            fd = (Fp - Fm) / (2 * h)
            an = J[:, j * b + v]
            # 1e-5 relative + the FD cancellation floor of each row
            noise = 64 * np.finfo(float).eps * (np.abs(Fp) + np.abs(Fm)) / (2 * h)
            tol = 1e-5 * np.maximum(np.abs(an), np.abs(fd)) + noise
            bad = np.abs(fd - an) > tol
            assert not bad.any(), (j, v, np.flatnonzero(bad), fd[bad], an[bad], tol[bad])
    o.set_u(cur)


def test_flux_antisymmetry_and_zero_states():
    c = pkg.Case(1, nx=2, ny=1)
    o = Oracle(c)
    s = c.init_state()
    o.set_state(s, DAY)  # same state: zero accumulation
    cg = pkg.Case(1, nx=2, ny=1)
    F, *_ = o.assemble_raw(np.arange(2, dtype=np.int32))
    # both cells are fracture+well cells in this tiny c1: F = well term only
    wi = cg.well_wi
    rho = cg.fluid.rho_ref[1]
    mu = cg.fluid.mu[1]
    expect = wi * rho / mu * (s.u[0] - cg.graph.bhp)
    assert F == pytest.approx(expect, rel=1e-14)


def test_single_phase_flux_kat():
    # two matrix cells, no wells: flux = Υ ρ_up/μ (p_i - p_j), antisymmetric
    c = pkg.Case(5, nx=2, ny=1, nz=1)
    o = Oracle(c)
    s = c.init_state()
    o.set_state(s, DAY)
    cur = s.copy()
    cur.u[0] += 1e5
    o.set_u(cur)
    F0, D, rp, col, val = o.assemble_raw(np.arange(2, dtype=np.int32))
    o.set_u(s)
    f = c.fluid
    rho0 = f.rho_ref[1] * math.exp(f.c_f[1] * (cur.u[0] - f.p_ref))
    flux = c.tx[0] * (rho0 / f.mu[1]) * 1e5
    acc0 = c.pv[0] * (rho0 - f.rho_ref[1]) / DAY
    assert F0[0] == pytest.approx(acc0 + flux, rel=1e-12)
    assert F0[1] == pytest.approx(-flux, rel=1e-12)
    # equal pressures -> zero flux
    o.set_u(s)
    F1 = o.assemble_raw(np.arange(2, dtype=np.int32))[0]
    assert not F1.any()


def test_accumulation_doubling_dt_halves_exactly():
    c = pkg.Case(5, nx=3, ny=1, nz=1)
    o = Oracle(c)
    s = c.init_state()
    cur = s.copy()
    cur.u[:] += 3e5  # uniform: no flux
    for dt, F in ((DAY, None), (2 * DAY, None)):
        o.set_state(s, dt)
        o.set_u(cur)
        if dt == DAY:
            F1 = o.assemble_raw(np.arange(3, dtype=np.int32))[0]
        else:
            F2 = o.assemble_raw(np.arange(3, dtype=np.int32))[0]
    assert np.array_equal(F2, 0.5 * F1)


def test_well_kat():
    c = pkg.Case(1, nx=10, ny=4)
    o = Oracle(c)
    s = c.init_state()
    o.set_state(s, DAY)
    act = np.arange(c.n, dtype=np.int32)
    F = o.assemble_raw(act)[0]
    wells = np.flatnonzero(c.well_wi > 0)
    assert (F[wells] > 0).all()
    g2 = pkg.GraphDesc.from_buffer_copy(c.graph)
    wi2 = c.well_wi * 2
    g2.well_wi = wi2.ctypes.data_as(g2.well_wi.__class__)
    o2 = Oracle(graph=g2, fluid=c.fluid)
    o2.set_state(s, DAY)
    F2 = o2.assemble_raw(act)[0]
    assert np.allclose(F2[wells], 2 * F[wells], rtol=1e-14)  # 2·WI -> 2·rate
    g3 = pkg.GraphDesc.from_buffer_copy(c.graph)
    g3.bhp = float(s.u[0])
    o3 = Oracle(graph=g3, fluid=c.fluid)
    o3.set_state(s, DAY)
    assert not o3.assemble_raw(act)[0].any()  # p = bhp -> 0


def test_assembly_pattern_3x3_and_single_cell():
    c = pkg.Case(5, nx=3, ny=3, nz=1)
    o = Oracle(c)
    s = _state(c, 5)
    o.set_state(s, DAY)
    F, D, rp, col, val = o.assemble_raw(np.arange(9, dtype=np.int32))
    assert D.shape[0] == 9 and len(col) == 24  # 9 diagonal + 24 off-diagonal blocks
    F1, D1, rp1, col1, _ = o.assemble_raw(np.array([4], np.int32))  # interior cell, neighbours frozen
    assert len(col1) == 0 and F1[0] == F[4]  # accumulation + 4 frozen fluxes


@pytest.mark.parametrize("cfg", [dict(config=2, nx=16, ny=16, n_dfn=8), dict(config=4, nx=8, ny=8, nz=2, n_dfn=4)])
def test_restriction_consistency(cfg):
    # assemble(V_A) rows bit-identical to the full assembly
    c = pkg.Case(**cfg)
    o = Oracle(c)
    o.set_state(_state(c, 1), DAY)
    o.set_u(_state(c, 2))
    full = o.assemble(np.arange(c.n, dtype=np.int32))
    rng = np.random.default_rng(9)
    act = np.sort(rng.choice(c.n, c.n // 3, replace=False)).astype(np.int32)
    sub = o.assemble(act)
    b = c.b
    g2l = -np.ones(c.n, int)
    g2l[act] = np.arange(len(act))
    for l, i in enumerate(act):
        assert np.array_equal(sub[0][l * b:(l + 1) * b], full[0][i * b:(i + 1) * b])
        assert np.array_equal(sub[1][l * b:(l + 1) * b], full[1][i * b:(i + 1) * b])
        fc = full[3][full[2][i]:full[2][i + 1]]
        fv = full[4].reshape(-1, b, b)[full[2][i]:full[2][i + 1]]
        keep = g2l[fc] >= 0
        sc = sub[3][sub[2][l]:sub[2][l + 1]]
        sv = sub[4].reshape(-1, b, b)[sub[2][l]:sub[2][l + 1]]
        assert np.array_equal(sc, g2l[fc[keep]])
        assert np.array_equal(sv, fv[keep])


# ---------------------------------------------------------------- linear_solver
def _dense(c, act, rp, col, val):
    b = c.b
    nA = len(act)
    M = np.eye(nA * b)
    V = val.reshape(-1, b, b)
    for l in range(nA):
        for q in range(rp[l], rp[l + 1]):
            M[l * b:(l + 1) * b, col[q] * b:(col[q] + 1) * b] += V[q]
    return M


@pytest.mark.parametrize("cfg", [dict(config=1, nx=10, ny=5), dict(config=2, nx=8, ny=8, n_dfn=4),
                                 dict(config=4, nx=4, ny=4, nz=2, n_dfn=2)])
def test_bicgstab_matches_dense_lu(cfg):
    # SPEC.md:319 (random well-conditioned system vs dense LU to 1e-10)
    c = pkg.Case(**cfg)
    o = Oracle(c)
    o.set_state(_state(c, 1), DAY)
    o.set_u(_state(c, 2))
    act = np.arange(min(c.n, 50), dtype=np.int32)
    F, rhs, rp, col, val = o.assemble(act)
    M = _dense(c, act, rp, col, val)
    x_lu = np.linalg.solve(M, rhs)
    opts = c.solver_opts(lin_rtol=1e-14, lin_maxit=2000)
    rc, x, it, rr = o.linear_solve(len(act), opts)
    assert rc == 0
    assert np.abs(x - x_lu).max() <= 1e-10 * np.abs(x_lu).max()
    rc2, x2, it2, rr2 = o.linear_solve(len(act), opts)
    assert np.array_equal(x, x2) and it == it2  # determinism


def test_solve_isolated_cells_is_elementwise():
    # diagonal (block-diagonal) system -> elementwise division
    c = pkg.Case(5, nx=9, ny=1, nz=1)
    o = Oracle(c)
    o.set_state(_state(c, 1), DAY)
    o.set_u(_state(c, 2))
    act = np.array([0, 2, 4, 6, 8], np.int32)
    F, rhs, rp, col, val = o.assemble(act)
    assert len(col) == 0
    rc, x, it, rr = o.linear_solve(len(act), c.solver_opts())
    assert rc == 0 and np.array_equal(x, rhs)


def test_canonical_sum_order():
    # the canonical tree of blockops.h restated in numpy must give the same bits
    def chunk(v):
        t = [float(v[i]) if i < len(v) else 0.0 for i in range(256)]
        w = []
        for wp in range(8):
            L = t[32 * wp:32 * wp + 32]
            off = 16
            while off >= 1:
                for lane in range(off):
                    L[lane] = L[lane] + L[lane + off]
                off //= 2
            w.append(L[0])
        off = 4
        while off >= 1:
            for k in range(off):
                w[k] = w[k] + w[k + off]
            off //= 2
        return w[0]

    def canon(v):
        if len(v) <= 256:
            return chunk(v)
        parts = [chunk(v[i:i + 256]) for i in range(0, len(v), 256)]
        return canon(np.array(parts))

    rng = np.random.default_rng(1)
    for n in (0, 1, 7, 256, 257, 2049, 70000):
        v = rng.standard_normal(n) * 10.0 ** rng.integers(-5, 5, n)
        assert oracle.canon_sum(v) == canon(v)
        assert oracle.canon_sum(v) == pytest.approx(math.fsum(v), rel=1e-10, abs=1e-12)


# ---------------------------------------------------------------- nonlinear_locality
def test_support_set_kat():
    # SPEC.md:365-367
    out = np.zeros(3, np.int32)
    dp = np.array([0.0, 0.5, 0.29])
    L = oracle.lib()
    k = L.orc_support_set(dp.ctypes.data_as(oracle.d), 3, 0.3, out.ctypes.data_as(oracle.i32))
    assert list(out[:k]) == [1]
    assert L.orc_support_set(np.zeros(3).ctypes.data_as(oracle.d), 3, 0.3, out.ctypes.data_as(oracle.i32)) == 0
    dp = np.array([0.3, 0.1, 0.3])
    k = L.orc_support_set(dp.ctypes.data_as(oracle.d), 3, 0.3, out.ctypes.data_as(oracle.i32))
    assert list(out[:k]) == [0, 2]  # equality included


def test_boundary_and_halo_kat():
    c = pkg.Case(5, nx=10, ny=10, nz=1)
    o = Oracle(c)
    full = np.arange(100, dtype=np.int32)
    assert len(o.boundary_layer(full)) == 0 and len(o.outer_halo(full)) == 0
    assert list(o.boundary_layer([55])) == [55]
    assert len(o.outer_halo([55])) == 4
    blk = np.array([r * 10 + q for r in (4, 5, 6) for q in (4, 5, 6)], np.int32)
    ring = o.boundary_layer(blk)
    assert len(ring) == 8 and 55 not in ring
    h1, h2 = o.outer_halo([11]), o.outer_halo([88])
    assert np.array_equal(o.outer_halo([11, 88]), np.union1d(h1, h2))


def test_expand_active_kat():
    c = pkg.Case(5, nx=12, ny=12, nz=1)
    o = Oracle(c)
    va = np.array([r * 12 + q for r in range(4, 8) for q in range(4, 8)], np.int32)
    dp = np.zeros(c.n)
    dp[va] = 0.01
    na, nb, ex = o.estimate_active(va, dp, 0.3, 2)
    assert not ex and len(na) == 0  # all below ε -> shrink to supp ∪ pinned
    dp[va] = 0.01
    dp[4 * 12 + 4] = 1.0  # one flagged boundary cell (corner of the block)
    na, nb, ex = o.estimate_active(va, dp, 0.3, 2)
    assert ex
    assert np.array_equal(na, np.union1d(va, bfs(c, [4 * 12 + 4], 2)))
    na2, _, ex2 = o.estimate_active(na, np.where(np.isin(np.arange(c.n), na), 0.0, 0.0) + dp * 0, 0.3, 2, False)
    assert not ex2


def test_newton_standard_kats():
    # converged initial guess (BHP = p_init, no change) -> 1 iteration
    c = pkg.Case(1, nx=12, ny=12)
    g = pkg.GraphDesc.from_buffer_copy(c.graph)
    s = c.init_state()
    g.bhp = float(s.u[0])
    o = Oracle(graph=g, fluid=c.fluid)
    opts = c.solver_opts()
    s1, rep, rc = o.newton_standard(s, DAY, opts)
    assert rc == 0 and rep.iterations == 1 and np.array_equal(s1.u, s.u)
    # single-cell closed system converges in <= 3 iterations
    c1 = pkg.Case(5, nx=1, ny=1, nz=1)
    o1 = Oracle(c1)
    s = c1.init_state()
    s.u[0] -= 1e6
    s1, rep, rc = o1.newton_standard(s, DAY, c1.solver_opts(eps_p=0.2, eps_set=0.2))
    assert rc == 0 and rep.iterations <= 3


def test_newton_localized_kats():
    c = pkg.Case(1, nx=20, ny=20)
    o = Oracle(c)
    s0 = c.init_state()
    dt = float(c.schedule()[2])
    opts = c.solver_opts()
    full = np.arange(c.n, dtype=np.int32)
    s_std, r_std, _ = o.newton_standard(s0, dt, opts)
    s_loc, r_loc, rc = o.newton_localized(s0, dt, full, 2, opts.eps_set, opts)
    a, b = r_std.records()[0], r_loc.records()[0]
    assert a["dp_inf_A"] == b["dp_inf_A"] and a["f_norm2"] == b["f_norm2"]  # V_A = full
    # zero production: V_A never grows beyond V_A_init
    g = pkg.GraphDesc.from_buffer_copy(c.graph)
    g.bhp = float(s0.u[0])
    oz = Oracle(graph=g, fluid=c.fluid)
    va = oz.initial_active(None, opts.eps_set, 2)
    _, rep, rc = oz.newton_localized(s0, dt, va, 2, opts.eps_set, opts)
    assert rc == 0 and all(r["n_active"] <= len(va) for r in rep.records())


@pytest.mark.parametrize("solver", [1, 2])
def test_solution_equivalence_and_invariants(solver):
    # SPEC.md:433-438 on a small c1 run: ‖p_loc - p_std‖∞ <= 2ε_p every step,
    # inactive complement bit-immutable, mode monotone, M_A accounting.
    c = pkg.Case(1, nx=30, ny=30, n_steps=8)
    o_std, o_loc = Oracle(c), Oracle(c)
    opts = c.solver_opts()
    s = c.init_state()
    s_std, s_loc = s.copy(), s.copy()
    p_prev = None
    for k, dt in enumerate(c.schedule()):
        s_std, r_std, rc = o_std.newton_standard(s_std, dt, opts)
        assert rc == 0
        total, avg = pkg.compute_ma(r_std, c.n)
        assert total == r_std.iterations and avg == 1.0
        va = o_loc.initial_active(p_prev, opts.eps_set, 2) if k else o_loc.initial_active(None, opts.eps_set, 2)
        o_loc.set_state(s_loc, dt)
        start = s_loc.copy()
        if solver == 1:
            s_new, rep, rc = o_loc.newton_localized(s_loc, dt, va, 2, opts.eps_set, opts)
            modes = [r["mode_expand"] for r in rep.records()]
            assert modes == sorted(modes, reverse=True)  # once shrink, never expand again
        else:
            s_new, rep, rc, labels = o_loc.adaptive_nonlinear_dd(s_loc, dt, va, 4, opts.eps_set,
                                                                 c.solver_opts(m=4))
            assert rc == 0
            lab = labels[labels >= 0]
            assert set(np.unique(lab)) == set(range(rep.n_subdomains))  # partition of V_T
            outside = labels < 0
            assert np.array_equal(s_new.u[outside], start.u[outside])  # immutability
        assert rc == 0
        p_prev = start.u.copy()
        s_loc = s_new
        assert np.abs(s_loc.u - s_std.u).max() <= 2 * opts.eps_p


def test_compute_ma_and_schedule():
    class R:
        def __init__(self, recs):
            self._r = recs

        def records(self):
            return self._r
    assert pkg.compute_ma(R([{"n_active": 100}] * 156), 100) == (156.0, 1.0)
    assert pkg.compute_ma(R([{"n_active": 50}]), 100) == (0.5, 0.5)
    d = pkg.timestep_schedule(10.0, 1.2, 5, 10.0)
    assert np.array_equal(d, np.full(5, 10.0))  # Δt0 = Δt_max -> uniform
    c = pkg.Case(1)
    assert c.schedule().sum() / DAY == pytest.approx(66.48513460159302, rel=1e-12)


def test_mass_balance_closed_system():
    # closed system (no wells) -> Σ residual = Σ accumulation at convergence
    c = pkg.Case(5, nx=12, ny=10, nz=2)
    o = Oracle(c)
    s = c.init_state()
    s.u[: c.n // 2] -= 3e6
    s1, rep, rc = o.newton_standard(s, DAY, c.solver_opts(eps_p=1e-6, eps_set=1e-6, lin_rtol=1e-13))
    assert rc == 0
    o.set_state(s, DAY)
    o.set_u(s1)
    F = o.assemble_raw(np.arange(c.n, dtype=np.int32))[0]
    mass = c.pv.sum() * c.fluid.rho_ref[1]
    assert abs(F.sum()) * DAY <= 1e-10 * mass


def test_oracle_gmres_solves_the_system():
    """GMRES(30) in the oracle: the solution satisfies Â x = rhs to the
    tolerance (dense check), and agrees with BiCGSTAB's solution."""
    import scipy.sparse as sp
    case = pkg.Case(2, nx=24, ny=24, n_dfn=6)
    orc = Oracle(case)
    s = case.init_state()
    s.u[::2] -= np.linspace(0, 2e6, case.n)
    orc.set_state(s, 86400.0)
    act = np.arange(case.n, dtype=np.int32)
    F, rhs, rp, col, val = orc.assemble(act)
    b = case.b
    A = (sp.identity(case.n * b) + sp.bsr_matrix((val.reshape(-1, b, b), col, rp),
                                                 shape=(case.n * b, case.n * b))).tocsr()
    for pc in (0, 2):
        o = case.solver_opts(lin_method=1, precond=pc, lin_rtol=1e-11)
        rc, x, it, rr = orc.linear_solve(case.n, o)
        assert rc == 0 and it > 0
        assert np.linalg.norm(A @ x - rhs) <= 1e-9 * np.linalg.norm(rhs)
        o2 = case.solver_opts(lin_method=0, precond=pc, lin_rtol=1e-11)
        _, x2, _, _ = orc.linear_solve(case.n, o2)
        assert np.allclose(x, x2, rtol=1e-6, atol=1e-9 * np.abs(x2).max())
