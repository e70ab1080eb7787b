"""GPU (sm_100a, through the C-ABI) vs CPU oracle parity.

The bar (BASELINE.json north star): active-set flags and partition labels
bit-exact given the same Newton update; identical Newton and linear iteration
counts; residual norms within 1e-10 relative; final p/S within 1e-8 relative.
By construction (shared cell-local arithmetic, canonical reduction order,
no FMA contraction) every comparison here is BIT-EXACT, which is stricter.
"""
import numpy as np
import pytest

import paper_2008_01539_b200 as pkg
from oracle import Oracle

pytestmark = pytest.mark.gpu

CASES = {
    "c1": dict(config=1),
    "c1s": dict(config=1, nx=40, ny=40),
    "c2s": dict(config=2, nx=64, ny=64, n_dfn=20),
    "c3s": dict(config=3, nx=32, ny=32, nz=4),
    "c4s": dict(config=4, nx=32, ny=32, nz=4, n_dfn=10),
    "c5m": dict(config=5, nx=64, ny=64, nz=8),      # 32768 rows: cooperative-grid Krylov path
    "c2m": dict(config=2, nx=160, ny=160, n_dfn=30),  # 25600 rows, b=2: cooperative-grid path
    # K7 layouts: row-group kernels (large vec4 grids, with and without NNC), per-cell path (nx % 4 != 0)
    "c5rg": dict(config=5, nx=256, ny=256, nz=40),
    "c4rg": dict(config=4, nx=256, ny=256, nz=40, n_dfn=20),
    "c1x": dict(config=1, nx=102, ny=50),
    "c5mid": dict(config=5, nx=64, ny=128, nz=40),  # > 4096 row tiles, < 16*148 row groups: separate row kernels
}


def perturbed_state(case, seed):
    """A non-trivial state: init + smooth pressure drawdown + saturation noise,
    mixed black-oil statuses."""
    rng = np.random.default_rng(seed)
    s = case.init_state()
    b, n = case.b, case.n
    p = s.u[::b]
    p -= rng.uniform(0, 5e6, n)
    if b >= 2:
        s.u[1::b] = np.clip(s.u[1::b] + rng.uniform(-0.05, 0.1, n), 0.0, 1.0)
    if b == 3:
        sat = rng.random(n) < 0.4
        s.status[:] = np.where(sat, 1, 0).astype(np.uint8)
        s.u[2::b] = np.where(sat, rng.uniform(0.0, 0.2, n), case.fluid.rs_b * rng.uniform(0.8, 1.0, n))
    return s


def random_active(case, seed, frac=0.3):
    rng = np.random.default_rng(seed + 1)
    a = np.sort(np.flatnonzero(rng.random(case.n) < frac)).astype(np.int32)
    pin = np.flatnonzero(case.pinned())
    return np.union1d(a, pin).astype(np.int32)


@pytest.mark.parametrize("name", [k for k in CASES if not k.endswith("rg") and k != "c5mid"])
def test_assemble_and_solve_bit_exact(name):
    case = pkg.Case(**CASES[name])
    s = perturbed_state(case, 7)
    dt = 86400.0
    act = random_active(case, 3)
    orc = Oracle(case)
    orc.set_state(s, dt)
    Fo, ro, rpo, co, vo = orc.assemble(act)
    sim = pkg.GpuSimulator(case)
    sim.set_state(s, dt)
    st = sim.set_active(act)
    assert st.n_active == len(act)
    assert np.array_equal(sim.active(), act)
    sim.assemble()
    Fg, rg, rpg, cg, vg = sim.system(len(act))
    assert np.array_equal(rpg, rpo)
    assert np.array_equal(cg, co)
    assert np.array_equal(Fg, Fo), np.abs(Fg - Fo).max()
    assert np.array_equal(rg, ro)
    assert np.array_equal(vg, vo), np.abs(vg - vo).max()
    opts = case.solver_opts()
    rc_o, xo, it_o, rr_o = orc.linear_solve(len(act), opts)
    sim.linear_solve(opts)
    gst = sim.stats()
    xg = sim.solution(len(act))
    assert gst.status == rc_o  # (a Neumann-1 breakdown falls back to block-Jacobi on both sides)
    assert rc_o == 0
    assert gst.lin_iters == it_o
    assert np.array_equal(xg, xo), np.abs(xg - xo).max()
    assert gst.lin_relres == rr_o
    sim.close()


@pytest.mark.parametrize("name", ["c1", "c2s", "c3s", "c5rg", "c4rg", "c1x", "c5mid"])
@pytest.mark.parametrize("m", [1, 2, 4])
@pytest.mark.parametrize("shrink_locked", [False, True])
def test_estimate_active_flags_bit_exact(name, m, shrink_locked):
    case = pkg.Case(**CASES[name])
    rng = np.random.default_rng(m)
    orc = Oracle(case)
    sim = pkg.GpuSimulator(case)
    va = random_active(case, 11, 0.05)
    dp = np.zeros(case.n)
    dp[va] = rng.lognormal(-2.0, 2.0, len(va)) * rng.choice([-1, 1], len(va))
    eps = 0.2
    dp[va[::17]] = eps  # equality is included (Eq. 14)
    oa, ob, oex = orc.estimate_active(va, dp, eps, m, shrink_locked)
    sim.set_active(va)
    sim.upload_dp(dp)
    sim.threshold(eps)
    st = sim.estimate_active(eps, m, shrink_locked)
    assert bool(st.expand) == oex
    assert np.array_equal(sim.active(), oa)
    assert np.array_equal(sim.boundary(), ob)
    sim.close()


def _cmp_reports(rg, ro):
    assert rg.iterations == ro.iterations
    recg, reco = rg.records(), ro.records()
    for a, b in zip(recg, reco):
        assert a["n_active"] == b["n_active"], (a, b)
        assert a["lin_iters"] == b["lin_iters"], (a, b)
        assert a["mode_expand"] == b["mode_expand"], (a, b)
        assert a["dp_inf_A"] == b["dp_inf_A"], (a, b)
        assert a["f_norm2"] == b["f_norm2"], (a, b)
        assert a["f_norminf"] == b["f_norminf"], (a, b)


@pytest.mark.parametrize("name", ["c1", "c2s", "c3s", "c4s"])
def test_newton_solvers_bit_exact(name):
    case = pkg.Case(**CASES[name])
    s0 = case.init_state()
    dts = case.schedule()
    opts = case.solver_opts()
    orc = Oracle(case)
    sim = pkg.GpuSimulator(case)
    for k in (0, 4):
        dt = float(dts[k])
        so, ro, rco = orc.newton_standard(s0, dt, opts)
        sg, rg = sim.newton_standard(s0, dt, opts)
        assert rg.status == rco
        _cmp_reports(rg, ro)
        assert np.array_equal(sg.u, so.u) and np.array_equal(sg.status, so.status)
        va = orc.initial_active(None, opts.eps_set, 2)
        so, ro, rco = orc.newton_localized(s0, dt, va, 2, opts.eps_set, opts)
        sg, rg = sim.newton_localized(s0, dt, va, 2, opts.eps_set, opts)
        assert rg.status == rco
        _cmp_reports(rg, ro)
        assert np.array_equal(sg.u, so.u) and np.array_equal(sg.status, so.status)
        so, ro, rco, lab = orc.adaptive_nonlinear_dd(s0, dt, va, 4, opts.eps_set, opts)
        sg, rg = sim.adaptive_nonlinear_dd(s0, dt, va, 4, opts.eps_set, opts)
        assert rg.status == rco
        assert rg.n_subdomains == ro.n_subdomains
        assert rg.outer_iterations == ro.outer_iterations
        _cmp_reports(rg, ro)
        assert np.array_equal(sim.labels(), lab)
        assert np.array_equal(sg.u, so.u) and np.array_equal(sg.status, so.status)
    sim.close()


@pytest.mark.parametrize("name,solver,precond", [("c1", 0, 0), ("c1", 1, 0), ("c1", 2, 0), ("c2s", 1, 0), ("c4s", 1, 0),
                                                 ("c1", 1, 2), ("c2s", 1, 2), ("c2s", 2, 2), ("c4s", 1, 2)])
def test_run_case_bit_exact(name, solver, precond):
    case = pkg.Case(**CASES[name])
    s0 = case.init_state()
    dts = case.schedule()
    opts = case.solver_opts(precond=precond)
    if solver == 2:
        opts.m = 4
    orc = Oracle(case)
    ro = orc.run_case(solver, s0, dts, opts)
    sim = pkg.GpuSimulator(case)
    rg = sim.run_case(solver, s0, dts, opts)
    assert rg["status"] == ro["status"] == 0
    for k in ("iterations", "sum_na", "lin_iters", "cuts"):
        assert rg[k] == ro[k], (k, rg[k], ro[k])
    assert rg["total_ma"] == ro["total_ma"]
    assert np.array_equal(rg["states"].u, ro["states"].u)
    sim.close()


@pytest.mark.parametrize("name", ["c1", "c2s", "c5mid"])
def test_set_update_paths_agree(name, monkeypatch):
    """The single-kernel cooperative K7 (small grids) and the multi-kernel path
    give identical sets: run the same estimate with RSIM_NO_COOP_K7 in a child."""
    import subprocess, sys, json, os
    code = f"""
import json, numpy as np, paper_2008_01539_b200 as pkg
from tests.test_gpu_parity import CASES, random_active
case = pkg.Case(**CASES[{name!r}])
sim = pkg.GpuSimulator(case)
rng = np.random.default_rng(5)
va = random_active(case, 11, 0.05)
dp = np.zeros(case.n); dp[va] = rng.lognormal(-2.0, 2.0, len(va))
sim.set_active(va); sim.upload_dp(dp); sim.threshold(0.2)
st = sim.estimate_active(0.2, 2, False)
print(json.dumps({{"a": sim.active().tolist(), "b": sim.boundary().tolist(), "ex": int(st.expand)}}))
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env in ({}, {"RSIM_NO_SMEM_K7": "1"}, {"RSIM_NO_SMEM_K7": "1", "RSIM_NO_COOP_K7": "1"}):
        e = dict(os.environ, **env, PYTHONPATH=root)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=e, cwd=root, timeout=600)
        assert r.returncode == 0, r.stderr
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0] == outs[1]


@pytest.mark.parametrize("dims", [(1024, 304, 1),   # 2D full set: 256x4 tile kernel
                                  (256, 64, 19),    # 3D full set: z-marching tile kernel, partial last z-chunk
                                  (512, 32, 24)])
def test_full_set_tile_assembly_bit_exact(dims):
    """Full-set b=1 assembly above the row-kernel threshold runs the tile kernel
    (k_assemble_full1, 256 x 4 tiles of a plane): F, rhs, the scaled
    blocks and the canonical (F,F) partials must equal the oracle's."""
    nx, ny, nz = dims
    case = pkg.Case(5, nx=nx, ny=ny, nz=nz)
    assert case.n >= 148 * 2048
    s = perturbed_state(case, 5)
    dt = 86400.0
    orc = Oracle(case)
    orc.set_state(s, dt)
    Fo, ro, rpo, co, vo = orc.assemble(np.arange(case.n, dtype=np.int32))
    sim = pkg.GpuSimulator(case)
    assert sim.L.rsim_gpu_set_debug(sim._ctx, 1) == 0  # keep the raw residual for the download
    sim.set_state(s, dt)
    sim.set_active(None)
    sim.assemble()
    Fg, rg, rpg, cg, vg = sim.system(case.n)
    assert np.array_equal(rpg, rpo) and np.array_equal(cg, co)
    assert np.array_equal(Fg, Fo), np.abs(Fg - Fo).max()
    assert np.array_equal(rg, ro)
    assert np.array_equal(vg, vo), np.abs(vg - vo).max()
    # ‖F‖₂ from the kernel's canonical chunk partials (no raw-F re-read) must be the oracle's bits
    sim.L.rsim_gpu_set_debug(sim._ctx, 0)
    sim.assemble()
    opts = case.solver_opts(precond=pkg.PREC_BJACOBI, fixed_lin_iters=2, lin_maxit=2)
    rc_o, xo, it_o, rr_o = orc.linear_solve(case.n, opts)
    sim.linear_solve(opts)
    g = sim.stats()
    assert g.lin_iters == it_o
    assert np.array_equal(sim.solution(case.n), xo)
    assert g.lin_relres == rr_o
    sim.close()


@pytest.mark.parametrize("dims", [(1024, 512, 1), (256, 64, 32)])
def test_partial_set_tile_assembly_bit_exact(dims):
    """Partial-set b=1 assembly above the row-kernel threshold (k_assemble_row<1, false>,
    canonical (F,F) chunk partials) on an irregular active set (blocks + sprinkled cells):
    F, rhs, the ELL columns (frozen neighbours -1), the scaled blocks and a 2-iteration
    Krylov solve equal the oracle's."""
    nx, ny, nz = dims
    case = pkg.Case(5, nx=nx, ny=ny, nz=nz)
    s = perturbed_state(case, 7)
    dt = 86400.0
    i = np.arange(case.n)
    ix, iy, iz = i % nx, (i // nx) % ny, i // (nx * ny)
    rng = np.random.default_rng(11)
    mask = ((ix // 37 + iy // 11 + iz) % 3 != 0) | (rng.random(case.n) < 0.02)
    act = np.flatnonzero(mask).astype(np.int32)
    assert len(act) >= 148 * 2048 and len(act) < case.n
    orc = Oracle(case)
    orc.set_state(s, dt)
    Fo, ro, rpo, co, vo = orc.assemble(act)
    sim = pkg.GpuSimulator(case)
    assert sim.L.rsim_gpu_set_debug(sim._ctx, 1) == 0
    sim.set_state(s, dt)
    sim.set_active(act)
    sim.assemble()
    Fg, rg, rpg, cg, vg = sim.system(len(act))
    assert np.array_equal(rpg, rpo) and np.array_equal(cg, co)
    assert np.array_equal(Fg, Fo), np.abs(Fg - Fo).max()
    assert np.array_equal(rg, ro)
    assert np.array_equal(vg, vo), np.abs(vg - vo).max()
    sim.L.rsim_gpu_set_debug(sim._ctx, 0)
    sim.assemble()
    opts = case.solver_opts(precond=pkg.PREC_BJACOBI, fixed_lin_iters=2, lin_maxit=2)
    rc_o, xo, it_o, rr_o = orc.linear_solve(len(act), opts)
    sim.linear_solve(opts)
    g = sim.stats()
    assert g.lin_iters == it_o and g.lin_relres == rr_o
    assert np.array_equal(sim.solution(len(act)), xo)
    sim.close()


def _dilate_np(mask, m):
    """m hops of 6-neighbour (4 in 2D) dilation on a (nz, ny, nx) boolean grid."""
    out = mask.copy()
    for _ in range(m):
        cur = out.copy()
        for ax in range(3):
            if cur.shape[ax] > 1:
                sl_a = [slice(None)] * 3
                sl_b = [slice(None)] * 3
                sl_a[ax], sl_b[ax] = slice(1, None), slice(None, -1)
                out[tuple(sl_a)] |= cur[tuple(sl_b)]
                out[tuple(sl_b)] |= cur[tuple(sl_a)]
    return out


@pytest.mark.parametrize("frac,m", [(0.05, 2), (0.2, 1), (0.5, 3), (1.0, 2)])
def test_support_active_c5_field(frac, m):
    """Config-5 set update (fused reset + seed, bitmap dilation on large grids,
    count / scan / scatter): V_A = m-hop dilation of {|δp| >= ε} and its
    boundary layer, against a numpy restatement."""
    import ctypes as C
    case = pkg.Case(5, nx=256, ny=256, nz=40)
    eps = 1e-3
    dp, _, _ = case.c5_field(frac, m, eps)
    sim = pkg.GpuSimulator(case)
    sim.upload_dp(dp)
    st = pkg.GpuStats()
    assert sim.L.rsim_gpu_support_active(sim._ctx, eps, m, C.byref(st)) == 0
    shape = (case.nz, case.ny, case.nx)
    a = _dilate_np((np.abs(dp) >= eps).reshape(shape), m)
    act = np.flatnonzero(a.ravel()).astype(np.int32)
    ga = sim.active()
    assert st.n_active == len(act)
    assert np.array_equal(ga, act)
    inner = ~_dilate_np(~a, 1)  # active cells whose every neighbour is active
    bnd = np.flatnonzero((a & ~inner).ravel()).astype(np.int32)
    assert np.array_equal(sim.boundary(), bnd)
    sim.close()
