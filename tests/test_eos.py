"""Peng-Robinson property functions and flash (
SPEC.md:135-177), include/rsim/eos.h.

CPU: the oracle's functions against the SPEC known answers and against an
independent numpy restatement (np.roots for the cubic, np.log, a dense
tangent-plane-distance scan for stability, scipy brentq for Rachford-Rice).
GPU: the sm_100a flash kernel (rsim_eos_flash, C-ABI) is bit-identical to the
oracle on seeded batches of cells.
"""
import ctypes as C

import numpy as np
import pytest

import paper_2008_01539_b200 as pkg
from paper_2008_01539_b200 import _abi as A

R = 8.31446261815324
PSI = 6894.757293168361
T3 = 340.0  # Case 3 temperature (§5 Case 3)


def _orc():
    import oracle
    return oracle.lib()


def _params(nc, comps):
    """Component table: (Tc K, Pc Pa, omega) per component."""
    e = A.EosParams()
    e.nc = nc
    for i, (tc, pc, w) in enumerate(comps):
        e.tc[i], e.pc[i], e.omega[i], e.mw[i] = tc, pc, w, 0.1
    e.flash_tol, e.flash_maxit, e.stab_maxit = 1e-8, 500, 200
    return e


C1, C4, C10 = (190.56, 4.599e6, 0.0115), (425.12, 3.796e6, 0.2002), (617.7, 2.110e6, 0.4923)


# ---- numpy restatement (independent code path: np.roots, np.log) ----------
def np_terms(e, T):
    nc = e.nc
    tc, pc, w = (np.array(v[:nc]) for v in (e.tc, e.pc, e.omega))
    kap = np.where(w <= 0.49, 0.37464 + 1.54226 * w - 0.26992 * w * w,
                   0.379642 + 1.48503 * w - 0.164423 * w * w + 0.016666 * w ** 3)
    ai = 0.457235529 * (R * tc) ** 2 / pc * (1 + kap * (1 - np.sqrt(T / tc))) ** 2
    bi = 0.0777960739 * R * tc / pc
    kij = np.array([[e.kij[i][j] for j in range(nc)] for i in range(nc)])
    aij = np.sqrt(np.outer(ai, ai)) * (1 - kij)
    return aij, bi


def np_roots(Aa, B):
    r = np.roots([1.0, -(1 - B), Aa - 3 * B * B - 2 * B, -(Aa * B - B * B - B ** 3)])
    r = np.sort(r[np.abs(r.imag) < 1e-10 * np.maximum(1, np.abs(r.real))].real)
    return r[r > B]


def np_lnphi(e, T, p, x, sel):
    aij, bi = np_terms(e, T)
    am, bm = x @ aij @ x, x @ bi
    Aa, B = am * p / (R * T) ** 2, bm * p / (R * T)
    r = np_roots(Aa, B)
    Z = r[0] if sel == 0 else r[-1]
    s2 = np.sqrt(2.0)
    lp = bi / bm * (Z - 1) - np.log(Z - B) - Aa / (2 * s2 * B) * (2 * (aij @ x) / am - bi / bm) * np.log(
        (Z + (1 + s2) * B) / (Z + (1 - s2) * B))
    return Z, lp


def orc_phase(e, T, p, x, sel, min_g=0):
    Z, lp = C.c_double(), np.zeros(e.nc)
    x = np.ascontiguousarray(x, np.float64)
    rc = _orc().orc_eos_phase(C.byref(e), T, p, A.ptr(x, C.c_double), sel, min_g, C.byref(Z), A.ptr(lp, C.c_double))
    return rc, Z.value, lp


# ---- CPU: oracle vs SPEC known answers and the numpy restatement ----------
def test_rlog_matches_log():
    rng = np.random.default_rng(1)
    x = np.concatenate([10.0 ** rng.uniform(-300, 300, 20000), rng.uniform(0.5, 2.0, 20000), [1.0, 2.0, 0.5,
                                                                                               5e-324, 1e-310]])
    L = _orc()
    got = np.array([L.orc_eos_rlog(v) for v in x])
    ref = np.log(x)
    err = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)
    assert np.max(np.where(ref != 0, err, np.abs(got))) < 1e-15
    assert L.orc_eos_rlog(1.0) == 0.0


def test_cubic_roots_match_np_roots():
    rng = np.random.default_rng(2)
    L = _orc()
    r = np.zeros(3)
    for _ in range(3000):
        Aa, B = rng.uniform(0, 12), rng.uniform(1e-4, 0.35)
        n = L.orc_eos_cubic_roots(Aa, B, A.ptr(r, C.c_double))
        ref = np_roots(Aa, B)
        if n != len(ref):  # only near a double root may the counts differ
            assert np.min(np.abs(np.diff(np.roots([1.0, -(1 - B), Aa - 3 * B * B - 2 * B,
                                                   -(Aa * B - B * B - B ** 3)])))) < 1e-4
            continue
        np.testing.assert_allclose(r[:n], ref, rtol=1e-9, atol=1e-12)
    assert L.orc_eos_cubic_roots(0.0, 0.0, A.ptr(r, C.c_double)) == 1 and r[0] == 1.0  # ideal limit Z = 1


def test_z_factor_kats():
    c1 = _params(1, [C1])
    rc, Z, lp = orc_phase(c1, T3, 101325.0, [1.0], 1)
    # SPEC.md:141 says within 1e-3 of 1; PR with the standard C1 constants gives
    # 0.99858 here (the numpy restatement agrees), i.e. 1.4e-3: asserted as 2e-3
    assert rc == 0 and abs(Z - 1.0) < 2e-3 and abs(Z - np_lnphi(c1, T3, 101325.0, np.array([1.0]), 1)[0]) < 1e-14
    rc, Z, lp = orc_phase(c1, T3, 0.0, [1.0], 1)  # ideal limit: Z = 1, φ = 1
    assert rc == 0 and Z == 1.0 and lp[0] == 0.0
    c10 = _params(1, [C10])
    _, Zl, _ = orc_phase(c10, T3, 2e7, [1.0], 0)
    _, Zv, _ = orc_phase(c10, T3, 2e7, [1.0], 1)
    assert Zl <= Zv  # SPEC.md:142 root ordering
    twin = _params(2, [C4, C4])
    _, _, lp = orc_phase(twin, T3, 5e6, [0.5, 0.5], 0)
    assert lp[0] == lp[1]  # SPEC.md:149 symmetry


@pytest.mark.parametrize("comps", [[C1, C10], [C1, C4, C10], [C1, C4, C10, C4]])
def test_lnphi_matches_numpy(comps):
    e = _params(len(comps), comps)
    rng = np.random.default_rng(len(comps))
    for _ in range(200):
        x = rng.dirichlet(np.ones(e.nc))
        p = rng.uniform(1e5, 3e7)
        for sel in (0, 1):
            rc, Z, lp = orc_phase(e, T3, p, x, sel)
            Zr, lr = np_lnphi(e, T3, p, x, sel)
            assert rc == 0
            assert abs(Z - Zr) <= 1e-10 * Zr
            np.testing.assert_allclose(lp, lr, rtol=1e-8, atol=1e-10)


def test_rachford_rice_kats():
    L = _orc()
    nu = C.c_double()
    z = np.array([0.5, 0.5])
    for K in ([2.0, 0.5], [4.0, 0.25]):
        K = np.array(K)
        assert L.orc_eos_rachford_rice(2, A.ptr(z, C.c_double), A.ptr(K, C.c_double), C.byref(nu)) == 0
        assert abs(nu.value - 0.5) < 1e-14
    K = np.array([1.0, 1.0])
    assert L.orc_eos_rachford_rice(2, A.ptr(z, C.c_double), A.ptr(K, C.c_double), C.byref(nu)) != 0
    from scipy.optimize import brentq
    rng = np.random.default_rng(4)
    for _ in range(300):
        z = rng.dirichlet(np.ones(3))
        K = np.array([rng.uniform(1.2, 20), rng.uniform(0.05, 0.9), rng.uniform(0.1, 5)])
        g = lambda v: np.sum(z * (K - 1) / (1 + v * (K - 1)))  # noqa: E731
        lo, hi = 1 / (1 - K.max()), 1 / (1 - K.min())
        ref = brentq(g, lo + 1e-12 * (hi - lo), hi - 1e-12 * (hi - lo), xtol=1e-15)
        assert L.orc_eos_rachford_rice(3, A.ptr(z, C.c_double), A.ptr(K, C.c_double), C.byref(nu)) == 0
        assert abs(nu.value - ref) <= 1e-12 * max(1.0, abs(ref))


def _stable(e, p, z):
    K, st = np.zeros(e.nc), C.c_int32()
    z = np.ascontiguousarray(z, np.float64)
    assert _orc().orc_eos_stability(C.byref(e), T3, p, A.ptr(z, C.c_double), A.ptr(K, C.c_double), C.byref(st)) == 0
    return bool(st.value)


def _tpd_scan_unstable(e, p, z):
    """Dense tangent-plane-distance scan over binary trial compositions (0.001 grid)."""
    Zz, lz = np_lnphi(e, T3, p, np.asarray(z), 0)
    Zv, lv = np_lnphi(e, T3, p, np.asarray(z), 1)
    if Zv != Zz and np.dot(z, lv) < np.dot(z, lz):
        lz = lv
    d = np.log(z) + lz
    tpd_min = np.inf
    for w in np.arange(0.001, 1.0, 0.001):
        y = np.array([w, 1 - w])
        for sel in (0, 1):
            _, ly = np_lnphi(e, T3, p, y, sel)
            tpd_min = min(tpd_min, float(np.dot(y, np.log(y) + ly - d)))
    return tpd_min < -1e-10


def test_stability_kats_and_tpd_scan():
    e = pkg.eos_case3()
    assert _stable(_params(2, [C1, C10]), 2e6, [1.0, 0.0])  # pure component
    assert _stable(e, 2900 * PSI, [0.5, 0.5])               # Case 3 initial state
    assert not _stable(e, 1000 * PSI, [0.5, 0.5])           # below the bubble point
    for p_psi in (2900, 2500, 2000, 1000, 300):
        assert _stable(e, p_psi * PSI, [0.5, 0.5]) == (not _tpd_scan_unstable(e, p_psi * PSI, np.array([0.5, 0.5])))


@pytest.mark.parametrize("comps", [[C1, C10], [C1, C4, C10]])
def test_flash_material_balance_and_fugacity_equality(comps):
    import oracle
    e = _params(len(comps), comps)
    rng = np.random.default_rng(7)
    n = 400
    p = rng.uniform(50, 3000, n) * PSI
    z = rng.dirichlet(np.ones(e.nc), n)
    o = oracle.eos_flash(e, T3, p, z)
    two = o["status"] == 2
    assert two.sum() > 50 and (~two).sum() > 20
    x, y = o["x"].reshape(n, e.nc), o["y"].reshape(n, e.nc)
    nu = o["nu_g"]
    for i in np.flatnonzero(two):
        assert 0.0 < nu[i] < 1.0
        np.testing.assert_allclose((1 - nu[i]) * x[i] + nu[i] * y[i], z[i], rtol=0, atol=1e-10)
        _, lo = np_lnphi(e, T3, p[i], x[i], 0)
        _, lg = np_lnphi(e, T3, p[i], y[i], 1)
        fo, fg = x[i] * np.exp(lo) * p[i], y[i] * np.exp(lg) * p[i]
        np.testing.assert_allclose(fo, fg, rtol=1e-7)  # SPEC.md:115, :150 (flash tol 1e-8 on the ratio)
        assert y[i][0] > x[i][0]  # gas enriched in the light component
    for i in np.flatnonzero(~two):  # single phase: composition of the phase is z
        assert np.array_equal(x[i], z[i]) and np.array_equal(y[i], z[i])
        assert o["nu_g"][i] in (0.0, 1.0)


def test_case3_depletion_sequence():
    import oracle
    e = pkg.eos_case3()
    p = np.array([2900, 2500, 2000, 1500, 1000, 500, 100]) * PSI
    o = oracle.eos_flash(e, T3, p, np.tile([0.5, 0.5], (len(p), 1)))
    assert o["status"][0] == 0 and o["status"][-1] == 2  # undersaturated oil, then gas appears (§5 Case 3)
    nu = o["nu_g"][o["status"] == 2]
    assert np.all(np.diff(nu) > 0)  # more gas as pressure drops


# ---- GPU: the sm_100a flash kernel is bit-identical to the oracle ----------
@pytest.mark.gpu
@pytest.mark.parametrize("comps", [[C1, C10], [C1, C4, C10], [C1, C4, C10, C4], [C10]])
def test_gpu_flash_bit_exact(comps):
    import oracle
    e = _params(len(comps), comps)
    rng = np.random.default_rng(11)
    n = 50000
    p = rng.uniform(14.7, 3500, n) * PSI
    z = rng.dirichlet(np.ones(e.nc), n) if e.nc > 1 else np.ones((n, 1))
    g = pkg.eos_flash(e, T3, p, z)
    o = oracle.eos_flash(e, T3, p, z)
    for k in ("status", "nu_g", "x", "y", "zfac", "iters"):
        assert np.array_equal(g[k], o[k]), k
    if e.nc > 1:
        assert (g["status"] == 2).sum() > 0
