"""ctypes wrapper of the CPU oracle (oracle/_build/liborsim.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product
package paper_2008_01539_b200.  The oracle restates SPEC.md + PAPER.md
Algorithms 1-2 in C++ (oracle/oracle.cpp, each function cites its source).
Parity pinning: SPEC known-answer examples and invariants only — the
reference ships no implementation or golden vectors.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from paper_2008_01539_b200 import _abi as A

LIB_PATH = Path(__file__).resolve().parent / "_build" / "liborsim.so"
P = C.c_void_p
d, i32, u8, i64 = A.dptr, A.i32ptr, A.u8ptr, A.i64ptr

PROTOS = {
    "orc_build_matrix_grid": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double,
                                        d, d, d, d, d, d]),
    "orc_create": (P, [C.POINTER(A.GraphDesc), C.POINTER(A.FluidParams)]),
    "orc_destroy": (None, [P]),
    "orc_set_threads": (None, [C.c_int]),
    "orc_threads": (C.c_int, []),
    "orc_set_state": (C.c_int, [P, d, u8, C.c_double]),
    "orc_get_state": (C.c_int, [P, d, u8]),
    "orc_set_dt": (C.c_int, [P, C.c_double]),
    "orc_assemble": (C.c_int64, [P, i32, C.c_int32, d, d, i32, i32, d, C.c_int64]),
    "orc_linear_solve": (C.c_int, [P, C.POINTER(A.SolverOpts), d, i32, d]),
    "orc_canon_sum": (C.c_double, [d, C.c_int64]),
    "orc_neighbor_set": (C.c_int32, [P, C.c_int32, C.c_int32, i32]),
    "orc_support_set": (C.c_int32, [d, C.c_int32, C.c_double, i32]),
    "orc_boundary_layer": (C.c_int32, [P, i32, C.c_int32, i32]),
    "orc_outer_halo": (C.c_int32, [P, i32, C.c_int32, i32]),
    "orc_estimate_active": (C.c_int32, [P, i32, C.c_int32, d, C.c_double, C.c_int32, C.c_int32, i32, i32, i32,
                                        i32]),
    "orc_newton_standard": (C.c_int, [P, C.c_double, C.POINTER(A.SolverOpts), C.POINTER(A.NewtonReport)]),
    "orc_newton_localized": (C.c_int, [P, C.c_double, i32, C.c_int32, C.POINTER(A.SolverOpts),
                                       C.POINTER(A.NewtonReport)]),
    "orc_adaptive_dd": (C.c_int, [P, C.c_double, i32, C.c_int32, C.POINTER(A.SolverOpts),
                                  C.POINTER(A.NewtonReport), i32]),
    "orc_initial_active": (C.c_int32, [P, d, C.c_double, C.c_int32, i32]),
    "orc_run_case": (C.c_int, [P, C.c_int32, d, C.c_int32, C.POINTER(A.SolverOpts), i32, d, i64, i32, i32]),
    "orc_full_residual": (C.c_int, [P, d]),
    "orc_rexp": (C.c_double, [C.c_double]),
    "orc_corey": (None, [C.c_double, C.c_double, C.c_double, d, d]),
    "orc_props": (C.c_int, [C.POINTER(A.FluidParams), d, C.c_uint8, d, d, d, d]),
    "orc_set_u": (C.c_int, [P, d, u8]),
    "orc_assemble_raw": (C.c_int64, [P, i32, C.c_int32, d, d, i32, i32, d, C.c_int64]),
    "orc_eos_rlog": (C.c_double, [C.c_double]),
    "orc_eos_cubic_roots": (C.c_int, [C.c_double, C.c_double, d]),
    "orc_eos_phase": (C.c_int, [C.POINTER(A.EosParams), C.c_double, C.c_double, d, C.c_int32, C.c_int32, d, d]),
    "orc_eos_rachford_rice": (C.c_int, [C.c_int32, d, d, d]),
    "orc_eos_stability": (C.c_int, [C.POINTER(A.EosParams), C.c_double, C.c_double, d, d, i32]),
    "orc_eos_flash": (C.c_int, [C.POINTER(A.EosParams), C.c_double, C.c_int64, d, d, u8, d, d, d, d, i32]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build()")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in PROTOS.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def canon_sum(v: np.ndarray) -> float:
    v = np.ascontiguousarray(v, np.float64)
    return float(lib().orc_canon_sum(A.ptr(v, C.c_double), len(v)))


def set_threads(n: int) -> None:
    lib().orc_set_threads(n)


def build_matrix_grid(nx, ny, nz, dx, dy, dz, kx, ky, kz):
    n = nx * ny * nz
    tx, ty, tz = np.zeros(n), np.zeros(n), np.zeros(n)
    kx, ky, kz = (np.ascontiguousarray(k, np.float64) for k in (kx, ky, kz))
    rc = lib().orc_build_matrix_grid(nx, ny, nz, dx, dy, dz, A.ptr(kx, C.c_double), A.ptr(ky, C.c_double),
                                     A.ptr(kz, C.c_double), A.ptr(tx, C.c_double), A.ptr(ty, C.c_double),
                                     A.ptr(tz, C.c_double))
    if rc != 0:
        raise ValueError("build_matrix_grid: configuration error")
    return tx, ty, tz


def rexp(x: float) -> float:
    return float(lib().orc_rexp(x))


def corey(s: float, s_r: float, den: float) -> tuple[float, float]:
    kr, dkr = C.c_double(), C.c_double()
    lib().orc_corey(s, s_r, den, C.byref(kr), C.byref(dkr))
    return kr.value, dkr.value


def props(fluid, u, st=0):
    """(A, dA, L, dL) of one cell (include/rsim/physics.h)."""
    b = int(fluid.kind)
    u = np.ascontiguousarray(u, np.float64)
    Aa, dA, L, dL = np.zeros(b), np.zeros(b * b), np.zeros(b), np.zeros(b * b)
    lib().orc_props(C.byref(fluid), A.ptr(u, C.c_double), st, A.ptr(Aa, C.c_double), A.ptr(dA, C.c_double),
                    A.ptr(L, C.c_double), A.ptr(dL, C.c_double))
    return Aa, dA.reshape(b, b), L, dL.reshape(b, b)


class Oracle:
    """CPU restatement bound to one graph + fluid (mirrors GpuSimulator)."""

    def __init__(self, case=None, graph=None, fluid=None):
        self.L = lib()
        g = graph if graph is not None else case.graph
        f = fluid if fluid is not None else case.fluid
        self.case = case
        self.b = int(f.kind)
        self.n = int(g.nx) * int(g.ny) * int(g.nz)
        self._h = self.L.orc_create(C.byref(g), C.byref(f))
        if not self._h:
            raise ValueError("orc_create failed")

    def __del__(self):
        if getattr(self, "_h", None):
            self.L.orc_destroy(self._h)
            self._h = None

    def set_state(self, states, dt):
        self.L.orc_set_state(self._h, A.ptr(states.u, C.c_double), A.ptr(states.status, C.c_uint8), dt)

    def get_state(self):
        from paper_2008_01539_b200 import CellStates
        s = CellStates(np.zeros(self.n * self.b), np.zeros(self.n, np.uint8))
        self.L.orc_get_state(self._h, A.ptr(s.u, C.c_double), A.ptr(s.status, C.c_uint8))
        return s

    def assemble(self, act: np.ndarray):
        act = np.ascontiguousarray(act, np.int32)
        nA, b = len(act), self.b
        F, rhs, rp = np.zeros(nA * b), np.zeros(nA * b), np.zeros(nA + 1, np.int32)
        nnz = self.L.orc_assemble(self._h, A.ptr(act, C.c_int32), nA, A.ptr(F, C.c_double),
                                  A.ptr(rhs, C.c_double), A.ptr(rp, C.c_int32), None, None, 0)
        if nnz < 0:
            raise ArithmeticError("singular diagonal block")
        col = np.zeros(max(nnz, 1), np.int32)
        val = np.zeros(max(nnz, 1) * b * b)
        self.L.orc_assemble(self._h, A.ptr(act, C.c_int32), nA, None, None, None, A.ptr(col, C.c_int32),
                            A.ptr(val, C.c_double), nnz)
        return F, rhs, rp, col[:nnz], val[: nnz * b * b]

    def set_u(self, states):
        self.L.orc_set_u(self._h, A.ptr(states.u, C.c_double), A.ptr(states.status, C.c_uint8))

    def assemble_raw(self, act: np.ndarray):
        act = np.ascontiguousarray(act, np.int32)
        nA, b = len(act), self.b
        F, D, rp = np.zeros(nA * b), np.zeros(nA * b * b), np.zeros(nA + 1, np.int32)
        nnz = self.L.orc_assemble_raw(self._h, A.ptr(act, C.c_int32), nA, A.ptr(F, C.c_double),
                                      A.ptr(D, C.c_double), A.ptr(rp, C.c_int32), None, None, 0)
        if nnz < 0:
            raise ArithmeticError("singular")
        col = np.zeros(max(nnz, 1), np.int32)
        val = np.zeros(max(nnz, 1) * b * b)
        self.L.orc_assemble_raw(self._h, A.ptr(act, C.c_int32), nA, None, None, None, A.ptr(col, C.c_int32),
                                A.ptr(val, C.c_double), nnz)
        return F, D.reshape(nA, b, b), rp, col[:nnz], val[: nnz * b * b].reshape(-1, b, b)

    def linear_solve(self, nA: int, opts):
        x = np.zeros(max(nA * self.b, 1))
        it = C.c_int32()
        rr = C.c_double()
        rc = self.L.orc_linear_solve(self._h, C.byref(opts), A.ptr(x, C.c_double), C.byref(it), C.byref(rr))
        return rc, x[: nA * self.b], it.value, rr.value

    def neighbor_set(self, i: int, m: int) -> np.ndarray:
        out = np.zeros(self.n, np.int32)
        k = self.L.orc_neighbor_set(self._h, i, m, A.ptr(out, C.c_int32))
        return out[:k].copy()

    def boundary_layer(self, va) -> np.ndarray:
        va = np.ascontiguousarray(va, np.int32)
        out = np.zeros(self.n, np.int32)
        k = self.L.orc_boundary_layer(self._h, A.ptr(va, C.c_int32), len(va), A.ptr(out, C.c_int32))
        return out[:k].copy()

    def outer_halo(self, va) -> np.ndarray:
        va = np.ascontiguousarray(va, np.int32)
        out = np.zeros(self.n, np.int32)
        k = self.L.orc_outer_halo(self._h, A.ptr(va, C.c_int32), len(va), A.ptr(out, C.c_int32))
        return out[:k].copy()

    def estimate_active(self, va, dp_global, eps, m, shrink_locked=False):
        va = np.ascontiguousarray(va, np.int32)
        dp = np.ascontiguousarray(dp_global, np.float64)
        oa, ob = np.zeros(self.n, np.int32), np.zeros(self.n, np.int32)
        nb, ex = C.c_int32(), C.c_int32()
        k = self.L.orc_estimate_active(self._h, A.ptr(va, C.c_int32), len(va), A.ptr(dp, C.c_double), eps, m,
                                       int(shrink_locked), A.ptr(oa, C.c_int32), A.ptr(ob, C.c_int32),
                                       C.byref(nb), C.byref(ex))
        return oa[:k].copy(), ob[: nb.value].copy(), bool(ex.value)

    def initial_active(self, p_prev, eps, m) -> np.ndarray:
        out = np.zeros(self.n, np.int32)
        pp = None if p_prev is None else np.ascontiguousarray(p_prev, np.float64)
        k = self.L.orc_initial_active(self._h, A.ptr(pp, C.c_double), eps, m, A.ptr(out, C.c_int32))
        return out[:k].copy()

    def newton_standard(self, states, dt, opts):
        self.set_state(states, dt)
        rep = A.NewtonReport()
        rc = self.L.orc_newton_standard(self._h, dt, C.byref(opts), C.byref(rep))
        return self.get_state(), rep, rc

    def newton_localized(self, states, dt, va_init, m, eps, opts):
        o = A.SolverOpts.from_buffer_copy(opts)
        o.m, o.eps_set = m, eps
        self.set_state(states, dt)
        va = np.ascontiguousarray(va_init, np.int32)
        rep = A.NewtonReport()
        rc = self.L.orc_newton_localized(self._h, dt, A.ptr(va, C.c_int32), len(va), C.byref(o), C.byref(rep))
        return self.get_state(), rep, rc

    def adaptive_nonlinear_dd(self, states, dt, va_init, m, eps, opts):
        o = A.SolverOpts.from_buffer_copy(opts)
        o.m, o.eps_set = m, eps
        self.set_state(states, dt)
        va = np.ascontiguousarray(va_init, np.int32)
        rep = A.NewtonReport()
        labels = np.full(self.n, -1, np.int32)
        rc = self.L.orc_adaptive_dd(self._h, dt, A.ptr(va, C.c_int32), len(va), C.byref(o), C.byref(rep),
                                    A.ptr(labels, C.c_int32))
        return self.get_state(), rep, rc, labels

    def run_case(self, solver, states, dts, opts) -> dict:
        self.set_state(states, float(dts[0]))
        d = np.ascontiguousarray(dts, np.float64)
        it, lin, cuts = C.c_int32(), C.c_int32(), C.c_int32()
        ma, na = C.c_double(), C.c_int64()
        rc = self.L.orc_run_case(self._h, solver, A.ptr(d, C.c_double), len(d), C.byref(opts), C.byref(it),
                                 C.byref(ma), C.byref(na), C.byref(lin), C.byref(cuts))
        return {"status": rc, "states": self.get_state(), "iterations": it.value, "total_ma": ma.value,
                "sum_na": na.value, "lin_iters": lin.value, "cuts": cuts.value}

    def full_residual(self) -> np.ndarray:
        F = np.zeros(self.n * self.b)
        self.L.orc_full_residual(self._h, A.ptr(F, C.c_double))
        return F


def eos_flash(e, T: float, p: np.ndarray, z: np.ndarray) -> dict:
    """CPU flash of every cell (oracle, OpenMP): same outputs as pkg.eos_flash."""
    n, nc = len(p), e.nc
    p = np.ascontiguousarray(p, np.float64)
    z = np.ascontiguousarray(z, np.float64).reshape(n * nc)
    out = dict(status=np.zeros(n, np.uint8), nu_g=np.zeros(n), x=np.zeros(n * nc), y=np.zeros(n * nc),
               zfac=np.zeros(2 * n), iters=np.zeros(n, np.int32))
    rc = lib().orc_eos_flash(C.byref(e), T, n, A.ptr(p, C.c_double), A.ptr(z, C.c_double),
                             A.ptr(out["status"], C.c_uint8), A.ptr(out["nu_g"], C.c_double),
                             A.ptr(out["x"], C.c_double), A.ptr(out["y"], C.c_double),
                             A.ptr(out["zfac"], C.c_double), A.ptr(out["iters"], C.c_int32))
    assert rc == 0, rc
    return out
