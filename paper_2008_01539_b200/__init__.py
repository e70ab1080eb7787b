"""paper_2008_01539_b200 — B200-native localized FIM Newton (arXiv 2008.01539).

Host-side Python mirror of the reference's solver interface (SPEC.md
modules nonlinear_locality / sim_driver_cli) over the C-ABI of
lib/librsim.so (include/rsim/gpu_abi.h).  Every compute step runs in
hand-written sm_100a kernels; there is no CPU fallback: on a machine without
a B200 the GPU entry points raise RsimError(RSIM_ECUDA).

SPEC operation            -> this module
  newton_standard  GpuSimulator.newton_standard
  newton_localized  GpuSimulator.newton_localized
  adaptive_nonlinear_dd (:413)    GpuSimulator.adaptive_nonlinear_dd
  run_case          GpuSimulator.run_case
  timestep_schedule timestep_schedule
  compute_ma        compute_ma
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi as A
from ._abi import (DIRECT_MAX, FLUID_BLACKOIL, FLUID_OILWATER, FLUID_SINGLE, LIN_BICGSTAB, LIN_DIRECT, LIN_GMRES, PREC_BJACOBI, PREC_ILU0,
                   PREC_NEUMANN1, RSIM_EARG, RSIM_ECUDA,
                   RSIM_ENOCONV, RSIM_ENUM, RSIM_OK, FluidParams, GpuStats, GraphDesc, NewtonReport, SolverOpts)

__all__ = [
    "Case", "CellStates", "GpuSimulator", "RsimError", "compute_ma", "timestep_schedule", "SolverOpts",
    "NewtonReport", "FluidParams", "GraphDesc", "RSIM_OK", "RSIM_EARG", "RSIM_ECUDA", "RSIM_ENUM", "RSIM_ENOCONV",
    "FLUID_SINGLE", "FLUID_OILWATER", "FLUID_BLACKOIL", "PREC_BJACOBI", "PREC_ILU0", "PREC_NEUMANN1", "DAY",
    "LIN_BICGSTAB", "LIN_GMRES", "LIN_DIRECT", "DIRECT_MAX",
]

DAY = 86400.0


class RsimError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"rsim error {code}: {msg}")
        self.code = code


def _check(rc: int, what: str) -> None:
    if rc != RSIM_OK:
        err = A.lib().rsim_gpu_last_error()
        raise RsimError(rc, f"{what}: {err.decode() if err else ''}")


def timestep_schedule(dt0: float, growth: float, nsteps: int, dt_max: float = float("inf")) -> np.ndarray:
    """Δt_k = min(Δt0·g^k, Δt_max), k < nsteps."""
    return np.array([min(dt0 * growth**k, dt_max) for k in range(nsteps)], dtype=np.float64)


def compute_ma(report: NewtonReport, n: int) -> tuple[float, float]:
    """(total M_A, average per iteration) = (Σ n_A/n, total/iterations)."""
    recs = report.records()
    total = sum(r["n_active"] / n for r in recs)
    return total, (total / len(recs) if recs else 0.0)


@dataclass
class CellStates:
    """Natural-variable state: u[n*b] cell-major, status u8[n]."""
    u: np.ndarray
    status: np.ndarray

    def copy(self) -> "CellStates":
        return CellStates(self.u.copy(), self.status.copy())

    def pressure(self, b: int) -> np.ndarray:
        return self.u[::b]


class Case:
    """Seeded synthetic input for one BASELINE.json config (include/rsim/cases.h)."""

    def __init__(self, config: int, nx: int = 0, ny: int = 0, nz: int = 0, seed: int = 0, n_dfn: int = -1,
                 n_steps: int = -1, lib=None, _handle=None):
        # lib: any library exporting include/rsim/cases.h (librsim.so by default; the
        # oracle's own liborsim.so links the same host-only generator, so the CPU
        # reference arm builds its inputs without loading the product library)
        L = lib if lib is not None else A.lib()
        self._L = L
        if _handle is not None:  # Case.from_file / Case.from_text
            self._h = _handle
        else:
            o = A.CaseOpts(config, nx, ny, nz, seed, n_dfn, n_steps)
            self._h = L.rsim_case_create(C.byref(o))
        if not self._h:
            raise RsimError(RSIM_EARG, f"bad case config {config}")
        self.config = config
        info = A.CaseInfo()
        L.rsim_case_info(self._h, C.byref(info))
        self.n_live, self.n_frac, self.n_dead = int(info.n_live), int(info.n_frac), int(info.n_dead)
        self.default_solver, self.default_m = int(info.solver), int(info.m)
        self.n = int(L.rsim_case_n(self._h))
        d = np.zeros(3, np.int32)
        s = np.zeros(3, np.float64)
        L.rsim_case_dims(self._h, A.ptr(d, C.c_int32), A.ptr(s, C.c_double))
        self.nx, self.ny, self.nz = (int(v) for v in d)
        self.dx, self.dy, self.dz = (float(v) for v in s)
        self.graph = GraphDesc()
        L.rsim_case_graph(self._h, C.byref(self.graph))
        self.fluid = FluidParams()
        L.rsim_case_fluid(self._h, C.byref(self.fluid))
        self.b = int(self.fluid.kind)
        self.n_nnc = int(L.rsim_case_n_nnc(self._h))

    @classmethod
    def from_text(cls, text: str, lib=None) -> "Case":
        """A case file's text (grammar: include/rsim/cases.h; EDFM fractures)."""
        L = lib if lib is not None else A.lib()
        err = C.create_string_buffer(512)
        h = L.rsim_case_from_text(text.encode(), err, 512)
        if not h:
            raise RsimError(RSIM_EARG, "case file: " + err.value.decode())
        return cls(0, lib=L, _handle=h)

    @classmethod
    def from_file(cls, path: str, lib=None) -> "Case":
        with open(path) as f:
            return cls.from_text(f.read(), lib=lib)

    def connections(self):
        """(i, j, Υ) of every connection with Υ > 0, i < j (Cartesian faces, then NNCs)."""
        k = int(self._L.rsim_case_connections(self._h, None, None, None, 0))
        i, j, t = np.zeros(k, np.int32), np.zeros(k, np.int32), np.zeros(k)
        self._L.rsim_case_connections(self._h, A.ptr(i, C.c_int32), A.ptr(j, C.c_int32), A.ptr(t, C.c_double), k)
        return i, j, t

    def well_rates(self, states: "CellStates") -> np.ndarray:
        """Surface production rates (water, oil, gas) in m^3/s at `states`."""
        q = np.zeros(3)
        _check(A.lib().rsim_well_rates(self._h, A.ptr(states.u, C.c_double), A.ptr(states.status, C.c_uint8),
                                       A.ptr(q, C.c_double)), "well_rates")
        return q

    def __del__(self):
        if getattr(self, "_h", None):
            self._L.rsim_case_destroy(self._h)
            self._h = None

    # borrowed arrays (copies, so they outlive nothing)
    def _arr(self, p, n, dt):
        if not p:
            return None
        return np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True)

    @property
    def tx(self): return self._arr(self.graph.tx, self.n, np.float64)
    @property
    def ty(self): return self._arr(self.graph.ty, self.n, np.float64)
    @property
    def tz(self): return self._arr(self.graph.tz, self.n, np.float64)
    @property
    def pv(self): return self._arr(self.graph.pv, self.n, np.float64)
    @property
    def kind(self): return self._arr(self.graph.kind, self.n, np.uint8)
    @property
    def well_wi(self): return self._arr(self.graph.well_wi, self.n, np.float64)

    def nnc(self):
        if not self.graph.nnc_ptr:
            return None
        ptr_ = self._arr(self.graph.nnc_ptr, self.n + 1, np.int32)
        m = int(ptr_[-1])
        return ptr_, self._arr(self.graph.nnc_nbr, m, np.int32), self._arr(self.graph.nnc_t, m, np.float64)

    def perm(self, axis: int) -> np.ndarray:
        return self._arr(self._L.rsim_case_perm(self._h, axis), self.n, np.float64)

    def pinned(self) -> np.ndarray:
        return (self.kind == 1) | (self.well_wi > 0)

    def init_state(self) -> CellStates:
        u = np.zeros(self.n * self.b, np.float64)
        st = np.zeros(self.n, np.uint8)
        self._L.rsim_case_init_state(self._h, A.ptr(u, C.c_double), A.ptr(st, C.c_uint8))
        return CellStates(u, st)

    def schedule(self) -> np.ndarray:
        buf = np.zeros(4096, np.float64)
        k = self._L.rsim_case_schedule(self._h, A.ptr(buf, C.c_double), 4096)
        return buf[:k].copy()

    def solver_opts(self, **kw) -> SolverOpts:
        o = SolverOpts()
        self._L.rsim_case_solver_opts(self._h, C.byref(o))
        for k, v in kw.items():
            setattr(o, k, v)
        return o

    def c5_field(self, target: float, m: int = 2, eps: float = 1e-3):
        dp = np.zeros(self.n, np.float64)
        R = C.c_double(0.0)
        f = self._L.rsim_case_c5_field(self._h, target, m, eps, A.ptr(dp, C.c_double), C.byref(R))
        return dp, float(f), float(R.value)


class GpuSimulator:
    """One B200 context bound to a graph + fluid (the SPEC's implicit context)."""

    def __init__(self, case: Case | None = None, graph: GraphDesc | None = None, fluid: FluidParams | None = None):
        self.L = A.lib()
        self.case = case
        g = graph if graph is not None else case.graph
        f = fluid if fluid is not None else case.fluid
        self.b = int(f.kind)
        self.n = int(g.nx) * int(g.ny) * int(g.nz)
        self._ctx = C.c_void_p()
        _check(self.L.rsim_gpu_create(C.byref(self._ctx), C.byref(g), C.byref(f)), "rsim_gpu_create")

    def close(self):
        if getattr(self, "_ctx", None) and self._ctx.value:
            self.L.rsim_gpu_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- SPEC solver entry points ---------------------------------------
    def newton_standard(self, states: CellStates, dt: float, opts: SolverOpts):
        s = states.copy()
        rep = NewtonReport()
        rc = self.L.rsim_newton_standard(self._ctx, A.ptr(s.u, C.c_double), A.ptr(s.status, C.c_uint8), dt,
                                         C.byref(opts), C.byref(rep))
        if rc in (RSIM_ECUDA, RSIM_EARG):
            _check(rc, "newton_standard")
        return s, rep

    def newton_localized(self, states: CellStates, dt: float, va_init: np.ndarray, m: int, eps: float,
                         opts: SolverOpts):
        s = states.copy()
        va = np.ascontiguousarray(va_init, np.int32)
        rep = NewtonReport()
        rc = self.L.rsim_newton_localized(self._ctx, A.ptr(s.u, C.c_double), A.ptr(s.status, C.c_uint8), dt,
                                          A.ptr(va, C.c_int32), len(va), m, eps, C.byref(opts), C.byref(rep))
        if rc in (RSIM_ECUDA, RSIM_EARG):
            _check(rc, "newton_localized")
        return s, rep

    def adaptive_nonlinear_dd(self, states: CellStates, dt: float, va_init: np.ndarray, m: int, eps: float,
                              opts: SolverOpts):
        s = states.copy()
        va = np.ascontiguousarray(va_init, np.int32)
        rep = NewtonReport()
        rc = self.L.rsim_adaptive_nonlinear_dd(self._ctx, A.ptr(s.u, C.c_double), A.ptr(s.status, C.c_uint8),
                                               dt, A.ptr(va, C.c_int32), len(va), m, eps, C.byref(opts),
                                               C.byref(rep))
        if rc in (RSIM_ECUDA, RSIM_EARG):
            _check(rc, "adaptive_nonlinear_dd")
        return s, rep

    def run_case(self, solver: int, states: CellStates, dts: np.ndarray, opts: SolverOpts) -> dict:
        s = states.copy()
        d = np.ascontiguousarray(dts, np.float64)
        it, lin, cuts = C.c_int32(), C.c_int32(), C.c_int32()
        ma = C.c_double()
        na = C.c_int64()
        rc = self.L.rsim_run_case(self._ctx, solver, A.ptr(s.u, C.c_double), A.ptr(s.status, C.c_uint8),
                                  A.ptr(d, C.c_double), len(d), C.byref(opts), C.byref(it), C.byref(ma),
                                  C.byref(na), C.byref(lin), C.byref(cuts))
        if rc in (RSIM_ECUDA, RSIM_EARG):
            _check(rc, "run_case")
        return {"status": rc, "states": s, "iterations": it.value, "total_ma": ma.value, "sum_na": na.value,
                "lin_iters": lin.value, "cuts": cuts.value}

    # ---- kernel-level hooks (tests, bench) -------------------------------
    def set_state(self, states: CellStates, dt: float):
        _check(self.L.rsim_gpu_set_state(self._ctx, A.ptr(states.u, C.c_double), A.ptr(states.status, C.c_uint8),
                                         dt), "set_state")

    def get_state(self) -> CellStates:
        s = CellStates(np.zeros(self.n * self.b), np.zeros(self.n, np.uint8))
        _check(self.L.rsim_gpu_get_state(self._ctx, A.ptr(s.u, C.c_double), A.ptr(s.status, C.c_uint8)),
               "get_state")
        return s

    def set_active(self, sorted_cells: np.ndarray | None) -> GpuStats:
        st = GpuStats()
        if sorted_cells is None:
            _check(self.L.rsim_gpu_set_active(self._ctx, None, -1, C.byref(st)), "set_active")
        else:
            a = np.ascontiguousarray(sorted_cells, np.int32)
            _check(self.L.rsim_gpu_set_active(self._ctx, A.ptr(a, C.c_int32), len(a), C.byref(st)), "set_active")
        return st

    def initial_active(self, first: bool, eps: float, m: int) -> GpuStats:
        st = GpuStats()
        _check(self.L.rsim_gpu_initial_active(self._ctx, int(first), eps, m, C.byref(st)), "initial_active")
        return st

    def assemble(self):
        _check(self.L.rsim_gpu_assemble(self._ctx), "assemble")

    def linear_solve(self, opts: SolverOpts):
        _check(self.L.rsim_gpu_linear_solve(self._ctx, C.byref(opts)), "linear_solve")

    def update(self, eps: float):
        _check(self.L.rsim_gpu_update(self._ctx, eps), "update")

    def threshold(self, eps: float):
        _check(self.L.rsim_gpu_threshold(self._ctx, eps), "threshold")

    def estimate_active(self, eps: float, m: int, shrink_locked: bool = False) -> GpuStats:
        st = GpuStats()
        _check(self.L.rsim_gpu_estimate_active(self._ctx, eps, m, int(shrink_locked), C.byref(st)),
               "estimate_active")
        return st

    def stats(self) -> GpuStats:
        st = GpuStats()
        _check(self.L.rsim_gpu_stats_get(self._ctx, C.byref(st)), "stats")
        return st

    def active(self) -> np.ndarray:
        n = C.c_int32()
        self.L.rsim_gpu_download_active(self._ctx, None, C.byref(n))
        a = np.zeros(max(n.value, 1), np.int32)
        _check(self.L.rsim_gpu_download_active(self._ctx, A.ptr(a, C.c_int32), C.byref(n)), "download_active")
        return a[: n.value]

    def boundary(self) -> np.ndarray:
        a = np.zeros(self.n, np.int32)
        n = C.c_int32()
        _check(self.L.rsim_gpu_download_boundary(self._ctx, A.ptr(a, C.c_int32), C.byref(n)), "download_boundary")
        return a[: n.value].copy()

    def categories(self) -> np.ndarray:
        a = np.zeros(self.n, np.uint8)
        _check(self.L.rsim_gpu_download_flags(self._ctx, A.ptr(a, C.c_uint8)), "download_flags")
        return a

    def labels(self) -> np.ndarray:
        a = np.zeros(self.n, np.int32)
        _check(self.L.rsim_gpu_download_labels(self._ctx, A.ptr(a, C.c_int32)), "download_labels")
        return a

    def upload_dp(self, dp: np.ndarray):
        d = np.ascontiguousarray(dp, np.float64)
        _check(self.L.rsim_gpu_upload_dp(self._ctx, A.ptr(d, C.c_double)), "upload_dp")

    def dp(self) -> np.ndarray:
        d = np.zeros(self.n, np.float64)
        _check(self.L.rsim_gpu_download_dp(self._ctx, A.ptr(d, C.c_double)), "download_dp")
        return d

    def solution(self, nA: int) -> np.ndarray:
        x = np.zeros(max(nA * self.b, 1), np.float64)
        _check(self.L.rsim_gpu_download_solution(self._ctx, A.ptr(x, C.c_double)), "download_solution")
        return x[: nA * self.b]

    def system(self, nA: int):
        """Last assembled system: (F_raw, rhs, rowptr, col, val) in canonical CSR order."""
        b = self.b
        F = np.zeros(nA * b)
        rhs = np.zeros(nA * b)
        rp = np.zeros(nA + 1, np.int32)
        nnz = self.L.rsim_gpu_download_system(self._ctx, None, None, None, None, None, 0)
        col = np.zeros(max(nnz, 1), np.int32)
        val = np.zeros(max(nnz, 1) * b * b)
        nnz2 = self.L.rsim_gpu_download_system(self._ctx, A.ptr(F, C.c_double), A.ptr(rhs, C.c_double),
                                               A.ptr(rp, C.c_int32), A.ptr(col, C.c_int32),
                                               A.ptr(val, C.c_double), nnz)
        if nnz2 < 0:
            raise RsimError(RSIM_ECUDA, "download_system")
        return F, rhs, rp, col[:nnz], val[: nnz * b * b]

    def timers(self, enable: int = -1):
        ms = np.zeros(4)
        n = C.c_int32()
        _check(self.L.rsim_gpu_timers(self._ctx, enable, A.ptr(ms, C.c_double), C.byref(n)), "timers")
        return ms, n.value

    # DD hooks
    def dd_partition(self, n_sub: int) -> np.ndarray:
        sizes = np.zeros(n_sub, np.int32)
        _check(self.L.rsim_gpu_dd_partition(self._ctx, n_sub, A.ptr(sizes, C.c_int32)), "dd_partition")
        return sizes


def device_info() -> dict:
    name = C.create_string_buffer(256)
    sm, ma, mi = C.c_int32(), C.c_int32(), C.c_int32()
    _check(A.lib().rsim_gpu_device_info(name, 256, C.byref(sm), C.byref(ma), C.byref(mi)), "device_info")
    return {"name": name.value.decode(), "sm_count": sm.value, "cc": (ma.value, mi.value)}


SOLVERS = {"standard": 0, "localized": 1, "adaptive_dd": 2}


def simulate(config: int, solver: str = "localized", out_dir: str | None = None, *, nx: int = 0, ny: int = 0,
             nz: int = 0, seed: int = 0, n_dfn: int = -1, m: int = 0, eps_p: float = 0.0, n_steps: int = 0,
             precond: int = -1, report_every_days: float = 0.0, write_fields: bool = True,
             lin_method: int = -1, trace_flags: bool = False) -> dict:
    """Case runner (SPEC.md sim_driver_cli run_case, include/rsim/simulate.h): run a seeded
    config on the GPU with the named solver; writes rates.csv / metrics.csv / summary.txt
    (+ field dumps) into out_dir when given.  eps_p in Pa (0 -> case default)."""
    co = A.CaseOpts(config, nx, ny, nz, seed, n_dfn, -1)
    so = A.SimOpts(SOLVERS[solver], m, eps_p, n_steps, precond, report_every_days, int(write_fields), lin_method,
                   int(trace_flags))
    mt = A.RunMetrics()
    rc = A.lib().rsim_simulate(C.byref(co), C.byref(so), (out_dir or "").encode(), C.byref(mt))
    _check(rc, "simulate")
    return {f: getattr(mt, f) for f, _ in A.RunMetrics._fields_ if f != "pad"}


def simulate_file(case_file: str, solver: str | None = None, out_dir: str | None = None, *, m: int = 0,
                  eps_p: float = 0.0, n_steps: int = 0, precond: int = -1, report_every_days: float = 0.0,
                  write_fields: bool = True, lin_method: int = -1, trace_flags: bool = False) -> dict:
    """Case runner on a case file (SPEC.md sim_driver_cli `simulate <case-file>`): EDFM
    fractures, the file's schedule and [solver] defaults (solver None -> the file's)."""
    so = A.SimOpts(SOLVERS[solver] if solver else -1, m, eps_p, n_steps, precond, report_every_days,
                   int(write_fields), lin_method, int(trace_flags))
    mt = A.RunMetrics()
    rc = A.lib().rsim_simulate_file(case_file.encode(), C.byref(so), (out_dir or "").encode(), C.byref(mt))
    _check(rc, "simulate_file")
    return {f: getattr(mt, f) for f, _ in A.RunMetrics._fields_ if f != "pad"}


def eos_case3() -> A.EosParams:
    """Paper Case 3 fluid: C1 / C10 Peng-Robinson components (include/rsim/eos.h)."""
    e = A.EosParams()
    _check(A.lib().rsim_eos_case3(C.byref(e)), "eos_case3")
    return e


def eos_flash(e: A.EosParams, T: float, p: np.ndarray, z: np.ndarray) -> dict:
    """Peng-Robinson flash of every cell on the GPU: two-sided
    Michelsen stability test, then successive substitution.  p[n] in Pa,
    z[n, nc] overall mole fractions.  Returns status (RSIM_PH_*: 0 oil, 1 gas,
    2 two-phase), nu_g, x, y ([n*nc]), zfac ([2n]: Z_o, Z_g), iters."""
    n, nc = len(p), e.nc
    p = np.ascontiguousarray(p, np.float64)
    z = np.ascontiguousarray(z, np.float64).reshape(n * nc)
    out = dict(status=np.zeros(n, np.uint8), nu_g=np.zeros(n), x=np.zeros(n * nc), y=np.zeros(n * nc),
               zfac=np.zeros(2 * n), iters=np.zeros(n, np.int32))
    _check(A.lib().rsim_eos_flash(C.byref(e), T, n, A.ptr(p, C.c_double), A.ptr(z, C.c_double),
                                  A.ptr(out["status"], C.c_uint8), A.ptr(out["nu_g"], C.c_double),
                                  A.ptr(out["x"], C.c_double), A.ptr(out["y"], C.c_double),
                                  A.ptr(out["zfac"], C.c_double), A.ptr(out["iters"], C.c_int32)), "eos_flash")
    return out
