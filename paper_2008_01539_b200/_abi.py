"""ctypes mirror of include/rsim/{types,gpu_abi,cases}.h.

Plain C structs and function prototypes only; the Python API built on top is
in paper_2008_01539_b200/__init__.py.  The library is the in-tree
lib/librsim.so (built by build.py for sm_100a); there is no Python or CPU
fallback for any kernel.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("RSIM_LIB") or (Path(__file__).resolve().parent / "lib" / "librsim.so"))  # RSIM_LIB: A/B experiments only

RSIM_OK, RSIM_EARG, RSIM_ECUDA, RSIM_ENUM, RSIM_ENOCONV = 0, 1, 2, 3, 4
FLUID_SINGLE, FLUID_OILWATER, FLUID_BLACKOIL = 1, 2, 3
LIN_BICGSTAB, LIN_GMRES, LIN_DIRECT = 0, 1, 2
DIRECT_MAX = 4096  # RSIM_DIRECT_MAX (include/rsim/types.h)
PREC_BJACOBI, PREC_ILU0, PREC_NEUMANN1 = 0, 1, 2
MAX_ITER_RECORDS = 4096

dptr = C.POINTER(C.c_double)
i32ptr = C.POINTER(C.c_int32)
u8ptr = C.POINTER(C.c_uint8)
i64ptr = C.POINTER(C.c_int64)


class FluidParams(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("p_ref", C.c_double), ("c_r", C.c_double),
        ("rho_ref", C.c_double * 3), ("c_f", C.c_double * 3), ("mu", C.c_double * 3),
        ("swc", C.c_double), ("sor", C.c_double), ("sgc", C.c_double),
        ("p_bub", C.c_double), ("rs_b", C.c_double), ("bo_alpha", C.c_double), ("p_gas", C.c_double),
        ("dp_max_rel", C.c_double), ("ds_max", C.c_double),
    ]


class GraphDesc(C.Structure):
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
        ("tx", dptr), ("ty", dptr), ("tz", dptr), ("pv", dptr), ("kind", u8ptr),
        ("nnc_ptr", i32ptr), ("nnc_nbr", i32ptr), ("nnc_t", dptr),
        ("well_wi", dptr), ("bhp", C.c_double),
    ]


class IterRecord(C.Structure):
    _fields_ = [
        ("n_active", C.c_int32), ("lin_iters", C.c_int32), ("subdomain", C.c_int32), ("mode_expand", C.c_int32),
        ("dp_inf_A", C.c_double), ("dp_inf_B", C.c_double), ("f_norm2", C.c_double),
        ("f_norminf", C.c_double), ("lin_res", C.c_double),
    ]


class NewtonReport(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32), ("outer_iterations", C.c_int32), ("n_subdomains", C.c_int32),
        ("converged", C.c_int32), ("status", C.c_int32), ("lin_iters_total", C.c_int32),
        ("sum_na_over_n", C.c_double), ("sum_na", C.c_int64), ("n_records", C.c_int32),
        ("rec", IterRecord * MAX_ITER_RECORDS),
    ]

    def records(self) -> list[dict]:
        out = []
        for k in range(self.n_records):
            r = self.rec[k]
            out.append({f: getattr(r, f) for f, _ in IterRecord._fields_})
        return out


class SolverOpts(C.Structure):
    _fields_ = [
        ("max_newton", C.c_int32), ("max_outer", C.c_int32), ("lin_method", C.c_int32), ("precond", C.c_int32),
        ("lin_maxit", C.c_int32), ("lin_rtol", C.c_double), ("eps_p", C.c_double), ("eps_set", C.c_double),
        ("m", C.c_int32), ("fixed_lin_iters", C.c_int32),
    ]


class GpuStats(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("bad_cell", C.c_int32), ("lin_iters", C.c_int32), ("n_active", C.c_int32),
        ("n_boundary", C.c_int32), ("expand", C.c_int32), ("n_new", C.c_int32), ("pad", C.c_int32),
        ("lin_relres", C.c_double), ("f_norm2", C.c_double), ("f_norminf", C.c_double),
        ("dp_inf_A", C.c_double), ("dp_inf_B", C.c_double), ("halo_max", C.c_double),
    ]


class CaseOpts(C.Structure):
    _fields_ = [
        ("config", C.c_int32), ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32),
        ("seed", C.c_uint64), ("n_dfn", C.c_int32), ("n_steps", C.c_int32),
    ]


class SimOpts(C.Structure):
    _fields_ = [
        ("solver", C.c_int32), ("m", C.c_int32), ("eps_p", C.c_double), ("n_steps", C.c_int32),
        ("precond", C.c_int32), ("report_every_days", C.c_double), ("write_fields", C.c_int32),
        ("lin_method", C.c_int32), ("trace_flags", C.c_int32),
    ]


class CaseInfo(C.Structure):
    _fields_ = [
        ("n_live", C.c_int64), ("n_frac", C.c_int64), ("n_dead", C.c_int64), ("solver", C.c_int32),
        ("m", C.c_int32), ("eps_p", C.c_double), ("total_time", C.c_double),
    ]


class RunMetrics(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("timesteps", C.c_int32), ("total_iters", C.c_int32), ("total_lin", C.c_int32),
        ("cuts", C.c_int32), ("pad", C.c_int32), ("sum_na", C.c_int64), ("total_ma", C.c_double),
        ("avg_ma", C.c_double), ("sim_days", C.c_double), ("cum_oil_m3", C.c_double),
        ("cum_water_m3", C.c_double), ("cum_gas_m3", C.c_double), ("wall_s", C.c_double),
        ("total_outer", C.c_int64),
    ]


EOS_NCMAX = 4


class EosParams(C.Structure):
    _fields_ = [
        ("nc", C.c_int32), ("tc", C.c_double * EOS_NCMAX), ("pc", C.c_double * EOS_NCMAX),
        ("omega", C.c_double * EOS_NCMAX), ("mw", C.c_double * EOS_NCMAX),
        ("kij", (C.c_double * EOS_NCMAX) * EOS_NCMAX), ("flash_tol", C.c_double), ("flash_maxit", C.c_int32),
        ("stab_maxit", C.c_int32),
    ]


# name -> (restype, argtypes); every symbol declared in include/rsim/*.h
P = C.c_void_p
PROTOS: dict[str, tuple] = {
    # cases.h
    "rsim_case_create": (P, [C.POINTER(CaseOpts)]),
    "rsim_case_destroy": (None, [P]),
    "rsim_case_n": (C.c_int64, [P]),
    "rsim_case_dims": (C.c_int, [P, i32ptr, dptr]),
    "rsim_case_graph": (C.c_int, [P, C.POINTER(GraphDesc)]),
    "rsim_case_fluid": (C.c_int, [P, C.POINTER(FluidParams)]),
    "rsim_case_perm": (dptr, [P, C.c_int32]),
    "rsim_case_init_state": (C.c_int, [P, dptr, u8ptr]),
    "rsim_case_schedule": (C.c_int32, [P, dptr, C.c_int32]),
    "rsim_case_solver_opts": (C.c_int, [P, C.POINTER(SolverOpts)]),
    "rsim_case_n_nnc": (C.c_int64, [P]),
    "rsim_case_from_text": (P, [C.c_char_p, C.c_char_p, C.c_int32]),
    "rsim_case_from_file": (P, [C.c_char_p, C.c_char_p, C.c_int32]),
    "rsim_case_info": (C.c_int, [P, C.POINTER(CaseInfo)]),
    "rsim_case_connections": (C.c_int64, [P, i32ptr, i32ptr, dptr, C.c_int64]),
    "rsim_edfm_avg_distance": (C.c_double, [C.c_double] * 8),
    # simulate.h (case runner, SPEC.md sim_driver_cli)
    "rsim_well_rates": (C.c_int, [P, dptr, u8ptr, dptr]),
    "rsim_simulate": (C.c_int, [C.POINTER(CaseOpts), C.POINTER(SimOpts), C.c_char_p, C.POINTER(RunMetrics)]),
    "rsim_simulate_file": (C.c_int, [C.c_char_p, C.POINTER(SimOpts), C.c_char_p, C.POINTER(RunMetrics)]),
    # eos.h (Peng-Robinson flash)
    "rsim_eos_case3": (C.c_int, [C.POINTER(EosParams)]),
    "rsim_eos_flash": (C.c_int, [C.POINTER(EosParams), C.c_double, C.c_int64, dptr, dptr, u8ptr, dptr, dptr, dptr,
                                 dptr, i32ptr]),
    "rsim_eos_flash_dev": (C.c_int, [C.POINTER(EosParams), C.c_double, C.c_int64, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p]),
    "rsim_case_c5_field": (C.c_double, [P, C.c_double, C.c_int32, C.c_double, dptr, dptr]),
    # gpu_abi.h
    "rsim_gpu_set_device": (C.c_int, [C.c_int32]),
    "rsim_gpu_counters": (C.c_int, [P, i64ptr, C.c_int32]),
    "rsim_gpu_block_counters": (C.c_int, [P, i64ptr, C.c_int32]),
    "rsim_gpu_create": (C.c_int, [C.POINTER(P), C.POINTER(GraphDesc), C.POINTER(FluidParams)]),
    "rsim_gpu_destroy": (C.c_int, [P]),
    "rsim_gpu_last_error": (C.c_char_p, []),
    "rsim_gpu_device_info": (C.c_int, [C.c_char_p, C.c_int32, i32ptr, i32ptr, i32ptr]),
    "rsim_gpu_set_state": (C.c_int, [P, dptr, u8ptr, C.c_double]),
    "rsim_gpu_set_dt": (C.c_int, [P, C.c_double]),
    "rsim_gpu_get_state": (C.c_int, [P, dptr, u8ptr]),
    "rsim_gpu_restore_state": (C.c_int, [P]),
    "rsim_gpu_set_active": (C.c_int, [P, i32ptr, C.c_int32, C.POINTER(GpuStats)]),
    "rsim_gpu_initial_active": (C.c_int, [P, C.c_int32, C.c_double, C.c_int32, C.POINTER(GpuStats)]),
    "rsim_gpu_estimate_active": (C.c_int, [P, C.c_double, C.c_int32, C.c_int32, C.POINTER(GpuStats)]),
    "rsim_gpu_assemble": (C.c_int, [P]),
    "rsim_gpu_linear_solve": (C.c_int, [P, C.POINTER(SolverOpts)]),
    "rsim_gpu_update": (C.c_int, [P, C.c_double]),
    "rsim_gpu_stats_get": (C.c_int, [P, C.POINTER(GpuStats)]),
    "rsim_gpu_dd_expand": (C.c_int, [P, C.c_double, C.c_int32, C.c_int32, C.POINTER(GpuStats)]),
    "rsim_gpu_dd_partition": (C.c_int, [P, C.c_int32, i32ptr]),
    "rsim_gpu_dd_select": (C.c_int, [P, C.c_int32, C.POINTER(GpuStats)]),
    "rsim_gpu_dd_skip": (C.c_int, [P, C.c_int32]),
    "rsim_gpu_download_labels": (C.c_int, [P, i32ptr]),
    "rsim_gpu_download_active": (C.c_int, [P, i32ptr, i32ptr]),
    "rsim_gpu_download_flags": (C.c_int, [P, u8ptr]),
    "rsim_gpu_download_boundary": (C.c_int, [P, i32ptr, i32ptr]),
    "rsim_gpu_download_system": (C.c_int64, [P, dptr, dptr, i32ptr, i32ptr, dptr, C.c_int64]),
    "rsim_gpu_download_solution": (C.c_int, [P, dptr]),
    "rsim_gpu_upload_dp": (C.c_int, [P, dptr]),
    "rsim_gpu_threshold": (C.c_int, [P, C.c_double]),
    "rsim_gpu_download_dp": (C.c_int, [P, dptr]),
    "rsim_gpu_timers": (C.c_int, [P, C.c_int32, dptr, i32ptr]),
    "rsim_gpu_mark": (C.c_int, [P, C.c_int32]),
    "rsim_gpu_ktrace": (C.c_int, [P, C.POINTER(C.c_ulonglong)]),
    "rsim_gpu_set_debug": (C.c_int, [P, C.c_int32]),
    "rsim_gpu_elapsed": (C.c_int, [P, C.c_int32, C.c_int32, dptr]),
    "rsim_gpu_flush_l2": (C.c_int, [P]),
    "rsim_gpu_checkpoint": (C.c_int, [P, C.c_int32]),
    "rsim_gpu_support_active": (C.c_int, [P, C.c_double, C.c_int32, C.POINTER(GpuStats)]),
    "rsim_gpu_state_from_dp": (C.c_int, [P, C.c_double, C.c_double]),
    "rsim_run_case_dev": (C.c_int, [P, C.c_int32, dptr, C.c_int32, C.POINTER(SolverOpts), i32ptr, dptr, i64ptr,
                                    i32ptr, i32ptr]),
    "rsim_newton_standard": (C.c_int, [P, dptr, u8ptr, C.c_double, C.POINTER(SolverOpts), C.POINTER(NewtonReport)]),
    "rsim_newton_localized": (C.c_int, [P, dptr, u8ptr, C.c_double, i32ptr, C.c_int32, C.c_int32, C.c_double,
                                        C.POINTER(SolverOpts), C.POINTER(NewtonReport)]),
    "rsim_adaptive_nonlinear_dd": (C.c_int, [P, dptr, u8ptr, C.c_double, i32ptr, C.c_int32, C.c_int32,
                                             C.c_double, C.POINTER(SolverOpts), C.POINTER(NewtonReport)]),
    "rsim_newton_standard_dev": (C.c_int, [P, C.POINTER(SolverOpts), C.POINTER(NewtonReport)]),
    "rsim_newton_localized_dev": (C.c_int, [P, C.POINTER(SolverOpts), C.POINTER(NewtonReport)]),
    "rsim_adaptive_nonlinear_dd_dev": (C.c_int, [P, C.POINTER(SolverOpts), C.POINTER(NewtonReport)]),
    "rsim_run_case": (C.c_int, [P, C.c_int32, dptr, u8ptr, dptr, C.c_int32, C.POINTER(SolverOpts), i32ptr,
                                dptr, i64ptr, i32ptr, i32ptr]),
}

_lib = None


def lib() -> C.CDLL:
    """Load lib/librsim.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in PROTOS.items():
            if os.environ.get("RSIM_LIB") and not hasattr(L, name):
                continue  # A/B against an older build: tolerate symbols it predates
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def ptr(a: np.ndarray | None, ct):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ct))
