/*
 * rsim/types.h — plain-C data descriptors shared by the GPU C-ABI
 * (include/rsim/gpu_abi.h), the host solver API (include/rsim/simulator.hpp)
 * and the CPU oracle's C API (oracle/oracle_api.h).
 *
 * Everything here is POD: plain pointers + sizes, no torch/STL types.
 *
 * Reference anchors (/root/reference):
 *   ConnectivityGraph  SPEC.md:37-40   (cells, connections with Υ, volumes, kind)
 *   CellState          SPEC.md:107-110 (natural variables + status tag)
 *   WellSpec           SPEC.md:236-239 (bhp, connected cells, WI per connection)
 *   NewtonReport       SPEC.md:353-356 (iterations, per-iteration n_A, ‖δp‖∞)
 *   LinearSolveReport
 */
#ifndef RSIM_TYPES_H
#define RSIM_TYPES_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Fluid model == block size b (unknowns per cell). */
enum {
  RSIM_FLUID_SINGLE   = 1, /* slightly compressible single phase, u = (p)            */
  RSIM_FLUID_OILWATER = 2, /* oil-water, mobile water, Corey n=2, u = (p, S_w)       */
  RSIM_FLUID_BLACKOIL = 3  /* water/oil/gas black-oil, u = (p, S_w, X), X = S_g|R_s */
};

/* Black-oil phase status (variable-substitution tag, SPEC.md:103-106 adapted). */
enum { RSIM_BO_UNDERSAT = 0, RSIM_BO_SAT = 1 };

/* Cell kind (SPEC.md:38 cell_kind). Fracture cells are always active. */
enum { RSIM_KIND_MATRIX = 0, RSIM_KIND_FRACTURE = 1, RSIM_KIND_DEAD = 2 };  /* DEAD: EDFM fracture-plane filler (no connections, never active) */

/* Linear solver selectors. */
enum { RSIM_LIN_BICGSTAB = 0, RSIM_LIN_GMRES = 1, RSIM_LIN_DIRECT = 2 };
/* Exact (direct) solve of small active systems:
 * dense LU with partial pivoting, n_A*b unknowns at most. */
#define RSIM_DIRECT_MAX 4096
#define RSIM_GMRES_M 30 /* GMRES restart length (SPEC-free choice: GMRES(30)) */
enum { RSIM_PREC_BJACOBI = 0, RSIM_PREC_ILU0 = 1, RSIM_PREC_NEUMANN1 = 2 };

/* Return codes of every C-ABI call. */
enum {
  RSIM_OK = 0,
  RSIM_EARG = 1,        /* bad argument                                        */
  RSIM_ECUDA = 2,       /* CUDA error                                          */
  RSIM_ENUM = 3,        /* numerical failure: Krylov breakdown / singular block */
  RSIM_ENOCONV = 4      /* not converged (iteration cap → timestep cut)        */
};

typedef struct {
  int32_t kind;        /* RSIM_FLUID_*                                          */
  double p_ref;        /* Pa, reference pressure for densities and porosity      */
  double c_r;          /* rock compressibility 1/Pa: φ = φ_ref (1 + c_r (p-p_ref)) */
  /* phase index 0 = water, 1 = oil, 2 = gas.  Single-phase uses index 1 (oil). */
  double rho_ref[3];   /* kg/m^3 at p_ref (single, oil-water)                    */
  double c_f[3];       /* fluid compressibility 1/Pa                             */
  double mu[3];        /* Pa s                                                   */
  double swc, sor, sgc;/* residual saturations (Corey, exponent 2)               */
  /* black-oil PVT (model defined by this repo) */
  double p_bub;        /* Pa, bubble point of the initial oil                    */
  double rs_b;         /* sm3/sm3, Rs at p_bub;  Rs_sat(p) = rs_b * p / p_bub     */
  double bo_alpha;     /* 1/(sm3/sm3): b_o = exp(c_o (p-p_ref)) / (1 + alpha Rs) */
  double p_gas;        /* Pa: b_g = p / p_gas                                     */
  /* Newton update limiter (Appleyard chop per cell, DESIGN.md §5 item 11); 0 = off.
   * The cell's update δu is scaled by w = min(1, dp_max_rel·|p|/|δp|, ds_max/max|δS|). */
  double dp_max_rel;   /* max |δp| per iteration relative to the cell pressure   */
  double ds_max;       /* max |δS_w|, |δS_g| per iteration                       */
} rsim_fluid_params;

/* The immutable connection graph, Cartesian part as face
 * arrays + optional symmetric NNC CSR.  Cell i = (iz*ny + iy)*nx + ix. */
typedef struct {
  int32_t nx, ny, nz;
  const double* tx;      /* [n] Υ between i and i+1      (0 on the +x boundary) */
  const double* ty;      /* [n] Υ between i and i+nx     (0 on the +y boundary) */
  const double* tz;      /* [n] Υ between i and i+nx*ny  (0 on the +z boundary) */
  const double* pv;      /* [n] pore volume at p_ref, V * φ_ref (m^3)           */
  const uint8_t* kind;   /* [n] RSIM_KIND_*                                     */
  const int32_t* nnc_ptr;/* [n+1] or NULL: symmetric NNC CSR, rows sorted       */
  const int32_t* nnc_nbr;/* [nnc_ptr[n]] neighbour cell, ascending per row      */
  const double*  nnc_t;  /* [nnc_ptr[n]] Υ                                      */
  const double* well_wi; /* [n] well index (m^3) of a perforation, 0 elsewhere  */
  double bhp;            /* Pa, producer bottom-hole pressure      */
} rsim_graph_desc;

/* One Newton iteration record (SPEC.md:353-356 extended per SURVEY §5). */
typedef struct {
  int32_t n_active;      /* n_A: cells assembled/solved this iteration          */
  int32_t lin_iters;     /* Krylov iterations                                   */
  int32_t subdomain;     /* DD: subdomain id (-1: expansion / Newton iteration)  */
  int32_t mode_expand;   /* localized: 1 = expand, 0 = shrink after this iter   */
  double  dp_inf_A;      /* ‖δp‖∞ over V_A                                      */
  double  dp_inf_B;      /* ‖δp‖∞ over V_B (boundary layer)                     */
  double  f_norm2;       /* ‖F_A‖₂ (raw residual, before the update)            */
  double  f_norminf;     /* ‖F_A‖∞                                              */
  double  lin_res;       /* final scaled ‖r‖₂ / ‖b‖₂                            */
} rsim_iter_record;

#define RSIM_MAX_ITER_RECORDS 4096

typedef struct {
  int32_t iterations;    /* Newton iterations (DD: inner iterations = local solves) */
  int32_t outer_iterations; /* DD: Phase-2 sweeps (0 otherwise)                   */
  int32_t n_subdomains;  /* DD: N                                                */
  int32_t converged;     /* 1 on success                                         */
  int32_t status;        /* RSIM_* code of the failing step (0 on success)       */
  int32_t lin_iters_total;
  double  sum_na_over_n; /* Σ n_A / n  (M_A of this timestep)   */
  int64_t sum_na;        /* Σ n_A                                                */
  int32_t n_records;
  rsim_iter_record rec[RSIM_MAX_ITER_RECORDS];
} rsim_newton_report;

/* Solver settings shared by the GPU host solvers and the oracle. */
typedef struct {
  int32_t max_newton;    /* iteration cap (default 25)              */
  int32_t max_outer;     /* DD outer cap (default 50)               */
  int32_t lin_method;    /* RSIM_LIN_*                                           */
  int32_t precond;       /* RSIM_PREC_*                                          */
  int32_t lin_maxit;     /* Krylov iteration cap                                 */
  double  lin_rtol;      /* on ‖r̂‖₂/‖b̂‖₂ of the block-Jacobi-scaled system        */
  double  eps_p;         /* Newton tolerance on ‖δp‖∞              */
  double  eps_set;       /* active-set cutoff ε (= eps_p by default) */
  int32_t m;             /* neighbour layers for expansion          */
  int32_t fixed_lin_iters; /* >0: run exactly this many Krylov iterations (c5)   */
} rsim_solver_opts;

#ifdef __cplusplus
}
#endif
#endif /* RSIM_TYPES_H */
