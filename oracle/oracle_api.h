/*
 * oracle/oracle_api.h — C API of the CPU oracle (TEST INFRASTRUCTURE ONLY).
 *
 * This library is the parity checker for the sm_100a path.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  The product library (paper_2008_01539_b200/lib/librsim.so)
 * never links or calls it.
 *
 * The reference (/root/reference) ships no implementation, so
 * this is a C++ restatement of SPEC.md + PAPER.md Algorithms 1-2; every
 * entry point cites the SPEC operation it restates.  "Parity pinned" only
 * to the SPEC known-answer examples and invariants (tests/test_oracle_*.py);
 * there are no reference golden vectors to pin against.
 */
#ifndef RSIM_ORACLE_API_H
#define RSIM_ORACLE_API_H

#include "rsim/eos.h"
#include <stdint.h>
#include "rsim/types.h"

#ifdef __cplusplus
extern "C" {
#endif

/* TPFA face transmissibilities: Υ = harmonic mean of
 * half-transmissibilities k·A/(d/2) of the two cells. */
int orc_build_matrix_grid(int32_t nx, int32_t ny, int32_t nz, double dx, double dy, double dz,
                          const double* kx, const double* ky, const double* kz,
                          double* tx, double* ty, double* tz);

void* orc_create(const rsim_graph_desc* g, const rsim_fluid_params* f);
void  orc_destroy(void* h);
void  orc_set_threads(int n);      /* OpenMP threads (1 = serial oracle) */
int   orc_threads(void);

int orc_set_state(void* h, const double* u, const uint8_t* st, double dt);
int orc_get_state(void* h, double* u, uint8_t* st);
int orc_set_dt(void* h, double dt);

/* assemble(target_set) over a sorted active list.  Writes
 * the raw residual F (nA*b), the block-Jacobi-scaled rhs = -D^-1 F, and the
 * scaled off-diagonal blocks D^-1 J_ij in canonical order as CSR.
 * Returns nnzb (>=0) or -(RSIM_ENUM) on a singular diagonal block. */
int64_t orc_assemble(void* h, const int32_t* act, int32_t nA, double* F_raw, double* rhs,
                     int32_t* rowptr, int32_t* col, double* val, int64_t cap_nnzb);

/* Solve the system of the last orc_assemble (BiCGSTAB, canonical reductions). */
int orc_linear_solve(void* h, const rsim_solver_opts* o, double* x, int32_t* iters, double* relres);

/* Canonical sum of per-row values (blockops.h). */
double orc_canon_sum(const double* v, int64_t n);

/* Set operations.  Output lists sorted; return count. */
int32_t orc_neighbor_set(void* h, int32_t i, int32_t m, int32_t* out);
int32_t orc_support_set(const double* dp, int32_t n, double eps, int32_t* out);
int32_t orc_boundary_layer(void* h, const int32_t* va, int32_t n, int32_t* out);
int32_t orc_outer_halo(void* h, const int32_t* va, int32_t n, int32_t* out);
/* Algorithm 1 lines 7-18 for one iteration: given V_A, the global δp and the
 * current mode, return the next V_A (sorted) and V_B, and the next mode. */
int32_t orc_estimate_active(void* h, const int32_t* va, int32_t n, const double* dp_global,
                            double eps, int32_t m, int32_t shrink_locked,
                            int32_t* va_out, int32_t* vb_out, int32_t* nb_out, int32_t* expand_out);

/* The three solvers.  State is the handle's current state;
 * on success it holds the new state. */
int orc_newton_standard(void* h, double dt, const rsim_solver_opts* o, rsim_newton_report* rep);
int orc_newton_localized(void* h, double dt, const int32_t* va_init, int32_t n_init,
                         const rsim_solver_opts* o, rsim_newton_report* rep);
int orc_adaptive_dd(void* h, double dt, const int32_t* va_init, int32_t n_init,
                    const rsim_solver_opts* o, rsim_newton_report* rep, int32_t* labels_out);

/* Initial active set of a timestep: step 0 -> pinned cells and
 * their m-halo; later -> {|p - p_prev| >= eps} ∪ pinned.  p_prev may be NULL
 * for step 0.  Returns count. */
int32_t orc_initial_active(void* h, const double* p_prev, double eps, int32_t m, int32_t* out);

/* One full case run (minimal): solver 0 standard,
 * 1 localized, 2 adaptive DD.  dts: schedule; on failure the step is halved.
 * Per-step reports are summarised into the outputs. */
int orc_run_case(void* h, int32_t solver, const double* dts, int32_t nsteps,
                 const rsim_solver_opts* o, int32_t* total_iters, double* total_ma,
                 int64_t* total_na, int32_t* total_lin, int32_t* n_cuts);
int orc_run_steps(void* h, int32_t solver, const double* dts, int32_t nsteps, const rsim_solver_opts* o,
                  double* p_prev_io, int32_t* has_prev, int32_t* total_iters, double* total_ma, int64_t* total_na,
                  int32_t* total_lin, int32_t* n_cuts);

/* Property-suite hooks. */
double orc_rexp(double x);
void orc_corey(double s, double s_r, double den, double* kr, double* dkr);
/* Cell properties for the fluid's b: A[b], dA[b*b], L[b], dL[b*b]. */
int orc_props(const rsim_fluid_params* f, const double* u, uint8_t st, double* A, double* dA, double* L, double* dL);
/* Set the current iterate WITHOUT touching the old-time accumulation. */
int orc_set_u(void* h, const double* u, const uint8_t* st);
/* Unscaled assembly: raw F, raw diagonal blocks (nA*b*b) and raw
 * off-diagonal blocks in canonical CSR order.  Returns nnzb. */
int64_t orc_assemble_raw(void* h, const int32_t* act, int32_t nA, double* F_raw, double* diag,
                         int32_t* rowptr, int32_t* col, double* val, int64_t cap_nnzb);

/* Residual of the current state on the FULL cell set (for mass balance /
 * restriction tests); F_raw has n*b entries. */
int orc_full_residual(void* h, double* F_raw);

/* Peng-Robinson EoS (arithmetic in include/rsim/eos.h). */
double orc_eos_rlog(double x);
int orc_eos_cubic_roots(double A, double B, double* r3);
int orc_eos_phase(const rsim_eos_params* e, double T, double p, const double* x, int32_t sel, int32_t min_g,
                  double* Z, double* lnphi);
int orc_eos_rachford_rice(int32_t nc, const double* z, const double* K, double* nu);
int orc_eos_stability(const rsim_eos_params* e, double T, double p, const double* z, double* K, int32_t* stable);
int orc_eos_flash(const rsim_eos_params* e, double T, int64_t n, const double* p, const double* z, uint8_t* status,
                  double* nu_g, double* x, double* y, double* zfac, int32_t* iters);

#ifdef __cplusplus
}
#endif
#endif
