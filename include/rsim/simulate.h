/*
 * rsim/simulate.h — case runner (SPEC.md:460-531,
 * module sim_driver_cli).  Host C++ in librsim.so over the C-ABI solvers:
 * runs a seeded synthetic case (rsim/cases.h) on the GPU with the selected
 * nonlinear solver and writes the SPEC's output files.
 *
 *   rsim_simulate   ← run_case(cfg) -> RunMetrics + output files
 *   rsim_well_rates ← well_rates(states, wells)
 *
 * Output files in out_dir (SPEC.md "External Interfaces"):
 *   rates.csv    time_days, oil_rate, gas_rate, bhp, water_rate, oil_rate_bbl
 *                (surface m^3/day; bhp in psi; one row per committed timestep)
 *   metrics.csv  step, time_days, dt_days, iterations, sum_nA_over_n, sum_nA,
 *                lin_iters, n_subdomains
 *   iterations.csv  step, attempt, committed, dt_days, iter, n_active,
 *                active_fraction, lin_iters, subdomain, mode_expand, dp_inf_A,
 *                dp_inf_B, f_norm2, f_norminf, lin_relres — one row per Newton
 *                iteration (DD: per local solve) of every attempt, cut ones
 *                included (committed = 0): the per-iteration active fraction
 *   summary.txt  Tables-2..6-style totals (timesteps, total iterations,
 *                total M_A, average M_A per iteration, cuts, cumulative oil)
 *   pressure_t<days>.txt / satwater_t / satgas_t / phasestatus_t
 *                row-major matrices (one row per y line, layers stacked) at
 *                every report time (report_every_days > 0) and at the end.
 *   flags_t<days>_iter<k>.txt  (trace_flags) Fig. 8 category of every cell
 *                after Newton iteration k of the step ending at <days>:
 *                0 inactive, 1 active, 2 boundary, 3 active + updated,
 *                4 boundary + updated, -1 dead EDFM filler position.
 * Units: SI inside, psi / days / bbl externally (SPEC.md design decision).
 * Surface rates: single phase and oil-water models conserve mass, so the
 * mass rate is divided by the phase reference density; the black-oil model
 * conserves surface volumes directly.
 *
 * Return codes: RSIM_* (0 ok, 1 bad argument, 2 CUDA / no sm_100 device,
 * 3 numerical failure after cuts, 4 not converged).  The CLI
 * (csrc/simulate_main.cpp) maps them to SPEC exit codes 0 / 2 / 3.
 */
#ifndef RSIM_SIMULATE_H
#define RSIM_SIMULATE_H

#include <stdint.h>
#include "cases.h"
#include "gpu_abi.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t solver;            /* 0 standard, 1 localized, 2 adaptive DD          */
  int32_t m;                 /* dilation hops; <= 0 -> case default (DD: 4)      */
  double eps_p;              /* Pa; <= 0 -> case default (also the set cutoff)   */
  int32_t n_steps;           /* <= 0 -> the case's whole schedule                */
  int32_t precond;           /* -1 -> case default (RSIM_PREC_*)                 */
  double report_every_days;  /* field dumps every this many days; 0 -> end only */
  int32_t write_fields;      /* 0: no field dumps at all                         */
  int32_t lin_method;        /* -1 -> case default (RSIM_LIN_*; DIRECT: n_A·b <= RSIM_DIRECT_MAX) */
  int32_t trace_flags;       /* 1: flags_t<days>_iter<k>.txt after every Newton iteration (Fig. 8 categories) */
} rsim_sim_opts;

typedef struct {
  int32_t status;            /* RSIM_*                                           */
  int32_t timesteps;         /* committed timesteps                              */
  int32_t total_iters;       /* Newton (inner) iterations, cut attempts included */
  int32_t total_lin;         /* Krylov iterations                                */
  int32_t cuts;
  int32_t pad;
  int64_t sum_na;            /* Σ n_A                                            */
  double total_ma;           /* Σ n_A / n                                        */
  double avg_ma;             /* total_ma / total_iters                           */
  double sim_days;
  double cum_oil_m3, cum_water_m3, cum_gas_m3;  /* surface volumes               */
  double wall_s;             /* host wall time of the solver loop                */
  int64_t total_outer;       /* DD outer (Schwarz sweep) iterations of the committed steps */
} rsim_run_metrics;

/* Surface-condition production rates of the case's producer at state (u, st):
 * q[0] water, q[1] oil, q[2] gas, m^3/s. */
int rsim_well_rates(const rsim_case* c, const double* u, const uint8_t* st, double* q);

/* Run the case on the GPU; out_dir NULL or "" -> no files. */
int rsim_simulate(const rsim_case_opts* co, const rsim_sim_opts* so, const char* out_dir, rsim_run_metrics* out);

/* The same for a case file (rsim/cases.h grammar; EDFM fractures): so->solver
 * -1 and so->m / so->eps_p <= 0 take the case file's [solver] defaults.
 * RSIM_EARG (message in rsim_gpu_last_error) on a configuration error. */
int rsim_simulate_file(const char* case_file, const rsim_sim_opts* so, const char* out_dir, rsim_run_metrics* out);

#ifdef __cplusplus
}
#endif
#endif
