/*
 * rsim/gpu_abi.h — the thin extern "C" boundary between host solver control
 * (C++ rsim::Simulator, include/rsim/simulator.hpp) and the hand-written
 * sm_100a fp64 kernels (paper_2008_01539_b200/csrc/ *.cu files).
 *
 * The reference has no FFI: its interface is the SPEC
 * operation list.  Each call below replaces the SPEC operation cited beside
 * it; the solver-level entry points at the bottom keep the SPEC signatures
 * newton_standard / newton_localized / adaptive_nonlinear_dd verbatim
 * (SPEC.md:395, :404, :413), with the graph/fluid/wells bound in the context
 * ("implicit context" per SURVEY.md §8b).
 *
 * Conventions
 *   - every function returns int: RSIM_OK / RSIM_EARG / RSIM_ECUDA /
 *     RSIM_ENUM (Krylov breakdown, singular block) / RSIM_ENOCONV;
 *     rsim_gpu_last_error() returns a thread-local message.
 *   - ownership: all device memory belongs to the opaque ctx; host pointers
 *     are borrowed for the duration of the call only.
 *   - threading: one host thread per ctx, one CUDA stream per ctx; not
 *     re-entrant.  There is NO CPU fallback: without a usable sm_100a device
 *     rsim_gpu_create fails with RSIM_ECUDA.
 *   - state layout: u[n*b] cell-major interleaved (p, S_w, X), status u8[n].
 */
#ifndef RSIM_GPU_ABI_H
#define RSIM_GPU_ABI_H

#include <stdint.h>
#include "types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rsim_gpu_ctx rsim_gpu_ctx;

/* Scalar struct returned once per Newton iteration (the only per-iteration
 * device->host transfer). */
typedef struct {
  int32_t status;        /* RSIM_* of the last kernel sequence                */
  int32_t bad_cell;      /* cell of a singular diagonal block (-1)            */
  int32_t lin_iters;     /* Krylov iterations                                 */
  int32_t n_active;      /* |V_A| after the last set update                   */
  int32_t n_boundary;    /* |V_B|                                             */
  int32_t expand;        /* 1: the last set update expanded                   */
  int32_t n_new;         /* DD: cells added to V_T by the last expansion      */
  int32_t pad;
  double  lin_relres;    /* ‖r̂‖₂/‖b̂‖₂                                         */
  double  f_norm2;       /* ‖F_A‖₂ (raw residual of the last assembly)        */
  double  f_norminf;     /* ‖F_A‖∞                                            */
  double  dp_inf_A;      /* ‖δp‖∞ over the solved set (last update)           */
  double  dp_inf_B;      /* ‖δp‖∞ over V_B                                    */
  double  halo_max;      /* DD: max latest |δp| over the selected halo        */
} rsim_gpu_stats;

/* ---- context / data movement ------------------------------------------ */
/* Select the CUDA device of the calling thread (one process per GPU). */
int rsim_gpu_set_device(int32_t device);
int rsim_gpu_create(rsim_gpu_ctx** ctx, const rsim_graph_desc* g, const rsim_fluid_params* f);
int rsim_gpu_destroy(rsim_gpu_ctx* ctx);
const char* rsim_gpu_last_error(void);
int rsim_gpu_device_info(char* name, int32_t cap, int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);

/* Upload a state and precompute the old-time accumulation. */
int rsim_gpu_set_state(rsim_gpu_ctx* ctx, const double* u, const uint8_t* status, double dt);
int rsim_gpu_set_dt(rsim_gpu_ctx* ctx, double dt);     /* recompute M^n for a new Δt */
int rsim_gpu_get_state(rsim_gpu_ctx* ctx, double* u, uint8_t* status);
int rsim_gpu_restore_state(rsim_gpu_ctx* ctx);          /* back to the last set_state (timestep cut) */

/* ---- active set -------------------------------------- */
/* V_A := sorted ∪ pinned (fracture + perforated cells); computes V_B, the
 * compacted list and g2l.  n = -1 selects every cell (newton_standard). */
int rsim_gpu_set_active(rsim_gpu_ctx* ctx, const int32_t* sorted, int32_t n, rsim_gpu_stats* st);
/* Initial set of a timestep: step0 -> pinned + m-halo,
 * else {|p - p_step_start_prev| >= eps} ∪ pinned, using the pressure saved
 * by the previous set_state. */
int rsim_gpu_initial_active(rsim_gpu_ctx* ctx, int32_t first_step, double eps, int32_t m, rsim_gpu_stats* st);
/* Algorithm 1 lines 7-18 (support_set, expand_active, shrink, boundary_layer):
 * from the δp of the last update.  shrink_locked forces shrink. */
int rsim_gpu_estimate_active(rsim_gpu_ctx* ctx, double eps, int32_t m, int32_t shrink_locked, rsim_gpu_stats* st);

/* ---- one Newton iteration's kernels ------------------------------------ */
int rsim_gpu_assemble(rsim_gpu_ctx* ctx);                                   /* K1 (+K2 pattern)  */
/* solve: o->lin_method BICGSTAB / GMRES (persistent Krylov kernels, K3/K4/K5) or
 * DIRECT (exact dense LU with partial pivoting, n_A*b <= RSIM_DIRECT_MAX, else RSIM_EARG). */
int rsim_gpu_linear_solve(rsim_gpu_ctx* ctx, const rsim_solver_opts* o);
int rsim_gpu_update(rsim_gpu_ctx* ctx, double eps);                         /* K6                */
int rsim_gpu_stats_get(rsim_gpu_ctx* ctx, rsim_gpu_stats* st);              /* sync + D2H scalars */

/* ---- dynamic DD (Algorithm 2) ------------------------------------------ */
/* Phase-1 set update over V_T: expand by m layers from flagged boundary
 * cells, label fresh cells with `round` (K8). */
int rsim_gpu_dd_expand(rsim_gpu_ctx* ctx, double eps, int32_t m, int32_t round, rsim_gpu_stats* st);
/* Build the N subdomain cell lists + halos from the labels (device). */
int rsim_gpu_dd_partition(rsim_gpu_ctx* ctx, int32_t n_sub, int32_t* sizes_out);
/* Select subdomain k as the active set; st->halo_max = max latest |δp| on its halo. */
int rsim_gpu_dd_select(rsim_gpu_ctx* ctx, int32_t k, rsim_gpu_stats* st);
/* Mark subdomain k skipped: its latest |δp| := 0 (SPEC.md:444 ledger). */
int rsim_gpu_dd_skip(rsim_gpu_ctx* ctx, int32_t k);
int rsim_gpu_download_labels(rsim_gpu_ctx* ctx, int32_t* labels);

/* ---- debug / parity downloads ------------------------------------------ */
int rsim_gpu_download_active(rsim_gpu_ctx* ctx, int32_t* act, int32_t* n);
int rsim_gpu_download_flags(rsim_gpu_ctx* ctx, uint8_t* flags);   /* Fig. 8 categories 0..4 */
int rsim_gpu_download_boundary(rsim_gpu_ctx* ctx, int32_t* vb, int32_t* n);
/* Last assembled system in canonical CSR order (see oracle_api.h). */
int64_t rsim_gpu_download_system(rsim_gpu_ctx* ctx, double* F_raw, double* rhs, int32_t* rowptr,
                                 int32_t* col, double* val, int64_t cap_nnzb);
int rsim_gpu_download_solution(rsim_gpu_ctx* ctx, double* x);
int rsim_gpu_upload_dp(rsim_gpu_ctx* ctx, const double* dp_global);  /* test hook for K7 parity */
/* K7 threshold from the uploaded δp (FLAG/seed bits, ‖δp‖∞ over V_A, V_B) — test hook. */
int rsim_gpu_threshold(rsim_gpu_ctx* ctx, double eps);
int rsim_gpu_download_dp(rsim_gpu_ctx* ctx, double* dp_global);

/* ---- timing hooks (bench) ----------------------------------------------- */
/* Device time (ms) of the kernels launched since the last reset, per phase:
 * [0] set/compaction, [1] assembly, [2] Krylov, [3] update. */
int rsim_gpu_timers(rsim_gpu_ctx* ctx, int32_t enable, double* ms4, int32_t* launches);

/* Work counters accumulated by the host solvers since the last reset:
 * [0] rows assembled, [1] Krylov row-iterations Σ n_A·its, [2] Krylov solves,
 * [3] Krylov launches' rows Σ n_A, [4] set-update passes (full-grid scans). */
int rsim_gpu_counters(rsim_gpu_ctx* ctx, int64_t* out5, int32_t reset);
/* b > 1, accumulated with the counters above: [0] Σ its · off-diagonal ELL
 * blocks stored by the assembly (active Cartesian neighbours), [1] Σ its · the
 * pressure-only ones among them (blockops.h col0_only; statistics only: the
 * Krylov kernels load and multiply them whole). */
int rsim_gpu_block_counters(rsim_gpu_ctx* ctx, int64_t* out2, int32_t reset);

/* Debug flags: bit 0 = the large-set assembly also stores the raw residual F
 * (otherwise only ‖F‖ partials are kept; rsim_gpu_download_system needs F). */
int rsim_gpu_set_debug(rsim_gpu_ctx* ctx, int32_t flags);

/* Debug: cycle counters of the cluster Krylov phases (RSIM_KTRACE=1 at create). */
#define RSIM_KTRACE_N 136 /* 8 phase counters (CTA 0) + 16 CTAs x 8 per-CTA counters */
int rsim_gpu_ktrace(rsim_gpu_ctx* ctx, unsigned long long* out);

/* CUDA events on the ctx stream (bench timing on the launching stream). */
int rsim_gpu_mark(rsim_gpu_ctx* ctx, int32_t slot);                 /* slot < 64 */
int rsim_gpu_elapsed(rsim_gpu_ctx* ctx, int32_t a, int32_t b, double* ms);
/* Write a 512 MB scratch buffer (> 126 MB L2) on the ctx stream. */
int rsim_gpu_flush_l2(rsim_gpu_ctx* ctx);
/* Device-side checkpoint of (u, status): 0 = save, 1 = restore. */
int rsim_gpu_checkpoint(rsim_gpu_ctx* ctx, int32_t restore);
/* Config-5 style set estimation from an uploaded global δp: seeds =
 * {|δp| >= eps} over ALL cells, m-hop dilation, compaction (support_set +
 * neighbor_set + compaction of SPEC.md:359-394 on the whole grid). */
int rsim_gpu_support_active(rsim_gpu_ctx* ctx, double eps, int32_t m, rsim_gpu_stats* st);
/* Set p := p_hi - dp_scale * δp (global δp already uploaded), for c5. */
int rsim_gpu_state_from_dp(rsim_gpu_ctx* ctx, double p_hi, double dp_scale);

/* ---- solver-level entry points (SPEC signatures) ----------------------- */
/* states in/out are host buffers (u[n*b], status[n]); Δt in seconds. */
int rsim_newton_standard(rsim_gpu_ctx* ctx, double* u, uint8_t* status, double dt,
                         const rsim_solver_opts* o, rsim_newton_report* rep);
int rsim_newton_localized(rsim_gpu_ctx* ctx, double* u, uint8_t* status, double dt,
                          const int32_t* va_init, int32_t n_init, int32_t m, double eps,
                          const rsim_solver_opts* o, rsim_newton_report* rep);
int rsim_adaptive_nonlinear_dd(rsim_gpu_ctx* ctx, double* u, uint8_t* status, double dt,
                               const int32_t* va_init, int32_t n_init, int32_t m, double eps,
                               const rsim_solver_opts* o, rsim_newton_report* rep);
/* Device-resident variants used by run_case: state stays on the device,
 * V_A_init from rsim_gpu_initial_active. */
int rsim_newton_standard_dev(rsim_gpu_ctx* ctx, const rsim_solver_opts* o, rsim_newton_report* rep);
int rsim_newton_localized_dev(rsim_gpu_ctx* ctx, const rsim_solver_opts* o, rsim_newton_report* rep);
int rsim_adaptive_nonlinear_dd_dev(rsim_gpu_ctx* ctx, const rsim_solver_opts* o, rsim_newton_report* rep);

/* run_case (minimal): whole schedule on the device with
 * timestep cuts; solver 0 standard, 1 localized, 2 adaptive DD. */
int rsim_run_case(rsim_gpu_ctx* ctx, int32_t solver, double* u, uint8_t* status, const double* dts,
                  int32_t nsteps, const rsim_solver_opts* o, int32_t* total_iters, double* total_ma,
                  int64_t* total_na, int32_t* total_lin, int32_t* n_cuts);

/* run_case on the state already resident on the device (no H2D/D2H). */
int rsim_run_case_dev(rsim_gpu_ctx* ctx, int32_t solver, const double* dts, int32_t nsteps,
                      const rsim_solver_opts* o, int32_t* total_iters, double* total_ma,
                      int64_t* total_na, int32_t* total_lin, int32_t* n_cuts);

#ifdef __cplusplus
}
#endif
#endif
