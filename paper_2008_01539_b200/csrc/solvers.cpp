// solvers.cpp — host C++ control of the three nonlinear solvers over the
// C-ABI kernels.  This is the product's restatement of
//   newton_standard
//   newton_localized       SPEC.md:404-412, Algorithm 1
//   adaptive_nonlinear_dd  SPEC.md:413-430, Algorithm 2
//   run_case (minimal)
// with the ledgered decisions of DESIGN.md §Ambiguities (shared with the
// oracle, which restates the same control independently).
//
// Per Newton iteration exactly ONE device->host transfer happens (the scalar
// struct of rsim_gpu_stats); the expand/shrink decision and
// all set logic stay on the device.
#include <algorithm>
#include <cstring>
#include <deque>
#include <vector>

#include "rsim/gpu_abi.h"

// internal hooks (abi.cu)
int rsim_internal_begin_step(rsim_gpu_ctx* c, double dt);
int rsim_internal_commit_step(rsim_gpu_ctx* c);
int rsim_internal_dd_begin(rsim_gpu_ctx* c);
int64_t rsim_internal_n(const rsim_gpu_ctx* c);
int rsim_internal_iter_hook(rsim_gpu_ctx* c, int32_t iter, int32_t subdomain);
int rsim_internal_b(const rsim_gpu_ctx* c);
int32_t rsim_internal_nA(const rsim_gpu_ctx* c);
extern "C" int rsim_internal_add_row_iters(rsim_gpu_ctx* c, int64_t nA, int64_t its);
extern "C" int rsim_internal_solve_update(rsim_gpu_ctx* c, const rsim_solver_opts* o, double eps);
// hook after every timestep attempt: committed = 1 (accepted) or 0 (failed, about to be cut)
typedef int (*rsim_step_cb)(void* user, double dt, const rsim_newton_report* rep, int committed);
extern "C" int rsim_internal_run_case_cb(rsim_gpu_ctx* c, int32_t solver, const double* dts, int32_t nsteps,
                                         const rsim_solver_opts* o, int32_t* total_iters, double* total_ma,
                                         int64_t* total_na, int32_t* total_lin, int32_t* n_cuts, rsim_step_cb cb,
                                         void* user);

namespace {

#define TRY(x)                    \
  do {                            \
    int _r = (x);                 \
    if (_r != RSIM_OK) return _r; \
  } while (0)

void rep_init(rsim_newton_report* rep) { std::memset(rep, 0, sizeof(*rep)); }

void rep_push(rsim_newton_report* rep, const rsim_iter_record& r, int64_t n) {
  if (rep->n_records < RSIM_MAX_ITER_RECORDS) rep->rec[rep->n_records++] = r;
  rep->iterations += 1;
  rep->lin_iters_total += r.lin_iters;
  rep->sum_na += r.n_active;
  rep->sum_na_over_n += (double)r.n_active / (double)n;
}

// assemble -> Krylov -> update over the current device active list.
int local_step(rsim_gpu_ctx* c, const rsim_solver_opts* o) {
  TRY(rsim_gpu_assemble(c));
  TRY(rsim_internal_solve_update(c, o, o->eps_set));
  return RSIM_OK;
}

void fill_rec(rsim_iter_record& rec, int32_t nA, const rsim_gpu_stats& s, rsim_gpu_ctx* c) {
  rsim_internal_add_row_iters(c, nA, s.lin_iters);
  rec.n_active = nA;
  rec.lin_iters = s.lin_iters;
  rec.dp_inf_A = s.dp_inf_A;
  rec.dp_inf_B = s.dp_inf_B;
  rec.f_norm2 = s.f_norm2;
  rec.f_norminf = s.f_norminf;
  rec.lin_res = s.lin_relres;
}

int standard_dev(rsim_gpu_ctx* c, const rsim_solver_opts* o, rsim_newton_report* rep) {
  rep_init(rep);
  const int64_t n = rsim_internal_n(c);
  rsim_gpu_stats s{};
  TRY(rsim_gpu_set_active(c, nullptr, -1, &s));
  for (int it = 0; it < o->max_newton; ++it) {
    TRY(local_step(c, o));
    TRY(rsim_internal_iter_hook(c, it, -1));
    TRY(rsim_gpu_stats_get(c, &s));
    rsim_iter_record rec{};
    rec.subdomain = -1;
    fill_rec(rec, (int32_t)n, s, c);
    rec.dp_inf_B = 0.0;
    rep_push(rep, rec, n);
    if (s.status != RSIM_OK) { rep->status = s.status; return s.status; }
    if (s.dp_inf_A < o->eps_p) { rep->converged = 1; return RSIM_OK; }
  }
  rep->status = RSIM_ENOCONV;
  return RSIM_ENOCONV;
}

// Algorithm 1 with the active set already on the device.
int localized_dev(rsim_gpu_ctx* c, const rsim_solver_opts* o, rsim_newton_report* rep) {
  rep_init(rep);
  const int64_t n = rsim_internal_n(c);
  int shrink_locked = 0;
  rsim_gpu_stats s{};
  for (int it = 0; it < o->max_newton; ++it) {
    const int32_t nA = rsim_internal_nA(c);
    TRY(local_step(c, o));
    TRY(rsim_internal_iter_hook(c, it, -1));
    // set update for the next iteration (device-side mode decision) + the
    // single scalar D2H of this iteration
    TRY(rsim_gpu_estimate_active(c, o->eps_set, o->m, shrink_locked, &s));
    rsim_iter_record rec{};
    rec.subdomain = -1;
    fill_rec(rec, nA, s, c);
    rec.mode_expand = s.expand;
    rep_push(rep, rec, n);
    if (s.status != RSIM_OK) { rep->status = s.status; return s.status; }
    if (!s.expand) shrink_locked = 1;
    const bool conv = s.dp_inf_A < o->eps_p;
    if (!s.expand && conv) { rep->converged = 1; return RSIM_OK; }
  }
  rep->status = RSIM_ENOCONV;
  return RSIM_ENOCONV;
}

// Algorithm 2 (phase 1 over the cumulative V_T, phase 2 multiplicative
// Schwarz with the skip check), active set already on the device = V_T^0.
int dd_dev(rsim_gpu_ctx* c, const rsim_solver_opts* o, rsim_newton_report* rep) {
  rep_init(rep);
  const int64_t n = rsim_internal_n(c);
  TRY(rsim_internal_dd_begin(c));
  rsim_gpu_stats s{};
  int k = 0, inner = 0;
  while (true) {
    if (inner >= o->max_newton) { rep->status = RSIM_ENOCONV; return RSIM_ENOCONV; }
    const int32_t nA = rsim_internal_nA(c);
    TRY(local_step(c, o));
    TRY(rsim_internal_iter_hook(c, inner, -1));
    ++inner;
    TRY(rsim_gpu_dd_expand(c, o->eps_set, o->m, k + 1, &s));
    rsim_iter_record rec{};
    rec.subdomain = -1;
    fill_rec(rec, nA, s, c);
    rec.mode_expand = s.expand;
    rep_push(rep, rec, n);
    if (s.status != RSIM_OK) { rep->status = s.status; return s.status; }
    if (!s.expand) break;
    ++k;
  }
  const int N = k + 1;
  rep->n_subdomains = N;
  std::vector<int32_t> sizes(N);
  TRY(rsim_gpu_dd_partition(c, N, sizes.data()));
  std::vector<double> normA(N, 0.0);
  bool first = true;
  int outer = 0;
  while (true) {
    if (outer >= o->max_outer) { rep->outer_iterations = outer; rep->status = RSIM_ENOCONV; return RSIM_ENOCONV; }
    ++outer;
    bool any_big = false;
    for (int sd = 0; sd < N; ++sd) {
      TRY(rsim_gpu_dd_select(c, sd, &s));
      const double hmax = s.halo_max;
      if (first || normA[sd] >= o->eps_set || hmax >= o->eps_set) {
        TRY(local_step(c, o));
        TRY(rsim_internal_iter_hook(c, rep->iterations, sd));
        TRY(rsim_gpu_stats_get(c, &s));
        rsim_iter_record rec{};
        rec.subdomain = sd;
        fill_rec(rec, sizes[sd], s, c);
        rec.dp_inf_B = hmax;
        rep_push(rep, rec, n);
        if (s.status != RSIM_OK) { rep->outer_iterations = outer; rep->status = s.status; return s.status; }
        normA[sd] = s.dp_inf_A;
        if (normA[sd] >= o->eps_p) any_big = true;
      } else {
        normA[sd] = 0.0;
        TRY(rsim_gpu_dd_skip(c, sd));
      }
    }
    first = false;
    if (!any_big) break;
  }
  rep->outer_iterations = outer;
  rep->converged = 1;
  return RSIM_OK;
}

rsim_solver_opts with_m_eps(const rsim_solver_opts* o, int32_t m, double eps) {
  rsim_solver_opts q = *o;
  q.m = m;
  q.eps_set = eps;
  return q;
}

}  // namespace

extern "C" {

int rsim_newton_standard_dev(rsim_gpu_ctx* c, const rsim_solver_opts* o, rsim_newton_report* rep) {
  return standard_dev(c, o, rep);
}
int rsim_newton_localized_dev(rsim_gpu_ctx* c, const rsim_solver_opts* o, rsim_newton_report* rep) {
  return localized_dev(c, o, rep);
}
int rsim_adaptive_nonlinear_dd_dev(rsim_gpu_ctx* c, const rsim_solver_opts* o, rsim_newton_report* rep) {
  return dd_dev(c, o, rep);
}

int rsim_newton_standard(rsim_gpu_ctx* c, double* u, uint8_t* status, double dt, const rsim_solver_opts* o,
                         rsim_newton_report* rep) {
  if (!c || !u || !status || !o || !rep) return RSIM_EARG;
  TRY(rsim_gpu_set_state(c, u, status, dt));
  int r = standard_dev(c, o, rep);
  if (r == RSIM_OK) TRY(rsim_gpu_get_state(c, u, status));
  return r;
}

int rsim_newton_localized(rsim_gpu_ctx* c, double* u, uint8_t* status, double dt, const int32_t* va_init,
                          int32_t n_init, int32_t m, double eps, const rsim_solver_opts* o, rsim_newton_report* rep) {
  if (!c || !u || !status || !o || !rep || (n_init > 0 && !va_init)) return RSIM_EARG;
  rsim_solver_opts q = with_m_eps(o, m, eps);
  TRY(rsim_gpu_set_state(c, u, status, dt));
  TRY(rsim_gpu_set_active(c, va_init, n_init, nullptr));
  int r = localized_dev(c, &q, rep);
  if (r == RSIM_OK) TRY(rsim_gpu_get_state(c, u, status));
  return r;
}

int rsim_adaptive_nonlinear_dd(rsim_gpu_ctx* c, double* u, uint8_t* status, double dt, const int32_t* va_init,
                               int32_t n_init, int32_t m, double eps, const rsim_solver_opts* o,
                               rsim_newton_report* rep) {
  if (!c || !u || !status || !o || !rep || (n_init > 0 && !va_init)) return RSIM_EARG;
  rsim_solver_opts q = with_m_eps(o, m, eps);
  TRY(rsim_gpu_set_state(c, u, status, dt));
  TRY(rsim_gpu_set_active(c, va_init, n_init, nullptr));
  int r = dd_dev(c, &q, rep);
  if (r == RSIM_OK) TRY(rsim_gpu_get_state(c, u, status));
  return r;
}

int rsim_run_case_dev(rsim_gpu_ctx* c, int32_t solver, const double* dts, int32_t nsteps, const rsim_solver_opts* o,
                      int32_t* total_iters, double* total_ma, int64_t* total_na, int32_t* total_lin,
                      int32_t* n_cuts) {
  return rsim_internal_run_case_cb(c, solver, dts, nsteps, o, total_iters, total_ma, total_na, total_lin, n_cuts,
                                   nullptr, nullptr);
}

// run_case with a hook called after every committed timestep (the case
// runner's per-step outputs, simulate.cpp); cb returning non-zero aborts.
int rsim_internal_run_case_cb(rsim_gpu_ctx* c, int32_t solver, const double* dts, int32_t nsteps,
                              const rsim_solver_opts* o, int32_t* total_iters, double* total_ma, int64_t* total_na,
                              int32_t* total_lin, int32_t* n_cuts, rsim_step_cb cb, void* user) {
  if (!c || !dts || !o || nsteps < 1) return RSIM_EARG;
  *total_iters = 0; *total_ma = 0.0; *total_na = 0; *total_lin = 0; *n_cuts = 0;
  rsim_newton_report* rep = new rsim_newton_report;
  int r = RSIM_OK;
  std::deque<double> q(dts, dts + nsteps);
  bool first = true;
  int status_out = RSIM_OK;
  while (r == RSIM_OK && !q.empty()) {
    const double dt = q.front();
    q.pop_front();
    rsim_gpu_stats s{};
    if (solver != 0) {
      r = rsim_gpu_initial_active(c, first ? 1 : 0, o->eps_set, o->m, &s);
      if (r != RSIM_OK) break;
    }
    r = rsim_internal_begin_step(c, dt);
    if (r != RSIM_OK) break;
    int st;
    if (solver == 0) st = standard_dev(c, o, rep);
    else if (solver == 1) st = localized_dev(c, o, rep);
    else st = dd_dev(c, o, rep);
    *total_iters += rep->iterations;
    *total_ma += rep->sum_na_over_n;
    *total_na += rep->sum_na;
    *total_lin += rep->lin_iters_total;
    if (st == RSIM_ECUDA || st == RSIM_EARG) { status_out = st; break; }
    if (st != RSIM_OK) {
      if (cb) {
        r = cb(user, dt, rep, 0);
        if (r != RSIM_OK) break;
      }
      r = rsim_gpu_restore_state(c);
      if (dt * 0.5 < 1e-4 * 86400.0) { status_out = st; break; }
      ++*n_cuts;
      q.push_front(dt * 0.5);
      q.push_front(dt * 0.5);
      continue;
    }
    r = rsim_internal_commit_step(c);
    first = false;
    if (r == RSIM_OK && cb) r = cb(user, dt, rep, 1);
  }
  delete rep;
  if (r != RSIM_OK) return r;
  return status_out;
}

int rsim_run_case(rsim_gpu_ctx* c, int32_t solver, double* u, uint8_t* status, const double* dts, int32_t nsteps,
                  const rsim_solver_opts* o, int32_t* total_iters, double* total_ma, int64_t* total_na,
                  int32_t* total_lin, int32_t* n_cuts) {
  if (!c || !u || !status || !dts || !o || nsteps < 1) return RSIM_EARG;
  TRY(rsim_gpu_set_state(c, u, status, dts[0]));
  int r = rsim_run_case_dev(c, solver, dts, nsteps, o, total_iters, total_ma, total_na, total_lin, n_cuts);
  if (r == RSIM_ECUDA || r == RSIM_EARG) return r;
  TRY(rsim_gpu_get_state(c, u, status));
  return r;
}

}  // extern "C"
