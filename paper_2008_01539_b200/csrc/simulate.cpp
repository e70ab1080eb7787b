// simulate.cpp — the case runner (SPEC.md:460-531,
// module sim_driver_cli): timestep schedule → GPU nonlinear solver per step
// (rsim_run_case's loop with a per-step hook) → rates / metrics / summary /
// field files.  Host C++ only; every solve runs through the C-ABI kernels.
//
//   run_case(cfg)   SPEC.md:484-487   rsim_simulate
//   well_rates      SPEC.md:501-507   rsim_well_rates
//   compute_ma      SPEC.md:493-501   total / average M_A in rsim_run_metrics
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "rsim/physics.h"
#include "rsim/simulate.h"

// hook after every timestep attempt: committed = 1 (accepted) or 0 (failed, about to be cut)
typedef int (*rsim_step_cb)(void* user, double dt, const rsim_newton_report* rep, int committed);
extern "C" void rsim_set_error_c(const char* msg);
void rsim_internal_set_iter_hook(rsim_gpu_ctx* c, int (*fn)(void*, int32_t, int32_t), void* user);
double rsim_internal_dt(const rsim_gpu_ctx* c);
extern "C" int rsim_internal_run_case_cb(rsim_gpu_ctx* c, int32_t solver, const double* dts, int32_t nsteps,
                                         const rsim_solver_opts* o, int32_t* total_iters, double* total_ma,
                                         int64_t* total_na, int32_t* total_lin, int32_t* n_cuts, rsim_step_cb cb,
                                         void* user);

namespace {

constexpr double kDay = 86400.0;
constexpr double kPsi = 6894.757293168361;  // Pa
constexpr double kBbl = 0.158987294928;     // m^3

int block_size(int32_t kind) { return kind == RSIM_FLUID_SINGLE ? 1 : (kind == RSIM_FLUID_OILWATER ? 2 : 3); }

template <int B>
void rates_b(const rsim_graph_desc& g, const rsim::phys::Fluid& f, int64_t n, const double* u, const uint8_t* st,
             double* q) {
  double s[3] = {0.0, 0.0, 0.0};
  for (int64_t i = 0; i < n; ++i) {
    const double wi = g.well_wi[i];
    if (!(wi > 0.0)) continue;
    rsim::phys::Props<B> P;
    rsim::phys::props(f, &u[i * B], st[i], P);
    double qe[B];
    rsim::phys::well_rate<B>(wi, u[i * B], g.bhp, P, qe);
    for (int e = 0; e < B; ++e) s[e] += qe[e];
  }
  // equation e -> surface phase: B=1 (oil) mass; B=2 (water, oil) mass; B=3 surface volumes
  if (B == 1) {
    q[0] = 0.0; q[1] = s[0] / f.rho_ref[1]; q[2] = 0.0;
  } else if (B == 2) {
    q[0] = s[0] / f.rho_ref[0]; q[1] = s[1] / f.rho_ref[1]; q[2] = 0.0;
  } else {
    q[0] = s[0]; q[1] = s[1]; q[2] = s[2];
  }
}

struct Run {
  const rsim_case* cs = nullptr;
  rsim_gpu_ctx* ctx = nullptr;
  rsim_graph_desc g{};
  rsim::phys::Fluid fl;
  int b = 1;
  int64_t n = 0;
  int32_t nxyz[3] = {0, 0, 0};
  std::string dir;
  double report_every = 0.0, next_report = 0.0;
  bool fields = false;
  double t = 0.0;  // seconds
  mutable double last_dump = -1.0;
  int step = 0;
  std::vector<double> u;
  std::vector<uint8_t> st;
  FILE* rates = nullptr;
  FILE* metrics = nullptr;
  FILE* iters = nullptr;
  int attempt = 0;
  rsim_run_metrics* m = nullptr;
  bool trace = false;            // --trace-flags: flags_t<days>_iter<k>.txt per Newton iteration
  std::vector<uint8_t> cat;      // Fig. 8 categories of the last iteration
};

bool mkdir_p(const std::string& d) {
  if (d.empty()) return true;
  std::string cur;
  for (size_t k = 0; k <= d.size(); ++k) {
    if (k == d.size() || d[k] == '/') {
      if (!cur.empty()) {
        struct stat sb;
        if (stat(cur.c_str(), &sb) != 0 && mkdir(cur.c_str(), 0755) != 0) return false;
      }
    }
    if (k < d.size()) cur += d[k];
  }
  return true;
}

// row-major matrix dump: one line per (layer, y) row, nx values per line
template <class F>
int dump(const Run& R, const char* what, F&& val) {
  char name[512];
  std::snprintf(name, sizeof(name), "%s/%s_t%.6g.txt", R.dir.c_str(), what, R.t / kDay);
  FILE* f = std::fopen(name, "w");
  if (!f) return RSIM_EARG;
  const int64_t nx = R.nxyz[0], rows = R.n / nx;
  for (int64_t r = 0; r < rows; ++r) {
    for (int64_t x = 0; x < nx; ++x) {
      if (x) std::fputc(' ', f);
      val(f, r * nx + x);
    }
    std::fputc('\n', f);
  }
  std::fclose(f);
  return RSIM_OK;
}

// --trace-flags (Figs. 8-9, 11): the Fig. 8 category of every cell
// after Newton iteration k of the timestep ending at t days — 0 inactive,
// 1 active, 2 boundary layer, 3 active + updated (|δp| >= ε), 4 boundary +
// updated; -1 marks dead EDFM filler positions.  Integer matrix, same layout
// as the field dumps.  DD local solves are numbered in solve order.
int trace_flags(void* user, int32_t iter, int32_t subdomain) {
  (void)subdomain;
  Run& R = *static_cast<Run*>(user);
  R.cat.resize((size_t)R.n);
  int r = rsim_gpu_download_flags(R.ctx, R.cat.data());
  if (r != RSIM_OK) return r;
  char name[512];
  std::snprintf(name, sizeof(name), "%s/flags_t%.6g_iter%d.txt", R.dir.c_str(),
                (R.t + rsim_internal_dt(R.ctx)) / kDay, iter);
  FILE* f = std::fopen(name, "w");
  if (!f) return RSIM_EARG;
  const int64_t nx = R.nxyz[0], rows = R.n / nx;
  for (int64_t row = 0; row < rows; ++row) {
    for (int64_t x = 0; x < nx; ++x) {
      const int64_t i = row * nx + x;
      std::fprintf(f, x ? " %d" : "%d", R.g.kind[i] == RSIM_KIND_DEAD ? -1 : (int)R.cat[i]);
    }
    std::fputc('\n', f);
  }
  std::fclose(f);
  return RSIM_OK;
}

int dump_fields(const Run& R) {
  const int b = R.b;
  R.last_dump = R.t;
  int r = dump(R, "pressure", [&](FILE* f, int64_t i) { std::fprintf(f, "%.17g", R.u[i * b] / kPsi); });
  if (r == RSIM_OK && b >= 2)
    r = dump(R, "satwater", [&](FILE* f, int64_t i) { std::fprintf(f, "%.17g", R.u[i * b + 1]); });
  if (r == RSIM_OK && b == 3) {
    r = dump(R, "satgas", [&](FILE* f, int64_t i) {
      std::fprintf(f, "%.17g", R.st[i] == RSIM_BO_SAT ? R.u[i * b + 2] : 0.0);
    });
    if (r == RSIM_OK) r = dump(R, "phasestatus", [&](FILE* f, int64_t i) { std::fprintf(f, "%d", (int)R.st[i]); });
  }
  return r;
}

// iterations.csv: one row per Newton iteration / local solve of every attempt
void log_iterations(Run& R, double dt, const rsim_newton_report* rep, int committed) {
  if (!R.iters) return;
  ++R.attempt;
  for (int32_t k = 0; k < rep->n_records; ++k) {
    const rsim_iter_record& q = rep->rec[k];
    std::fprintf(R.iters, "%d,%d,%d,%.10g,%d,%d,%.8g,%d,%d,%d,%.10g,%.10g,%.10g,%.10g,%.6g\n", R.step + 1, R.attempt,
                 committed, dt / kDay, k, q.n_active, (double)q.n_active / (double)R.n, q.lin_iters, q.subdomain,
                 q.mode_expand, q.dp_inf_A, q.dp_inf_B, q.f_norm2, q.f_norminf, q.lin_res);
  }
}

int on_step(void* user, double dt, const rsim_newton_report* rep, int committed) {
  Run& R = *static_cast<Run*>(user);
  log_iterations(R, dt, rep, committed);
  if (!committed) return RSIM_OK;
  R.attempt = 0;
  R.t += dt;
  ++R.step;
  int r = rsim_gpu_get_state(R.ctx, R.u.data(), R.st.data());
  if (r != RSIM_OK) return r;
  double q[3];
  rsim_well_rates(R.cs, R.u.data(), R.st.data(), q);
  rsim_run_metrics& m = *R.m;
  m.cum_water_m3 += q[0] * dt;
  m.cum_oil_m3 += q[1] * dt;
  m.cum_gas_m3 += q[2] * dt;
  m.timesteps += 1;
  m.total_outer += rep->outer_iterations;
  if (R.rates)
    std::fprintf(R.rates, "%.10g,%.10g,%.10g,%.10g,%.10g,%.10g\n", R.t / kDay, q[1] * kDay, q[2] * kDay,
                 R.g.bhp / kPsi, q[0] * kDay, q[1] * kDay / kBbl);
  if (R.metrics)
    std::fprintf(R.metrics, "%d,%.10g,%.10g,%d,%.10g,%lld,%d,%d\n", R.step, R.t / kDay, dt / kDay, rep->iterations,
                 rep->sum_na_over_n, (long long)rep->sum_na, rep->lin_iters_total, rep->n_subdomains);
  if (R.fields && R.report_every > 0.0 && R.t >= R.next_report * (1.0 - 1e-12)) {
    r = dump_fields(R);
    while (R.next_report <= R.t * (1.0 + 1e-12)) R.next_report += R.report_every;
  }
  return r;
}

}  // namespace

extern "C" {

int rsim_well_rates(const rsim_case* c, const double* u, const uint8_t* st, double* q) {
  if (!c || !u || !st || !q) return RSIM_EARG;
  rsim_graph_desc g;
  rsim_fluid_params fp;
  rsim_case_graph(c, &g);
  rsim_case_fluid(c, &fp);
  const rsim::phys::Fluid f(fp);
  const int64_t n = rsim_case_n(c);
  switch (block_size(fp.kind)) {
    case 1: rates_b<1>(g, f, n, u, st, q); break;
    case 2: rates_b<2>(g, f, n, u, st, q); break;
    default: rates_b<3>(g, f, n, u, st, q); break;
  }
  return RSIM_OK;
}

}  // extern "C"

namespace {

// run_case(cfg) of an already built case; takes ownership of cs.
int run_sim(rsim_case* cs, const char* label, const rsim_sim_opts* so_in, const char* out_dir, rsim_run_metrics* out) {
  rsim_case_info_t info;
  rsim_case_info(cs, &info);
  rsim_sim_opts sov = *so_in;
  const rsim_sim_opts* so = &sov;
  if (sov.solver < 0) sov.solver = info.solver;  // case default (case files: [solver] solver)
  Run R;
  R.cs = cs;
  R.m = out;
  rsim_fluid_params fp;
  rsim_case_graph(cs, &R.g);
  rsim_case_fluid(cs, &fp);
  R.fl = rsim::phys::Fluid(fp);
  R.b = block_size(fp.kind);
  R.n = rsim_case_n(cs);
  double dxyz[3];
  rsim_case_dims(cs, R.nxyz, dxyz);
  R.u.resize((size_t)R.n * R.b);
  R.st.resize((size_t)R.n);
  rsim_case_init_state(cs, R.u.data(), R.st.data());
  std::vector<double> dts(100000);
  int32_t ns = rsim_case_schedule(cs, dts.data(), (int32_t)dts.size());
  if (so->n_steps > 0 && so->n_steps < ns) ns = so->n_steps;
  rsim_solver_opts o;
  rsim_case_solver_opts(cs, &o);
  if (so->eps_p > 0.0) o.eps_p = o.eps_set = so->eps_p;
  o.m = so->m > 0 ? so->m : (so->solver == 2 && info.solver != 2 ? 4 : o.m);  // DD: m = 4
  if (so->precond >= 0) o.precond = so->precond;
  if (so->lin_method >= 0) o.lin_method = so->lin_method;
  int r = RSIM_OK;
  const bool files = out_dir && *out_dir;
  if (files) {
    R.dir = out_dir;
    if (!mkdir_p(R.dir)) r = RSIM_EARG;
    R.fields = so->write_fields != 0;
    R.report_every = so->report_every_days * kDay;
    R.next_report = R.report_every;
    if (r == RSIM_OK) {
      R.rates = std::fopen((R.dir + "/rates.csv").c_str(), "w");
      R.metrics = std::fopen((R.dir + "/metrics.csv").c_str(), "w");
      R.iters = std::fopen((R.dir + "/iterations.csv").c_str(), "w");
      if (!R.rates || !R.metrics || !R.iters) r = RSIM_EARG;
    }
    if (R.iters)
      std::fprintf(R.iters, "step,attempt,committed,dt_days,iter,n_active,active_fraction,lin_iters,subdomain,"
                            "mode_expand,dp_inf_A,dp_inf_B,f_norm2,f_norminf,lin_relres\n");
    if (R.rates) std::fprintf(R.rates, "time_days,oil_rate,gas_rate,bhp,water_rate,oil_rate_bbl\n");
    if (R.metrics) std::fprintf(R.metrics, "step,time_days,dt_days,iterations,sum_nA_over_n,sum_nA,lin_iters,n_subdomains\n");
    R.trace = so->trace_flags != 0;
  }
  if (r == RSIM_OK) r = rsim_gpu_create(&R.ctx, &R.g, &fp);
  if (r == RSIM_OK && R.trace) rsim_internal_set_iter_hook(R.ctx, trace_flags, &R);
  if (r == RSIM_OK) r = rsim_gpu_set_state(R.ctx, R.u.data(), R.st.data(), dts[0]);
  if (r == RSIM_OK) {
    const auto t0 = std::chrono::steady_clock::now();
    r = rsim_internal_run_case_cb(R.ctx, so->solver, dts.data(), ns, &o, &out->total_iters, &out->total_ma,
                                  &out->sum_na, &out->total_lin, &out->cuts, on_step, &R);
    out->wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  out->status = r;
  out->sim_days = R.t / kDay;
  out->avg_ma = out->total_iters > 0 ? out->total_ma / out->total_iters : 0.0;
  if (files && R.fields && R.step > 0 && R.last_dump != R.t)
    dump_fields(R);  // final state (unless the last report already wrote it)
  if (files && (r == RSIM_OK || R.step > 0)) {
    FILE* f = std::fopen((R.dir + "/summary.txt").c_str(), "w");
    if (f) {
      static const char* names[3] = {"standard", "localized", "adaptive_dd"};
      std::fprintf(f, "case %s  grid %dx%dx%d  n %lld  live %lld  fracture_cells %lld  solver %s  m %d  eps_p %.6g Pa\n",
                   label, R.nxyz[0], R.nxyz[1], R.nxyz[2], (long long)R.n, (long long)info.n_live,
                   (long long)info.n_frac, names[so->solver], o.m, o.eps_p);
      std::fprintf(f, "status %d\ntimesteps %d\nsimulated_days %.10g\ncuts %d\n", r, out->timesteps, out->sim_days,
                   out->cuts);
      std::fprintf(f, "total_iterations %d\ntotal_linear_iterations %d\n", out->total_iters, out->total_lin);
      std::fprintf(f, "total_ratio_MA %.10g\naverage_ratio_MA_per_iteration %.10g\nsum_nA %lld\n", out->total_ma,
                   out->avg_ma, (long long)out->sum_na);
      std::fprintf(f, "cumulative_oil_m3 %.10g\ncumulative_oil_bbl %.10g\ncumulative_water_m3 %.10g\n"
                   "cumulative_gas_m3 %.10g\nsolver_wall_s %.6g\n",
                   out->cum_oil_m3, out->cum_oil_m3 / kBbl, out->cum_water_m3, out->cum_gas_m3, out->wall_s);
      std::fclose(f);
    }
  }
  if (R.rates) std::fclose(R.rates);
  if (R.metrics) std::fclose(R.metrics);
  if (R.iters) std::fclose(R.iters);
  if (R.ctx) rsim_gpu_destroy(R.ctx);
  rsim_case_destroy(cs);
  return r;
}

bool opts_ok(const rsim_sim_opts* so) {
  if (so->solver < -1 || so->solver > 2 || so->precond < -1 || so->precond > RSIM_PREC_NEUMANN1 ||
      so->lin_method < -1 || so->lin_method > RSIM_LIN_DIRECT) {
    rsim_set_error_c("rsim_simulate: solver / precond / lin_method out of range");
    return false;
  }
  return true;
}

}  // namespace

extern "C" {

int rsim_simulate(const rsim_case_opts* co, const rsim_sim_opts* so, const char* out_dir, rsim_run_metrics* out) {
  if (!co || !so || !out || so->solver < 0 || !opts_ok(so)) return RSIM_EARG;
  std::memset(out, 0, sizeof(*out));
  rsim_case* cs = rsim_case_create(co);
  if (!cs) return RSIM_EARG;
  char label[32];
  std::snprintf(label, sizeof(label), "config%d", co->config);
  return run_sim(cs, label, so, out_dir, out);
}

int rsim_simulate_file(const char* case_file, const rsim_sim_opts* so, const char* out_dir, rsim_run_metrics* out) {
  if (!case_file || !so || !out || !opts_ok(so)) return RSIM_EARG;
  std::memset(out, 0, sizeof(*out));
  char err[512] = {0};
  rsim_case* cs = rsim_case_from_file(case_file, err, sizeof(err));
  if (!cs) {
    rsim_set_error_c(err);
    return RSIM_EARG;
  }
  return run_sim(cs, case_file, so, out_dir, out);
}

}  // extern "C"
