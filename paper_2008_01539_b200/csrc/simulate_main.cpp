// simulate_main.cpp — command-line front end of the case runner
// (SPEC.md sim_driver_cli "External Interfaces"):
//
//   simulate <case-file> | --config N [--nx X --ny Y --nz Z --seed S --n-dfn K]
//            [--solver standard|localized|adaptive_dd] [--m N] [--eps-p PSI]
//            [--steps K] [--precond bj|neumann1|ilu0] [--lin bicgstab|gmres|direct] [--out DIR]
//            [--report-every DAYS] [--no-fields] [--trace-flags]
//
// A case is either a case file (the SPEC's key = value + fracture-table text,
// grammar in rsim/cases.h; EDFM fractures; cases/*.case hold the paper's
// Case 1 / Case 2 and the grid-sensitivity models) or one of the seeded
// synthetic configs of BASELINE.json with optional overrides.
// Exit codes: 0 success, 2 configuration error, 3 solver failure.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "rsim/simulate.h"

static int usage(const char* msg) {
  if (msg) std::fprintf(stderr, "simulate: %s\n", msg);
  std::fprintf(stderr,
               "usage: simulate <case-file> | --config N [--nx X --ny Y --nz Z --seed S --n-dfn K] "
               "[--solver standard|localized|adaptive_dd] [--m N] [--eps-p PSI] [--steps K] "
               "[--precond bj|neumann1|ilu0] [--lin bicgstab|gmres|direct] [--out DIR] [--report-every DAYS] "
               "[--no-fields] [--trace-flags]\n");
  return 2;
}

int main(int argc, char** argv) {
  rsim_case_opts co;
  std::memset(&co, 0, sizeof(co));
  co.n_dfn = -1;
  co.n_steps = -1;
  rsim_sim_opts so;
  std::memset(&so, 0, sizeof(so));
  so.solver = -1;  // case default (seeded configs: localized)
  so.precond = -1;
  so.lin_method = -1;
  so.write_fields = 1;
  std::string out, case_file;
  for (int k = 1; k < argc; ++k) {
    const std::string a = argv[k];
    auto next = [&]() -> const char* { return k + 1 < argc ? argv[++k] : nullptr; };
    const char* v = nullptr;
    if (a == "--no-fields") { so.write_fields = 0; continue; }
    if (a == "--trace-flags") { so.trace_flags = 1; continue; }
    if (a.size() && a[0] != '-') {
      if (!case_file.empty()) return usage("more than one case file");
      case_file = a;
      continue;
    }
    if (a == "-h" || a == "--help") return usage(nullptr), 0;
    if (!(v = next())) return usage(("missing value for " + a).c_str());
    char* end = nullptr;
    if (a == "--config") co.config = (int32_t)std::strtol(v, &end, 10);
    else if (a == "--nx") co.nx = (int32_t)std::strtol(v, &end, 10);
    else if (a == "--ny") co.ny = (int32_t)std::strtol(v, &end, 10);
    else if (a == "--nz") co.nz = (int32_t)std::strtol(v, &end, 10);
    else if (a == "--seed") co.seed = std::strtoull(v, &end, 10);
    else if (a == "--n-dfn") co.n_dfn = (int32_t)std::strtol(v, &end, 10);
    else if (a == "--m") so.m = (int32_t)std::strtol(v, &end, 10);
    else if (a == "--steps") so.n_steps = (int32_t)std::strtol(v, &end, 10);
    else if (a == "--eps-p") so.eps_p = std::strtod(v, &end) * 6894.757293168361;
    else if (a == "--report-every") so.report_every_days = std::strtod(v, &end);
    else if (a == "--out") { out = v; continue; }
    else if (a == "--solver") {
      const std::string s = v;
      if (s == "standard") so.solver = 0;
      else if (s == "localized") so.solver = 1;
      else if (s == "adaptive_dd") so.solver = 2;
      else return usage(("unknown solver " + s).c_str());
      continue;
    } else if (a == "--precond") {
      const std::string s = v;
      if (s == "bj") so.precond = RSIM_PREC_BJACOBI;
      else if (s == "neumann1") so.precond = RSIM_PREC_NEUMANN1;
      else if (s == "ilu0") so.precond = RSIM_PREC_ILU0;
      else return usage(("unknown preconditioner " + s).c_str());
      continue;
    } else if (a == "--lin") {
      const std::string s = v;
      if (s == "bicgstab") so.lin_method = RSIM_LIN_BICGSTAB;
      else if (s == "gmres") so.lin_method = RSIM_LIN_GMRES;
      else if (s == "direct") so.lin_method = RSIM_LIN_DIRECT;
      else return usage(("unknown linear solver " + s).c_str());
      continue;
    } else {
      return usage(("unknown option " + a).c_str());
    }
    if (!end || *end) return usage(("bad value for " + a).c_str());
  }
  if (case_file.empty() == (co.config == 0)) return usage("give either a case file or --config N");
  if (case_file.empty() && (co.config < 1 || co.config > 4))
    return usage("--config must be 1..4 (config 5 has no time loop)");
  if (so.eps_p < 0.0 || so.report_every_days < 0.0) return usage("negative --eps-p / --report-every");
  if (case_file.empty() && so.solver < 0) so.solver = 1;
  rsim_run_metrics m;
  const int r = case_file.empty() ? rsim_simulate(&co, &so, out.c_str(), &m)
                                  : rsim_simulate_file(case_file.c_str(), &so, out.c_str(), &m);
  if (r == RSIM_EARG) {
    const std::string why = std::string("invalid case or output directory: ") + rsim_gpu_last_error();
    return usage(why.c_str());
  }
  if (r != RSIM_OK) {
    std::fprintf(stderr, "simulate: solver failure (code %d): %s\n", r, rsim_gpu_last_error());
    return 3;
  }
  std::printf("timesteps %d  iterations %d  linear %d  cuts %d  total M_A %.6g  avg M_A %.6g  "
              "cum oil %.6g m3  wall %.3f s\n",
              m.timesteps, m.total_iters, m.total_lin, m.cuts, m.total_ma, m.avg_ma, m.cum_oil_m3, m.wall_s);
  return 0;
}
