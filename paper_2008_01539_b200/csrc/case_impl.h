// case_impl.h — the rsim_case object shared by the seeded config generator
// (cases.cpp) and the case-file / EDFM builder (edfm.cpp).  Host-only, private.
#ifndef RSIM_CASE_IMPL_H
#define RSIM_CASE_IMPL_H

#include <cstdint>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "rsim/cases.h"

namespace rsim_case_detail {
constexpr double kMilliDarcy = 9.869233e-16;  // m^2
constexpr double kDay = 86400.0;
constexpr double kCp = 1e-3;                  // Pa s
constexpr double kPsi = 6894.757293168361;    // Pa
}  // namespace rsim_case_detail

struct rsim_case {
  int config = 1;
  int32_t nx = 0, ny = 0, nz = 0;
  double dx = 10, dy = 10, dz = 1;
  int64_t n = 0;
  uint64_t seed = 0;
  std::vector<double> kx, ky, kz, phi, tx, ty, tz, pv, wi;
  std::vector<uint8_t> kind;
  std::vector<int32_t> nptr, nnbr;
  std::vector<double> nt;
  rsim_fluid_params fl{};
  double bhp = 0, p_init = 0, sw_init = 0;
  int n_steps = 20;
  double dt0 = 0.01 * rsim_case_detail::kDay, growth = 1.5, dt_max = 1e30;
  double eps = 0.2;
  int m = 2;
  std::map<std::pair<int64_t, int64_t>, double> nnc;
  // case files (edfm.cpp): whole-schedule time with the SPEC truncation rule,
  // the default solver, and the EDFM bookkeeping
  double total_time = 0.0;  // s; > 0: dt ramp truncated so that sum(dt) = total_time exactly
  int solver = 1;           // 0 standard, 1 localized, 2 adaptive DD (case file [solver] solver)
  std::string name;
  int64_t n_frac = 0, n_dead = 0;
};

// shared builders (cases.cpp)
void rsim_case_finalize_nnc(rsim_case& c);
void rsim_case_fluid_single(rsim_case& c);
void rsim_case_fluid_oilwater(rsim_case& c);

#endif
