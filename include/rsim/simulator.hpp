// rsim/simulator.hpp — header-only C++ drop-in for the reference's solver
// entry points, with the SPEC signatures verbatim:
//
//   newton_standard(states, Δt)              -> (states', NewtonReport)
//   newton_localized(states, Δt, V_A, m, ε)  -> (states', NewtonReport)
//   adaptive_nonlinear_dd(states, Δt, V_A, m, ε) -> (states', NewtonReport) SPEC.md:413-421
//   run_case(schedule) (minimal driver loop with timestep cuts)
//
// The graph, fluid and wells are the SPEC's implicit context: a Simulator
// binds them once (rsim_gpu_create) and every call runs on the B200 through
// the C ABI of include/rsim/gpu_abi.h (lib/librsim.so).  States are value
// types, freely copyable; the graph is shared read-only
// (SPEC.md:84).  Errors follow SPEC.md:399/:408/:417 (iteration cap or a
// numerical failure -> TimestepCut, the state is left unchanged) and :315
// (a singular pivot names its cell, NumericalError::cell).  There is no CPU
// fallback: without an sm_100 device the constructor throws DeviceError.
//
// Link: -I<repo>/include -L<repo>/paper_2008_01539_b200/lib -lrsim
#ifndef RSIM_SIMULATOR_HPP
#define RSIM_SIMULATOR_HPP

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gpu_abi.h"

namespace rsim {

// CellState: natural variables u[n*b] (cell-major p, S_w, X)
// plus the phase-status tag of every cell.
struct CellStates {
  std::vector<double> u;
  std::vector<uint8_t> status;
};

// IndexSet: sorted unique global cell indices.
using IndexSet = std::vector<int32_t>;

// NewtonReport: iterations, per-iteration n_A and ‖δp‖∞, ...
struct NewtonReport : rsim_newton_report {
  NewtonReport() : rsim_newton_report() {}
  std::vector<int32_t> n_active() const {
    std::vector<int32_t> v;
    for (int32_t k = 0; k < n_records; ++k) v.push_back(rec[k].n_active);
    return v;
  }
};

struct RunTotals {
  int32_t iterations = 0, lin_iters = 0, cuts = 0;
  double total_ma = 0.0;
  int64_t sum_na = 0;
};

// SPEC error taxonomy
struct DeviceError : std::runtime_error {
  int code;
  DeviceError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
struct TimestepCut : std::runtime_error {  // cap reached / numerical failure
  int code;
  NewtonReport report;
  TimestepCut(int c, const NewtonReport& r)
      : std::runtime_error(c == RSIM_ENOCONV ? "newton: iteration cap (timestep cut)"
                                             : "newton: numerical failure (timestep cut)"),
        code(c), report(r) {}
};
struct ArgumentError : std::invalid_argument {
  explicit ArgumentError(const std::string& m) : std::invalid_argument(m) {}
};

enum class Solver : int32_t { Standard = 0, Localized = 1, AdaptiveDD = 2 };

class Simulator {
 public:
  // Binds the immutable graph (ConnectivityGraph + WellSpec, SPEC.md:37-40,
  // :236-239) and the fluid; `opts` carries the tolerances / caps / Krylov
  // settings the SPEC leaves to the implementation.
  Simulator(const rsim_graph_desc& g, const rsim_fluid_params& f, const rsim_solver_opts& opts)
      : opts_(opts), n_((int64_t)g.nx * g.ny * g.nz), b_(f.kind) {
    const int rc = rsim_gpu_create(&ctx_, &g, &f);
    if (rc != RSIM_OK) {
      ctx_ = nullptr;
      throw DeviceError(rc, std::string("rsim_gpu_create: ") + rsim_gpu_last_error());
    }
  }
  ~Simulator() {
    if (ctx_) rsim_gpu_destroy(ctx_);
  }
  Simulator(const Simulator&) = delete;
  Simulator& operator=(const Simulator&) = delete;

  int64_t n() const { return n_; }
  int b() const { return b_; }
  rsim_solver_opts& options() { return opts_; }

  std::pair<CellStates, NewtonReport> newton_standard(CellStates states, double dt) {
    check_state(states);
    NewtonReport r;
    finish(rsim_newton_standard(ctx_, states.u.data(), states.status.data(), dt, &opts_, &r), r);
    return {std::move(states), r};
  }

  std::pair<CellStates, NewtonReport> newton_localized(CellStates states, double dt, const IndexSet& va_init, int m,
                                                       double eps) {
    check_state(states);
    NewtonReport r;
    finish(rsim_newton_localized(ctx_, states.u.data(), states.status.data(), dt, va_init.data(),
                                 (int32_t)va_init.size(), m, eps, &opts_, &r),
           r);
    return {std::move(states), r};
  }

  std::pair<CellStates, NewtonReport> adaptive_nonlinear_dd(CellStates states, double dt, const IndexSet& va_init,
                                                            int m, double eps) {
    check_state(states);
    NewtonReport r;
    finish(rsim_adaptive_nonlinear_dd(ctx_, states.u.data(), states.status.data(), dt, va_init.data(),
                                      (int32_t)va_init.size(), m, eps, &opts_, &r),
           r);
    return {std::move(states), r};
  }

  // The driver loop: one solver call per timestep, halving
  // on a cut down to 1e-4 day; V_A^init per SPEC.md:442 (DESIGN.md §5 item 4).
  RunTotals run_case(Solver solver, CellStates& states, const std::vector<double>& dts) {
    check_state(states);
    RunTotals t;
    const int rc = rsim_run_case(ctx_, (int32_t)solver, states.u.data(), states.status.data(), dts.data(),
                                 (int32_t)dts.size(), &opts_, &t.iterations, &t.total_ma, &t.sum_na, &t.lin_iters,
                                 &t.cuts);
    if (rc == RSIM_ECUDA) throw DeviceError(rc, rsim_gpu_last_error());
    if (rc == RSIM_EARG) throw ArgumentError(rsim_gpu_last_error());
    if (rc != RSIM_OK) throw TimestepCut(rc, NewtonReport());
    return t;
  }

  // Cell of the last singular diagonal block / pivot, -1 if none.
  int32_t bad_cell() {
    rsim_gpu_stats s{};
    rsim_gpu_stats_get(ctx_, &s);
    return s.bad_cell;
  }

  rsim_gpu_ctx* handle() { return ctx_; }

 private:
  void check_state(const CellStates& s) const {
    if ((int64_t)s.status.size() != n_ || (int64_t)s.u.size() != n_ * b_)
      throw ArgumentError("CellStates size does not match the bound graph");
  }
  static void finish(int rc, const NewtonReport& r) {
    if (rc == RSIM_OK) return;
    if (rc == RSIM_ENOCONV || rc == RSIM_ENUM) throw TimestepCut(rc, r);
    if (rc == RSIM_EARG) throw ArgumentError(rsim_gpu_last_error());
    throw DeviceError(rc, rsim_gpu_last_error());
  }

  rsim_gpu_ctx* ctx_ = nullptr;
  rsim_solver_opts opts_;
  int64_t n_;
  int b_;
};

}  // namespace rsim

#endif  // RSIM_SIMULATOR_HPP
