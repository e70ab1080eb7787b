// One localized-Newton timestep through the header-only C++ drop-in
// (include/rsim/simulator.hpp, the SPEC signatures) on config 1 at 40x40.
// Prints "iterations <k>", "n_active <a0> <a1> ...", "p_sum <%.17g>" so that
// tests/test_simulator_hpp.py can compare it with the Python / C-ABI path.
// Exit 3 when no sm_100 device is present (DeviceError), 1 on any other error.
#include <cstdio>
#include <vector>

#include "rsim/cases.h"
#include "rsim/simulator.hpp"

int main() {
  rsim_case_opts co{};
  co.config = 1; co.nx = 40; co.ny = 40; co.nz = 0; co.seed = 0; co.n_dfn = -1; co.n_steps = -1;
  rsim_case* cs = rsim_case_create(&co);
  if (!cs) return 1;
  rsim_graph_desc g;
  rsim_fluid_params f;
  rsim_solver_opts o;
  rsim_case_graph(cs, &g);
  rsim_case_fluid(cs, &f);
  rsim_case_solver_opts(cs, &o);
  const int64_t n = rsim_case_n(cs);
  rsim::CellStates s0;
  s0.u.resize(n * f.kind);
  s0.status.resize(n);
  rsim_case_init_state(cs, s0.u.data(), s0.status.data());
  std::vector<double> dts(64);
  rsim_case_schedule(cs, dts.data(), 64);
  try {
    rsim::Simulator sim(g, f, o);
    // V_A^init of the first step (pinned cells + m-hop halo, DESIGN.md §5 item 4), derived on the device
    rsim_gpu_stats st{};
    if (rsim_gpu_set_state(sim.handle(), s0.u.data(), s0.status.data(), dts[3]) != RSIM_OK) return 1;
    if (rsim_gpu_initial_active(sim.handle(), 1, o.eps_set, o.m, &st) != RSIM_OK) return 1;
    rsim::IndexSet va(n);
    int32_t na = 0;
    if (rsim_gpu_download_active(sim.handle(), va.data(), &na) != RSIM_OK) return 1;
    va.resize(na);
    auto [s1, rep] = sim.newton_localized(s0, dts[3], va, o.m, o.eps_set);
    double psum = 0.0;
    for (int64_t i = 0; i < n; ++i) psum += s1.u[i * f.kind];
    std::printf("iterations %d\nn_active", rep.iterations);
    for (int32_t a : rep.n_active()) std::printf(" %d", a);
    std::printf("\np_sum %.17g\nva_init %d\n", psum, na);
  } catch (const rsim::DeviceError& e) {
    std::printf("no device: %s\n", e.what());
    rsim_case_destroy(cs);
    return 3;
  } catch (const std::exception& e) {
    std::printf("error: %s\n", e.what());
    rsim_case_destroy(cs);
    return 1;
  }
  rsim_case_destroy(cs);
  return 0;
}
