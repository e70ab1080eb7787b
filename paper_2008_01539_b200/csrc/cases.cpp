// cases.cpp — seeded synthetic inputs for BASELINE.json configs 1-5.
//
// Host-only.  Gaps in the configs are filled per SURVEY.md Appendix A and
// recorded in DESIGN.md §Cases.  TPFA transmissibility = harmonic mean of the
// half-transmissibilities k·A/(d/2) (build_matrix_grid).
// Fracture lines/planes are either high-permeability cells (c1, c3, stage
// fractures of c4) or DFN conduits "embedded as connections to the matrix
// cells they cross" (c2, c4): consecutive crossed cells get Υ_f = k_f·a·h/d
// added to their shared face, or an NNC if they touch only at a corner.
// Crossed cells are tagged fracture => always active.
#include "rsim/cases.h"
#include "case_impl.h"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <utility>
#include <vector>

namespace {

using rsim_case_detail::kCp;
using rsim_case_detail::kDay;
using rsim_case_detail::kMilliDarcy;

// SplitMix64 keyed by (seed, stream, index): counter-based, so every cell's
// draw is independent of generation order.
inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
inline double u01(uint64_t seed, uint64_t stream, uint64_t idx) {
  uint64_t z = mix64(seed + 0x9E3779B97F4A7C15ULL * (stream * 0x100000001ULL + idx + 1));
  return ((z >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}
inline double normal(uint64_t seed, uint64_t stream, uint64_t idx) {
  double a = u01(seed, stream, 2 * idx), b = u01(seed, stream, 2 * idx + 1);
  return std::sqrt(-2.0 * std::log(a)) * std::cos(6.283185307179586 * b);
}

struct Line {
  double x0, y0, x1, y1, kf;
  bool well;
};

}  // namespace

namespace {

void build_tpfa(rsim_case& c) {
  const int64_t n = c.n, nxy = (int64_t)c.nx * c.ny;
  c.tx.assign(n, 0.0);
  c.ty.assign(n, 0.0);
  c.tz.assign(n, 0.0);
  auto harm = [](double a, double b) { return (a > 0.0 && b > 0.0) ? (a * b) / (a + b) : 0.0; };
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    int64_t ix = i % c.nx, iy = (i / c.nx) % c.ny, iz = i / nxy;
    if (ix < c.nx - 1) {
      double a = c.dy * c.dz, h = 0.5 * c.dx;
      c.tx[i] = harm(c.kx[i] * a / h, c.kx[i + 1] * a / h);
    }
    if (iy < c.ny - 1) {
      double a = c.dx * c.dz, h = 0.5 * c.dy;
      c.ty[i] = harm(c.ky[i] * a / h, c.ky[i + c.nx] * a / h);
    }
    if (iz < c.nz - 1) {
      double a = c.dx * c.dy, h = 0.5 * c.dz;
      c.tz[i] = harm(c.kz[i] * a / h, c.kz[i + nxy] * a / h);
    }
  }
}

void lognormal_perm(rsim_case& c, double kg_md, double sigma) {
  c.kx.resize(c.n);
  c.ky.resize(c.n);
  c.kz.resize(c.n);
  const double lkg = std::log(kg_md * kMilliDarcy);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < c.n; ++i) {
    double k = std::exp(lkg + sigma * normal(c.seed, 1, (uint64_t)i));
    c.kx[i] = c.ky[i] = c.kz[i] = k;
  }
}

// Walk a segment at sub-cell resolution, returning the sequence of distinct
// (ix,iy) cells crossed (clipped to the domain).
std::vector<std::pair<int, int>> rasterize(const rsim_case& c, const Line& L) {
  std::vector<std::pair<int, int>> cells;
  double len = std::hypot(L.x1 - L.x0, L.y1 - L.y0);
  int steps = std::max(1, (int)std::ceil(len / (0.05 * std::min(c.dx, c.dy))));
  for (int s = 0; s <= steps; ++s) {
    double t = (double)s / steps;
    double x = L.x0 + (L.x1 - L.x0) * t, y = L.y0 + (L.y1 - L.y0) * t;
    int ix = (int)std::floor(x / c.dx), iy = (int)std::floor(y / c.dy);
    if (ix < 0 || iy < 0 || ix >= c.nx || iy >= c.ny) continue;
    if (cells.empty() || cells.back() != std::make_pair(ix, iy)) cells.emplace_back(ix, iy);
  }
  return cells;
}

// Embed a vertical planar fracture (2D line extruded over all layers) as
// conduits between consecutive crossed cells.
void embed_line(rsim_case& c, const Line& L, double aperture, double wi) {
  auto cells = rasterize(c, L);
  const int64_t nxy = (int64_t)c.nx * c.ny;
  for (int iz = 0; iz < c.nz; ++iz) {
    for (size_t k = 0; k < cells.size(); ++k) {
      int64_t i = iz * nxy + (int64_t)cells[k].second * c.nx + cells[k].first;
      c.kind[i] = RSIM_KIND_FRACTURE;
      if (L.well && wi > 0.0) c.wi[i] = wi;
      if (k == 0) continue;
      int64_t j = iz * nxy + (int64_t)cells[k - 1].second * c.nx + cells[k - 1].first;
      int dix = cells[k].first - cells[k - 1].first, diy = cells[k].second - cells[k - 1].second;
      double d = std::hypot(dix * c.dx, diy * c.dy);
      double tf = L.kf * aperture * c.dz / d;
      int64_t a = std::min(i, j), b = std::max(i, j);
      if (std::abs(dix) + std::abs(diy) == 1) {
        if (dix != 0) c.tx[a] += tf;
        else c.ty[a] += tf;
      } else {
        c.nnc[{a, b}] += tf;
      }
    }
  }
}

void finalize_nnc(rsim_case& c) {
  std::vector<std::vector<std::pair<int32_t, double>>> rows;
  c.nptr.assign(c.n + 1, 0);
  if (c.nnc.empty()) return;
  for (auto& kv : c.nnc) {
    c.nptr[kv.first.first + 1]++;
    c.nptr[kv.first.second + 1]++;
  }
  for (int64_t i = 0; i < c.n; ++i) c.nptr[i + 1] += c.nptr[i];
  c.nnbr.assign(c.nptr[c.n], 0);
  c.nt.assign(c.nptr[c.n], 0.0);
  std::vector<int32_t> fill(c.nptr.begin(), c.nptr.end() - 1);
  for (auto& kv : c.nnc) {  // map order => ascending (a,b): rows end up sorted
    int64_t a = kv.first.first, b = kv.first.second;
    c.nnbr[fill[a]] = (int32_t)b; c.nt[fill[a]++] = kv.second;
    c.nnbr[fill[b]] = (int32_t)a; c.nt[fill[b]++] = kv.second;
  }
  for (int64_t i = 0; i < c.n; ++i) {  // sort each row by neighbour
    std::vector<std::pair<int32_t, double>> r;
    for (int32_t q = c.nptr[i]; q < c.nptr[i + 1]; ++q) r.emplace_back(c.nnbr[q], c.nt[q]);
    std::sort(r.begin(), r.end());
    for (size_t k = 0; k < r.size(); ++k) { c.nnbr[c.nptr[i] + k] = r[k].first; c.nt[c.nptr[i] + k] = r[k].second; }
  }
}

void set_fluid_single(rsim_case& c) {
  rsim_fluid_params& f = c.fl;
  std::memset(&f, 0, sizeof(f));
  f.kind = RSIM_FLUID_SINGLE;
  f.p_ref = c.p_init;
  f.c_r = 0.0;
  f.rho_ref[0] = 1000.0; f.rho_ref[1] = 800.0; f.rho_ref[2] = 1.0;
  f.c_f[0] = 1e-9; f.c_f[1] = 1e-9; f.c_f[2] = 0.0;
  f.mu[0] = 0.5 * kCp; f.mu[1] = 1.0 * kCp; f.mu[2] = 0.02 * kCp;
}

void set_fluid_oilwater(rsim_case& c) {
  set_fluid_single(c);
  c.fl.kind = RSIM_FLUID_OILWATER;
  c.fl.swc = 0.2;
  c.fl.sor = 0.2;
}

void set_fluid_blackoil(rsim_case& c) {
  set_fluid_single(c);
  rsim_fluid_params& f = c.fl;
  f.kind = RSIM_FLUID_BLACKOIL;
  f.c_f[0] = 4e-10; f.c_f[1] = 1e-9;
  f.swc = 0.2; f.sor = 0.2; f.sgc = 0.05;
  f.p_bub = 20e6;
  f.rs_b = 100.0;
  f.bo_alpha = 5e-3;
  f.p_gas = 1.1e5;
}

void common_init(rsim_case& c) {
  c.n = (int64_t)c.nx * c.ny * c.nz;
  c.kind.assign(c.n, RSIM_KIND_MATRIX);
  c.wi.assign(c.n, 0.0);
  c.phi.assign(c.n, 0.06);
}

void finish(rsim_case& c) {
  c.pv.resize(c.n);
  for (int64_t i = 0; i < c.n; ++i) c.pv[i] = c.dx * c.dy * c.dz * c.phi[i];
  finalize_nnc(c);
}

// ---- config builders ------------------------------------------------------
void build_c1(rsim_case& c) {  // 2D single phase, line of high-perm cells
  common_init(c);
  lognormal_perm(c, 1e-4, 1.0);
  int iy = c.ny / 2, x0 = c.nx / 5, x1 = (4 * c.nx) / 5;
  for (int ix = x0; ix < x1; ++ix) {
    int64_t i = (int64_t)iy * c.nx + ix;
    c.kx[i] = c.ky[i] = c.kz[i] = 1e4 * kMilliDarcy;
    c.kind[i] = RSIM_KIND_FRACTURE;
    c.wi[i] = 1e-10;
  }
  build_tpfa(c);
  c.p_init = 30e6; c.bhp = 10e6;
  set_fluid_single(c);
  c.n_steps = 20;
  c.eps = 1e-8 * (c.p_init - c.bhp);
  finish(c);
}

void build_dfn(rsim_case& c, int n_dfn, bool well_line, double zc_unused) {
  (void)zc_unused;
  const double W = c.nx * c.dx, H = c.ny * c.dy;
  const double scale = std::sqrt((double)c.nx * c.ny / (256.0 * 256.0));
  std::vector<Line> lines;
  if (well_line) {  // producer fracture through the centre ("producer at the centre")
    double hl = 150.0 * std::min(1.0, scale);
    lines.push_back({W / 2 - hl, H / 2 + 0.5 * c.dy, W / 2 + hl, H / 2 + 0.5 * c.dy, 1e4 * kMilliDarcy, true});
  }
  for (int k = 0; k < n_dfn; ++k) {
    double cx = u01(c.seed, 2, 6 * k) * W, cy = u01(c.seed, 2, 6 * k + 1) * H;
    double len = (50.0 + 350.0 * u01(c.seed, 2, 6 * k + 2)) * std::min(1.0, scale);
    double th = 3.141592653589793 * u01(c.seed, 2, 6 * k + 3);
    double kf = std::exp(std::log(1e3) + (std::log(1e5) - std::log(1e3)) * u01(c.seed, 2, 6 * k + 4)) * kMilliDarcy;
    double hx = 0.5 * len * std::cos(th), hy = 0.5 * len * std::sin(th);
    lines.push_back({cx - hx, cy - hy, cx + hx, cy + hy, kf, false});
  }
  for (auto& L : lines) embed_line(c, L, 1e-3, 1e-10);
}

void build_c2(rsim_case& c, int n_dfn) {  // 2D oil-water with DFN
  common_init(c);
  lognormal_perm(c, 1e-3, 1.5);
  build_tpfa(c);
  build_dfn(c, n_dfn, true, 0);
  c.p_init = 30e6; c.bhp = 10e6; c.sw_init = 0.35;
  set_fluid_oilwater(c);
  c.n_steps = 30;
  c.dt_max = 100.0 * kDay;
  c.eps = 1e-8 * (c.p_init - c.bhp);
  finish(c);
}

// Transverse full-height planar fractures along a horizontal well in x at
// (iy_w, iz_w): plane x = ix_c, iy in [iy_w - h, iy_w + h], all layers.
void stage_fractures(rsim_case& c, int n_stage, int per_stage, double x_lo, double x_hi, double kf_md,
                     int stream) {
  const int64_t nxy = (int64_t)c.nx * c.ny;
  int iy_w = c.ny / 2, iz_w = c.nz / 2;
  double cell_scale = c.ny / 256.0;
  int fidx = 0;
  for (int s = 0; s < n_stage; ++s) {
    double xc = x_lo + (x_hi - x_lo) * (s + 0.5) / n_stage;
    for (int k = 0; k < per_stage; ++k) {
      int ix = (int)std::lround(xc) + (k - per_stage / 2) * 3;
      ix = std::max(0, std::min(c.nx - 1, ix));
      double hl = 100.0 + 100.0 * u01(c.seed, stream, fidx++);
      int h = std::max(1, (int)std::lround(hl / c.dy * cell_scale));
      for (int iz = 0; iz < c.nz; ++iz)
        for (int iy = std::max(0, iy_w - h); iy <= std::min(c.ny - 1, iy_w + h); ++iy) {
          int64_t i = iz * nxy + (int64_t)iy * c.nx + ix;
          c.kx[i] = c.ky[i] = c.kz[i] = kf_md * kMilliDarcy;
          c.kind[i] = RSIM_KIND_FRACTURE;
        }
      c.wi[iz_w * nxy + (int64_t)iy_w * c.nx + ix] = 1e-10;
    }
  }
}

void build_c3(rsim_case& c) {  // 3D two-phase multi-stage HF
  common_init(c);
  lognormal_perm(c, 5e-4, 1.0);
  stage_fractures(c, 12, 3, 28.0 / 256.0 * c.nx, 228.0 / 256.0 * c.nx, 5e3, 3);
  build_tpfa(c);
  c.p_init = 30e6; c.bhp = 10e6; c.sw_init = 0.35;
  set_fluid_oilwater(c);
  c.n_steps = 20;
  c.eps = 1e-8 * (c.p_init - c.bhp);
  finish(c);
}

void build_c4(rsim_case& c, int n_dfn) {  // 3D black-oil, DFN + stage fractures
  common_init(c);
  lognormal_perm(c, 1e-3, 1.0);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < c.n; ++i)
    c.phi[i] = std::min(0.3, std::max(0.01, 0.06 * std::exp(0.25 * normal(c.seed, 4, (uint64_t)i))));
  stage_fractures(c, 20, 1, 56.0 / 512.0 * c.nx, 456.0 / 512.0 * c.nx, 5e3, 5);
  build_tpfa(c);
  build_dfn(c, n_dfn, false, 0);
  c.p_init = 21e6; c.bhp = 8e6; c.sw_init = 0.2;
  set_fluid_blackoil(c);
  c.fl.p_ref = c.p_init;
  // Newton update limiter (DESIGN.md §5 item 11); RSIM_C4_LIMITER="dp_rel,ds" overrides (tuning only)
  c.fl.dp_max_rel = 0.5;
  c.fl.ds_max = 0.2;
  if (const char* e = std::getenv("RSIM_C4_LIMITER")) std::sscanf(e, "%lf,%lf", &c.fl.dp_max_rel, &c.fl.ds_max);
  c.n_steps = 20;
  c.eps = 1e-8 * (c.p_init - c.bhp);
  finish(c);
}

void build_c5(rsim_case& c) {  // scaling stress, single phase, no Newton loop
  common_init(c);
  lognormal_perm(c, 1e-3, 1.0);
  build_tpfa(c);
  c.p_init = 30e6; c.bhp = 10e6;
  set_fluid_single(c);
  c.n_steps = 1;
  c.dt0 = kDay;
  c.eps = 1e-3;
  finish(c);
}

}  // namespace

void rsim_case_finalize_nnc(rsim_case& c) { finalize_nnc(c); }
void rsim_case_fluid_single(rsim_case& c) { set_fluid_single(c); }
void rsim_case_fluid_oilwater(rsim_case& c) { set_fluid_oilwater(c); }

extern "C" {

rsim_case* rsim_case_create(const rsim_case_opts* o) {
  if (!o || o->config < 1 || o->config > 5) return nullptr;
  rsim_case* c = new rsim_case();
  c->config = o->config;
  c->seed = o->seed ? o->seed : 2008015390ULL + (uint64_t)o->config;
  static const int def[6][3] = {{0, 0, 0}, {100, 100, 1}, {256, 256, 1}, {256, 256, 32}, {512, 512, 16}, {1024, 1024, 32}};
  c->nx = o->nx > 0 ? o->nx : def[o->config][0];
  c->ny = o->ny > 0 ? o->ny : def[o->config][1];
  c->nz = o->nz > 0 ? o->nz : def[o->config][2];
  c->dx = 10.0; c->dy = 10.0; c->dz = (o->config >= 3) ? 2.0 : 1.0;
  double area = (double)c->nx * c->ny;
  switch (o->config) {
    case 1: build_c1(*c); break;
    case 2: build_c2(*c, o->n_dfn >= 0 ? o->n_dfn : std::max(1, (int)std::lround(40 * area / 65536.0))); break;
    case 3: build_c3(*c); break;
    case 4: build_c4(*c, o->n_dfn >= 0 ? o->n_dfn : std::max(1, (int)std::lround(400 * area / 262144.0))); break;
    case 5: build_c5(*c); break;
  }
  if (o->n_steps > 0) c->n_steps = o->n_steps;
  return c;
}

void rsim_case_destroy(rsim_case* c) { delete c; }
int64_t rsim_case_n(const rsim_case* c) { return c->n; }
int64_t rsim_case_n_nnc(const rsim_case* c) { return c->nptr.empty() ? 0 : c->nptr[c->n]; }

int rsim_case_dims(const rsim_case* c, int32_t* nxyz, double* dxyz) {
  nxyz[0] = c->nx; nxyz[1] = c->ny; nxyz[2] = c->nz;
  dxyz[0] = c->dx; dxyz[1] = c->dy; dxyz[2] = c->dz;
  return 0;
}

int rsim_case_graph(const rsim_case* c, rsim_graph_desc* g) {
  g->nx = c->nx; g->ny = c->ny; g->nz = c->nz;
  g->tx = c->tx.data(); g->ty = c->ty.data(); g->tz = c->tz.data();
  g->pv = c->pv.data();
  g->kind = c->kind.data();
  bool has = !c->nptr.empty() && c->nptr[c->n] > 0;
  g->nnc_ptr = has ? c->nptr.data() : nullptr;
  g->nnc_nbr = has ? c->nnbr.data() : nullptr;
  g->nnc_t = has ? c->nt.data() : nullptr;
  g->well_wi = c->wi.data();
  g->bhp = c->bhp;
  return 0;
}

int rsim_case_fluid(const rsim_case* c, rsim_fluid_params* f) { *f = c->fl; return 0; }

const double* rsim_case_perm(const rsim_case* c, int32_t axis) {
  return axis == 0 ? c->kx.data() : axis == 1 ? c->ky.data() : c->kz.data();
}

int rsim_case_init_state(const rsim_case* c, double* u, uint8_t* st) {
  const int b = c->fl.kind;
  for (int64_t i = 0; i < c->n; ++i) {
    u[i * b] = c->p_init;
    if (b >= 2) u[i * b + 1] = c->sw_init;
    if (b == 3) u[i * b + 2] = c->fl.rs_b;  // undersaturated oil with bubble point p_bub
    st[i] = (b == 3) ? RSIM_BO_UNDERSAT : 0;
  }
  return 0;
}

// timestep_schedule: Δt_k = min(Δt_0·g^k, Δt_max); with a
// total time T the ramp is truncated so that Σ Δt = T exactly (last step
// shortened); otherwise n_steps steps.
int32_t rsim_case_schedule(const rsim_case* c, double* dts, int32_t cap) {
  double dt = c->dt0;
  int32_t k = 0;
  if (c->total_time > 0.0) {
    double t = 0.0;
    for (; t < c->total_time && k < cap; ++k) {
      double d = std::min(dt, c->dt_max);
      if (t + d >= c->total_time * (1.0 - 1e-12)) d = c->total_time - t;
      dts[k] = d;
      t += d;
      dt *= c->growth;
    }
    return k;
  }
  for (; k < c->n_steps && k < cap; ++k) {
    dts[k] = std::min(dt, c->dt_max);
    dt *= c->growth;
  }
  return k;
}

int rsim_case_solver_opts(const rsim_case* c, rsim_solver_opts* o) {
  std::memset(o, 0, sizeof(*o));
  o->max_newton = 25;
  o->max_outer = 50;
  o->lin_method = RSIM_LIN_BICGSTAB;
  o->precond = RSIM_PREC_NEUMANN1;  // block-Jacobi scaling + 1st-order Neumann polynomial
  o->lin_maxit = 4000;
  o->lin_rtol = 1e-9;
  o->eps_p = c->eps;
  o->eps_set = c->eps;
  o->m = c->m;
  o->fixed_lin_iters = 0;
  return 0;
}

double rsim_case_c5_field(const rsim_case* c, double target, int32_t m, double eps, double* dp, double* R_out) {
  const int64_t n = c->n, nxy = (int64_t)c->nx * c->ny;
  const double W = c->nx * c->dx, H = c->ny * c->dy, Z = c->nz * c->dz;
  double sx[64], sy[64], sz[64];
  for (int s = 0; s < 64; ++s) {
    sx[s] = u01(c->seed, 7, 3 * s) * W;
    sy[s] = u01(c->seed, 7, 3 * s + 1) * H;
    sz[s] = u01(c->seed, 7, 3 * s + 2) * Z;
  }
  std::vector<float> d2(n);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double x = ((i % c->nx) + 0.5) * c->dx, y = (((i / c->nx) % c->ny) + 0.5) * c->dy, z = ((i / nxy) + 0.5) * c->dz;
    double best = 1e300;
    for (int s = 0; s < 64; ++s) {
      double ddx = x - sx[s], ddy = y - sy[s], ddz = z - sz[s];
      best = std::min(best, ddx * ddx + ddy * ddy + ddz * ddz);
    }
    d2[i] = (float)best;
  }
  // post-dilation fraction for a distance threshold rho
  std::vector<uint8_t> a(n), b(n);
  auto frac_for = [&](double rho) {
    float r2 = (float)(rho * rho);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) a[i] = d2[i] <= r2;
    for (int r = 0; r < m; ++r) {
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) {
        int64_t ix = i % c->nx, iy = (i / c->nx) % c->ny, iz = i / nxy;
        uint8_t v = a[i];
        if (!v && ix > 0) v = a[i - 1];
        if (!v && ix < c->nx - 1) v = a[i + 1];
        if (!v && iy > 0) v = a[i - c->nx];
        if (!v && iy < c->ny - 1) v = a[i + c->nx];
        if (!v && iz > 0) v = a[i - nxy];
        if (!v && iz < c->nz - 1) v = a[i + nxy];
        b[i] = v;
      }
      std::swap(a, b);
    }
    int64_t cnt = 0;
#pragma omp parallel for reduction(+ : cnt) schedule(static)
    for (int64_t i = 0; i < n; ++i) cnt += a[i];
    return (double)cnt / (double)n;
  };
  const double kfac = std::sqrt(2.0 * std::log(1.0 / eps));  // δp >= eps  <=>  d <= kfac R
  double lo = 0.0, hi = std::sqrt(W * W + H * H + Z * Z), rho = hi, f = 1.0;
  if (target < 1.0) {
    for (int it = 0; it < 60; ++it) {
      rho = 0.5 * (lo + hi);
      f = frac_for(rho);
      if (std::fabs(f - target) <= 1e-3 * target) break;
      if (f < target) lo = rho; else hi = rho;
    }
  } else {
    f = 1.0;
  }
  double R = rho / kfac;
  if (R_out) *R_out = R;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) dp[i] = std::exp(-(double)d2[i] / (2.0 * R * R));
  return f;
}

}  // extern "C"
