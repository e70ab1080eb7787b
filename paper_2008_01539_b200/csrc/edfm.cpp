// edfm.cpp — case files and the embedded discrete fracture model (EDFM).
//
// Restates, host-only (shared by librsim.so and the oracle library):
//   discretize_fractures(grid, segments)   SPEC.md:52-60 (+ :81, :91)
//   CaseConfig / case-file parsing         SPEC.md:463-466, :522-524 ("flat
//                                          structured-text format: key = value
//                                          sections + fracture table")
//   timestep_schedule with total time      SPEC.md:475-483 (cases.cpp)
//
// EDFM on this repo's Cartesian + NNC graph layout: the 2D
// matrix grid is plane z = 0; the fracture cell of (segment s, matrix cell c)
// sits at (c, plane p) with p = 1, 2, ... the order in which segments reach c,
// so a fracture cell lies "above" its host matrix cell.  Then
//   * matrix-fracture Υ = k_eff·A_f/⟨d⟩ is the z-face (c,0)-(c,1) for p = 1,
//     an NNC otherwise;
//   * fracture-fracture Υ along a segment (TPFA over the pieces' half lengths,
//     cross-section aperture·thickness) is an x/y face of plane p when the two
//     pieces share a plane and an edge, an NNC otherwise;
//   * two segments crossing inside c meet at (c,p)-(c,p') — a z-face when the
//     planes are adjacent, an NNC otherwise — with Υ from the two
//     half-transmissibilities at the intersection point;
//   * every other position of a fracture plane is a DEAD cell (RSIM_KIND_DEAD):
//     no connection (all faces 0), never active, not a graph neighbour and not
//     counted in M_A's n.
// Fracture cells are RSIM_KIND_FRACTURE, hence always active.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "case_impl.h"
#include "rsim/cases.h"

using rsim_case_detail::kCp;
using rsim_case_detail::kDay;
using rsim_case_detail::kPsi;

namespace {

struct Segment {
  double x0, y0, x1, y1, aperture, kf, phi;
};

struct Piece {  // the part of a segment inside one matrix cell
  int ix, iy;
  double ta, tb, len;  // parameter range on the segment, length (m)
  int plane;           // 1.. (fracture plane of its fracture cell)
};

struct CaseError {
  std::string msg;
};

[[noreturn]] void fail(const std::string& m) { throw CaseError{m}; }

// Pieces of segment S in grid cells (exact crossings of the grid lines).
std::vector<Piece> pieces_of(const Segment& S, int nx, int ny, double dx, double dy) {
  const double len = std::hypot(S.x1 - S.x0, S.y1 - S.y0);
  std::vector<double> ts = {0.0, 1.0};
  auto cross = [&](double a0, double a1, double h, int nlines) {
    if (a0 == a1) return;
    for (int k = 1; k < nlines; ++k) {
      const double t = (k * h - a0) / (a1 - a0);
      if (t > 0.0 && t < 1.0) ts.push_back(t);
    }
  };
  cross(S.x0, S.x1, dx, nx);
  cross(S.y0, S.y1, dy, ny);
  std::sort(ts.begin(), ts.end());
  std::vector<Piece> out;
  for (size_t k = 0; k + 1 < ts.size(); ++k) {
    const double ta = ts[k], tb = ts[k + 1];
    const double L = (tb - ta) * len;
    if (!(L > 1e-12 * len)) continue;  // zero-length intersection (a grid corner): skipped
    const double tm = 0.5 * (ta + tb);
    const double mx = S.x0 + (S.x1 - S.x0) * tm, my = S.y0 + (S.y1 - S.y0) * tm;
    const int ix = std::min(nx - 1, std::max(0, (int)std::floor(mx / dx)));
    const int iy = std::min(ny - 1, std::max(0, (int)std::floor(my / dy)));
    if (!out.empty() && out.back().ix == ix && out.back().iy == iy) {
      out.back().tb = tb;
      out.back().len += L;
    } else {
      out.push_back(Piece{ix, iy, ta, tb, L, 0});
    }
  }
  return out;
}

// Intersection parameters (u on A, v on B) of two segments; false if parallel or disjoint.
bool seg_cross(const Segment& A, const Segment& B, double& u, double& v) {
  const double rx = A.x1 - A.x0, ry = A.y1 - A.y0, sx = B.x1 - B.x0, sy = B.y1 - B.y0;
  const double den = rx * sy - ry * sx;
  if (std::fabs(den) <= 1e-14 * std::hypot(rx, ry) * std::hypot(sx, sy)) return false;
  const double qx = B.x0 - A.x0, qy = B.y0 - A.y0;
  u = (qx * sy - qy * sx) / den;
  v = (qx * ry - qy * rx) / den;
  return u >= 0.0 && u <= 1.0 && v >= 0.0 && v <= 1.0;
}

const Piece* piece_at(const std::vector<Piece>& P, double t) {
  for (const Piece& p : P)
    if (t >= p.ta && t <= p.tb) return &p;
  return nullptr;
}

// ⟨d⟩: mean normal distance of the points of cell [cx, cx+dx] x [cy, cy+dy] to the
// line through the segment, 8x8 midpoint quadrature (SPEC.md:59 design decision).
double avg_distance(double cx, double cy, double dx, double dy, const Segment& S) {
  const double len = std::hypot(S.x1 - S.x0, S.y1 - S.y0);
  const double nx_ = -(S.y1 - S.y0) / len, ny_ = (S.x1 - S.x0) / len;
  double sum = 0.0;
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b) {
      const double px = cx + (a + 0.5) * dx / 8.0, py = cy + (b + 0.5) * dy / 8.0;
      sum += std::fabs(nx_ * (px - S.x0) + ny_ * (py - S.y0));
    }
  return sum / 64.0;
}

// ------------------------------------------------------------------ parser
struct Parsed {
  std::map<std::string, std::map<std::string, std::string>> kv;  // section -> key -> value
  std::vector<std::vector<double>> fractures;
};

std::string trim(const std::string& s) {
  size_t a = s.find_first_not_of(" \t\r"), b = s.find_last_not_of(" \t\r");
  return a == std::string::npos ? std::string() : s.substr(a, b - a + 1);
}

Parsed parse(const std::string& text) {
  Parsed P;
  std::string sec;
  std::istringstream in(text);
  std::string line;
  int ln = 0;
  while (std::getline(in, line)) {
    ++ln;
    const size_t h = line.find('#');
    if (h != std::string::npos) line = line.substr(0, h);
    line = trim(line);
    if (line.empty()) continue;
    if (line.front() == '[') {
      if (line.back() != ']') fail("line " + std::to_string(ln) + ": bad section header");
      sec = trim(line.substr(1, line.size() - 2));
      continue;
    }
    if (sec.empty()) fail("line " + std::to_string(ln) + ": entry outside a section");
    if (sec == "fractures") {
      std::istringstream r(line);
      std::vector<double> row;
      double x;
      while (r >> x) row.push_back(x);
      if (!r.eof() || row.size() < 6 || row.size() > 7)
        fail("line " + std::to_string(ln) + ": fracture row needs x0 y0 x1 y1 aperture perm [porosity]");
      P.fractures.push_back(row);
      continue;
    }
    const size_t eq = line.find('=');
    if (eq == std::string::npos) fail("line " + std::to_string(ln) + ": expected key = value");
    P.kv[sec][trim(line.substr(0, eq))] = trim(line.substr(eq + 1));
  }
  return P;
}

struct Getter {
  const Parsed& P;
  bool has(const std::string& s, const std::string& k) const {
    auto it = P.kv.find(s);
    return it != P.kv.end() && it->second.count(k);
  }
  std::string str(const std::string& s, const std::string& k, const std::string& d) const {
    return has(s, k) ? P.kv.at(s).at(k) : d;
  }
  double num(const std::string& s, const std::string& k, double d, bool required = false) const {
    if (!has(s, k)) {
      if (required) fail("missing [" + s + "] " + k);
      return d;
    }
    const std::string v = P.kv.at(s).at(k);
    char* end = nullptr;
    const double x = std::strtod(v.c_str(), &end);
    if (end == v.c_str() || trim(end).size()) fail("[" + s + "] " + k + ": not a number: " + v);
    return x;
  }
  std::vector<double> nums(const std::string& s, const std::string& k) const {
    std::vector<double> out;
    if (!has(s, k)) return out;
    std::istringstream r(P.kv.at(s).at(k));
    double x;
    while (r >> x) out.push_back(x);
    return out;
  }
};

uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// ------------------------------------------------------------------ builder
void build_from(rsim_case& c, const Parsed& P) {
  const Getter G{P};
  c.config = 0;
  c.name = G.str("case", "name", "case");
  c.nx = (int32_t)G.num("grid", "nx", 0, true);
  c.ny = (int32_t)G.num("grid", "ny", 0, true);
  c.dx = G.num("grid", "dx", 0, true);
  c.dy = G.num("grid", "dy", 0, true);
  c.dz = G.num("grid", "thickness", 1.0);  // fractures fully penetrate: 2D areal x thickness
  if (c.nx < 1 || c.ny < 1 || !(c.dx > 0) || !(c.dy > 0) || !(c.dz > 0)) fail("[grid]: non-positive geometry");
  const double W = c.nx * c.dx, H = c.ny * c.dy;
  // ---- segments and their pieces
  std::vector<Segment> segs;
  for (const auto& r : P.fractures) {
    Segment S{r[0], r[1], r[2], r[3], r[4], r[5], r.size() > 6 ? r[6] : 1.0};
    if (!(S.aperture > 0) || !(S.kf > 0) || !(S.phi > 0)) fail("fracture: aperture, permeability and porosity must be > 0");
    if (S.x0 == S.x1 && S.y0 == S.y1) fail("fracture: endpoints must be distinct");
    for (double x : {S.x0, S.x1})
      if (x < 0.0 || x > W) fail("fracture: segment outside the grid");
    for (double y : {S.y0, S.y1})
      if (y < 0.0 || y > H) fail("fracture: segment outside the grid");
    segs.push_back(S);
  }
  std::vector<std::vector<Piece>> pcs(segs.size());
  std::vector<int> planes((size_t)c.nx * c.ny, 0);
  int np = 0;
  for (size_t s = 0; s < segs.size(); ++s) {
    pcs[s] = pieces_of(segs[s], c.nx, c.ny, c.dx, c.dy);
    for (Piece& p : pcs[s]) {
      p.plane = ++planes[(size_t)p.iy * c.nx + p.ix];
      np = std::max(np, p.plane);
    }
  }
  c.nz = 1 + np;
  c.n = (int64_t)c.nx * c.ny * c.nz;
  const int64_t nxy = (int64_t)c.nx * c.ny;
  auto gid = [&](int ix, int iy, int pl) { return (int64_t)pl * nxy + (int64_t)iy * c.nx + ix; };
  // ---- matrix plane
  c.kind.assign(c.n, RSIM_KIND_DEAD);
  c.wi.assign(c.n, 0.0);
  c.phi.assign(c.n, 0.0);
  c.kx.assign(c.n, 0.0);
  c.tx.assign(c.n, 0.0);
  c.ty.assign(c.n, 0.0);
  c.tz.assign(c.n, 0.0);
  c.pv.assign(c.n, 0.0);
  const double phi_m = G.num("rock", "porosity", 0.05);
  const std::vector<double> ln = G.nums("rock", "perm_lognormal");  // geometric mean (m^2), sigma_ln, seed
  const double km_u = G.num("rock", "perm", 1e-19);
  if (!(phi_m > 0) || (ln.empty() && !(km_u > 0))) fail("[rock]: porosity and permeability must be > 0");
  const uint64_t seed = ln.size() > 2 ? (uint64_t)ln[2] : 2008015390ULL;
  for (int64_t i = 0; i < nxy; ++i) {
    c.kind[i] = RSIM_KIND_MATRIX;
    c.phi[i] = phi_m;
    double k = km_u;
    if (!ln.empty()) {  // ln k ~ N(ln kg, sigma^2), Box-Muller on SplitMix64 counters
      auto u01 = [&](uint64_t idx) {
        uint64_t z = mix64(seed + 0x9E3779B97F4A7C15ULL * (0x100000001ULL + idx + 1));
        return ((z >> 11) + 0.5) * (1.0 / 9007199254740992.0);
      };
      const double a = u01(2 * (uint64_t)i), b = u01(2 * (uint64_t)i + 1);
      k = std::exp(std::log(ln[0]) + ln[1] * std::sqrt(-2.0 * std::log(a)) * std::cos(6.283185307179586 * b));
    }
    c.kx[i] = k;
    c.pv[i] = c.dx * c.dy * c.dz * phi_m;
  }
  auto harm = [](double a, double b) { return (a > 0.0 && b > 0.0) ? (a * b) / (a + b) : 0.0; };
  for (int iy = 0; iy < c.ny; ++iy)
    for (int ix = 0; ix < c.nx; ++ix) {  // build_matrix_grid
      const int64_t i = gid(ix, iy, 0);
      if (ix < c.nx - 1) c.tx[i] = harm(c.kx[i] * c.dy * c.dz / (0.5 * c.dx), c.kx[i + 1] * c.dy * c.dz / (0.5 * c.dx));
      if (iy < c.ny - 1)
        c.ty[i] = harm(c.kx[i] * c.dx * c.dz / (0.5 * c.dy), c.kx[i + c.nx] * c.dx * c.dz / (0.5 * c.dy));
    }
  // dead filler cells: a positive pore volume (they are never assembled), nothing else
  for (int64_t i = nxy; i < c.n; ++i) c.pv[i] = c.dx * c.dy * c.dz * phi_m;
  // ---- connections: a Cartesian face when (i, j) are grid neighbours, an NNC otherwise
  auto connect = [&](int64_t i, int64_t j, double T) {
    if (!(T > 0.0) || i == j) return;
    const int64_t a = std::min(i, j), b = std::max(i, j), d = b - a;
    const int64_t ax = a % c.nx, ay = (a / c.nx) % c.ny;
    if (d == 1 && ax < c.nx - 1) c.tx[a] += T;
    else if (d == c.nx && ay < c.ny - 1 && (a / nxy) == (b / nxy)) c.ty[a] += T;
    else if (d == nxy) c.tz[a] += T;
    else c.nnc[{a, b}] += T;
  };
  c.n_frac = 0;
  for (size_t s = 0; s < segs.size(); ++s) {
    const Segment& S = segs[s];
    const double cs = S.aperture * c.dz;  // fracture cross-section
    for (size_t k = 0; k < pcs[s].size(); ++k) {
      const Piece& p = pcs[s][k];
      const int64_t f = gid(p.ix, p.iy, p.plane), m = gid(p.ix, p.iy, 0);
      c.kind[f] = RSIM_KIND_FRACTURE;
      c.phi[f] = S.phi;
      c.kx[f] = S.kf;
      c.pv[f] = p.len * cs * S.phi;
      ++c.n_frac;
      // matrix-fracture: k_eff A_f / <d>, A_f = 2 L h, k_eff = harmonic mean of k_m and k_f
      const double km = c.kx[m];
      const double keff = 2.0 * km * S.kf / (km + S.kf);
      const double dav = avg_distance(p.ix * c.dx, p.iy * c.dy, c.dx, c.dy, S);
      connect(m, f, keff * 2.0 * p.len * c.dz / std::max(dav, 1e-12 * c.dx));
      // fracture-fracture along the segment: half-transmissibilities k_f a h / (L/2)
      if (k > 0) {
        const Piece& q = pcs[s][k - 1];
        const double T1 = S.kf * cs / (0.5 * q.len), T2 = S.kf * cs / (0.5 * p.len);
        connect(gid(q.ix, q.iy, q.plane), f, harm(T1, T2));
      }
    }
  }
  // intersections: Υ from the half-transmissibilities at the intersection point
  for (size_t s = 0; s < segs.size(); ++s)
    for (size_t t = s + 1; t < segs.size(); ++t) {
      double u, v;
      if (!seg_cross(segs[s], segs[t], u, v)) continue;
      const Piece* ps = piece_at(pcs[s], u);
      const Piece* pt = piece_at(pcs[t], v);
      if (!ps || !pt) continue;
      auto half = [&](const Segment& S, const Piece& p, double tx) {
        const double len = std::hypot(S.x1 - S.x0, S.y1 - S.y0);
        const double L1 = (tx - p.ta) * len, L2 = (p.tb - tx) * len;
        const double d = std::max((L1 * L1 + L2 * L2) / (2.0 * (L1 + L2)), 1e-12 * c.dx);
        return S.kf * S.aperture * c.dz / d;
      };
      connect(gid(ps->ix, ps->iy, ps->plane), gid(pt->ix, pt->iy, pt->plane),
              harm(half(segs[s], *ps, u), half(segs[t], *pt, v)));
    }
  c.n_dead = 0;
  for (int64_t i = 0; i < c.n; ++i) c.n_dead += c.kind[i] == RSIM_KIND_DEAD;
  // ---- fluid, rock compressibility, initial state, well
  const std::string model = G.str("fluid", "model", "oilwater");
  c.p_init = G.num("initial", "pressure", 0, true) * kPsi;
  if (model == "single") rsim_case_fluid_single(c);
  else if (model == "oilwater") rsim_case_fluid_oilwater(c);
  else fail("[fluid] model must be single or oilwater");
  rsim_fluid_params& f = c.fl;
  f.p_ref = c.p_init;
  f.c_r = G.num("rock", "c_r", 0.0) / kPsi;
  f.mu[0] = G.num("fluid", "mu_w", 0.5) * kCp;
  f.mu[1] = G.num("fluid", "mu_o", 1.0) * kCp;
  f.c_f[0] = G.num("fluid", "c_w", 1e-9 * kPsi) / kPsi;
  f.c_f[1] = G.num("fluid", "c_o", 1e-9 * kPsi) / kPsi;
  f.rho_ref[0] = G.num("fluid", "rho_w", 1000.0);
  f.rho_ref[1] = G.num("fluid", "rho_o", 800.0);
  if (model == "oilwater") {
    f.swc = G.num("fluid", "swc", 0.2);
    f.sor = G.num("fluid", "sor", 0.2);
  }
  c.sw_init = G.num("initial", "sw", model == "oilwater" ? f.swc : 0.0);
  c.bhp = G.num("well", "bhp", 0, true) * kPsi;
  const double wi = G.num("well", "wi", 1e-11);
  const std::vector<double> tr = G.nums("well", "trajectory");  // x0 y0 x1 y1: perforates the fracture cells it crosses
  if (tr.size() != 4) fail("[well] trajectory = x0 y0 x1 y1");
  const Segment Wl{tr[0], tr[1], tr[2], tr[3], 1.0, 1.0, 1.0};
  int nperf = 0;
  for (size_t s = 0; s < segs.size(); ++s) {
    double u, v;
    if (!seg_cross(segs[s], Wl, u, v)) continue;
    const Piece* p = piece_at(pcs[s], u);
    if (!p) continue;
    c.wi[gid(p->ix, p->iy, p->plane)] = wi;
    ++nperf;
  }
  if (nperf == 0) fail("[well] trajectory crosses no fracture");
  // ---- time and solver defaults
  c.total_time = G.num("time", "total", 0, true) * kDay;
  c.dt0 = G.num("time", "dt0", 0.1) * kDay;
  c.growth = G.num("time", "growth", 1.2);
  c.dt_max = G.num("time", "dt_max", 100.0) * kDay;
  if (!(c.dt0 > 0) || !(c.dt0 <= c.dt_max) || !(c.dt_max <= c.total_time) || !(c.growth >= 1.0))
    fail("[time]: need 0 < dt0 <= dt_max <= total and growth >= 1");
  c.n_steps = 0;
  const std::string sv = G.str("solver", "solver", "localized");
  c.solver = sv == "standard" ? 0 : sv == "localized" ? 1 : sv == "adaptive_dd" ? 2 : -1;
  if (c.solver < 0) fail("[solver] solver must be standard, localized or adaptive_dd");
  c.m = (int)G.num("solver", "m", c.solver == 2 ? 4 : 2);
  c.eps = G.num("solver", "eps_p", 0.3) * kPsi;
  c.ky = c.kx;
  c.kz = c.kx;
  rsim_case_finalize_nnc(c);
}

rsim_case* from_text(const std::string& text, char* err, int32_t errlen) {
  rsim_case* c = new rsim_case();
  try {
    build_from(*c, parse(text));
    return c;
  } catch (const CaseError& e) {
    if (err && errlen > 0) std::snprintf(err, (size_t)errlen, "%s", e.msg.c_str());
    delete c;
    return nullptr;
  }
}

}  // namespace

extern "C" {

rsim_case* rsim_case_from_text(const char* text, char* err, int32_t errlen) {
  if (!text) return nullptr;
  return from_text(text, err, errlen);
}

rsim_case* rsim_case_from_file(const char* path, char* err, int32_t errlen) {
  std::ifstream f(path ? path : "");
  if (!f) {
    if (err && errlen > 0) std::snprintf(err, (size_t)errlen, "cannot read case file %s", path ? path : "(null)");
    return nullptr;
  }
  std::stringstream ss;
  ss << f.rdbuf();
  return from_text(ss.str(), err, errlen);
}

int rsim_case_info(const rsim_case* c, rsim_case_info_t* out) {
  if (!c || !out) return RSIM_EARG;
  out->n_live = c->n - c->n_dead;
  out->n_frac = c->n_frac;
  out->n_dead = c->n_dead;
  out->solver = c->solver;
  out->m = c->m;
  out->eps_p = c->eps;
  out->total_time = c->total_time;
  return RSIM_OK;
}

// Every connection of the graph with Υ > 0 (Cartesian faces + NNCs), i < j.
int64_t rsim_case_connections(const rsim_case* c, int32_t* ci, int32_t* cj, double* ct, int64_t cap) {
  int64_t k = 0;
  auto put = [&](int64_t i, int64_t j, double T) {
    if (!(T > 0.0)) return;
    if (k < cap && ci) { ci[k] = (int32_t)i; cj[k] = (int32_t)j; ct[k] = T; }
    ++k;
  };
  const int64_t nxy = (int64_t)c->nx * c->ny;
  for (int64_t i = 0; i < c->n; ++i) {
    const int64_t ix = i % c->nx, iy = (i / c->nx) % c->ny, iz = i / nxy;
    if (ix < c->nx - 1) put(i, i + 1, c->tx[i]);
    if (iy < c->ny - 1) put(i, i + c->nx, c->ty[i]);
    if (iz < c->nz - 1) put(i, i + nxy, c->tz[i]);
    if (!c->nptr.empty())
      for (int32_t q = c->nptr[i]; q < c->nptr[i + 1]; ++q)
        if (c->nnbr[q] > i) put(i, c->nnbr[q], c->nt[q]);
  }
  return k;
}

double rsim_edfm_avg_distance(double cx, double cy, double dx, double dy, double x0, double y0, double x1,
                              double y1) {
  return avg_distance(cx, cy, dx, dy, Segment{x0, y0, x1, y1, 1.0, 1.0, 1.0});
}

}  // extern "C"
