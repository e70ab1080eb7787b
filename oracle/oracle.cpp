// oracle/oracle.cpp — CPU restatement of the localized FIM Newton path.
//
// TEST INFRASTRUCTURE ONLY (see oracle_api.h): the parity checker for the
// sm_100a product path, and the CPU baseline that bench.py times.
//
// Restates (reference = /root/reference, no implementation ships there):
//   build_matrix_grid
//   neighbor_set             SPEC.md:61-69 (graph distance)
//   assemble                 SPEC.md:269-277, PAPER.md:252-256 (Eq. 16), :861-884
//   solve                    SPEC.md:311-319, replaced by BiCGSTAB per the north
//                            star (BASELINE.json), block-Jacobi-scaled system
//   support_set              SPEC.md:359-367 (Eq. 14, inclusive >=)
//   boundary_layer
//   outer_halo
//   expand_active
//   newton_standard
//   newton_localized         SPEC.md:404-412, Algorithm 1 PAPER.md:273-308,
//                            decisions SPEC.md:440-447, :455
//   adaptive_nonlinear_dd    SPEC.md:413-430, Algorithm 2 PAPER.md:372-442,
//                            decisions SPEC.md:444, :456
//   timestep cut / run_case
//
// Shared with the product: ONLY include/rsim/physics.h, include/rsim/eos.h (cell-local
// constitutive relations) and include/rsim/blockops.h (b×b block arithmetic
// and the canonical reduction order).  Traversal, set logic, Krylov and
// Newton control below are written independently of the CUDA code.
#include "oracle_api.h"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <deque>
#include <vector>

#include "rsim/blockops.h"
#include "rsim/physics.h"

using namespace rsim;

namespace {

struct Graph {
  int32_t nx = 0, ny = 0, nz = 0;
  int64_t n = 0;
  bool d3 = false;
  int nslot = 0;
  std::vector<double> tx, ty, tz, pv, wi;
  std::vector<uint8_t> kind, pinned, dead;  // dead: RSIM_KIND_DEAD filler cells (no connections)
  int64_t n_live = 0;                       // cells of the model (n minus dead fillers): M_A's n
  std::vector<int32_t> nptr, nnbr;
  std::vector<double> nt;
  bool has_nnc = false;
  double bhp = 0.0;

  // Canonical connection order of a cell: Cartesian neighbours in ascending
  // column order (-z,-y,-x,+x,+y,+z), then NNCs in ascending neighbour order.
  template <class F>
  void each(int64_t i, F&& f) const {
    const int64_t nxy = (int64_t)nx * ny;
    const int64_t ix = i % nx, iy = (i / nx) % ny, iz = i / nxy;
    if (d3 && iz > 0) f(i - nxy, tz[i - nxy]);
    if (iy > 0) f(i - nx, ty[i - nx]);
    if (ix > 0) f(i - 1, tx[i - 1]);
    if (ix < nx - 1) f(i + 1, tx[i]);
    if (iy < ny - 1) f(i + nx, ty[i]);
    if (d3 && iz < nz - 1) f(i + nxy, tz[i]);
    if (has_nnc)
      for (int32_t q = nptr[i]; q < nptr[i + 1]; ++q) f((int64_t)nnbr[q], nt[q]);
  }
  // Graph neighbours for the set logic: as each(), without the
  // structural Cartesian neighbours that are dead filler cells (EDFM planes).
  template <class F>
  void each_live(int64_t i, F&& f) const {
    each(i, [&](int64_t j, double T) { if (!dead[j]) f(j, T); });
  }
};

struct Model {
  Graph g;
  phys::Fluid fl;  // params + reciprocals (physics.h)
  int b = 1;
  std::vector<double> u, mold, dp;
  std::vector<uint8_t> st;
  double dt = 1.0;
  // last assembled local system
  int32_t nA = 0;
  std::vector<int32_t> act, g2l, rowptr, col;
  std::vector<double> val, Fraw, rhs;
  int bad_cell = -1;
  bool raw = false;            // unscaled assembly (property tests)
  std::vector<double> diag;    // raw diagonal blocks when raw
};

// ---------------------------------------------------------------- reductions
// Canonical reduction (blockops.h): 256-row chunks, warp trees with offsets
// 16..1, then the 8 warp sums with offsets 4..1; recursive over partials.
static double chunk_tree(double* t) {
  double w[8];
  for (int wp = 0; wp < 8; ++wp) {
    double* L = t + 32 * wp;
    for (int off = 16; off >= 1; off >>= 1)
      for (int lane = 0; lane < off; ++lane) L[lane] = L[lane] + L[lane + off];
    w[wp] = L[0];
  }
  for (int off = 4; off >= 1; off >>= 1)
    for (int k = 0; k < off; ++k) w[k] = w[k] + w[k + off];
  return w[0];
}

template <class RowFn>
static double chunk_reduce_fn(int64_t base, int64_t m, RowFn&& fn) {
  double t[256];
  for (int th = 0; th < 256; ++th) t[th] = th < m ? fn(base + th) : 0.0;
  return chunk_tree(t);
}

static double canon_sum_arr(const double* v, int64_t n);

template <class RowFn>
static double canon_reduce(int64_t n, RowFn&& fn) {
  if (n <= RSIM_RED_CHUNK) return chunk_reduce_fn(0, n, fn);
  int64_t nc = (n + RSIM_RED_CHUNK - 1) / RSIM_RED_CHUNK;
  std::vector<double> part(nc);
#pragma omp parallel for schedule(static)
  for (int64_t c = 0; c < nc; ++c)
    part[c] = chunk_reduce_fn(c * RSIM_RED_CHUNK, std::min<int64_t>(RSIM_RED_CHUNK, n - c * RSIM_RED_CHUNK), fn);
  return canon_sum_arr(part.data(), nc);
}

static double canon_sum_arr(const double* v, int64_t n) {
  return canon_reduce(n, [v](int64_t l) { return v[l]; });
}

// ---------------------------------------------------------------- set ops
static std::vector<int32_t> to_list(const std::vector<uint8_t>& f) {
  std::vector<int32_t> out;
  for (int64_t i = 0; i < (int64_t)f.size(); ++i)
    if (f[i]) out.push_back((int32_t)i);
  return out;
}

// Multi-source BFS truncated at depth m (neighbor_set).
static void dilate(const Graph& g, const std::vector<int32_t>& seeds, int m, std::vector<uint8_t>& mark) {
  std::vector<int32_t> dist(g.n, -1);
  std::deque<int32_t> q;
  for (int32_t s : seeds)
    if (dist[s] < 0) { dist[s] = 0; q.push_back(s); }
  while (!q.empty()) {
    int32_t i = q.front();
    q.pop_front();
    mark[i] = 1;
    if (dist[i] >= m) continue;
    g.each_live(i, [&](int64_t j, double) {
      if (dist[j] < 0) { dist[j] = dist[i] + 1; q.push_back((int32_t)j); }
    });
  }
}

static std::vector<uint8_t> boundary_of(const Graph& g, const std::vector<uint8_t>& A) {
  std::vector<uint8_t> B(g.n, 0);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < g.n; ++i) {
    if (!A[i]) continue;
    bool out = false;
    g.each_live(i, [&](int64_t j, double) { if (!A[j]) out = true; });
    B[i] = out;
  }
  return B;
}

// ---------------------------------------------------------------- assembly
template <int B>
static bool assemble_row(Model& M, int32_t l) {
  const Graph& g = M.g;
  const int64_t i = M.act[l];
  const double* ui = &M.u[i * B];
  phys::Props<B> Pi;
  phys::props(M.fl, ui, M.st[i], Pi);
  double R[B], D[B][B], O[B][B];
  phys::accum_row<B>(M.fl, g.pv[i], ui[0], Pi, &M.mold[i * B], 1.0 / M.dt, R, D);
  int64_t pos = M.rowptr[l];
  g.each(i, [&](int64_t j, double T) {
    const double* uj = &M.u[j * B];
    double dpij = ui[0] - uj[0];
    bool up_i = !(dpij < 0.0);
    if (up_i) {
      phys::flux_conn<B>(T, dpij, true, Pi, R, D, O);
    } else {
      phys::Props<B> Pj;
      phys::props(M.fl, uj, M.st[j], Pj);
      phys::flux_conn<B>(T, dpij, false, Pj, R, D, O);
    }
    if (M.g2l[j] >= 0) {
      M.col[pos] = M.g2l[j];
      double* V = &M.val[pos * B * B];
      for (int r = 0; r < B; ++r)
        for (int c = 0; c < B; ++c) V[r * B + c] = O[r][c];
      ++pos;
    }
  });
  phys::well_row<B>(g.wi[i], ui[0], g.bhp, Pi, R, D);
  if (M.raw) {
    for (int e = 0; e < B; ++e) {
      M.Fraw[(int64_t)l * B + e] = R[e];
      for (int v = 0; v < B; ++v) M.diag[((int64_t)l * B + e) * B + v] = D[e][v];
    }
    return true;
  }
  double Di[B][B];
  if (!blk::inv(D, Di)) return false;
  double y[B];
  blk::gemv<B>(Di, R, y);
  for (int e = 0; e < B; ++e) {
    M.Fraw[(int64_t)l * B + e] = R[e];
    M.rhs[(int64_t)l * B + e] = -y[e];
  }
  for (int64_t p = M.rowptr[l]; p < M.rowptr[l + 1]; ++p) {
    double* V = &M.val[p * B * B];
    double Oc[B][B], S[B][B];
    for (int r = 0; r < B; ++r)
      for (int c = 0; c < B; ++c) Oc[r][c] = V[r * B + c];
    blk::gemm<B>(Di, Oc, S);
    for (int r = 0; r < B; ++r)
      for (int c = 0; c < B; ++c) V[r * B + c] = S[r][c];
  }
  return true;
}

template <int B>
static int assemble(Model& M, const int32_t* act, int32_t nA) {
  const Graph& g = M.g;
  for (int32_t l = 0; l < M.nA; ++l) M.g2l[M.act[l]] = -1;
  M.act.assign(act, act + nA);
  M.nA = nA;
  for (int32_t l = 0; l < nA; ++l) M.g2l[act[l]] = l;
  M.rowptr.assign(nA + 1, 0);
#pragma omp parallel for schedule(static)
  for (int32_t l = 0; l < nA; ++l) {
    int32_t c = 0;
    g.each(act[l], [&](int64_t j, double) { if (M.g2l[j] >= 0) ++c; });
    M.rowptr[l + 1] = c;
  }
  for (int32_t l = 0; l < nA; ++l) M.rowptr[l + 1] += M.rowptr[l];
  int64_t nnzb = M.rowptr[nA];
  M.col.assign(nnzb, 0);
  M.val.assign(nnzb * B * B, 0.0);
  M.Fraw.assign((int64_t)nA * B, 0.0);
  M.rhs.assign((int64_t)nA * B, 0.0);
  if (M.raw) M.diag.assign((int64_t)nA * B * B, 0.0);
  int32_t bad = -1;
#pragma omp parallel for schedule(static)
  for (int32_t l = 0; l < nA; ++l)
    if (!assemble_row<B>(M, l)) {
#pragma omp critical
      if (bad < 0 || act[l] < bad) bad = act[l];
    }
  M.bad_cell = bad;
  return bad >= 0 ? -RSIM_ENUM : 0;
}

static int assemble_any(Model& M, const int32_t* act, int32_t nA) {
  switch (M.b) {
    case 1: return assemble<1>(M, act, nA);
    case 2: return assemble<2>(M, act, nA);
    default: return assemble<3>(M, act, nA);
  }
}

// ---------------------------------------------------------------- Krylov
template <int B>
static void spmv(const Model& M, const double* x, double* y) {
#pragma omp parallel for schedule(static)
  for (int32_t l = 0; l < M.nA; ++l) {
    double acc[B];
    for (int c = 0; c < B; ++c) acc[c] = x[(int64_t)l * B + c];
    for (int64_t p = M.rowptr[l]; p < M.rowptr[l + 1]; ++p)
      blk::gemv_acc_flat<B>(&M.val[p * B * B], &x[(int64_t)M.col[p] * B], acc);
    for (int c = 0; c < B; ++c) y[(int64_t)l * B + c] = acc[c];
  }
}

template <int B>
static double dotc(int64_t nrows, const double* a, const double* b) {
  return canon_reduce(nrows, [a, b](int64_t l) { return blk::rowdot<B>(a + l * B, b + l * B); });
}

// Block ILU(0) of the unit-block-diagonal Â in the local (natural) ordering
// (north star "level-scheduled ILU(0)"): rows in ascending
// order (IKJ); row i: for each lower entry k (ascending column) L_ik = A_ik
// D_k^{-1}, then A_ij -= L_ik U_kj over row k's upper entries (ascending j) that
// exist in row i (j == i: the diagonal block).  A GPU level schedule computes
// each row with exactly these operations in this order, so the factors and the
// triangular solves are bit-identical whatever the schedule.
template <int B>
struct Ilu0 {
  std::vector<int64_t> ptr;   // rows: entries sorted by column, diagonal excluded
  std::vector<int32_t> col;
  std::vector<double> val;    // L (col < row) / U (col > row) blocks
  std::vector<double> dinv;   // inverse diagonal blocks of U
  std::vector<double> tmp;
};

template <int B>
static bool ilu0_factor(const Model& M, Ilu0<B>& F) {
  const int32_t n = M.nA;
  constexpr int BB = B * B;
  F.ptr.assign(n + 1, 0);
  F.col.resize(M.col.size());
  F.val.resize(M.val.size());
  for (int32_t l = 0; l < n; ++l) {
    const int64_t a = M.rowptr[l], e = M.rowptr[l + 1];
    std::vector<std::pair<int32_t, int64_t>> ent;
    for (int64_t p = a; p < e; ++p) ent.emplace_back(M.col[p], p);
    std::stable_sort(ent.begin(), ent.end(), [](auto& x, auto& y) { return x.first < y.first; });
    F.ptr[l + 1] = e;
    for (int64_t k = 0; k < e - a; ++k) {
      F.col[a + k] = ent[k].first;
      for (int q = 0; q < BB; ++q) F.val[(a + k) * BB + q] = M.val[ent[k].second * BB + q];
    }
  }
  F.dinv.assign((int64_t)n * BB, 0.0);
  std::vector<double> dg(BB);
  for (int32_t i = 0; i < n; ++i) {
    for (int q = 0; q < BB; ++q) dg[q] = (q % (B + 1) == 0) ? 1.0 : 0.0;
    for (int64_t p = F.ptr[i]; p < F.ptr[i + 1] && F.col[p] < i; ++p) {
      const int32_t k = F.col[p];
      double L[BB];
      blk::gemm_flat<B>(&F.val[p * BB], &F.dinv[(int64_t)k * BB], L);
      for (int q = 0; q < BB; ++q) F.val[p * BB + q] = L[q];
      for (int64_t r = F.ptr[k]; r < F.ptr[k + 1]; ++r) {
        const int32_t j = F.col[r];
        if (j <= k) continue;
        if (j == i) {
          blk::gemm_sub_flat<B>(L, &F.val[r * BB], dg.data());
        } else {
          for (int64_t t = F.ptr[i]; t < F.ptr[i + 1]; ++t)
            if (F.col[t] == j) { blk::gemm_sub_flat<B>(L, &F.val[r * BB], &F.val[t * BB]); break; }
        }
      }
    }
    if (!blk::inv_flat<B>(dg.data(), &F.dinv[(int64_t)i * BB])) return false;
  }
  F.tmp.assign((int64_t)n * B, 0.0);
  return true;
}

// out = (LU)^{-1} z: forward (unit L) then backward (U) substitution
template <int B>
static void ilu0_apply(const Ilu0<B>& F, int32_t n, const double* z, double* out, std::vector<double>& y) {
  constexpr int BB = B * B;
  for (int32_t i = 0; i < n; ++i) {
    double t[B];
    for (int c = 0; c < B; ++c) t[c] = z[(int64_t)i * B + c];
    for (int64_t p = F.ptr[i]; p < F.ptr[i + 1] && F.col[p] < i; ++p)
      blk::gemv_sub_flat<B>(&F.val[p * BB], &y[(int64_t)F.col[p] * B], t);
    for (int c = 0; c < B; ++c) y[(int64_t)i * B + c] = t[c];
  }
  for (int32_t i = n - 1; i >= 0; --i) {
    double t[B];
    for (int c = 0; c < B; ++c) t[c] = y[(int64_t)i * B + c];
    for (int64_t p = F.ptr[i]; p < F.ptr[i + 1]; ++p)
      if (F.col[p] > i) blk::gemv_sub_flat<B>(&F.val[p * BB], &out[(int64_t)F.col[p] * B], t);
    blk::gemv_flat<B>(&F.dinv[(int64_t)i * BB], t, &out[(int64_t)i * B]);
  }
}

// BiCGSTAB (van der Vorst) on the scaled system  Â x = rhs,  x0 = 0.
// Element formulas and reduction order are the contract the GPU kernel
// (csrc/krylov.cu) follows.
template <int B>
static int bicgstab_once(const Model& M, const rsim_solver_opts& o, int pk, double* x, int32_t* iters,
                         double* relres) {
  const int64_t nr = M.nA, N = nr * B;
  const bool neu = pk != RSIM_PREC_BJACOBI;  // a preconditioner on top of the fused block-Jacobi
  std::vector<double> r(M.rhs), r0(M.rhs), p(N, 0.0), v(N, 0.0), s(N), t(N), ph, sh, y;
  if (neu) { ph.assign(N, 0.0); sh.assign(N, 0.0); y.assign(N, 0.0); }
  Ilu0<B> F;
  if (pk == RSIM_PREC_ILU0 && !ilu0_factor<B>(M, F)) { *iters = 0; return RSIM_ENUM; }
  // Neumann-1: M^{-1} z = z + (z - Â z) (first-order polynomial on the unit-diagonal system);
  // ILU(0): M^{-1} z = (LU)^{-1} z
  auto prec = [&](const std::vector<double>& z, std::vector<double>& out) {
    if (pk == RSIM_PREC_ILU0) {
      ilu0_apply<B>(F, M.nA, z.data(), out.data(), y);
      return;
    }
    spmv<B>(M, z.data(), y.data());
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < N; ++e) out[e] = z[e] + (z[e] - y[e]);
  };
  std::fill(x, x + N, 0.0);
  double bb = dotc<B>(nr, r.data(), r.data());
  double bnorm = std::sqrt(bb);
  *iters = 0;
  *relres = 0.0;
  if (bnorm == 0.0) return RSIM_OK;
  const bool fixed = o.fixed_lin_iters > 0;
  const int maxit = fixed ? o.fixed_lin_iters : o.lin_maxit;
  const double tol = o.lin_rtol * bnorm;
  // Two global reductions per iteration: (r0,v) travels with
  // the LAGGED (r,r) of the previous iterate, and rho_{k+1} = (r0,s) - w (r0,t)
  // is formed from quantities reduced together with (s,s), (t,s), (t,t).
  double rho = 1.0, alpha = 1.0, omega = 1.0, rho_new = bb;
  for (int it = 1; it <= maxit; ++it) {
    if (it == 1) {
#pragma omp parallel for schedule(static)
      for (int64_t e = 0; e < N; ++e) p[e] = r[e];
    } else {
      double beta = (rho_new / rho) * (alpha / omega);
#pragma omp parallel for schedule(static)
      for (int64_t e = 0; e < N; ++e) p[e] = r[e] + beta * (p[e] - omega * v[e]);
    }
    const std::vector<double>& pp = neu ? (prec(p, ph), ph) : p;
    spmv<B>(M, pp.data(), v.data());
    double r0v = dotc<B>(nr, r0.data(), v.data());
    if (it > 1) {  // convergence of the previous iterate (reduced with (r0,v))
      const double rr = dotc<B>(nr, r.data(), r.data());
      if (!fixed && std::sqrt(rr) <= tol) {
        *iters = it - 1;
        *relres = std::sqrt(rr) / bnorm;
        return RSIM_OK;
      }
    }
    if (r0v == 0.0 || !std::isfinite(r0v)) { *iters = it; return RSIM_ENUM; }
    alpha = rho_new / r0v;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < N; ++e) s[e] = r[e] - alpha * v[e];
    const std::vector<double>& ss_ = neu ? (prec(s, sh), sh) : s;
    spmv<B>(M, ss_.data(), t.data());
    double ss = dotc<B>(nr, s.data(), s.data());
    double ts = dotc<B>(nr, t.data(), s.data());
    double tt = dotc<B>(nr, t.data(), t.data());
    double r0s = dotc<B>(nr, r0.data(), s.data());
    double r0t = dotc<B>(nr, r0.data(), t.data());
    if (!fixed && std::sqrt(ss) <= tol) {
#pragma omp parallel for schedule(static)
      for (int64_t e = 0; e < N; ++e) x[e] = x[e] + alpha * pp[e];
      *iters = it;
      *relres = std::sqrt(ss) / bnorm;
      return RSIM_OK;
    }
    if (tt == 0.0 || !std::isfinite(tt)) { *iters = it; return RSIM_ENUM; }
    omega = ts / tt;
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < N; ++e) {
      x[e] = (x[e] + alpha * pp[e]) + omega * ss_[e];
      r[e] = s[e] - omega * t[e];
    }
    rho = rho_new;
    rho_new = r0s - omega * r0t;
    *iters = it;
    if (omega == 0.0 || rho_new == 0.0 || !std::isfinite(rho_new)) return RSIM_ENUM;
  }
  {  // iteration cap: residual of the last iterate
    const double rr = dotc<B>(nr, r.data(), r.data());
    *relres = std::sqrt(rr) / bnorm;
    if (!fixed && std::sqrt(rr) <= tol) return RSIM_OK;
  }
  return fixed ? RSIM_OK : RSIM_ENOCONV;
}

// GMRES(m), m = RSIM_GMRES_M, right-preconditioned (block-Jacobi fused into Â:
// M = I; or the Neumann-1 polynomial), x0 = 0, classical Gram-Schmidt (the
// j+1 projections (w, v_i) are reduced together, then w -= Σ h_ij v_i in
// ascending i), Givens rotations on the Hessenberg column, restart from the
// true residual r = b − Â x.  Convergence on the Givens residual estimate
// |g_{j+1}| <= rtol·‖b‖ (also a happy breakdown h_{j+1,j} = 0).  Element
// formulas and reduction order are the contract krylov_gmres.cu follows.
template <int B>
static int gmres(const Model& M, const rsim_solver_opts& o, int pk, double* x, int32_t* iters, double* relres) {
  constexpr int MM = RSIM_GMRES_M;
  const int64_t nr = M.nA, N = nr * B;
  std::vector<double> r(M.rhs), V((int64_t)(MM + 1) * N), z(N), w(N), y(N), u(N);
  Ilu0<B> F;
  if (pk == RSIM_PREC_ILU0 && !ilu0_factor<B>(M, F)) { *iters = 0; return RSIM_ENUM; }
  auto prec = [&](const double* in, double* out) {  // out = M^{-1} in
    if (pk == RSIM_PREC_BJACOBI) {
      std::copy(in, in + N, out);
      return;
    }
    if (pk == RSIM_PREC_ILU0) {
      ilu0_apply<B>(F, M.nA, in, out, y);
      return;
    }
    spmv<B>(M, in, y.data());
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < N; ++e) out[e] = in[e] + (in[e] - y[e]);
  };
  std::fill(x, x + N, 0.0);
  double beta = std::sqrt(dotc<B>(nr, r.data(), r.data()));
  const double bnorm = beta;
  *iters = 0;
  *relres = 0.0;
  if (bnorm == 0.0) return RSIM_OK;
  const bool fixed = o.fixed_lin_iters > 0;
  const int maxit = fixed ? o.fixed_lin_iters : o.lin_maxit;
  const double tol = o.lin_rtol * bnorm;
  double H[MM + 1][MM], cs[MM], sn[MM], g[MM + 1], yy[MM];
  int total = 0;
  for (;;) {
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < N; ++e) V[e] = r[e] / beta;
    for (int q = 0; q <= MM; ++q) g[q] = 0.0;
    g[0] = beta;
    int k = 0;
    bool done = false;
    double resid = beta;
    for (int j = 0; j < MM; ++j) {
      const double* vj = &V[(int64_t)j * N];
      prec(vj, z.data());
      spmv<B>(M, z.data(), w.data());
      for (int i = 0; i <= j; ++i) H[i][j] = dotc<B>(nr, w.data(), &V[(int64_t)i * N]);
#pragma omp parallel for schedule(static)
      for (int64_t e = 0; e < N; ++e) {
        double we = w[e];
        for (int i = 0; i <= j; ++i) we = we - H[i][j] * V[(int64_t)i * N + e];
        w[e] = we;
      }
      const double hn = std::sqrt(dotc<B>(nr, w.data(), w.data()));
      H[j + 1][j] = hn;
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * H[i][j] + sn[i] * H[i + 1][j];
        H[i + 1][j] = -sn[i] * H[i][j] + cs[i] * H[i + 1][j];
        H[i][j] = t;
      }
      const double den = std::sqrt(H[j][j] * H[j][j] + hn * hn);
      if (den == 0.0 || !std::isfinite(den)) { *iters = total + 1; return RSIM_ENUM; }
      cs[j] = H[j][j] / den;
      sn[j] = hn / den;
      H[j][j] = cs[j] * H[j][j] + sn[j] * hn;
      H[j + 1][j] = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++total;
      k = j + 1;
      resid = std::fabs(g[j + 1]);
      if (hn == 0.0 || (!fixed && resid <= tol) || total >= maxit) { done = true; break; }
#pragma omp parallel for schedule(static)
      for (int64_t e = 0; e < N; ++e) V[(int64_t)(j + 1) * N + e] = w[e] / hn;
    }
    for (int i = k - 1; i >= 0; --i) {  // back substitution
      double t = g[i];
      for (int l = i + 1; l < k; ++l) t = t - H[i][l] * yy[l];
      yy[i] = t / H[i][i];
    }
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < N; ++e) {
      double ue = yy[0] * V[e];
      for (int i = 1; i < k; ++i) ue = ue + yy[i] * V[(int64_t)i * N + e];
      u[e] = ue;
    }
    prec(u.data(), z.data());
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < N; ++e) x[e] = x[e] + z[e];
    *iters = total;
    *relres = resid / bnorm;
    if (done && (fixed ? total >= maxit : (resid <= tol || resid == 0.0))) return RSIM_OK;
    if (total >= maxit) return fixed ? RSIM_OK : RSIM_ENOCONV;
    // restart from the true residual
    spmv<B>(M, x, y.data());
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < N; ++e) r[e] = M.rhs[e] - y[e];
    beta = std::sqrt(dotc<B>(nr, r.data(), r.data()));
    if (beta == 0.0) return RSIM_OK;
  }
}

// Neumann-1 preconditioned solve with a deterministic fallback: if it breaks
// down or hits the cap, the solve restarts from x0 = 0 with block-Jacobi only
// (the Neumann polynomial is not guaranteed positive on non-M-matrix blocks,
// e.g. black-oil).  Iterations of both attempts are reported.
template <int B>
static int bicgstab(const Model& M, const rsim_solver_opts& o, double* x, int32_t* iters, double* relres) {
  const int pk = o.precond;
  const bool gm = o.lin_method == RSIM_LIN_GMRES;
  auto once = [&](int k, int32_t* it) {
    return gm ? gmres<B>(M, o, k, x, it, relres) : bicgstab_once<B>(M, o, k, x, it, relres);
  };
  int st = once(pk, iters);
  if (pk != RSIM_PREC_BJACOBI && (st == RSIM_ENUM || st == RSIM_ENOCONV)) {
    int32_t it2 = 0;
    st = once(RSIM_PREC_BJACOBI, &it2);
    *iters += it2;
  }
  return st;
}

// Exact solve of the assembled system (SPEC.md:311-325:
// solve(J, F) "exact" for small active systems, the Krylov cross-check).
// Dense LU with partial pivoting of Â = D⁻¹J (unit block diagonal + the scaled
// off-diagonal blocks; entries of one row block added in CSR order), column-
// major, right-looking, k ascending:
//   pivot  = the first row i ≥ k of maximal |w_ik| (any non-finite entry in the
//            column, or a zero pivot => RSIM_ENUM);
//   swap rows k and piv across ALL columns (multipliers included);
//   l_ik   = w_ik / w_kk  (a division, stored in place);
//   w_ij   = w_ij − l_ik·w_kj for j > k, i > k (one product, one subtraction).
// Solve: b ← P b (the swaps in k order); forward, column-oriented:
// b_i −= l_ik·b_k (k ascending); backward: b_k /= u_kk, then b_i −= u_ik·b_k for
// i < k (k descending).  Every w_ij sees its updates in k order, so any
// schedule that keeps that order (the GPU: one column owner per CTA, one grid
// barrier per k) reproduces these bits.  iters = 1, relres = 0 (not formed).
template <int B>
static int direct_solve(Model& M, double* x, int32_t* iters, double* relres) {
  *iters = 1;
  *relres = 0.0;
  const int64_t N = (int64_t)M.nA * B;
  if (N > RSIM_DIRECT_MAX) return RSIM_EARG;
  if (N == 0) return RSIM_OK;
  std::vector<double> W((size_t)(N * N), 0.0);
  for (int64_t e = 0; e < N; ++e) W[e * N + e] = 1.0;
  for (int32_t l = 0; l < M.nA; ++l)
    for (int64_t p = M.rowptr[l]; p < M.rowptr[l + 1]; ++p)
      for (int r = 0; r < B; ++r)
        for (int c = 0; c < B; ++c) {
          double& w = W[((int64_t)M.col[p] * B + c) * N + (int64_t)l * B + r];
          w = w + M.val[p * B * B + r * B + c];
        }
  std::vector<int32_t> piv((size_t)N);
  for (int64_t k = 0; k < N; ++k) {
    double* ck = &W[k * N];
    int64_t pv = k;
    double best = -1.0;
    bool bad = false;
    for (int64_t i = k; i < N; ++i) {
      if (!std::isfinite(ck[i])) bad = true;
      else if (std::fabs(ck[i]) > best) { best = std::fabs(ck[i]); pv = i; }
    }
    if (bad || best == 0.0) {  // singular / non-finite pivot column: name its cell
      M.bad_cell = M.act[k / B];
      return RSIM_ENUM;
    }
    piv[k] = (int32_t)pv;
    if (pv != k)
      for (int64_t j = 0; j < N; ++j) std::swap(W[j * N + k], W[j * N + pv]);
    const double d = ck[k];
    for (int64_t i = k + 1; i < N; ++i) ck[i] = ck[i] / d;
    for (int64_t j = k + 1; j < N; ++j) {
      double* cj = &W[j * N];
      const double ukj = cj[k];
      for (int64_t i = k + 1; i < N; ++i) cj[i] = cj[i] - ck[i] * ukj;
    }
  }
  for (int64_t e = 0; e < N; ++e) x[e] = M.rhs[e];
  for (int64_t k = 0; k < N; ++k)
    if (piv[k] != k) std::swap(x[k], x[piv[k]]);
  for (int64_t k = 0; k < N; ++k)
    for (int64_t i = k + 1; i < N; ++i) x[i] = x[i] - W[k * N + i] * x[k];
  for (int64_t k = N - 1; k >= 0; --k) {
    x[k] = x[k] / W[k * N + k];
    for (int64_t i = 0; i < k; ++i) x[i] = x[i] - W[k * N + i] * x[k];
  }
  return RSIM_OK;
}

static int linsolve_any(Model& M, const rsim_solver_opts& o, double* x, int32_t* it, double* rr) {
  // the exact solve covers n_A·b <= RSIM_DIRECT_MAX; larger active sets fall
  // back to BiCGSTAB (same rule as krylov.cu launch_krylov)
  if (o.lin_method == RSIM_LIN_DIRECT && (int64_t)M.nA * M.b <= RSIM_DIRECT_MAX) {
    switch (M.b) {
      case 1: return direct_solve<1>(M, x, it, rr);
      case 2: return direct_solve<2>(M, x, it, rr);
      default: return direct_solve<3>(M, x, it, rr);
    }
  }
  switch (M.b) {
    case 1: return bicgstab<1>(M, o, x, it, rr);
    case 2: return bicgstab<2>(M, o, x, it, rr);
    default: return bicgstab<3>(M, o, x, it, rr);
  }
}

// ---------------------------------------------------------------- update
// u_A += δu_A, variable substitution per updated cell;
// returns ‖δp‖∞ over the active rows, records δp per cell.
template <int B>
static void update(Model& M, const double* x) {
#pragma omp parallel for schedule(static)
  for (int32_t l = 0; l < M.nA; ++l) {
    int64_t i = M.act[l];
    M.dp[i] = phys::apply_update<B>(M.fl, &M.u[i * B], M.st[i], &x[(int64_t)l * B]);
  }
}
static void update_any(Model& M, const double* x) {
  switch (M.b) {
    case 1: update<1>(M, x); break;
    case 2: update<2>(M, x); break;
    default: update<3>(M, x); break;
  }
}

template <int B>
static void set_mold(Model& M) {
  for (int64_t i = 0; i < M.g.n; ++i) {
    phys::Props<B> P;
    phys::props(M.fl, &M.u[i * B], M.st[i], P);
    phys::mass<B>(M.fl, M.g.pv[i], M.u[i * B], P, &M.mold[i * B]);
  }
}
static void set_mold_any(Model& M) {
  switch (M.b) {
    case 1: set_mold<1>(M); break;
    case 2: set_mold<2>(M); break;
    default: set_mold<3>(M); break;
  }
}

// One local Newton iteration over the given sorted active list:
// assemble, solve, extend + update.  Fills the record; returns status.
static int local_step(Model& M, const std::vector<int32_t>& act, const rsim_solver_opts& o,
                      rsim_iter_record& rec, std::vector<double>& xbuf) {
  const int B = M.b;
  rec.n_active = (int32_t)act.size();
  int st = assemble_any(M, act.data(), (int32_t)act.size());
  if (st < 0) return RSIM_ENUM;
  const int64_t nr = M.nA;
  double f2 = 0.0, finf = 0.0;
  switch (B) {
    case 1: f2 = dotc<1>(nr, M.Fraw.data(), M.Fraw.data()); break;
    case 2: f2 = dotc<2>(nr, M.Fraw.data(), M.Fraw.data()); break;
    default: f2 = dotc<3>(nr, M.Fraw.data(), M.Fraw.data()); break;
  }
  for (double f : M.Fraw) finf = std::max(finf, std::fabs(f));
  rec.f_norm2 = std::sqrt(f2);
  rec.f_norminf = finf;
  xbuf.assign(nr * B, 0.0);
  int32_t it = 0;
  double rr = 0.0;
  int ls = linsolve_any(M, o, xbuf.data(), &it, &rr);
  rec.lin_iters = it;
  rec.lin_res = rr;
  if (ls != RSIM_OK) return ls;
  update_any(M, xbuf.data());
  double mA = 0.0;
  for (int32_t i : act) mA = std::max(mA, std::fabs(M.dp[i]));
  rec.dp_inf_A = mA;
  return RSIM_OK;
}

static void rep_init(rsim_newton_report* rep) {
  std::memset(rep, 0, sizeof(*rep));
}
static void rep_push(rsim_newton_report* rep, const rsim_iter_record& r, int64_t n) {
  if (rep->n_records < RSIM_MAX_ITER_RECORDS) rep->rec[rep->n_records++] = r;
  rep->iterations += 1;
  rep->lin_iters_total += r.lin_iters;
  rep->sum_na += r.n_active;
  rep->sum_na_over_n += (double)r.n_active / (double)n;
}

static std::vector<uint8_t> initial_flags(const Model& M, const int32_t* va, int32_t n) {
  std::vector<uint8_t> A(M.g.n, 0);
  for (int32_t k = 0; k < n; ++k) A[va[k]] = 1;
  for (int64_t i = 0; i < M.g.n; ++i)
    if (M.g.pinned[i]) A[i] = 1;
  return A;
}

// newton_standard: V_A = all cells every iteration.
static int newton_standard(Model& M, const rsim_solver_opts& o, rsim_newton_report* rep) {
  std::vector<int32_t> all;  // every live cell (dead filler cells are not cells of the model)
  for (int64_t i = 0; i < M.g.n; ++i)
    if (!M.g.dead[i]) all.push_back((int32_t)i);
  std::vector<double> x;
  for (int it = 0; it < o.max_newton; ++it) {
    rsim_iter_record rec{};
    rec.subdomain = -1;
    int st = local_step(M, all, o, rec, x);
    rec.dp_inf_B = 0.0;
    rec.mode_expand = 0;
    rep_push(rep, rec, M.g.n_live);
    if (st != RSIM_OK) { rep->status = st; return st; }
    if (rec.dp_inf_A < o.eps_p) { rep->converged = 1; return RSIM_OK; }
  }
  rep->status = RSIM_ENOCONV;
  return RSIM_ENOCONV;
}

// Algorithm 1 set logic for one iteration (lines 7-18) — shared by the
// solver and orc_estimate_active.  Modifies A in place, returns expand flag.
static bool estimate_active(const Model& M, std::vector<uint8_t>& A, const std::vector<uint8_t>& Bf,
                            const std::vector<double>& dp, double eps, int m, bool shrink_locked,
                            double* maxB_out) {
  const Graph& g = M.g;
  double maxB = 0.0;
  std::vector<int32_t> seeds;
  for (int64_t i = 0; i < g.n; ++i)
    if (Bf[i]) {
      double a = std::fabs(dp[i]);
      maxB = std::max(maxB, a);
      if (a >= eps) seeds.push_back((int32_t)i);
    }
  if (maxB_out) *maxB_out = maxB;
  bool expand = !shrink_locked && maxB >= eps;
  if (expand) {
    std::vector<uint8_t> mark(g.n, 0);
    dilate(g, seeds, m, mark);
    for (int64_t i = 0; i < g.n; ++i) A[i] = A[i] | mark[i];
  } else {
    for (int64_t i = 0; i < g.n; ++i)
      A[i] = (uint8_t)((A[i] && std::fabs(dp[i]) >= eps) || g.pinned[i]);
  }
  return expand;
}

// newton_localized (Algorithm 1).
static int newton_localized(Model& M, const int32_t* va_init, int32_t n_init, const rsim_solver_opts& o,
                            rsim_newton_report* rep) {
  std::vector<uint8_t> A = initial_flags(M, va_init, n_init);
  std::vector<uint8_t> Bf = boundary_of(M.g, A);
  std::vector<int32_t> act = to_list(A);
  bool shrink_locked = false;
  std::vector<double> x;
  std::fill(M.dp.begin(), M.dp.end(), 0.0);
  for (int it = 0; it < o.max_newton; ++it) {
    rsim_iter_record rec{};
    rec.subdomain = -1;
    int st = local_step(M, act, o, rec, x);
    if (st != RSIM_OK) { rep_push(rep, rec, M.g.n_live); rep->status = st; return st; }
    bool conv = rec.dp_inf_A < o.eps_p;
    double maxB = 0.0;
    bool expand = estimate_active(M, A, Bf, M.dp, o.eps_set, o.m, shrink_locked, &maxB);
    if (!expand) shrink_locked = true;
    rec.dp_inf_B = maxB;
    rec.mode_expand = expand ? 1 : 0;
    rep_push(rep, rec, M.g.n_live);
    if (!expand && conv) { rep->converged = 1; return RSIM_OK; }
    Bf = boundary_of(M.g, A);
    act = to_list(A);
  }
  rep->status = RSIM_ENOCONV;
  return RSIM_ENOCONV;
}

// adaptive_nonlinear_dd (Algorithm 2) with the SPEC.md:444/:456 resolutions
// (DESIGN.md §DD): Phase 1 solves over the cumulative V_T, the fresh m-layer
// increment of each round becomes subdomain k (label = round); Phase 2 is a
// multiplicative Schwarz sweep with the skip check of SPEC.md:422-430,
// δu of a skipped subdomain := 0, halo change = latest |δp| of halo cells.
static int adaptive_dd(Model& M, const int32_t* va_init, int32_t n_init, const rsim_solver_opts& o,
                       rsim_newton_report* rep, int32_t* labels_out) {
  const Graph& g = M.g;
  std::vector<uint8_t> T = initial_flags(M, va_init, n_init);
  std::vector<int32_t> label(g.n, -1);
  for (int64_t i = 0; i < g.n; ++i)
    if (T[i]) label[i] = 0;
  std::vector<double> x;
  std::fill(M.dp.begin(), M.dp.end(), 0.0);
  int k = 0;
  int inner = 0;
  // ---- Phase 1: expansion over V_T
  while (true) {
    if (inner >= o.max_newton) { rep->status = RSIM_ENOCONV; return RSIM_ENOCONV; }
    std::vector<int32_t> act = to_list(T);
    std::vector<uint8_t> Bf = boundary_of(g, T);
    rsim_iter_record rec{};
    rec.subdomain = -1;
    int st = local_step(M, act, o, rec, x);
    ++inner;
    if (st != RSIM_OK) { rep_push(rep, rec, g.n_live); rep->status = st; return st; }
    double maxB = 0.0;
    std::vector<int32_t> seeds;
    for (int64_t i = 0; i < g.n; ++i)
      if (Bf[i]) {
        double a = std::fabs(M.dp[i]);
        maxB = std::max(maxB, a);
        if (a >= o.eps_set) seeds.push_back((int32_t)i);
      }
    rec.dp_inf_B = maxB;
    bool expand = maxB >= o.eps_set;
    rec.mode_expand = expand;
    rep_push(rep, rec, g.n_live);
    if (!expand) break;
    std::vector<uint8_t> mark(g.n, 0);
    dilate(g, seeds, o.m, mark);
    ++k;
    for (int64_t i = 0; i < g.n; ++i)
      if (mark[i] && !T[i]) { T[i] = 1; label[i] = k; }
  }
  const int N = k + 1;
  rep->n_subdomains = N;
  // ---- Phase 2: multiplicative Schwarz sweeps
  std::vector<std::vector<int32_t>> sub(N), halo(N);
  for (int64_t i = 0; i < g.n; ++i)
    if (label[i] >= 0) sub[label[i]].push_back((int32_t)i);
  for (int s = 0; s < N; ++s) {
    std::vector<uint8_t> in(g.n, 0), h(g.n, 0);
    for (int32_t i : sub[s]) in[i] = 1;
    for (int32_t i : sub[s])
      g.each_live(i, [&](int64_t j, double) { if (!in[j]) h[j] = 1; });
    halo[s] = to_list(h);
  }
  std::vector<double> last(g.n, 0.0);
  for (int64_t i = 0; i < g.n; ++i)
    if (T[i]) last[i] = std::fabs(M.dp[i]);
  std::vector<double> normA(N, 0.0);
  bool first = true;
  int outer = 0;
  while (true) {
    if (outer >= o.max_outer) { rep->outer_iterations = outer; rep->status = RSIM_ENOCONV; return RSIM_ENOCONV; }
    ++outer;
    bool any_big = false;
    for (int s = 0; s < N; ++s) {
      double hmax = 0.0;
      for (int32_t i : halo[s]) hmax = std::max(hmax, last[i]);
      if (first || normA[s] >= o.eps_set || hmax >= o.eps_set) {
        rsim_iter_record rec{};
        rec.subdomain = s;
        int st = local_step(M, sub[s], o, rec, x);
        rec.dp_inf_B = hmax;
        rep_push(rep, rec, g.n_live);
        if (st != RSIM_OK) { rep->outer_iterations = outer; rep->status = st; return st; }
        for (int32_t i : sub[s]) last[i] = std::fabs(M.dp[i]);
        normA[s] = rec.dp_inf_A;
        if (normA[s] >= o.eps_p) any_big = true;
      } else {
        normA[s] = 0.0;
        for (int32_t i : sub[s]) last[i] = 0.0;
      }
    }
    first = false;
    if (!any_big) break;
  }
  rep->outer_iterations = outer;
  rep->converged = 1;
  if (labels_out) std::memcpy(labels_out, label.data(), sizeof(int32_t) * g.n);
  return RSIM_OK;
}

static std::vector<int32_t> initial_active(const Model& M, const double* p_prev, double eps, int m) {
  const Graph& g = M.g;
  std::vector<uint8_t> A(g.n, 0);
  if (!p_prev) {
    std::vector<int32_t> seeds;
    for (int64_t i = 0; i < g.n; ++i)
      if (g.pinned[i]) seeds.push_back((int32_t)i);
    dilate(g, seeds, m, A);
  } else {
    const int B = M.b;
    for (int64_t i = 0; i < g.n; ++i)
      A[i] = (uint8_t)(std::fabs(M.u[i * B] - p_prev[i]) >= eps || g.pinned[i]);
  }
  return to_list(A);
}

}  // namespace

// =================================================================== C API
extern "C" {

int orc_build_matrix_grid(int32_t nx, int32_t ny, int32_t nz, double dx, double dy, double dz,
                          const double* kx, const double* ky, const double* kz, double* tx, double* ty,
                          double* tz) {
  if (nx < 1 || ny < 1 || nz < 1 || !(dx > 0) || !(dy > 0) || !(dz > 0)) return RSIM_EARG;
  const int64_t n = (int64_t)nx * ny * nz, nxy = (int64_t)nx * ny;
  // Υ_half = k A / (d/2); Υ = harmonic combination of the two halves.
  auto harm = [](double a, double b) { return (a > 0.0 && b > 0.0) ? (a * b) / (a + b) : 0.0; };
  for (int64_t i = 0; i < n; ++i) {
    int64_t ix = i % nx, iy = (i / nx) % ny, iz = i / nxy;
    tx[i] = ty[i] = tz[i] = 0.0;
    if (ix < nx - 1) {
      double a = dy * dz, h = 0.5 * dx;
      tx[i] = harm(kx[i] * a / h, kx[i + 1] * a / h);
    }
    if (iy < ny - 1) {
      double a = dx * dz, h = 0.5 * dy;
      ty[i] = harm(ky[i] * a / h, ky[i + nx] * a / h);
    }
    if (iz < nz - 1) {
      double a = dx * dy, h = 0.5 * dz;
      tz[i] = harm(kz[i] * a / h, kz[i + nxy] * a / h);
    }
  }
  return RSIM_OK;
}

void* orc_create(const rsim_graph_desc* gd, const rsim_fluid_params* f) {
  if (!gd || !f || f->kind < 1 || f->kind > 3) return nullptr;
  Model* M = new Model();
  Graph& g = M->g;
  g.nx = gd->nx; g.ny = gd->ny; g.nz = gd->nz;
  g.n = (int64_t)g.nx * g.ny * g.nz;
  g.d3 = g.nz > 1;
  g.nslot = g.d3 ? 6 : 4;
  g.tx.assign(gd->tx, gd->tx + g.n);
  g.ty.assign(gd->ty, gd->ty + g.n);
  g.tz.assign(gd->tz, gd->tz + g.n);
  g.pv.assign(gd->pv, gd->pv + g.n);
  g.kind.assign(gd->kind, gd->kind + g.n);
  g.wi.assign(gd->well_wi, gd->well_wi + g.n);
  g.bhp = gd->bhp;
  g.has_nnc = gd->nnc_ptr != nullptr && gd->nnc_ptr[g.n] > 0;
  if (g.has_nnc) {
    g.nptr.assign(gd->nnc_ptr, gd->nnc_ptr + g.n + 1);
    g.nnbr.assign(gd->nnc_nbr, gd->nnc_nbr + g.nptr[g.n]);
    g.nt.assign(gd->nnc_t, gd->nnc_t + g.nptr[g.n]);
  }
  g.pinned.resize(g.n);
  g.dead.resize(g.n);
  g.n_live = 0;
  for (int64_t i = 0; i < g.n; ++i) {
    g.pinned[i] = (uint8_t)(g.kind[i] == RSIM_KIND_FRACTURE || g.wi[i] > 0.0);
    g.dead[i] = (uint8_t)(g.kind[i] == RSIM_KIND_DEAD);
    g.n_live += !g.dead[i];
  }
  M->fl = phys::Fluid(*f);
  M->b = f->kind;
  M->u.assign(g.n * M->b, 0.0);
  M->mold.assign(g.n * M->b, 0.0);
  M->st.assign(g.n, 0);
  M->dp.assign(g.n, 0.0);
  M->g2l.assign(g.n, -1);
  return M;
}

void orc_destroy(void* h) { delete static_cast<Model*>(h); }
void orc_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }
int orc_threads(void) { return omp_get_max_threads(); }

int orc_set_state(void* h, const double* u, const uint8_t* st, double dt) {
  Model& M = *static_cast<Model*>(h);
  std::memcpy(M.u.data(), u, sizeof(double) * M.u.size());
  std::memcpy(M.st.data(), st, M.st.size());
  M.dt = dt;
  set_mold_any(M);
  return RSIM_OK;
}
int orc_get_state(void* h, double* u, uint8_t* st) {
  Model& M = *static_cast<Model*>(h);
  std::memcpy(u, M.u.data(), sizeof(double) * M.u.size());
  std::memcpy(st, M.st.data(), M.st.size());
  return RSIM_OK;
}
int orc_set_dt(void* h, double dt) {
  static_cast<Model*>(h)->dt = dt;
  return RSIM_OK;
}

int64_t orc_assemble(void* h, const int32_t* act, int32_t nA, double* F_raw, double* rhs, int32_t* rowptr,
                     int32_t* col, double* val, int64_t cap_nnzb) {
  Model& M = *static_cast<Model*>(h);
  int st = assemble_any(M, act, nA);
  if (st < 0) return st;
  const int B = M.b;
  int64_t nnzb = M.rowptr[nA];
  if (F_raw) std::memcpy(F_raw, M.Fraw.data(), sizeof(double) * nA * B);
  if (rhs) std::memcpy(rhs, M.rhs.data(), sizeof(double) * nA * B);
  if (rowptr) std::memcpy(rowptr, M.rowptr.data(), sizeof(int32_t) * (nA + 1));
  if (col && val && cap_nnzb >= nnzb) {
    std::memcpy(col, M.col.data(), sizeof(int32_t) * nnzb);
    std::memcpy(val, M.val.data(), sizeof(double) * nnzb * B * B);
  }
  return nnzb;
}

int orc_linear_solve(void* h, const rsim_solver_opts* o, double* x, int32_t* iters, double* relres) {
  Model& M = *static_cast<Model*>(h);
  return linsolve_any(M, *o, x, iters, relres);
}

double orc_canon_sum(const double* v, int64_t n) { return canon_sum_arr(v, n); }

int32_t orc_neighbor_set(void* h, int32_t i, int32_t m, int32_t* out) {
  Model& M = *static_cast<Model*>(h);
  std::vector<uint8_t> mark(M.g.n, 0);
  dilate(M.g, {i}, m, mark);
  std::vector<int32_t> l = to_list(mark);
  std::copy(l.begin(), l.end(), out);
  return (int32_t)l.size();
}

int32_t orc_support_set(const double* dp, int32_t n, double eps, int32_t* out) {
  int32_t c = 0;
  for (int32_t i = 0; i < n; ++i)
    if (std::fabs(dp[i]) >= eps) out[c++] = i;
  return c;
}

int32_t orc_boundary_layer(void* h, const int32_t* va, int32_t n, int32_t* out) {
  Model& M = *static_cast<Model*>(h);
  std::vector<uint8_t> A(M.g.n, 0);
  for (int32_t k = 0; k < n; ++k) A[va[k]] = 1;
  std::vector<int32_t> l = to_list(boundary_of(M.g, A));
  std::copy(l.begin(), l.end(), out);
  return (int32_t)l.size();
}

int32_t orc_outer_halo(void* h, const int32_t* va, int32_t n, int32_t* out) {
  Model& M = *static_cast<Model*>(h);
  std::vector<uint8_t> A(M.g.n, 0), H(M.g.n, 0);
  for (int32_t k = 0; k < n; ++k) A[va[k]] = 1;
  for (int32_t k = 0; k < n; ++k)
    M.g.each_live(va[k], [&](int64_t j, double) { if (!A[j]) H[j] = 1; });
  std::vector<int32_t> l = to_list(H);
  std::copy(l.begin(), l.end(), out);
  return (int32_t)l.size();
}

int32_t orc_estimate_active(void* h, const int32_t* va, int32_t n, const double* dp_global, double eps, int32_t m,
                            int32_t shrink_locked, int32_t* va_out, int32_t* vb_out, int32_t* nb_out,
                            int32_t* expand_out) {
  Model& M = *static_cast<Model*>(h);
  std::vector<uint8_t> A(M.g.n, 0);
  for (int32_t k = 0; k < n; ++k) A[va[k]] = 1;
  std::vector<uint8_t> Bf = boundary_of(M.g, A);
  std::vector<double> dp(M.g.n, 0.0);
  for (int32_t k = 0; k < n; ++k) dp[va[k]] = dp_global[va[k]];
  bool expand = estimate_active(M, A, Bf, dp, eps, m, shrink_locked != 0, nullptr);
  std::vector<int32_t> la = to_list(A), lb = to_list(boundary_of(M.g, A));
  std::copy(la.begin(), la.end(), va_out);
  if (vb_out) std::copy(lb.begin(), lb.end(), vb_out);
  if (nb_out) *nb_out = (int32_t)lb.size();
  if (expand_out) *expand_out = expand ? 1 : 0;
  return (int32_t)la.size();
}

int orc_newton_standard(void* h, double dt, const rsim_solver_opts* o, rsim_newton_report* rep) {
  Model& M = *static_cast<Model*>(h);
  rep_init(rep);
  M.dt = dt;
  return newton_standard(M, *o, rep);
}

int orc_newton_localized(void* h, double dt, const int32_t* va_init, int32_t n_init, const rsim_solver_opts* o,
                         rsim_newton_report* rep) {
  Model& M = *static_cast<Model*>(h);
  rep_init(rep);
  M.dt = dt;
  return newton_localized(M, va_init, n_init, *o, rep);
}

int orc_adaptive_dd(void* h, double dt, const int32_t* va_init, int32_t n_init, const rsim_solver_opts* o,
                    rsim_newton_report* rep, int32_t* labels_out) {
  Model& M = *static_cast<Model*>(h);
  rep_init(rep);
  M.dt = dt;
  return adaptive_dd(M, va_init, n_init, *o, rep, labels_out);
}

int32_t orc_initial_active(void* h, const double* p_prev, double eps, int32_t m, int32_t* out) {
  Model& M = *static_cast<Model*>(h);
  std::vector<int32_t> l = initial_active(M, p_prev, eps, m);
  std::copy(l.begin(), l.end(), out);
  return (int32_t)l.size();
}

// The driver loop over dts from the model's current state;
// p_prev = pressure at the start of the previous committed step (empty: the
// first-step rule of initial_active), updated in place.
static int run_steps(Model& M, int32_t solver, const double* dts, int32_t nsteps, const rsim_solver_opts* o,
                     std::vector<double>& p_prev, int32_t* total_iters, double* total_ma, int64_t* total_na,
                     int32_t* total_lin, int32_t* n_cuts) {
  const int B = M.b;
  const int64_t n = M.g.n;
  std::deque<double> q(dts, dts + nsteps);
  *total_iters = 0; *total_ma = 0.0; *total_na = 0; *total_lin = 0; *n_cuts = 0;
  std::vector<double> u_save;
  std::vector<uint8_t> st_save;
  rsim_newton_report* rep = new rsim_newton_report;
  int status = RSIM_OK;
  while (!q.empty()) {
    double dt = q.front();
    q.pop_front();
    std::vector<int32_t> va = initial_active(M, p_prev.empty() ? nullptr : p_prev.data(), o->eps_set, o->m);
    u_save = M.u;
    st_save = M.st;
    M.dt = dt;
    set_mold_any(M);
    rep_init(rep);
    int st;
    if (solver == 0) st = newton_standard(M, *o, rep);
    else if (solver == 1) st = newton_localized(M, va.data(), (int32_t)va.size(), *o, rep);
    else st = adaptive_dd(M, va.data(), (int32_t)va.size(), *o, rep, nullptr);
    *total_iters += rep->iterations;
    *total_ma += rep->sum_na_over_n;
    *total_na += rep->sum_na;
    *total_lin += rep->lin_iters_total;
    if (st != RSIM_OK) {
      M.u = u_save;
      M.st = st_save;
      if (dt * 0.5 < 1e-4 * 86400.0) { status = st; break; }
      ++*n_cuts;
      q.push_front(dt * 0.5);
      q.push_front(dt * 0.5);
      continue;
    }
    p_prev.resize(n);
    for (int64_t i = 0; i < n; ++i) p_prev[i] = u_save[i * B];
  }
  delete rep;
  return status;
}

int orc_run_case(void* h, int32_t solver, const double* dts, int32_t nsteps, const rsim_solver_opts* o,
                 int32_t* total_iters, double* total_ma, int64_t* total_na, int32_t* total_lin, int32_t* n_cuts) {
  std::vector<double> p_prev;
  return run_steps(*static_cast<Model*>(h), solver, dts, nsteps, o, p_prev, total_iters, total_ma, total_na,
                   total_lin, n_cuts);
}

// Continue a run one or more timesteps at a time (the bench's reference arm
// times single timesteps of the workload in sequence).  p_prev_io[n]: in, the
// pressure at the start of the previous committed step; out, updated.  *has_prev
// = 0 selects the first-step rule and is set to 1 after a committed step.
int orc_run_steps(void* h, int32_t solver, const double* dts, int32_t nsteps, const rsim_solver_opts* o,
                  double* p_prev_io, int32_t* has_prev, int32_t* total_iters, double* total_ma, int64_t* total_na,
                  int32_t* total_lin, int32_t* n_cuts) {
  Model& M = *static_cast<Model*>(h);
  std::vector<double> p_prev;
  if (*has_prev) p_prev.assign(p_prev_io, p_prev_io + M.g.n);
  const int r = run_steps(M, solver, dts, nsteps, o, p_prev, total_iters, total_ma, total_na, total_lin, n_cuts);
  if (!p_prev.empty()) {
    std::copy(p_prev.begin(), p_prev.end(), p_prev_io);
    *has_prev = 1;
  }
  return r;
}

double orc_rexp(double x) { return phys::rexp(x); }

void orc_corey(double s, double s_r, double den, double* kr, double* dkr) { phys::corey2(s, s_r, 1.0 / den, *kr, *dkr); }

}  // extern "C"

template <int B>
static void props_out(const rsim_fluid_params* f, const double* u, uint8_t st, double* A, double* dA, double* L,
                      double* dL) {
  phys::Props<B> P;
  phys::props(phys::Fluid(*f), u, st, P);
  for (int e = 0; e < B; ++e) {
    A[e] = P.A[e];
    L[e] = P.L[e];
    for (int v = 0; v < B; ++v) { dA[e * B + v] = P.dA[e][v]; dL[e * B + v] = P.dL[e][v]; }
  }
}

extern "C" {

int orc_props(const rsim_fluid_params* f, const double* u, uint8_t st, double* A, double* dA, double* L, double* dL) {
  switch (f->kind) {
    case 1: props_out<1>(f, u, st, A, dA, L, dL); return RSIM_OK;
    case 2: props_out<2>(f, u, st, A, dA, L, dL); return RSIM_OK;
    case 3: props_out<3>(f, u, st, A, dA, L, dL); return RSIM_OK;
    default: return RSIM_EARG;
  }
}

int orc_set_u(void* h, const double* u, const uint8_t* st) {
  Model& M = *static_cast<Model*>(h);
  std::memcpy(M.u.data(), u, sizeof(double) * M.u.size());
  std::memcpy(M.st.data(), st, M.st.size());
  return RSIM_OK;
}

int64_t orc_assemble_raw(void* h, const int32_t* act, int32_t nA, double* F_raw, double* diag, int32_t* rowptr,
                         int32_t* col, double* val, int64_t cap_nnzb) {
  Model& M = *static_cast<Model*>(h);
  M.raw = true;
  int st = assemble_any(M, act, nA);
  M.raw = false;
  if (st < 0) return st;
  const int B = M.b;
  int64_t nnzb = M.rowptr[nA];
  if (F_raw) std::memcpy(F_raw, M.Fraw.data(), sizeof(double) * nA * B);
  if (diag) std::memcpy(diag, M.diag.data(), sizeof(double) * nA * B * B);
  if (rowptr) std::memcpy(rowptr, M.rowptr.data(), sizeof(int32_t) * (nA + 1));
  if (col && val && cap_nnzb >= nnzb) {
    std::memcpy(col, M.col.data(), sizeof(int32_t) * nnzb);
    std::memcpy(val, M.val.data(), sizeof(double) * nnzb * B * B);
  }
  return nnzb;
}

int orc_full_residual(void* h, double* F_raw) {
  Model& M = *static_cast<Model*>(h);
  std::vector<int32_t> all(M.g.n);
  for (int64_t i = 0; i < M.g.n; ++i) all[i] = (int32_t)i;
  int st = assemble_any(M, all.data(), (int32_t)all.size());
  if (st < 0) return RSIM_ENUM;
  std::memcpy(F_raw, M.Fraw.data(), sizeof(double) * M.Fraw.size());
  return RSIM_OK;
}

}  // extern "C"

// ---- Peng-Robinson property functions and flash (
//      SPEC.md:135-177).  The cell-local arithmetic is include/rsim/eos.h,
//      shared with csrc/eos.cu (bit-identical results); these wrappers are the
//      CPU checker and the CPU baseline of the flash bench line.
#include "rsim/eos.h"

namespace {
template <class F>
int eos_dispatch(int nc, F&& f) {
  switch (nc) {
    case 1: return f(std::integral_constant<int, 1>{});
    case 2: return f(std::integral_constant<int, 2>{});
    case 3: return f(std::integral_constant<int, 3>{});
    case 4: return f(std::integral_constant<int, 4>{});
    default: return RSIM_EARG;
  }
}
}  // namespace

extern "C" {

double orc_eos_rlog(double x) { return rsim::eos::rlog(x); }

int orc_eos_cubic_roots(double A, double B, double* r3) { return rsim::eos::cubic_roots(A, B, r3); }

int orc_eos_phase(const rsim_eos_params* e, double T, double p, const double* x, int32_t sel, int32_t min_g,
                  double* Z, double* lnphi) {
  const rsim::eos::Terms t = rsim::eos::terms(*e, T);
  return eos_dispatch(e->nc, [&](auto NCc) {
    constexpr int NC = decltype(NCc)::value;
    return rsim::eos::phase_props<NC>(t, p, x, sel, min_g != 0, *Z, lnphi) ? RSIM_OK : RSIM_ENUM;
  });
}

int orc_eos_rachford_rice(int32_t nc, const double* z, const double* K, double* nu) {
  return eos_dispatch(nc, [&](auto NCc) {
    constexpr int NC = decltype(NCc)::value;
    return rsim::eos::rachford_rice<NC>(z, K, *nu) ? RSIM_OK : RSIM_EARG;
  });
}

int orc_eos_stability(const rsim_eos_params* e, double T, double p, const double* z, double* K, int32_t* stable) {
  const rsim::eos::Terms t = rsim::eos::terms(*e, T);
  return eos_dispatch(e->nc, [&](auto NCc) {
    constexpr int NC = decltype(NCc)::value;
    int its = 0;
    *stable = rsim::eos::stability<NC>(t, p, z, K, &its) ? 1 : 0;
    return RSIM_OK;
  });
}

int orc_eos_flash(const rsim_eos_params* e, double T, int64_t n, const double* p, const double* z, uint8_t* status,
                  double* nu_g, double* x, double* y, double* zfac, int32_t* iters) {
  if (!e || e->nc < 1 || e->nc > RSIM_EOS_NCMAX) return RSIM_EARG;
  const rsim::eos::Terms t = rsim::eos::terms(*e, T);
  return eos_dispatch(e->nc, [&](auto NCc) {
    constexpr int NC = decltype(NCc)::value;
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
      rsim::eos::Flash<NC> R;
      rsim::eos::flash<NC>(t, p[i], &z[i * NC], R);
      status[i] = (uint8_t)R.status;
      nu_g[i] = R.nu_g;
      for (int c = 0; c < NC; ++c) {
        x[i * NC + c] = R.x[c];
        y[i * NC + c] = R.y[c];
      }
      zfac[2 * i] = R.Zo;
      zfac[2 * i + 1] = R.Zg;
      if (iters) iters[i] = R.iters;
    }
    return RSIM_OK;
  });
}

}  // extern "C"
