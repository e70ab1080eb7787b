/*
 * rsim/physics.h — per-cell constitutive relations and per-connection flux
 * blocks, compiled identically for the host (g++) and sm_100a (nvcc).
 *
 * Why one header for both sides: the north star asks for GPU results that
 * match the CPU oracle with *identical* Newton and Krylov iteration counts,
 * which is only structural if the cell-local arithmetic is bit-identical
 * (SURVEY.md §7 H1).  So every formula below is written once, with a fixed
 * operation order; the host is compiled with -ffp-contract=off and the
 * device with --fmad=false so no side contracts a*b+c into an FMA, and the
 * only transcendental (exp) is implemented here (rexp) instead of libm.
 *
 * Divisions by model constants (μ, Δt, the Corey denominators, p_bub, p_gas)
 * are written as multiplications by the reciprocal, (1.0 / c), which the
 * compiler evaluates once per thread; both sides use the same expression.
 *
 * These functions are pure: no traversal, no set logic, no linear algebra.
 * The oracle (oracle/) shares ONLY this header and blockops.h with the
 * product; its assembly loop, set logic, Krylov solver and Newton control are
 * independent code.  The formulas themselves are pinned by the SPEC
 * known-answer tests and by central finite differences (tests/).
 *
 * Reference anchors (/root/reference):
 *   density  ρ = ρ_ref exp(c (p − p_ref))
 *   relperm  kr = ((s − s_r)/(1 − s_ro − s_rg))², clamp
 *   accumulation (V/Δt)[(φρ_T z)^{n+1} − (φρ_T z)^n],
 *            φ = φ_ref (1 + c_r (p − p_ref))
 *   flux_ppu F_l = Υ λ_l,up ρ_l,up (p_i − p_j), g = 0
 *   well     WI λ ρ (p − bhp) for p > bhp, else 0
 *   variable substitution (phase appearance/disappearance) SPEC.md:180-188
 *
 * Sign convention: R_i = (M_i − M_i^n)/Δt + Σ_j F_ij + Q_i, with F_ij the
 * outflow from i (positive when p_i > p_j) and Q_i the production rate.
 */
#ifndef RSIM_PHYSICS_H
#define RSIM_PHYSICS_H

#include <math.h>
#include <stdint.h>
#include "types.h"

#if defined(__CUDACC__)
#define RSIM_HD __host__ __device__ __forceinline__
#else
#define RSIM_HD inline
#endif

namespace rsim {
namespace phys {

/* exp(x) with a fixed operation sequence (Cody-Waite reduction + degree-13
 * Horner), so host and device return the same bits.  |rel err| < 3e-16 on
 * the reduced range; the ranges used here are |x| < 1. */
RSIM_HD double rexp(double x) {
  if (!(x < 709.0)) return (x != x) ? x : HUGE_VAL;
  if (x < -745.0) return 0.0;
  const double LOG2E = 1.4426950408889634;
  const double LN2_HI = 6.93147180369123816490e-01; /* 32 significant bits */
  const double LN2_LO = 1.90821492927058770002e-10;
  double kd = rint(x * LOG2E);
  double r = (x - kd * LN2_HI) - kd * LN2_LO;
  double q = 1.6059043836821613e-10;
  q = q * r + 2.08767569878681e-09;
  q = q * r + 2.505210838544172e-08;
  q = q * r + 2.755731922398589e-07;
  q = q * r + 2.7557319223985893e-06;
  q = q * r + 2.48015873015873e-05;
  q = q * r + 0.0001984126984126984;
  q = q * r + 0.001388888888888889;
  q = q * r + 0.008333333333333333;
  q = q * r + 0.041666666666666664;
  q = q * r + 0.16666666666666666;
  q = q * r + 0.5;
  q = q * r + 1.0;
  q = q * r + 1.0;
  const int k = (int)kd;
  if (k > -1000 && k < 1000) {  // q·2^k is a normal number: exact, the same bits as ldexp
#if defined(__CUDA_ARCH__)
    return q * __longlong_as_double((long long)(k + 1023) << 52);
#else
    union { long long i; double d; } e;
    e.i = (long long)(k + 1023) << 52;
    return q * e.d;
#endif
  }
  return ldexp(q, k);
}

/* Quadratic Corey curve on the normalised saturation (s − s_r)/den,
 * clamped to [0,1].  dkr is d kr / d s. */
RSIM_HD void corey2(double s, double s_r, double inv_den, double& kr, double& dkr) {
  double se = (s - s_r) * inv_den;
  if (!(se > 0.0)) { kr = 0.0; dkr = 0.0; }
  else if (!(se < 1.0)) { kr = 1.0; dkr = 0.0; }
  else { kr = se * se; dkr = (2.0 * se) * inv_den; }
}

/* Per-cell property block.
 *   A[e]      : amount of conserved quantity e per unit pore volume
 *   L[e]      : transport coefficient Σ_phases (fraction of e in phase)·ρ_l·λ_l
 *   dA, dL    : derivatives w.r.t. the cell's unknowns u[v].               */
template <int B>
struct Props {
  double A[B];
  double dA[B][B];
  double L[B];
  double dL[B][B];
};

/* Model constants plus the reciprocals the formulas use, formed ONCE per
 * context (host) and shipped to the kernels as a by-value argument: every
 * formula multiplies by these, so host and device use the same bits without
 * a division per evaluation. */
struct Fluid : rsim_fluid_params {
  double inv_mu[3];
  double inv_pbub, inv_pgas;
  double inv_den2;  /* 1 / (1 − swc − sor)        oil-water Corey  */
  double inv_den3;  /* 1 / (1 − swc − sor − sgc)  black-oil Corey  */
  RSIM_HD Fluid() : rsim_fluid_params(), inv_mu{0.0, 0.0, 0.0}, inv_pbub(0.0), inv_pgas(0.0), inv_den2(0.0), inv_den3(0.0) {}
  RSIM_HD explicit Fluid(const rsim_fluid_params& f) : rsim_fluid_params(f) {
    for (int k = 0; k < 3; ++k) inv_mu[k] = 1.0 / f.mu[k];
    inv_pbub = 1.0 / f.p_bub;
    inv_pgas = 1.0 / f.p_gas;
    inv_den2 = 1.0 / ((1.0 - f.swc) - f.sor);
    inv_den3 = 1.0 / (((1.0 - f.swc) - f.sor) - f.sgc);
  }
};

/* ---- Model 1: single phase slightly compressible, u = (p) ------------ */
RSIM_HD void props(const Fluid& f, const double* u, uint8_t /*st*/, Props<1>& P) {
  double p = u[0];
  double rho = f.rho_ref[1] * rexp(f.c_f[1] * (p - f.p_ref));
  double drho = f.c_f[1] * rho;
  P.A[0] = rho;
  P.dA[0][0] = drho;
  P.L[0] = rho * f.inv_mu[1];
  P.dL[0][0] = drho * f.inv_mu[1];
}

/* ---- Model 2: oil-water, u = (p, S_w); equations (water, oil) --------- */
RSIM_HD void props(const Fluid& f, const double* u, uint8_t /*st*/, Props<2>& P) {
  double p = u[0], sw = u[1];
  double rw = f.rho_ref[0] * rexp(f.c_f[0] * (p - f.p_ref));
  double drw = f.c_f[0] * rw;
  double ro = f.rho_ref[1] * rexp(f.c_f[1] * (p - f.p_ref));
  double dro = f.c_f[1] * ro;
  double so = 1.0 - sw;
  P.A[0] = rw * sw;
  P.dA[0][0] = drw * sw;
  P.dA[0][1] = rw;
  P.A[1] = ro * so;
  P.dA[1][0] = dro * so;
  P.dA[1][1] = -ro;
  double krw, dkrw, kro, dkro;
  corey2(sw, f.swc, f.inv_den2, krw, dkrw);
  corey2(so, f.sor, f.inv_den2, kro, dkro); /* d/dso; d so/d sw = -1 */
  P.L[0] = (rw * krw) * f.inv_mu[0];
  P.dL[0][0] = (drw * krw) * f.inv_mu[0];
  P.dL[0][1] = (rw * dkrw) * f.inv_mu[0];
  P.L[1] = (ro * kro) * f.inv_mu[1];
  P.dL[1][0] = (dro * kro) * f.inv_mu[1];
  P.dL[1][1] = -((ro * dkro) * f.inv_mu[1]);
}

/* ---- Model 3: black-oil, u = (p, S_w, X); equations (water, oil, gas) --
 * status SAT: X = S_g, R_s = R_s,sat(p);  UNDERSAT: X = R_s, S_g = 0.
 * Surface-volume conservation:  water φ S_w b_w;  oil φ S_o b_o;
 * gas φ (S_g b_g + R_s S_o b_o); b_l reciprocal formation volume factors.  */
RSIM_HD void props(const Fluid& f, const double* u, uint8_t st, Props<3>& P) {
  double p = u[0], sw = u[1], X = u[2];
  double bw = rexp(f.c_f[0] * (p - f.p_ref));
  double dbw = f.c_f[0] * bw;
  double eo = rexp(f.c_f[1] * (p - f.p_ref));
  double rs, drs_dp, drs_dx, sg, dsg_dx;
  if (st == RSIM_BO_SAT) {
    rs = (f.rs_b * p) * f.inv_pbub; drs_dp = f.rs_b * f.inv_pbub; drs_dx = 0.0;
    sg = X; dsg_dx = 1.0;
  } else {
    rs = X; drs_dp = 0.0; drs_dx = 1.0;
    sg = 0.0; dsg_dx = 0.0;
  }
  double so = (1.0 - sw) - sg;
  double dso_dx = -dsg_dx;
  double q = 1.0 + f.bo_alpha * rs;
  double bo = eo / q;
  double dbo_drs = -((f.bo_alpha * bo) / q);
  double dbo_dp = f.c_f[1] * bo + dbo_drs * drs_dp;
  double dbo_dx = dbo_drs * drs_dx;
  double bg = p * f.inv_pgas;
  double dbg = f.inv_pgas;

  P.A[0] = sw * bw;
  P.dA[0][0] = sw * dbw;
  P.dA[0][1] = bw;
  P.dA[0][2] = 0.0;
  P.A[1] = so * bo;
  P.dA[1][0] = so * dbo_dp;
  P.dA[1][1] = -bo;
  P.dA[1][2] = so * dbo_dx + dso_dx * bo;
  double sobo = so * bo;
  P.A[2] = sg * bg + rs * sobo;
  P.dA[2][0] = (sg * dbg + drs_dp * sobo) + rs * (so * dbo_dp);
  P.dA[2][1] = -(rs * bo);
  P.dA[2][2] = (dsg_dx * bg + drs_dx * sobo) + rs * P.dA[1][2];

  double krw, dkrw, kro, dkro, krg, dkrg;
  corey2(sw, f.swc, f.inv_den3, krw, dkrw);
  corey2(so, f.sor, f.inv_den3, kro, dkro);
  corey2(sg, f.sgc, f.inv_den3, krg, dkrg);
  double lo = (bo * kro) * f.inv_mu[1];
  double dlo_dp = (dbo_dp * kro) * f.inv_mu[1];
  double dlo_dsw = -((bo * dkro) * f.inv_mu[1]);
  double dlo_dx = (dbo_dx * kro + bo * (dkro * dso_dx)) * f.inv_mu[1];
  P.L[0] = (bw * krw) * f.inv_mu[0];
  P.dL[0][0] = (dbw * krw) * f.inv_mu[0];
  P.dL[0][1] = (bw * dkrw) * f.inv_mu[0];
  P.dL[0][2] = 0.0;
  P.L[1] = lo;
  P.dL[1][0] = dlo_dp;
  P.dL[1][1] = dlo_dsw;
  P.dL[1][2] = dlo_dx;
  double lg = (bg * krg) * f.inv_mu[2];
  P.L[2] = lg + rs * lo;
  P.dL[2][0] = ((dbg * krg) * f.inv_mu[2] + drs_dp * lo) + rs * dlo_dp;
  P.dL[2][1] = rs * dlo_dsw;
  P.dL[2][2] = ((bg * (dkrg * dsg_dx)) * f.inv_mu[2] + drs_dx * lo) + rs * dlo_dx;
}

/* Mass in place M_e = pv φ(p) A_e (used for the old-time accumulation). */
template <int B>
RSIM_HD void mass(const Fluid& f, double pv, double p, const Props<B>& P, double* M) {
  double pvp = pv * (1.0 + f.c_r * (p - f.p_ref));
  for (int e = 0; e < B; ++e) M[e] = pvp * P.A[e];
}

/* Accumulation: initialises the row residual R and diagonal block D. */
template <int B>
RSIM_HD void accum_row(const Fluid& f, double pv, double p, const Props<B>& P,
                       const double* Mold, double inv_dt, double* R, double (*D)[B]) {
  double pvp = pv * (1.0 + f.c_r * (p - f.p_ref));
  double pvc = pv * f.c_r;
  for (int e = 0; e < B; ++e) {
    R[e] = (pvp * P.A[e] - Mold[e]) * inv_dt;
    D[e][0] = (pvp * P.dA[e][0] + pvc * P.A[e]) * inv_dt;
    for (int v = 1; v < B; ++v) D[e][v] = (pvp * P.dA[e][v]) * inv_dt;
  }
}

/* Phase-potential-upwinded TPFA connection (i,j) with Υ = T, dp = p_i − p_j,
 * U = properties of the upwind cell (i when dp >= 0, else j).
 * flux_terms: the residual term Rc = T·L_up·dp, the diagonal term Dc and the
 * off-diagonal block O = ∂F_ij/∂u_j (not accumulated);
 * flux_conn: adds Rc to R and Dc to D of row i (the canonical order is the
 * order in which connections are visited). */
template <int B>
RSIM_HD void flux_terms(double T, double dp, bool up_i, const Props<B>& U, double* Rc, double (*Dc)[B],
                        double (*O)[B]) {
  for (int e = 0; e < B; ++e) {
    double tl = T * U.L[e];
    Rc[e] = tl * dp;
    for (int v = 0; v < B; ++v) {
      double c = (T * U.dL[e][v]) * dp;
      double di = up_i ? c : 0.0;
      double dj = up_i ? 0.0 : c;
      if (v == 0) { di = di + tl; dj = dj - tl; }
      Dc[e][v] = di;
      O[e][v] = dj;
    }
  }
}

template <int B>
RSIM_HD void flux_conn(double T, double dp, bool up_i, const Props<B>& U,
                       double* R, double (*D)[B], double (*O)[B]) {
  double Rc[B], Dc[B][B];
  flux_terms<B>(T, dp, up_i, U, Rc, Dc, O);
  for (int e = 0; e < B; ++e) {
    R[e] = R[e] + Rc[e];
    for (int v = 0; v < B; ++v) D[e][v] = D[e][v] + Dc[e][v];
  }
}

/* BHP producer, production only. */
template <int B>
RSIM_HD void well_row(double wi, double p, double bhp, const Props<B>& P, double* R, double (*D)[B]) {
  double dpw = p - bhp;
  if (wi > 0.0 && dpw > 0.0) {
    for (int e = 0; e < B; ++e) {
      double wl = wi * P.L[e];
      R[e] = R[e] + wl * dpw;
      for (int v = 0; v < B; ++v) {
        double c = (wi * P.dL[e][v]) * dpw;
        if (v == 0) c = c + wl;
        D[e][v] = D[e][v] + c;
      }
    }
  }
}

/* Production rate per equation (for rates / mass balance). */
template <int B>
RSIM_HD void well_rate(double wi, double p, double bhp, const Props<B>& P, double* q) {
  double dpw = p - bhp;
  for (int e = 0; e < B; ++e) q[e] = (wi > 0.0 && dpw > 0.0) ? (wi * P.L[e]) * dpw : 0.0;
}

/* Variable substitution after a Newton update (for the
 * black-oil model the saturated <-> undersaturated switch at the bubble
 * point).  Saturations are clamped to [0,1]. */
RSIM_HD double clamp01(double s) { return s < 0.0 ? 0.0 : (s > 1.0 ? 1.0 : s); }

template <int B>
RSIM_HD void substitute(const Fluid& f, double* u, uint8_t& st) {
  if (B >= 2) u[1] = clamp01(u[1]);
  if (B == 3) {
    double rs_sat = (f.rs_b * u[0]) * f.inv_pbub;
    if (st == RSIM_BO_UNDERSAT) {
      if (u[2] > rs_sat) { st = RSIM_BO_SAT; u[2] = 0.0; }
    } else {
      if (u[2] < 0.0) { st = RSIM_BO_UNDERSAT; u[2] = rs_sat; }
      else if (u[2] > 1.0 - u[1]) u[2] = 1.0 - u[1];
    }
  }
}

/* Newton update of one cell: u += w·δu, then variable substitution; returns
 * the applied pressure change w·δp (the value the support set, the flags and
 * ‖δp‖∞ see).  w is the per-cell Appleyard chop (DESIGN.md §5 item 11):
 *   w = min(1, dp_max_rel·|p| / |δp|, ds_max / max(|δS_w|, |δS_g|, |δS_o|))
 * with δS_g counted only in the saturated state (X = S_g) and δS_o = −(δS_w + δS_g).
 * Off (w = 1 exactly, so u + 1·δu == u + δu bit for bit) when both limits are 0,
 * which is every config but the black-oil one. */
template <int B>
RSIM_HD double apply_update(const Fluid& f, double* u, uint8_t& st, const double* x) {
  double w = 1.0;
  if (f.dp_max_rel > 0.0) {
    const double a = fabs(x[0]), lim = f.dp_max_rel * fabs(u[0]);
    if (a > lim) w = lim / a;
  }
  if (B >= 2 && f.ds_max > 0.0) {
    double a = fabs(x[1]);
    double so = x[1];
    if (B == 3 && st == RSIM_BO_SAT) {
      const double g = fabs(x[2]);
      if (g > a) a = g;
      so = so + x[2];
    }
    so = fabs(so);
    if (so > a) a = so;
    if (w * a > f.ds_max) w = f.ds_max / a;
  }
  for (int c = 0; c < B; ++c) u[c] = u[c] + w * x[c];
  substitute<B>(f, u, st);
  return w * x[0];
}

}  // namespace phys
}  // namespace rsim

#endif /* RSIM_PHYSICS_H */
