/*
 * rsim/eos.h — Peng-Robinson compositional property functions (SURVEY.md §8f
 * row 3, paper Case 3), cell-local and shared by the sm_100a
 * flash kernel (csrc/eos.cu) and the CPU oracle (oracle/oracle.cpp), for the
 * same reason as physics.h: bit-identical results on both sides need the same
 * operation order, no FMA contraction (--fmad=false / -ffp-contract=off) and
 * no libm transcendentals (rexp from physics.h, rlog here; sqrt is IEEE
 * exact everywhere).  The formulas are pinned independently by the SPEC
 * known answers and by a numpy restatement (np.roots, np.log, bisection) in
 * tests/test_eos.py.
 *
 *   pr_z_factor            SPEC.md:135-143   cubic_roots + phase_props (root selector)
 *   fugacity_coefficients  SPEC.md:144-151   lnphi
 *   stability_test         SPEC.md:152-160   stability (two-sided Michelsen, Wilson K)
 *   rachford_rice          SPEC.md:161-168   rachford_rice
 *   flash                  SPEC.md:169-177   flash (successive substitution)
 *
 * Temperature-only terms (a_i(T), b_i, a_ij, Wilson prefactors) are formed
 * ONCE on the host (terms()) and shipped by value, so the only per-cell
 * transcendental work is rlog / rexp.
 */
#ifndef RSIM_EOS_H
#define RSIM_EOS_H

#include <math.h>
#include <stdint.h>
#include "physics.h"

#define RSIM_EOS_NCMAX 4

#ifdef __cplusplus
extern "C" {
#endif

/* Components (SPEC.md:99-102 ComponentSpec) and solver controls. */
typedef struct {
  int32_t nc;                                /* 1..RSIM_EOS_NCMAX                        */
  double tc[RSIM_EOS_NCMAX];                 /* K                                        */
  double pc[RSIM_EOS_NCMAX];                 /* Pa                                       */
  double omega[RSIM_EOS_NCMAX];              /* acentric factor                          */
  double mw[RSIM_EOS_NCMAX];                 /* kg/mol                                   */
  double kij[RSIM_EOS_NCMAX][RSIM_EOS_NCMAX]; /* binary interaction, symmetric, 0 diagonal */
  double flash_tol;                          /* max_c |f_o/f_g - 1| (SPEC: 1e-8)          */
  int32_t flash_maxit;                       /* SPEC: 500                                */
  int32_t stab_maxit;                        /* Michelsen iterations per trial            */
} rsim_eos_params;

/* Phase status. */
enum { RSIM_PH_OIL = 0, RSIM_PH_GAS = 1, RSIM_PH_TWO = 2 };
/* Root selector of pr_z_factor. */
enum { RSIM_ROOT_LIQUID = 0, RSIM_ROOT_VAPOR = 1 };

/* Paper Case 3 fluid (§5 Case 3: C1 50 % / C10 50 %, 340 K): standard
 * critical constants of methane and n-decane, k_ij = 0 [choice]. */
int rsim_eos_case3(rsim_eos_params* out);

/* Batch flash on the GPU (one thread per cell), host buffers (copied in and
 * out inside the call).  z: [n*nc] cell-major; outputs: status[n] (RSIM_PH_*),
 * nu_g[n], x[n*nc], y[n*nc], zfac[2n] (Z_o, Z_g per cell), iters[n] (may be
 * NULL).  Returns RSIM_OK, RSIM_EARG, RSIM_ECUDA (no sm_100 device). */
int rsim_eos_flash(const rsim_eos_params* e, double T, int64_t n, const double* p, const double* z,
                   uint8_t* status, double* nu_g, double* x, double* y, double* zfac, int32_t* iters);
/* Same on device-resident buffers, enqueued on `stream` (cudaStream_t or NULL);
 * no synchronisation. */
int rsim_eos_flash_dev(const rsim_eos_params* e, double T, int64_t n, const double* p, const double* z,
                       uint8_t* status, double* nu_g, double* x, double* y, double* zfac, int32_t* iters,
                       void* stream);

#ifdef __cplusplus
}

namespace rsim {
namespace eos {

using rsim::phys::rexp;
constexpr double kR = 8.31446261815324;        /* J/(mol K) */
constexpr double kSqrt2 = 1.4142135623730951;

/* ln x for finite x > 0 without libm: x = m 2^e, m in [1/sqrt2, sqrt2),
 * ln m = 2 atanh(s), s = (m-1)/(m+1), |s| <= 0.1716 (odd series to s^23). */
RSIM_HD double rlog(double x) {
  if (!(x > 0.0)) return x == 0.0 ? -HUGE_VAL : (x - x) / (x - x);
  if (x == HUGE_VAL) return x;
  long long bits;
#if defined(__CUDA_ARCH__)
  bits = __double_as_longlong(x);
#else
  union { double d; long long i; } u;
  u.d = x;
  bits = u.i;
#endif
  int e = (int)((bits >> 52) & 0x7ff);
  double scale = 0.0;
  if (e == 0) {  // subnormal: renormalise by 2^54 (exact)
    x = x * 18014398509481984.0;
#if defined(__CUDA_ARCH__)
    bits = __double_as_longlong(x);
#else
    u.d = x;
    bits = u.i;
#endif
    e = (int)((bits >> 52) & 0x7ff);
    scale = -54.0;
  }
  long long mb = (bits & 0x000fffffffffffffLL) | 0x3ff0000000000000LL;  // m in [1, 2)
  double m;
#if defined(__CUDA_ARCH__)
  m = __longlong_as_double(mb);
#else
  u.i = mb;
  m = u.d;
#endif
  double k = (double)(e - 1023) + scale;
  if (m > kSqrt2) {
    m = m * 0.5;
    k = k + 1.0;
  }
  const double s = (m - 1.0) / (m + 1.0);
  const double s2 = s * s;
  double q = 1.0 / 23.0;
  q = q * s2 + 1.0 / 21.0;
  q = q * s2 + 1.0 / 19.0;
  q = q * s2 + 1.0 / 17.0;
  q = q * s2 + 1.0 / 15.0;
  q = q * s2 + 1.0 / 13.0;
  q = q * s2 + 1.0 / 11.0;
  q = q * s2 + 1.0 / 9.0;
  q = q * s2 + 1.0 / 7.0;
  q = q * s2 + 1.0 / 5.0;
  q = q * s2 + 1.0 / 3.0;
  q = q * s2 + 1.0;
  const double LN2_HI = 6.93147180369123816490e-01, LN2_LO = 1.90821492927058770002e-10;
  return (k * LN2_HI + (2.0 * s) * q) + k * LN2_LO;
}

/* Temperature-only terms, formed once per (params, T) on the host. */
struct Terms {
  int nc;
  double T, RT;
  double a[RSIM_EOS_NCMAX][RSIM_EOS_NCMAX];  /* a_ij = sqrt(a_i a_j)(1 - k_ij), Pa m^6/mol^2 */
  double b[RSIM_EOS_NCMAX];                  /* m^3/mol                                     */
  double kw[RSIM_EOS_NCMAX];                 /* Wilson: K_i = kw_i / p                       */
  double tc[RSIM_EOS_NCMAX];
  double tol;
  int maxit, stab_maxit;
};

inline Terms terms(const rsim_eos_params& P, double T) {  /* host */
  Terms t{};
  t.nc = P.nc;
  t.T = T;
  t.RT = kR * T;
  double ai[RSIM_EOS_NCMAX];
  for (int i = 0; i < P.nc; ++i) {
    const double w = P.omega[i];
    const double kap = w <= 0.49 ? (0.37464 + 1.54226 * w) - 0.26992 * w * w
                                 : ((0.379642 + 1.48503 * w) - 0.164423 * w * w) + 0.016666 * w * w * w;
    const double al = 1.0 + kap * (1.0 - sqrt(T / P.tc[i]));
    ai[i] = (0.457235529 * (kR * P.tc[i]) * (kR * P.tc[i]) / P.pc[i]) * (al * al);
    t.b[i] = 0.0777960739 * kR * P.tc[i] / P.pc[i];
    t.kw[i] = P.pc[i] * exp(5.373 * (1.0 + w) * (1.0 - P.tc[i] / T));
    t.tc[i] = P.tc[i];
  }
  for (int i = 0; i < P.nc; ++i)
    for (int j = 0; j < P.nc; ++j) t.a[i][j] = sqrt(ai[i] * ai[j]) * (1.0 - P.kij[i][j]);
  t.tol = P.flash_tol > 0.0 ? P.flash_tol : 1e-8;
  t.maxit = P.flash_maxit > 0 ? P.flash_maxit : 500;
  t.stab_maxit = P.stab_maxit > 0 ? P.stab_maxit : 200;
  return t;
}

/* Mixture parameters: A = a_m p/(RT)^2, B = b_m p/(RT); sa[i] = Σ_j x_j a_ij. */
template <int NC>
RSIM_HD void mix(const Terms& t, double p, const double* x, double& A, double& B, double& am, double& bm, double* sa) {
  am = 0.0;
  bm = 0.0;
  for (int i = 0; i < NC; ++i) {
    double s = 0.0;
    for (int j = 0; j < NC; ++j) s = s + x[j] * t.a[i][j];
    sa[i] = s;
    am = am + x[i] * s;
    bm = bm + x[i] * t.b[i];
  }
  A = am * p / (t.RT * t.RT);
  B = bm * p / t.RT;
}

/* Real roots of Z^3 - (1-B) Z^2 + (A - 3B^2 - 2B) Z - (AB - B^2 - B^3) that
 * exceed B, ascending: the largest by bracketed Newton from the Cauchy bound,
 * the others from the deflated quadratic, polished by Newton on the cubic.
 * Returns the count (0..3). */
RSIM_HD int cubic_roots(double A, double B, double* r) {
  const double c2 = -(1.0 - B), c1 = (A - 3.0 * B * B) - 2.0 * B, c0 = -((A * B - B * B) - B * B * B);
  auto f = [&](double z) { return ((z + c2) * z + c1) * z + c0; };
  auto df = [&](double z) { return (3.0 * z + 2.0 * c2) * z + c1; };
  // Largest root: Newton from the Cauchy bound, safeguarded by the bracket
  // [B, hi] (f(B) = -2B^2 <= 0 < f(hi)).  With three real roots the iterates
  // decrease monotonically onto the largest; with one real root left of the
  // inflection point a Newton step may leave the bracket and is replaced by
  // bisection.
  double lo = B, hi = 1.0 + fmax(fabs(c2), fmax(fabs(c1), fabs(c0)));
  double z = hi;
  for (int k = 0; k < 300; ++k) {
    const double fz = f(z);
    if (fz == 0.0) break;
    if (fz > 0.0) hi = z;
    else lo = z;
    const double d = df(z);
    double zn = d != 0.0 ? z - fz / d : 0.5 * (lo + hi);
    if (!(zn > lo && zn < hi)) zn = 0.5 * (lo + hi);
    if (fabs(zn - z) <= 1e-15 * fabs(z)) {
      z = zn;
      break;
    }
    z = zn;
  }
  const double z1 = z;
  const double pq = c2 + z1, qq = c1 + z1 * pq;  // Z^2 + pq Z + qq
  const double D = pq * pq - 4.0 * qq;
  double rr[3];
  int n = 0;
  rr[n++] = z1;
  if (D >= 0.0) {
    const double sd = sqrt(D);
    const double h = pq >= 0.0 ? -0.5 * (pq + sd) : -0.5 * (pq - sd);
    double z2 = h, z3 = h != 0.0 ? qq / h : 0.0;
    for (int it = 0; it < 2; ++it) {  // polish on the undeflated cubic
      const double d2 = df(z2), d3 = df(z3);
      if (d2 != 0.0) z2 = z2 - f(z2) / d2;
      if (d3 != 0.0) z3 = z3 - f(z3) / d3;
    }
    rr[n++] = z2;
    rr[n++] = z3;
  }
  int m = 0;
  for (int k = 0; k < n; ++k)
    if (rr[k] > B) r[m++] = rr[k];
  for (int i = 1; i < m; ++i)  // ascending (m <= 3)
    for (int j = i; j > 0 && r[j] < r[j - 1]; --j) {
      const double tmp = r[j];
      r[j] = r[j - 1];
      r[j - 1] = tmp;
    }
  return m;
}

/* ln φ_i (PR mixing rules). */
template <int NC>
RSIM_HD void lnphi(const Terms& t, double Z, double A, double B, double am, double bm, const double* sa, double* out) {
  const double lzb = rlog(Z - B);
  const double lr = rlog((Z + (1.0 + kSqrt2) * B) / (Z + (1.0 - kSqrt2) * B));
  const double pre = A / ((2.0 * kSqrt2) * B);
  for (int i = 0; i < NC; ++i) {
    const double bi = t.b[i] / bm;
    out[i] = (bi * (Z - 1.0) - lzb) - pre * ((2.0 * sa[i]) / am - bi) * lr;
  }
}

/* Z and ln φ of composition x at p with the given root selector; MIN_G picks
 * the root of lowest Gibbs energy Σ x_i ln φ_i instead.  Returns false when
 * no root exceeds B. */
/* Out of line on the device (RSIM_EOS_NI): it is called from six sites, and
 * inlining all of them overflows the instruction cache (ncu: "no_instructions"
 * was the top stall of the fully inlined kernel). */
#if defined(__CUDACC__)
#define RSIM_EOS_NI __host__ __device__ __noinline__
#else
#define RSIM_EOS_NI inline
#endif
template <int NC>
RSIM_EOS_NI bool phase_props(const Terms& t, double p, const double* x, int sel, bool min_g, double& Z, double* lp) {
  double A, B, am, bm, sa[NC];
  mix<NC>(t, p, x, A, B, am, bm, sa);
  double r[3];
  const int m = cubic_roots(A, B, r);
  if (m == 0) return false;
  if (B == 0.0 || am == 0.0) {  // ideal limit: Z = 1, φ = 1
    Z = r[m - 1];
    for (int i = 0; i < NC; ++i) lp[i] = 0.0;
    return true;
  }
  if (min_g && m > 1) {
    double l0[NC], l1[NC];
    lnphi<NC>(t, r[0], A, B, am, bm, sa, l0);
    lnphi<NC>(t, r[m - 1], A, B, am, bm, sa, l1);
    double g0 = 0.0, g1 = 0.0;
    for (int i = 0; i < NC; ++i) {
      g0 = g0 + x[i] * l0[i];
      g1 = g1 + x[i] * l1[i];
    }
    const bool lo = g0 <= g1;
    Z = lo ? r[0] : r[m - 1];
    for (int i = 0; i < NC; ++i) lp[i] = lo ? l0[i] : l1[i];
    return true;
  }
  Z = sel == RSIM_ROOT_LIQUID ? r[0] : r[m - 1];
  lnphi<NC>(t, Z, A, B, am, bm, sa, lp);
  return true;
}

/* Rachford-Rice: root of Σ z_i (K_i-1)/(1+ν(K_i-1)) in the
 * open window (1/(1-Kmax), 1/(1-Kmin)) by bracketed Newton / bisection.
 * Returns false when the precondition (some K > 1 and some K < 1) fails. */
template <int NC>
RSIM_HD bool rachford_rice(const double* z, const double* K, double& nu) {
  double kmax = 0.0, kmin = HUGE_VAL;
  for (int i = 0; i < NC; ++i)
    if (z[i] > 0.0) {
      kmax = fmax(kmax, K[i]);
      kmin = fmin(kmin, K[i]);
    }
  if (!(kmax > 1.0 && kmin < 1.0)) return false;
  double lo = 1.0 / (1.0 - kmax), hi = 1.0 / (1.0 - kmin);
  double v = 0.5 * (lo + hi);
  for (int it = 0; it < 300; ++it) {
    double g = 0.0, dg = 0.0;
    for (int i = 0; i < NC; ++i) {
      if (!(z[i] > 0.0)) continue;
      const double km = K[i] - 1.0;
      const double den = 1.0 + v * km;
      g = g + z[i] * km / den;
      dg = dg - z[i] * (km * km) / (den * den);
    }
    if (g == 0.0) break;
    if (g > 0.0) lo = v;  // g decreases in ν
    else hi = v;
    double vn = v - g / dg;
    if (!(vn > lo && vn < hi)) vn = 0.5 * (lo + hi);
    if (fabs(vn - v) <= 1e-15 * fmax(1.0, fabs(v)) || !(hi > lo)) {
      v = vn;
      break;
    }
    v = vn;
  }
  nu = v;
  return true;
}

/* Two-sided Michelsen stability test with Wilson initial K.
 * Returns true when stable; otherwise Kout holds the trial K of the most
 * negative tangent-plane distance. */
template <int NC>
RSIM_HD bool stability(const Terms& t, double p, const double* z, double* Kout, int* iters) {
  double Zz, lz[NC], d[NC];
  if (!phase_props<NC>(t, p, z, RSIM_ROOT_LIQUID, true, Zz, lz)) return true;
  double lzc[NC];
  for (int i = 0; i < NC; ++i) {
    lzc[i] = z[i] > 0.0 ? rlog(z[i]) : 0.0;
    d[i] = z[i] > 0.0 ? lzc[i] + lz[i] : 0.0;
  }
  bool stable = true;
  double best = 1.0 + 1e-10;  // ΣY > 1 <=> TPD < 0
  int its = 0;
  for (int trial = 0; trial < 2; ++trial) {  // 0: vapour-like Y = z K, 1: liquid-like Y = z / K
    double Y[NC];
    for (int i = 0; i < NC; ++i) {
      const double K = t.kw[i] / p;
      Y[i] = z[i] > 0.0 ? (trial == 0 ? z[i] * K : z[i] / K) : 0.0;
    }
    double sY = 0.0;
    bool trivial = false;
    for (int k = 0; k < t.stab_maxit; ++k) {
      ++its;
      sY = 0.0;
      for (int i = 0; i < NC; ++i) sY = sY + Y[i];
      double y[NC], ly[NC], Zy;
      for (int i = 0; i < NC; ++i) y[i] = Y[i] / sY;
      // trial phase root by the trial's side (vapour-like: largest, liquid-like: smallest)
      if (!phase_props<NC>(t, p, y, trial == 0 ? RSIM_ROOT_VAPOR : RSIM_ROOT_LIQUID, false, Zy, ly)) {
        trivial = true;
        break;
      }
      double err = 0.0, triv = 0.0;
      for (int i = 0; i < NC; ++i) {
        if (!(z[i] > 0.0)) continue;
        const double lY = d[i] - ly[i];  // ln Y_new
        const double Yn = rexp(lY);
        err = fmax(err, fabs(Yn / Y[i] - 1.0));
        const double lk = lY - lzc[i];     // ln(Y_new / z)
        triv = triv + lk * lk;
        Y[i] = Yn;
      }
      if (triv < 1e-8) {
        trivial = true;
        break;
      }
      if (err < 1e-10) break;
    }
    sY = 0.0;
    for (int i = 0; i < NC; ++i) sY = sY + Y[i];
    if (!trivial && sY > best) {
      best = sY;
      stable = false;
      for (int i = 0; i < NC; ++i)
        Kout[i] = z[i] > 0.0 ? (trial == 0 ? Y[i] / z[i] : z[i] / Y[i]) : 1.0;  // unnormalised Y: ΣzK ≠ 1
    }
  }
  *iters = its;
  return stable;
}

/* Flash result of one cell. */
template <int NC>
struct Flash {
  int status;        /* RSIM_PH_*                                  */
  double nu_g;       /* vapour mole fraction                        */
  double x[NC], y[NC];
  double Zo, Zg;     /* Z of the oil / gas phase (0 when absent)   */
  int iters;         /* stability + successive-substitution steps  */
};

/* Single-phase label of a stable mixture: the phase of its minimum-Gibbs root
 * when the cubic has several, else Kay's pseudo-critical temperature. */
template <int NC>
RSIM_HD int single_label(const Terms& t, double p, const double* z, double& Z) {
  double A, B, am, bm, sa[NC], lp[NC], r[3];
  mix<NC>(t, p, z, A, B, am, bm, sa);
  const int m = cubic_roots(A, B, r);
  phase_props<NC>(t, p, z, RSIM_ROOT_LIQUID, true, Z, lp);
  if (m > 1) return Z == r[0] ? RSIM_PH_OIL : RSIM_PH_GAS;
  double tpc = 0.0;
  for (int i = 0; i < NC; ++i) tpc = tpc + z[i] * t.tc[i];
  return t.T > tpc ? RSIM_PH_GAS : RSIM_PH_OIL;
}

/* flash(p, T, z): stability test, then successive
 * substitution K_i <- K_i f_o,i / f_g,i until max_i |f_o,i/f_g,i - 1| < tol.
 * Returns 0, or 1 on iteration cap (flash failure, single-phase result). */
template <int NC>
RSIM_HD int flash(const Terms& t, double p, const double* z, Flash<NC>& R) {
  double K[NC];
  int its = 0;
  R.nu_g = 0.0;
  R.Zo = 0.0;
  R.Zg = 0.0;
  auto single = [&]() {
    double Z;
    R.status = single_label<NC>(t, p, z, Z);
    R.nu_g = R.status == RSIM_PH_GAS ? 1.0 : 0.0;
    for (int i = 0; i < NC; ++i) { R.x[i] = z[i]; R.y[i] = z[i]; }
    if (R.status == RSIM_PH_GAS) R.Zg = Z;
    else R.Zo = Z;
  };
  if (stability<NC>(t, p, z, K, &its)) {
    single();
    R.iters = its;
    return 0;
  }
  int rc = 1;
  for (int k = 0; k < t.maxit; ++k) {
    ++its;
    double nu;
    if (!rachford_rice<NC>(z, K, nu)) {  // no sign change: no split
      single();
      R.iters = its;
      return 0;
    }
    // ν may lie outside (0, 1) while K settles (negative flash); the phase
    // split is decided on the converged ν below
    double x[NC], y[NC], sx = 0.0, sy = 0.0;
    for (int i = 0; i < NC; ++i) {
      x[i] = z[i] / (1.0 + nu * (K[i] - 1.0));
      y[i] = K[i] * x[i];
      sx = sx + x[i];
      sy = sy + y[i];
    }
    for (int i = 0; i < NC; ++i) { x[i] = x[i] / sx; y[i] = y[i] / sy; }
    double Zo, Zg, lo[NC], lg[NC];
    if (!phase_props<NC>(t, p, x, RSIM_ROOT_LIQUID, false, Zo, lo) ||
        !phase_props<NC>(t, p, y, RSIM_ROOT_VAPOR, false, Zg, lg))
      break;
    double err = 0.0, triv = 0.0;
    for (int i = 0; i < NC; ++i) {
      if (!(z[i] > 0.0)) continue;
      // f_o / f_g = (x φ_o) / (y φ_g)
      const double r = rexp((rlog(x[i]) + lo[i]) - (rlog(y[i]) + lg[i]));
      err = fmax(err, fabs(r - 1.0));
      K[i] = K[i] * r;
      const double lk = rlog(K[i]);
      triv = triv + lk * lk;
    }
    R.nu_g = nu;
    for (int i = 0; i < NC; ++i) { R.x[i] = x[i]; R.y[i] = y[i]; }
    R.Zo = Zo;
    R.Zg = Zg;
    if (triv < 1e-8) {  // trivial solution: declared stable
      single();
      R.iters = its;
      return 0;
    }
    if (err < t.tol) {
      if (!(nu > 0.0 && nu < 1.0)) {  // converged outside the two-phase window
        single();
        R.iters = its;
        return 0;
      }
      rc = 0;
      R.status = RSIM_PH_TWO;
      break;
    }
  }
  if (rc != 0) single();
  R.iters = its;
  return rc;
}

}  // namespace eos
}  // namespace rsim
#endif
#endif
