// krylov_dsm.cu — cluster-resident BiCGSTAB for small active systems.
//
// The localized solver's active systems are small (~10^2-10^4
// rows), so a Krylov iteration is bound by latency, not HBM.  This kernel runs
// the whole solve inside ONE thread-block cluster of G <= 16 CTAs:
//
//   * CTA g owns the contiguous local rows [g*RC, (g+1)*RC), RC = 64..1024
//     (RC/32 canonical warps, blockops.h); canonical warp sums are local, a
//     chunk partial is the 8-way tree of 8 warp sums
//     warp shuffles + an 8-way tree inside the CTA, and only the <= 64 chunk
//     partials cross DSMEM (one cluster barrier per reduction);
//   * the Krylov vectors and (when it fits) the ELL rows of each CTA live in
//     its shared memory for the whole solve — global traffic is the initial
//     load and the final store of x;
//   * SpMV reads neighbour entries from the owning CTA (own smem when local —
//     the usual case since the active list is sorted by cell — DSMEM else);
//   * the p- and s-updates are recomputed at the gather site from r, p_old,
//     v_old (same formulas, same bits), so an iteration needs 3 cluster
//     barriers instead of 5.
// Element formulas and reduction order are those of oracle/oracle.cpp
// bicgstab(); results are bit-identical to it and to krylov.cu.

#include <cooperative_groups.h>

#include <cstdlib>
#include <map>
#include <tuple>
#include <type_traits>

#include "ctx.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int GMAX = 16;
constexpr int NNCMAX = 256;             // NNC entries cached in smem per CTA
constexpr int NNC_GLOBAL = 0x40000000;  // flag in the range end: entries stay in global

struct DArgs {
  int32_t nA, nslot, maxit, fixed, LRC, nch, neu;
  int64_t cap;
  bool has_nnc;
  double rtol;
  const int32_t* ell_col;
  const double* ell_val;
  const int32_t* act;
  const int32_t* nptr;
  const int32_t* nnc_lcol;
  const double* nnc_val;
  const double* rhs;
  const double* F_raw;
  double* x;
  DevScalars* dsc;
  unsigned long long* trace;  // optional [8] cycle accumulators (RSIM_KTRACE)
};

template <int B, int NS, bool MS, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_krylov_dsm(const DArgs a) {
  extern __shared__ __align__(16) double dyn[];
  const int RC = 1 << a.LRC;
  // shared (read by neighbours): r, p[2], v[2]  (p, v double-buffered:
  // neighbours read the previous iterate while the owner writes the new one);
  // own-row-only vectors r0, x, s, t live in registers.
  double* vr = dyn;
  double* vp0 = vr + RC * B;
  double* vp1 = vp0 + RC * B;
  double* vv0 = vp1 + RC * B;
  double* vv1 = vv0 + RC * B;
  double* vph = vv1 + RC * B;  // M^-1 p  (Neumann-1 preconditioner only)
  double* vsh = vph + RC * B;  // M^-1 s
  double* mval = vsh + RC * B;                                    // [NS][RC][B*B]  (MS)
  int32_t* mcol = (int32_t*)(mval + (MS ? NS * RC * B * B : 0));   // [NS][RC]       (MS)
  int2* nrng = (int2*)(mcol + (MS ? NS * RC : 0));                // [RC] NNC ranges (has_nnc)
  double* nsv = (double*)(nrng + RC);                              // [NNCMAX][B*B] NNC blocks
  int32_t* nsc = (int32_t*)(nsv + NNCMAX * B * B);                 // [NNCMAX] NNC local columns
  __shared__ int nnc_cnt;

  __shared__ double* rb[GMAX];
  __shared__ double* pb[2][GMAX];
  __shared__ double* vb[2][GMAX];
  __shared__ double* wsb[GMAX];
  __shared__ double* phb[GMAX];
  __shared__ double* shb[GMAX];
  __shared__ double ws[2][3][32];  // [buf][q][warp]: canonical warp sums of this CTA
  __shared__ double res[3];

  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int G = (int)cluster.num_blocks();
  const int tid = threadIdx.x;
  const int w = tid >> 5, lane = tid & 31;
  const int64_t nr = a.nA;
  const int nch = a.nch;
  const int LWPC = a.LRC - 5;  // log2(warps per CTA)
  if (tid < G) {
    rb[tid] = cluster.map_shared_rank(vr, tid);
    pb[0][tid] = cluster.map_shared_rank(vp0, tid);
    pb[1][tid] = cluster.map_shared_rank(vp1, tid);
    vb[0][tid] = cluster.map_shared_rank(vv0, tid);
    vb[1][tid] = cluster.map_shared_rank(vv1, tid);
    wsb[tid] = cluster.map_shared_rank(&ws[0][0][0], tid);
    phb[tid] = cluster.map_shared_rank(vph, tid);
    shb[tid] = cluster.map_shared_rank(vsh, tid);
  }
  const int LSH = a.LRC;  // log2(RC)
  const int RCM = RC - 1;
  const int64_t row0 = (int64_t)rank * RC;
  const int64_t l = row0 + tid;
  const bool valid = l < nr;
  const int lam = tid;
  int wbuf = 0;

  // Canonical reduction of NQ per-row values (one per thread): warp trees
  // into shared memory, ONE cluster barrier (which also orders the CTA), then
  // warp 0 of every CTA gathers the 8 warp sums of each chunk via DSMEM and
  // finishes the canonical tree (8-way per chunk, then over the chunk
  // partials); one __syncthreads broadcasts the result.
  auto csync = [&]() {
    if (G == 1) __syncthreads();
    else cluster.sync();
  };
  auto reduce = [&](auto NQc, const double* val) {
    constexpr int NQ = decltype(NQc)::value;
    double v[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) v[q] = val[q];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
      for (int q = 0; q < NQ; ++q) v[q] = v[q] + __shfl_down_sync(0xffffffffu, v[q], off);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < NQ; ++q) ws[wbuf][q][w] = v[q];
    csync();
    for (int q = w; q < NQ; q += (1 << LWPC)) {  // warp w finishes quantities w, w+WPC, ...
      double cp[2] = {0.0, 0.0};
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // lane c holds chunk c (and c + 32)
        const int c = lane + 32 * h;
        if (c < nch) {
          double w8[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {  // canonical warp 8c+k lives on CTA gw >> LWPC
            const int gw = (c << 3) | k;
            w8[k] = ((int64_t)gw << 5) < nr ? wsb[gw >> LWPC][(wbuf * 3 + q) * 32 + (gw & ((1 << LWPC) - 1))]
                                            : 0.0;  // warp entirely past n_A: structural zero
          }
          cp[h] = tree8(w8);
        }
      }
      if (nch == 1) {
        if (lane == 0) res[q] = cp[0];
      } else {
        double W[8] = {warp_tree_n(cp[0], nch), warp_tree_n(cp[1], nch - 32), 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        if (lane == 0) res[q] = tree8(W);
      }
    }
    __syncthreads();
    wbuf ^= 1;
  };

  // neighbour value of the vector being multiplied, recomputed at the gather site:
  //   mode 0: p_new_j = r_j + beta (p_old_j - omega v_old_j)   (it > 1)
  //   mode 1: p_new_j = r_j                                     (it == 1)
  //   mode 2: s_j     = r_j - alpha v_new_j
  //   mode 3: (M^-1 p)_j, mode 4: (M^-1 s)_j   (stored by the owner, Neumann-1)
  auto gather = [&](int mode, int cur, int32_t j, double beta, double omega, double alpha, double* out) {
    const int g = j >> LSH;
    const int rr = (j & RCM) * B;
    const bool loc = g == rank;
    if (mode >= 3) {
      const double* X_ = (mode == 3 ? (loc ? vph : phb[g]) : (loc ? vsh : shb[g])) + rr;
#pragma unroll
      for (int e = 0; e < B; ++e) out[e] = X_[e];
      return;
    }
    const double* R_ = (loc ? vr : rb[g]) + rr;
    if (mode == 1) {
#pragma unroll
      for (int e = 0; e < B; ++e) out[e] = R_[e];
    } else if (mode == 0) {
      const double* P_ = (loc ? (cur ? vp0 : vp1) : pb[cur ^ 1][g]) + rr;
      const double* V_ = (loc ? (cur ? vv0 : vv1) : vb[cur ^ 1][g]) + rr;
#pragma unroll
      for (int e = 0; e < B; ++e) out[e] = R_[e] + beta * (P_[e] - omega * V_[e]);
    } else {
      const double* V_ = (loc ? (cur ? vv1 : vv0) : vb[cur][g]) + rr;
#pragma unroll
      for (int e = 0; e < B; ++e) out[e] = R_[e] - alpha * V_[e];
    }
  };

  // y = xown + Σ_slots Â_s x_col (+ NNC)
  auto spmv = [&](int mode, int cur, const double* xown, double beta, double omega, double alpha, double* y) {
    int32_t cl[NS];
    double xv[NS][B];
#pragma unroll
    for (int s = 0; s < NS; ++s) cl[s] = MS ? mcol[s * RC + lam] : __ldg(&a.ell_col[s * a.cap + l]);
#pragma unroll
    for (int s = 0; s < NS; ++s) gather(mode, cur, cl[s] < 0 ? (int32_t)l : cl[s], beta, omega, alpha, xv[s]);
    double acc[B];
#pragma unroll
    for (int e = 0; e < B; ++e) acc[e] = xown[e];
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (cl[s] >= 0) {
        const double* M = MS ? &mval[((size_t)s * RC + lam) * B * B] : &a.ell_val[((int64_t)s * a.cap + l) * B * B];
        rsim::blk::gemv_acc_flat<B>(M, xv[s], acc);
      }
    if (a.has_nnc) {
      const int2 rg = nrng[lam];
      if (rg.y & NNC_GLOBAL) {
        for (int32_t q = rg.x; q < (rg.y & ~NNC_GLOBAL); ++q) {
          const int32_t c2 = a.nnc_lcol[q];
          if (c2 >= 0) {
            double xn[B];
            gather(mode, cur, c2, beta, omega, alpha, xn);
            rsim::blk::gemv_acc_flat<B>(&a.nnc_val[(int64_t)q * B * B], xn, acc);
          }
        }
      } else {
        for (int32_t q = rg.x; q < rg.y; ++q) {
          double xn[B];
          gather(mode, cur, nsc[q], beta, omega, alpha, xn);
          rsim::blk::gemv_acc_flat<B>(&nsv[q * B * B], xn, acc);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < B; ++e) y[e] = acc[e];
  };

  double r0r[B], xr[B], sr[B], tr_[B];
#pragma unroll
  for (int e = 0; e < B; ++e) { r0r[e] = 0.0; xr[e] = 0.0; sr[e] = 0.0; tr_[e] = 0.0; }
  // ---- load: matrix rows (MS), rhs -> r, r0; x = 0; (b,b), (F,F)
  if (tid == 0) nnc_cnt = 0;
  __syncthreads();
  {
    double val[3] = {0.0, 0.0, 0.0};
    if (valid) {
      double bv[B], fv[B];
#pragma unroll
      for (int e = 0; e < B; ++e) {
        bv[e] = a.rhs[l * B + e];
        fv[e] = a.F_raw[l * B + e];
        vr[lam * B + e] = bv[e];
        r0r[e] = bv[e];
        xr[e] = 0.0;
        vp0[lam * B + e] = 0.0; vp1[lam * B + e] = 0.0;
        vv0[lam * B + e] = 0.0; vv1[lam * B + e] = 0.0;
      }
      val[0] = rsim::blk::rowdot<B>(bv, bv);
      val[1] = rsim::blk::rowdot<B>(fv, fv);
      if (a.has_nnc) {  // cache this row's active NNC blocks in smem (order preserved)
        const int64_t i = a.act[l];
        const int32_t q0 = a.nptr[i], q1 = a.nptr[i + 1];
        int k = 0;
        for (int32_t q = q0; q < q1; ++q) k += a.nnc_lcol[q] >= 0;
        const int base = k ? atomicAdd(&nnc_cnt, k) : 0;
        if (base + k <= NNCMAX) {
          int m = base;
          for (int32_t q = q0; q < q1; ++q) {
            const int32_t c2 = a.nnc_lcol[q];
            if (c2 < 0) continue;
            nsc[m] = c2;
#pragma unroll
            for (int e = 0; e < B * B; ++e) nsv[m * B * B + e] = a.nnc_val[(int64_t)q * B * B + e];
            ++m;
          }
          nrng[lam] = make_int2(base, base + k);
        } else {
          nrng[lam] = make_int2(q0, q1 | NNC_GLOBAL);
        }
      }
      if (MS) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const int32_t cl = (s < a.nslot) ? a.ell_col[s * a.cap + l] : -1;
          mcol[s * RC + lam] = cl;
          if (cl >= 0)
#pragma unroll
            for (int e = 0; e < B * B; ++e)
              mval[((size_t)s * RC + lam) * B * B + e] = a.ell_val[((int64_t)s * a.cap + l) * B * B + e];
        }
      }
    }
    reduce(std::integral_constant<int, 2>{}, val);
  }
  const double bb = res[0];
  if (rank == 0 && tid == 0) a.dsc->f2 = sqrt(res[1]);
  const double bnorm = sqrt(bb);
  const bool fixed = a.fixed > 0;
  const int maxit = fixed ? a.fixed : a.maxit;
  const double tol = a.rtol * bnorm;
  double rho = 1.0, alpha = 1.0, omega = 1.0, rho_new = bb;
  int status = RSIM_OK;
  int it = 0;
  double relres = 0.0;
  int cur = 0;  // buffer holding the current iteration's p, v
  if (bnorm != 0.0) {
    status = RSIM_ENOCONV;
    unsigned long long tc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const bool tr = a.trace && rank == 0 && tid == 0;
    long long t0 = clock64();
#define KT_MARK(k) do { if (tr) { long long t1 = clock64(); tc[k] += (unsigned long long)(t1 - t0); t0 = t1; } } while (0)
    int it_total = 0;
    // attempt 0: as configured; attempt 1 (only after a Neumann-1 breakdown or
    // cap): block-Jacobi only, restarted from x0 = 0 (same rule as the oracle)
    for (int attempt = 0; attempt < (a.neu ? 2 : 1); ++attempt) {
    const bool neu = a.neu && attempt == 0;
    if (attempt) {
      if (valid)
#pragma unroll
        for (int e = 0; e < B; ++e) {
          vr[lam * B + e] = a.rhs[l * B + e];
          xr[e] = 0.0;
        }
      rho = 1.0; alpha = 1.0; omega = 1.0; rho_new = bb;
      cur = 0;
      status = RSIM_ENOCONV;
      csync();
    }
    for (it = 1; it <= maxit; ++it) {
      KT_MARK(7);
      const double beta = (it == 1) ? 0.0 : (rho_new / rho) * (alpha / omega);
      double* vpc = cur ? vp1 : vp0;
      double* vvc = cur ? vv1 : vv0;
      const double* vpo = cur ? vp0 : vp1;
      const double* vvo = cur ? vv0 : vv1;
      // ---- p = r + β (p − ω v) (own + recomputed for neighbours)
      //      BJ:  v = Â p;   Neumann-1: ph = p + (p − Â p), barrier, v = Â ph;  (r0, v)
      double phr[B];
      {
        double val[3] = {0.0, 0.0, 0.0};
        double pown[B], y[B];
        if (valid) {
#pragma unroll
          for (int e = 0; e < B; ++e) {
            const int q = lam * B + e;
            pown[e] = (it == 1) ? vr[q] : vr[q] + beta * (vpo[q] - omega * vvo[q]);
            vpc[q] = pown[e];
          }
          spmv(it == 1 ? 1 : 0, cur, pown, beta, omega, 0.0, y);
        }
        if (neu) {
          if (valid)
#pragma unroll
            for (int e = 0; e < B; ++e) {
              phr[e] = pown[e] + (pown[e] - y[e]);
              vph[lam * B + e] = phr[e];
            }
          csync();
          if (valid) spmv(3, cur, phr, 0.0, 0.0, 0.0, y);
        } else {
#pragma unroll
          for (int e = 0; e < B; ++e) phr[e] = pown[e];
        }
        if (valid) {
#pragma unroll
          for (int e = 0; e < B; ++e) vvc[lam * B + e] = y[e];
          val[0] = rsim::blk::rowdot<B>(r0r, y);
        }
        KT_MARK(0);
        reduce(std::integral_constant<int, 1>{}, val);
        KT_MARK(1);
      }
      const double r0v = res[0];
      if (r0v == 0.0 || !isfinite(r0v)) { status = RSIM_ENUM; break; }
      alpha = rho_new / r0v;
      // ---- s = r − α v (own + recomputed for neighbours)
      //      BJ: t = Â s;  Neumann-1: sh = s + (s − Â s), barrier, t = Â sh;  (s,s), (t,s), (t,t)
      double shr[B];
      {
        double val[3] = {0.0, 0.0, 0.0};
        double y[B];
        if (valid) {
#pragma unroll
          for (int e = 0; e < B; ++e) sr[e] = vr[lam * B + e] - alpha * vvc[lam * B + e];
          spmv(2, cur, sr, 0.0, 0.0, alpha, y);
        }
        if (neu) {
          if (valid)
#pragma unroll
            for (int e = 0; e < B; ++e) {
              shr[e] = sr[e] + (sr[e] - y[e]);
              vsh[lam * B + e] = shr[e];
            }
          csync();
          if (valid) spmv(4, cur, shr, 0.0, 0.0, 0.0, y);
        } else {
#pragma unroll
          for (int e = 0; e < B; ++e) shr[e] = sr[e];
        }
        if (valid) {
#pragma unroll
          for (int e = 0; e < B; ++e) tr_[e] = y[e];
          val[0] = rsim::blk::rowdot<B>(sr, sr);
          val[1] = rsim::blk::rowdot<B>(y, sr);
          val[2] = rsim::blk::rowdot<B>(y, y);
        }
        KT_MARK(2);
        reduce(std::integral_constant<int, 3>{}, val);
        KT_MARK(3);
      }
      const double ssn = res[0], ts = res[1], tt = res[2];
      if (!fixed && sqrt(ssn) <= tol) {
        if (valid)
#pragma unroll
          for (int e = 0; e < B; ++e) xr[e] = xr[e] + alpha * phr[e];
        relres = sqrt(ssn) / bnorm;
        status = RSIM_OK;
        break;
      }
      if (tt == 0.0 || !isfinite(tt)) { status = RSIM_ENUM; break; }
      omega = ts / tt;
      // ---- x, r update ; (r, r), (r0, r)
      {
        double val[3] = {0.0, 0.0, 0.0};
        if (valid) {
          double rv[B];
#pragma unroll
          for (int e = 0; e < B; ++e) {
            xr[e] = (xr[e] + alpha * phr[e]) + omega * shr[e];
            rv[e] = sr[e] - omega * tr_[e];
            vr[lam * B + e] = rv[e];
          }
          val[0] = rsim::blk::rowdot<B>(rv, rv);
          val[1] = rsim::blk::rowdot<B>(r0r, rv);
        }
        KT_MARK(4);
        reduce(std::integral_constant<int, 2>{}, val);
        KT_MARK(5);
      }
      const double rr = res[0];
      rho = rho_new;
      rho_new = res[1];
      relres = sqrt(rr) / bnorm;
      if (!fixed && sqrt(rr) <= tol) { status = RSIM_OK; break; }
      if (omega == 0.0 || rho_new == 0.0 || !isfinite(rho_new)) { status = RSIM_ENUM; break; }
      cur ^= 1;
    }
    if (it > maxit) { it = maxit; status = fixed ? RSIM_OK : RSIM_ENOCONV; }
    it_total += it;
    if (!(neu && (status == RSIM_ENUM || status == RSIM_ENOCONV))) break;
    }
    it = it_total;
    if (tr)
      for (int k = 0; k < 8; ++k) atomicAdd(&a.trace[k], tc[k]);
#undef KT_MARK
  }
  if (valid)
#pragma unroll
    for (int e = 0; e < B; ++e) a.x[l * B + e] = xr[e];
  if (rank == 0 && tid == 0) {
    a.dsc->lin_iters = it;
    a.dsc->lin_relres = relres;
    if (status != RSIM_OK) a.dsc->status = status;
  }
  cluster.sync();  // keep every CTA's shared memory alive until all remote reads are done
}

size_t smem_bytes(int B, int NS, bool MS, int LRC) {
  const size_t R = (size_t)1 << LRC;
  size_t b = 7 * R * B * sizeof(double) + R * sizeof(int2) + NNCMAX * (B * B * sizeof(double) + sizeof(int32_t));
  if (MS) b += NS * R * B * B * sizeof(double) + NS * R * sizeof(int32_t);
  return b;
}

template <int B, int NS, bool MS, int MAXT>
int launch_t(rsim_gpu_ctx* c, const DArgs& a, int G, int TPB, size_t smem, bool* ok) {
  static std::map<std::tuple<int, int, size_t>, bool> fits;
  auto key = std::make_tuple(G, TPB, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G, 1, 1);
  cfg.blockDim = dim3(TPB, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // the dynamic-smem attribute is a per-kernel maximum: only ever raise it
  static size_t attr_max = 0;
  auto ensure_attr = [&](size_t need) -> cudaError_t {
    if (need <= attr_max) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k_krylov_dsm<B, NS, MS, MAXT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)need);
    if (e == cudaSuccess) attr_max = need;
    return e;
  };
  auto itf = fits.find(key);
  if (itf == fits.end()) {
    bool f = ensure_attr(smem) == cudaSuccess;
    cudaFuncSetAttribute(k_krylov_dsm<B, NS, MS, MAXT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int ncl = 0;
    f = f && cudaOccupancyMaxActiveClusters(&ncl, k_krylov_dsm<B, NS, MS, MAXT>, &cfg) == cudaSuccess && ncl >= 1;
    cudaGetLastError();
    itf = fits.emplace(key, f).first;
  }
  *ok = itf->second;
  if (!*ok) return RSIM_OK;
  RSIM_CUDA(ensure_attr(smem));
  RSIM_CUDA(cudaLaunchKernelEx(&cfg, k_krylov_dsm<B, NS, MS, MAXT>, a));
  return RSIM_OK;
}

template <int B, int NS>
int launch_bn(rsim_gpu_ctx* c, DArgs& a, int G, int TPB, bool* ok) {
  const size_t with_m = smem_bytes(B, NS, true, a.LRC), without = smem_bytes(B, NS, false, a.LRC);
  const size_t cap = 220 * 1024;
  if (with_m <= cap) {
    int r = TPB <= 512 ? launch_t<B, NS, true, 512>(c, a, G, TPB, with_m, ok)
                       : launch_t<B, NS, true, 1024>(c, a, G, TPB, with_m, ok);
    if (r != RSIM_OK || *ok) return r;
  }
  if (without <= cap)
    return TPB <= 512 ? launch_t<B, NS, false, 512>(c, a, G, TPB, without, ok)
                      : launch_t<B, NS, false, 1024>(c, a, G, TPB, without, ok);
  *ok = false;
  return RSIM_OK;
}

int dsm_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("RSIM_NO_CLUSTER");
    v = (e && *e == '1') ? 1 : 0;
  }
  return v;
}

}  // namespace

int launch_krylov_dsm(rsim_gpu_ctx* c, const rsim_solver_opts* o) {
  if (dsm_disabled() || c->nA <= 0) return RSIM_ENOTAPPLICABLE;
  const int nch = (c->nA + RSIM_RED_CHUNK - 1) / RSIM_RED_CHUNK;
  if (nch > 4 * GMAX) return RSIM_ENOTAPPLICABLE;
  DArgs a;
  a.nA = c->nA;
  a.nslot = c->nslot;
  a.maxit = o->lin_maxit;
  a.fixed = o->fixed_lin_iters;
  a.neu = o->precond == RSIM_PREC_NEUMANN1;
  a.nch = nch;
  a.cap = c->n;
  a.has_nnc = c->has_nnc;
  a.rtol = o->lin_rtol;
  a.ell_col = c->ell_col;
  a.ell_val = c->ell_val;
  a.act = c->act;
  a.nptr = c->nptr;
  a.nnc_lcol = c->nnc_lcol;
  a.nnc_val = c->nnc_val;
  a.rhs = c->rhs;
  a.F_raw = c->F_raw;
  a.x = c->x;
  a.trace = c->ktrace;
  a.dsc = c->dsc;
  // one chunk per CTA when possible (G = nch <= 16), else 2 or 4 chunks per CTA
  // (powers of two, so the owner of a row is a shift)
  // rows per CTA: the smallest power of two >= 64 that fits the system in
  // <= 16 CTAs (more CTAs = shorter per-CTA critical path)
  static int minl = -1;
  if (minl < 0) {
    const char* e = std::getenv("RSIM_DSM_MINLRC");
    minl = e ? std::atoi(e) : 6;
  }
  for (int LRC = minl; LRC <= 10; ++LRC) {
    const int RC = 1 << LRC;
    const int G = (c->nA + RC - 1) / RC;
    if (G > GMAX) continue;
    a.LRC = LRC;
    const int TPB = RC;
    bool ok = false;
    int r;
    switch (c->b * 10 + c->nslot) {
      case 14: r = launch_bn<1, 4>(c, a, G, TPB, &ok); break;
      case 16: r = launch_bn<1, 6>(c, a, G, TPB, &ok); break;
      case 24: r = launch_bn<2, 4>(c, a, G, TPB, &ok); break;
      case 26: r = launch_bn<2, 6>(c, a, G, TPB, &ok); break;
      case 34: r = launch_bn<3, 4>(c, a, G, TPB, &ok); break;
      default: r = launch_bn<3, 6>(c, a, G, TPB, &ok); break;
    }
    if (r != RSIM_OK) return r;
    if (ok) {
      c->launches++;
      RSIM_CUDA(cudaGetLastError());
      return RSIM_OK;
    }
  }
  return RSIM_ENOTAPPLICABLE;
}
