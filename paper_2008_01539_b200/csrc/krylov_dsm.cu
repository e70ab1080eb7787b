// krylov_dsm.cu — cluster-resident BiCGSTAB for small active systems.
//
// The localized solver's active systems are small (~10^2-10^4
// rows), so a Krylov iteration is bound by latency, not HBM.  This kernel runs
// the whole solve inside ONE thread-block cluster of G = 8 or 16 CTAs:
//
//   * the canonical reduction order (blockops.h) is mapped onto the cluster:
//     a 2048-row chunk is 8 "items" of 256 rows; item k of chunk c lives on
//     CTA ((c mod H) * 8 + k), row t of the item on thread t of that CTA's
//     segment (c div H).  The canonical per-thread sum Σ_k v[t + 256k] is
//     therefore a sum over the 8 CTAs' shared memories (DSMEM), in k order;
//   * the Krylov vectors r, r0, p, v, s, t, x and (when it fits) the ELL matrix
//     rows of each CTA live in its shared memory for the whole solve — the only
//     global traffic is the initial load and the final store of x;
//   * SpMV gathers neighbour entries from the owning CTA through DSMEM;
//   * phases are separated by the hardware cluster barrier (≈380 cycles)
//     instead of a grid-wide barrier; per-row reduction values are staged in
//     double-buffered shared memory so one barrier per phase suffices.
// Element formulas and reduction order are those of oracle/oracle.cpp
// bicgstab(); results are bit-identical to it and to krylov.cu.
#include <cooperative_groups.h>

#include <cstdlib>
#include <map>
#include <tuple>

#include "ctx.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int GMAX = 16;
constexpr int SEG = RSIM_RED_THREADS;  // 256 rows per (chunk, item)

struct DArgs {
  int32_t nA, nslot, maxit, fixed, S, H, nch;
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
};

__device__ __forceinline__ int owner_cta(int64_t j, int H) { return ((int)((j >> 11) & (H - 1)) << 3) | (int)((j >> 8) & 7); }
__device__ __forceinline__ int owner_row(int64_t j, int H) {
  return ((int)((j >> 11) >> (H - 1)) << 8) | (int)(j & 255);
}

template <int B, int NS, bool MS>
__global__ void __launch_bounds__(1024, 1) k_krylov_dsm(const DArgs a) {
  extern __shared__ __align__(16) double dyn[];
  const int R = a.S * SEG;
  double* vr = dyn;
  double* vp = vr + R * B;
  double* vv = vp + R * B;
  double* vs = vv + R * B;
  double* vt = vs + R * B;
  double* vr0 = vt + R * B;
  double* vx = vr0 + R * B;
  double* stg = vx + R * B;              // [2 buf][2 q][R]
  double* mval = stg + 4 * R;            // [NS][R][B*B]   (MS)
  int32_t* mcol = (int32_t*)(mval + (MS ? NS * R * B * B : 0));  // [NS][R] (MS)

  __shared__ double* pb[GMAX];
  __shared__ double* sb[GMAX];
  __shared__ double* stb[GMAX];
  __shared__ double wsum[2][4][8];
  __shared__ double part[2][32];
  __shared__ double res[2];

  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int G = (int)cluster.num_blocks();
  const int tid = threadIdx.x;
  const int H = a.H;
  const int64_t nr = a.nA;
  const int nch = a.nch;
  if (tid < G) {
    pb[tid] = cluster.map_shared_rank(vp, tid);
    sb[tid] = cluster.map_shared_rank(vs, tid);
    stb[tid] = cluster.map_shared_rank(stg, tid);
  }
  // my row
  const int sig = tid >> 8, t8 = tid & 255;
  const int64_t c_my = (int64_t)sig * H + (rank >> 3);
  const int64_t l = (c_my << 11) | ((int64_t)(rank & 7) << 8) | t8;
  const bool valid = l < nr;
  const int lam = tid;

  // canonical cluster reduction of NQ staged quantities in buffer `buf`
  auto reduce = [&](int NQ, int buf) {
    for (int c0 = 0; c0 < nch; c0 += a.S) {
      const int c = c0 + sig;
      double sq[2] = {0.0, 0.0};
      if (c < nch) {
        const int64_t base = (int64_t)c << 11;
        const int m = (int)(nr - base < RSIM_RED_CHUNK ? nr - base : RSIM_RED_CHUNK);
        const int g0 = (c & (H - 1)) << 3;
        const int lam0 = ((c >> (H - 1)) << 8) | t8;
#pragma unroll
        for (int k = 0; k < RSIM_RED_ITEMS; ++k) {
          const int idx = (k << 8) + t8;
          if (idx < m) {
            const double* src = stb[g0 + k] + (size_t)(buf * 2) * R + lam0;
            sq[0] = sq[0] + src[0];
            if (NQ > 1) sq[1] = sq[1] + src[R];
          }
        }
      }
      for (int q = 0; q < NQ; ++q) {
        double v = sq[q];
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) v = v + __shfl_down_sync(0xffffffffu, v, off);
        if ((tid & 31) == 0) wsum[q][sig][(tid >> 5) & 7] = v;
      }
      __syncthreads();
      if (tid < a.S * NQ) {
        const int sg = tid % a.S, q = tid / a.S;
        const int cc = c0 + sg;
        if (cc < nch) {
          double w[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) w[k] = wsum[q][sg][k];
#pragma unroll
          for (int off = 4; off >= 1; off >>= 1)
#pragma unroll
            for (int k = 0; k < off; ++k) w[k] = w[k] + w[k + off];
          part[q][cc] = w[0];
        }
      }
      __syncthreads();
    }
    // canonical reduction over the nch chunk partials (one 256-"thread" chunk)
    if (tid < 256) {
      for (int q = 0; q < NQ; ++q) {
        double v = (tid < nch) ? part[q][tid] : 0.0;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) v = v + __shfl_down_sync(0xffffffffu, v, off);
        if ((tid & 31) == 0) wsum[q][0][tid >> 5] = v;
      }
    }
    __syncthreads();
    if (tid < NQ) {
      double w[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) w[k] = wsum[tid][0][k];
#pragma unroll
      for (int off = 4; off >= 1; off >>= 1)
#pragma unroll
        for (int k = 0; k < off; ++k) w[k] = w[k] + w[k + off];
      res[tid] = w[0];
    }
    __syncthreads();
  };

  // SpMV row: y = x_own + Σ_slots Â_s x_col (+ NNC), x gathered via DSMEM
  auto spmv = [&](double* const* xb, const double* xloc, double* y) {
    double acc[B];
#pragma unroll
    for (int e = 0; e < B; ++e) acc[e] = xloc[lam * B + e];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int32_t cl = MS ? mcol[s * R + lam] : __ldg(&a.ell_col[s * a.cap + l]);
      if (cl >= 0) {
        const double* xr = xb[owner_cta(cl, H)] + owner_row(cl, H) * B;
        const double* M = MS ? &mval[((size_t)s * R + lam) * B * B] : &a.ell_val[((int64_t)s * a.cap + l) * B * B];
        rsim::blk::gemv_acc_flat<B>(M, xr, acc);
      }
    }
    if (a.has_nnc) {
      const int64_t i = a.act[l];
      const int32_t q0 = a.nptr[i], q1 = a.nptr[i + 1];
      for (int32_t q = q0; q < q1; ++q) {
        const int32_t cl = a.nnc_lcol[q];
        if (cl >= 0)
          rsim::blk::gemv_acc_flat<B>(&a.nnc_val[(int64_t)q * B * B], xb[owner_cta(cl, H)] + owner_row(cl, H) * B,
                                      acc);
      }
    }
#pragma unroll
    for (int e = 0; e < B; ++e) y[e] = acc[e];
  };

  // ---- load: matrix rows (MS), rhs -> r, r0; x = 0; stage (b,b), (F,F)
  int buf = 0;
  {
    double q0 = 0.0, q1 = 0.0;
    if (valid) {
      double bv[B], fv[B];
#pragma unroll
      for (int e = 0; e < B; ++e) {
        bv[e] = a.rhs[l * B + e];
        fv[e] = a.F_raw[l * B + e];
        vr[lam * B + e] = bv[e];
        vr0[lam * B + e] = bv[e];
        vx[lam * B + e] = 0.0;
        vp[lam * B + e] = 0.0;
        vv[lam * B + e] = 0.0;
      }
      q0 = rsim::blk::rowdot<B>(bv, bv);
      q1 = rsim::blk::rowdot<B>(fv, fv);
      if (MS) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const int32_t cl = (s < a.nslot) ? a.ell_col[s * a.cap + l] : -1;
          mcol[s * R + lam] = cl;
          if (cl >= 0)
#pragma unroll
            for (int e = 0; e < B * B; ++e)
              mval[((size_t)s * R + lam) * B * B + e] = a.ell_val[((int64_t)s * a.cap + l) * B * B + e];
        }
      }
    }
    stg[(buf * 2 + 0) * R + lam] = q0;
    stg[(buf * 2 + 1) * R + lam] = q1;
  }
  cluster.sync();
  reduce(2, buf);
  buf ^= 1;
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
  if (bnorm != 0.0) {
    status = RSIM_ENOCONV;
    for (it = 1; it <= maxit; ++it) {
      const double beta = (it == 1) ? 0.0 : (rho_new / rho) * (alpha / omega);
      // ---- p update
      if (valid)
#pragma unroll
        for (int e = 0; e < B; ++e) {
          const int q = lam * B + e;
          vp[q] = (it == 1) ? vr[q] : vr[q] + beta * (vp[q] - omega * vv[q]);
        }
      cluster.sync();
      // ---- v = Â p ; (r0, v)
      {
        double q0 = 0.0;
        if (valid) {
          double y[B];
          spmv(pb, vp, y);
#pragma unroll
          for (int e = 0; e < B; ++e) vv[lam * B + e] = y[e];
          q0 = rsim::blk::rowdot<B>(&vr0[lam * B], y);
        }
        stg[(buf * 2) * R + lam] = q0;
      }
      cluster.sync();
      reduce(1, buf);
      buf ^= 1;
      const double r0v = res[0];
      if (r0v == 0.0 || !isfinite(r0v)) { status = RSIM_ENUM; break; }
      alpha = rho_new / r0v;
      // ---- s = r − α v ; (s, s)
      {
        double q0 = 0.0;
        if (valid) {
          double sv[B];
#pragma unroll
          for (int e = 0; e < B; ++e) {
            const int q = lam * B + e;
            sv[e] = vr[q] - alpha * vv[q];
            vs[q] = sv[e];
          }
          q0 = rsim::blk::rowdot<B>(sv, sv);
        }
        stg[(buf * 2) * R + lam] = q0;
      }
      cluster.sync();
      reduce(1, buf);
      buf ^= 1;
      const double ssn = res[0];
      if (!fixed && sqrt(ssn) <= tol) {
        if (valid)
#pragma unroll
          for (int e = 0; e < B; ++e) vx[lam * B + e] = vx[lam * B + e] + alpha * vp[lam * B + e];
        relres = sqrt(ssn) / bnorm;
        status = RSIM_OK;
        break;
      }
      // ---- t = Â s ; (t, s), (t, t)
      {
        double q0 = 0.0, q1 = 0.0;
        if (valid) {
          double y[B];
          spmv(sb, vs, y);
#pragma unroll
          for (int e = 0; e < B; ++e) vt[lam * B + e] = y[e];
          q0 = rsim::blk::rowdot<B>(y, &vs[lam * B]);
          q1 = rsim::blk::rowdot<B>(y, y);
        }
        stg[(buf * 2) * R + lam] = q0;
        stg[(buf * 2 + 1) * R + lam] = q1;
      }
      cluster.sync();
      reduce(2, buf);
      buf ^= 1;
      const double ts = res[0], tt = res[1];
      if (tt == 0.0 || !isfinite(tt)) { status = RSIM_ENUM; break; }
      omega = ts / tt;
      // ---- x, r update ; (r, r), (r0, r)
      {
        double q0 = 0.0, q1 = 0.0;
        if (valid) {
          double rv[B];
#pragma unroll
          for (int e = 0; e < B; ++e) {
            const int q = lam * B + e;
            const double sq = vs[q];
            vx[q] = (vx[q] + alpha * vp[q]) + omega * sq;
            rv[e] = sq - omega * vt[q];
            vr[q] = rv[e];
          }
          q0 = rsim::blk::rowdot<B>(rv, rv);
          q1 = rsim::blk::rowdot<B>(&vr0[lam * B], rv);
        }
        stg[(buf * 2) * R + lam] = q0;
        stg[(buf * 2 + 1) * R + lam] = q1;
      }
      cluster.sync();
      reduce(2, buf);
      buf ^= 1;
      const double rr = res[0];
      rho = rho_new;
      rho_new = res[1];
      relres = sqrt(rr) / bnorm;
      if (!fixed && sqrt(rr) <= tol) { status = RSIM_OK; break; }
      if (omega == 0.0 || rho_new == 0.0 || !isfinite(rho_new)) { status = RSIM_ENUM; break; }
    }
    if (it > maxit) { it = maxit; status = fixed ? RSIM_OK : RSIM_ENOCONV; }
  }
  if (valid)
#pragma unroll
    for (int e = 0; e < B; ++e) a.x[l * B + e] = vx[lam * B + e];
  if (rank == 0 && tid == 0) {
    a.dsc->lin_iters = it;
    a.dsc->lin_relres = relres;
    if (status != RSIM_OK) a.dsc->status = status;
  }
  cluster.sync();  // keep every CTA's shared memory alive until all remote reads are done
}

size_t smem_bytes(int B, int NS, bool MS, int S) {
  const size_t R = (size_t)S * SEG;
  size_t b = (7 * R * B + 4 * R) * sizeof(double);
  if (MS) b += NS * R * B * B * sizeof(double) + NS * R * sizeof(int32_t);
  return b;
}

template <int B, int NS, bool MS>
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
  auto itf = fits.find(key);
  if (itf == fits.end()) {
    cudaFuncSetAttribute(k_krylov_dsm<B, NS, MS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_krylov_dsm<B, NS, MS>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int ncl = 0;
    bool f = cudaOccupancyMaxActiveClusters(&ncl, k_krylov_dsm<B, NS, MS>, &cfg) == cudaSuccess && ncl >= 1;
    cudaGetLastError();
    itf = fits.emplace(key, f).first;
  }
  *ok = itf->second;
  if (!*ok) return RSIM_OK;
  RSIM_CUDA(cudaFuncSetAttribute(k_krylov_dsm<B, NS, MS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  RSIM_CUDA(cudaLaunchKernelEx(&cfg, k_krylov_dsm<B, NS, MS>, a));
  return RSIM_OK;
}

template <int B, int NS>
int launch_bn(rsim_gpu_ctx* c, DArgs& a, int G, int TPB, bool* ok) {
  const size_t with_m = smem_bytes(B, NS, true, a.S), without = smem_bytes(B, NS, false, a.S);
  const size_t cap = 220 * 1024;
  if (with_m <= cap) {
    int r = launch_t<B, NS, true>(c, a, G, TPB, with_m, ok);
    if (r != RSIM_OK || *ok) return r;
  }
  if (without <= cap) return launch_t<B, NS, false>(c, a, G, TPB, without, ok);
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
  if (nch > 8) return RSIM_ENOTAPPLICABLE;
  DArgs a;
  a.nA = c->nA;
  a.nslot = c->nslot;
  a.maxit = o->lin_maxit;
  a.fixed = o->fixed_lin_iters;
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
  a.dsc = c->dsc;
  // prefer 16 CTAs (two chunk parities) when there are >= 2 chunks
  for (int H = (nch >= 2 ? 2 : 1); H >= 1; --H) {
    const int S = (nch + H - 1) / H;
    if (S > 4) continue;
    a.H = H;
    a.S = S;
    const int G = 8 * H, TPB = SEG * S;
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
