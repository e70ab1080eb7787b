// krylov_gmres.cu — GMRES(30) (north star / SURVEY.md §8 a10 alternative to
// BiCGSTAB) as ONE persistent cooperative kernel per linear solve.
//
// Right-preconditioned (block-Jacobi fused into Â: M = I; or the Neumann-1
// polynomial M^{-1} z = z + (z − Â z)), x0 = 0, classical Gram-Schmidt: the j+1
// projections (w, v_i) of an Arnoldi step are reduced TOGETHER (one grid
// barrier for all of them), then w −= Σ_i h_ij v_i in ascending i, then ‖w‖;
// Givens rotations on the Hessenberg column (computed redundantly by every
// CTA from the same canonical sums); restart from the true residual.
// Element formulas and reduction order follow oracle/oracle.cpp gmres() —
// results are bit-identical.  Latency-bound systems use BiCGSTAB (the
// default, krylov_dsm.cu); this kernel runs every size on the cooperative grid.
#include <cooperative_groups.h>

#include "ctx.cuh"
#include "ilu.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int GT = 1024;           // threads per CTA
constexpr int GCPR = GT / 256;     // canonical chunks per round
constexpr int MM = RSIM_GMRES_M;   // restart length
constexpr int NQMAX = MM + 1;      // quantities of one reduction (projections)

struct GArgs {
  int32_t nA, nslot, maxit, fixed, neu, ilu;
  IluArgs fa;
  int64_t cap;
  int32_t nx, ny, nz;
  bool d3, has_nnc, implicit, f2_parts;
  double rtol;
  const int32_t *ell_col, *act, *nptr, *nnc_lcol;
  const double *ell_val, *nnc_val, *rhs, *F_raw, *part_f2;
  double *x, *r, *z, *w, *u;
  double* V;  // (MM+1) vectors of cap*B
  double *part, *part2;
  int32_t pstride, pstride2;
  DevScalars* dsc;
};

struct GRed {
  double ws[NQMAX][32];
  double lvl[64];
  double res[NQMAX];
  double H[MM + 1][MM];
  double cs[MM], sn[MM], g[MM + 1], yy[MM];
  double resid, hn;
  int bad;
};

// y_l = x_l + Σ_slots Â_s x_col + NNC (canonical row order), x fully stored
template <int B>
__device__ __forceinline__ void spmv_row(const GArgs& a, int64_t l, const double* __restrict__ xv, double* y) {
  int32_t cl[6];
#pragma unroll
  for (int s = 0; s < 6; ++s) cl[s] = -1;
  if (a.implicit) {
    implicit_cols(a.nx, a.ny, a.nz, a.d3, l, cl);
  } else {
#pragma unroll
    for (int s = 0; s < 6; ++s)
      if (s < a.nslot) cl[s] = __ldg(&a.ell_col[s * a.cap + l]);
  }
#pragma unroll
  for (int e = 0; e < B; ++e) y[e] = xv[l * B + e];
#pragma unroll
  for (int s = 0; s < 6; ++s)
    if (cl[s] >= 0) {
      double M[B * B];
      ell_load<B>(a.ell_val, a.cap, s, l, M);
      rsim::blk::gemv_acc_flat<B>(M, &xv[(int64_t)cl[s] * B], y);
    }
  if (a.has_nnc) {
    const int64_t i = a.act[l];
    const int32_t q0 = a.nptr[i], q1 = a.nptr[i + 1];
    for (int32_t q = q0; q < q1; ++q) {
      const int32_t cc = a.nnc_lcol[q];
      if (cc >= 0) rsim::blk::gemv_acc_flat<B>(&a.nnc_val[(int64_t)q * B * B], &xv[(int64_t)cc * B], y);
    }
  }
}

// per-round commit: warp trees -> 8-way trees -> level-1 chunk partials
__device__ __forceinline__ void commit(GRed& R, int NQ, const double* val, int64_t chunk0, int64_t nch, double* part,
                                       int pstride) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = 0; q < NQ; ++q) {
    const double v = warp_tree(val[q]);
    if (lane == 0) R.ws[q][w] = v;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < GCPR * NQ; k += blockDim.x) {
    const int g = k % GCPR, q = k / GCPR;
    if (chunk0 + g < nch) part[q * pstride + chunk0 + g] = tree8(&R.ws[q][8 * g]);
  }
  __syncthreads();
}

// canonical reduction of P (<= 64*256) partials by one CTA -> R.res[q]
__device__ __forceinline__ void reduce_small(GRed& R, int q, const double* src, int P) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (P == 1) {
    if (threadIdx.x == 0) R.res[q] = src[0];
    __syncthreads();
    return;
  }
  const int P2 = (P + 255) / 256;
  for (int c0 = 0; c0 < P2; c0 += GCPR) {
    const int idx = c0 * 256 + threadIdx.x;
    const double v = warp_tree(idx < P ? src[idx] : 0.0);
    if (lane == 0) R.ws[q][w] = v;
    __syncthreads();
    if ((int)threadIdx.x < GCPR && c0 + (int)threadIdx.x < P2) R.lvl[c0 + threadIdx.x] = tree8(&R.ws[q][8 * threadIdx.x]);
    __syncthreads();
  }
  if (P2 == 1) {
    if (threadIdx.x == 0) R.res[q] = R.lvl[0];
  } else {
    const double v = warp_tree(threadIdx.x < (unsigned)P2 ? R.lvl[threadIdx.x] : 0.0);
    __syncthreads();
    if (lane == 0 && w < 8) R.ws[q][w] = v;
    __syncthreads();
    if (threadIdx.x == 0) R.res[q] = tree8(&R.ws[q][0]);
  }
  __syncthreads();
}

template <int B>
__global__ void __launch_bounds__(GT, 1) k_gmres(const GArgs a) {
  __shared__ GRed R;
  const bool single = gridDim.x == 1;
  auto sync = [&]() {
    if (single) __syncthreads();
    else cg::this_grid().sync();
  };
  const int64_t nr = a.nA;
  const int64_t nch = (nr + 255) / 256;
  const int64_t nrounds = (nch + GCPR - 1) / GCPR;
  const int tid = threadIdx.x;
  const int64_t N = nr * B;

  auto reduce = [&](int NQ, const double* src1) {
    sync();
    const int P1 = (int)nch;
    auto src = [&](int q) { return (q == 1 && src1) ? src1 : a.part + (int64_t)q * a.pstride; };
    if (P1 <= 64 * 256) {
      for (int q = 0; q < NQ; ++q) reduce_small(R, q, src(q), P1);
    } else {
      const int P2 = (P1 + 255) / 256;
      for (int64_t rr = blockIdx.x; rr * GCPR < P2; rr += gridDim.x) {
        const int64_t c2 = rr * GCPR + (tid >> 8);
        const int64_t idx = c2 * 256 + (tid & 255);
        double v[NQMAX];
        for (int q = 0; q < NQ; ++q) v[q] = idx < P1 ? src(q)[idx] : 0.0;
        commit(R, NQ, v, rr * GCPR, P2, a.part2, a.pstride2);
      }
      sync();
      for (int q = 0; q < NQ; ++q) reduce_small(R, q, a.part2 + (int64_t)q * a.pstride2, P2);
    }
  };
  // a pass over the own rows (no reduction)
#define GPASS_BEGIN                                                \
  for (int64_t rd = blockIdx.x; rd < nrounds; rd += gridDim.x) { \
    const int64_t l = rd * GT + tid;                               \
    if (l < nr) {
#define GPASS_END \
  }               \
  }
  // a pass with NQ per-row values reduced canonically
#define GRED_BEGIN                                                 \
  for (int64_t rd = blockIdx.x; rd < nrounds; rd += gridDim.x) { \
    const int64_t l = rd * GT + tid;                               \
    const bool ok = l < nr;                                        \
    double val[NQMAX];                                             \
    for (int q = 0; q < NQMAX; ++q) val[q] = 0.0;
#define GRED_END(NQ)                                                \
  commit(R, NQ, val, rd * GCPR, nch, a.part, a.pstride);            \
  }

  // ---- init: r = rhs, x = 0;  (rhs, rhs), (F, F)
  GRED_BEGIN
  if (ok) {
    double bv[B];
#pragma unroll
    for (int e = 0; e < B; ++e) { bv[e] = a.rhs[l * B + e]; a.r[l * B + e] = bv[e]; a.x[l * B + e] = 0.0; }
    val[0] = rsim::blk::rowdot<B>(bv, bv);
    if (!a.f2_parts) {
      double fv[B];
#pragma unroll
      for (int e = 0; e < B; ++e) fv[e] = a.F_raw[l * B + e];
      val[1] = rsim::blk::rowdot<B>(fv, fv);
    }
  }
  GRED_END(a.f2_parts ? 1 : 2)
  reduce(2, a.f2_parts ? a.part_f2 : nullptr);
  const double bnorm = sqrt(R.res[0]);
  if (blockIdx.x == 0 && tid == 0) a.dsc->f2 = sqrt(R.res[1]);
  const bool fixed = a.fixed > 0;
  const int maxit = fixed ? a.fixed : a.maxit;
  const double tol = a.rtol * bnorm;
  int status = RSIM_OK, total_all = 0;
  double relres = 0.0;
  if (bnorm != 0.0) {
    const bool ilu_bad = a.ilu && a.dsc->ilu_bad;
    for (int attempt = 0; attempt < ((a.neu || a.ilu) ? 2 : 1); ++attempt) {
      const bool neu = a.neu && attempt == 0;
      const bool ilu = a.ilu && attempt == 0;
      const bool prec = neu || ilu;
      if (ilu && ilu_bad) { status = RSIM_ENUM; continue; }  // singular pivot: block-Jacobi only
      if (attempt) {  // block-Jacobi only, from x0 = 0
        GPASS_BEGIN
#pragma unroll
        for (int e = 0; e < B; ++e) { a.r[l * B + e] = a.rhs[l * B + e]; a.x[l * B + e] = 0.0; }
        GPASS_END
        sync();
      }
      double beta = bnorm;
      int total = 0;
      status = RSIM_ENOCONV;
      for (;;) {
        // ---- v_0 = r / β
        GPASS_BEGIN
#pragma unroll
        for (int e = 0; e < B; ++e) a.V[l * B + e] = a.r[l * B + e] / beta;
        GPASS_END
        if (tid == 0) {
          for (int q = 0; q <= MM; ++q) R.g[q] = 0.0;
          R.g[0] = beta;
        }
        sync();
        int k = 0;
        bool done = false;
        double resid = beta;
        for (int j = 0; j < MM; ++j) {
          const double* vj = a.V + (int64_t)j * a.cap * B;
          const double* zsrc = vj;
          if (neu) {  // z = v_j + (v_j − Â v_j)
            GPASS_BEGIN
            double y[B];
            spmv_row<B>(a, l, vj, y);
#pragma unroll
            for (int e = 0; e < B; ++e) a.z[l * B + e] = vj[l * B + e] + (vj[l * B + e] - y[e]);
            GPASS_END
            sync();
            zsrc = a.z;
          } else if (ilu) {  // z = (LU)^{-1} v_j
            ilu_apply<B>(a.fa, vj, a.z, sync);
            zsrc = a.z;
          }
          // ---- w = Â z;  (w, v_i), i <= j
          GRED_BEGIN
          if (ok) {
            double y[B];
            spmv_row<B>(a, l, zsrc, y);
#pragma unroll
            for (int e = 0; e < B; ++e) a.w[l * B + e] = y[e];
            for (int i = 0; i <= j; ++i) val[i] = rsim::blk::rowdot<B>(y, &a.V[((int64_t)i * a.cap + l) * B]);
          }
          GRED_END(j + 1)
          reduce(j + 1, nullptr);
          if (tid == 0)
            for (int i = 0; i <= j; ++i) R.H[i][j] = R.res[i];
          __syncthreads();
          // ---- w −= Σ_i h_ij v_i (ascending i);  (w, w)
          GRED_BEGIN
          if (ok) {
            double wv[B];
#pragma unroll
            for (int e = 0; e < B; ++e) {
              double we = a.w[l * B + e];
              for (int i = 0; i <= j; ++i) we = we - R.H[i][j] * a.V[((int64_t)i * a.cap + l) * B + e];
              wv[e] = we;
              a.w[l * B + e] = we;
            }
            val[0] = rsim::blk::rowdot<B>(wv, wv);
          }
          GRED_END(1)
          reduce(1, nullptr);
          if (tid == 0) {  // Givens rotations (every CTA, identical sums)
            const double hn = sqrt(R.res[0]);
            R.H[j + 1][j] = hn;
            for (int i = 0; i < j; ++i) {
              const double t = R.cs[i] * R.H[i][j] + R.sn[i] * R.H[i + 1][j];
              R.H[i + 1][j] = -R.sn[i] * R.H[i][j] + R.cs[i] * R.H[i + 1][j];
              R.H[i][j] = t;
            }
            const double den = sqrt(R.H[j][j] * R.H[j][j] + hn * hn);
            R.bad = (den == 0.0 || !isfinite(den)) ? 1 : 0;
            if (!R.bad) {
              R.cs[j] = R.H[j][j] / den;
              R.sn[j] = hn / den;
              R.H[j][j] = R.cs[j] * R.H[j][j] + R.sn[j] * hn;
              R.H[j + 1][j] = 0.0;
              R.g[j + 1] = -R.sn[j] * R.g[j];
              R.g[j] = R.cs[j] * R.g[j];
            }
            R.hn = hn;
            R.resid = fabs(R.g[j + 1]);
          }
          __syncthreads();
          if (R.bad) { status = RSIM_ENUM; ++total; k = -1; break; }
          ++total;
          k = j + 1;
          resid = R.resid;
          const double hn = R.hn;
          if (hn == 0.0 || (!fixed && resid <= tol) || total >= maxit) { done = true; break; }
          double* vn = a.V + (int64_t)(j + 1) * a.cap * B;
          GPASS_BEGIN
#pragma unroll
          for (int e = 0; e < B; ++e) vn[l * B + e] = a.w[l * B + e] / hn;
          GPASS_END
          sync();
        }
        if (k < 0) break;  // breakdown
        if (tid == 0)
          for (int i = k - 1; i >= 0; --i) {  // back substitution
            double t = R.g[i];
            for (int q = i + 1; q < k; ++q) t = t - R.H[i][q] * R.yy[q];
            R.yy[i] = t / R.H[i][i];
          }
        __syncthreads();
        // ---- x += M^{-1} Σ_i y_i v_i
        GPASS_BEGIN
#pragma unroll
        for (int e = 0; e < B; ++e) {
          double ue = R.yy[0] * a.V[l * B + e];
          for (int i = 1; i < k; ++i) ue = ue + R.yy[i] * a.V[((int64_t)i * a.cap + l) * B + e];
          if (prec) a.u[l * B + e] = ue;
          else a.x[l * B + e] = a.x[l * B + e] + ue;
        }
        GPASS_END
        if (neu) {
          sync();
          GPASS_BEGIN
          double y[B];
          spmv_row<B>(a, l, a.u, y);
#pragma unroll
          for (int e = 0; e < B; ++e) {
            const double ue = a.u[l * B + e];
            a.x[l * B + e] = a.x[l * B + e] + (ue + (ue - y[e]));
          }
          GPASS_END
        } else if (ilu) {
          sync();
          ilu_apply<B>(a.fa, a.u, a.z, sync);
          GPASS_BEGIN
#pragma unroll
          for (int e = 0; e < B; ++e) a.x[l * B + e] = a.x[l * B + e] + a.z[l * B + e];
          GPASS_END
        }
        relres = resid / bnorm;
        if (done && (fixed ? total >= maxit : (resid <= tol || resid == 0.0))) { status = RSIM_OK; break; }
        if (total >= maxit) { status = fixed ? RSIM_OK : RSIM_ENOCONV; break; }
        sync();
        // ---- restart: r = rhs − Â x;  (r, r)
        GRED_BEGIN
        if (ok) {
          double y[B], rv[B];
          spmv_row<B>(a, l, a.x, y);
#pragma unroll
          for (int e = 0; e < B; ++e) { rv[e] = a.rhs[l * B + e] - y[e]; a.r[l * B + e] = rv[e]; }
          val[0] = rsim::blk::rowdot<B>(rv, rv);
        }
        GRED_END(1)
        reduce(1, nullptr);
        beta = sqrt(R.res[0]);
        if (beta == 0.0) { status = RSIM_OK; break; }
      }
      total_all += total;
      if (!(prec && (status == RSIM_ENUM || status == RSIM_ENOCONV))) break;
      sync();
    }
  }
  (void)N;
  if (blockIdx.x == 0 && tid == 0) {
    a.dsc->lin_iters = total_all;
    a.dsc->lin_relres = relres;
    if (status != RSIM_OK) a.dsc->status = status;
  }
#undef GPASS_BEGIN
#undef GPASS_END
#undef GRED_BEGIN
#undef GRED_END
}

template <int B>
int launch_g(rsim_gpu_ctx* c, const rsim_solver_opts* o) {
  const int64_t nch = (c->nA + 255) / 256, pstride = (c->n + 255) / 256, pstride2 = (pstride + 255) / 256;
  if (!c->gm_V) {
    RSIM_CUDA(cudaMalloc(&c->gm_V, sizeof(double) * (MM + 1) * c->n * c->b));
    RSIM_CUDA(cudaMalloc(&c->gm_part, sizeof(double) * NQMAX * (pstride + pstride2 + 1)));
  }
  GArgs a;
  a.nA = c->nA; a.nslot = c->nslot; a.maxit = o->lin_maxit; a.fixed = o->fixed_lin_iters;
  a.neu = o->precond == RSIM_PREC_NEUMANN1;
  a.ilu = o->precond == RSIM_PREC_ILU0;
  a.fa = ilu_args(c);
  a.cap = c->ell_cap;
  a.nx = c->nx; a.ny = c->ny; a.nz = c->nz; a.d3 = c->d3;
  a.has_nnc = c->has_nnc; a.implicit = c->cols_implicit; a.f2_parts = c->f2_parts;
  a.rtol = o->lin_rtol;
  a.ell_col = c->ell_col; a.act = c->act; a.nptr = c->nptr; a.nnc_lcol = c->nnc_lcol;
  a.ell_val = c->ell_val; a.nnc_val = c->nnc_val; a.rhs = c->rhs; a.F_raw = c->F_raw; a.part_f2 = c->part_f2;
  a.x = c->x; a.r = c->r; a.z = c->ph; a.w = c->t; a.u = c->s;
  a.V = c->gm_V;
  a.pstride = (int32_t)pstride; a.pstride2 = (int32_t)pstride2;
  a.part = c->gm_part; a.part2 = c->gm_part + NQMAX * pstride;
  a.dsc = c->dsc;
  const int64_t nrounds = (nch + GCPR - 1) / GCPR;
  static int per_sm[4] = {0, 0, 0, 0};
  if (per_sm[B] == 0) {
    RSIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[B], k_gmres<B>, GT, 0));
    if (per_sm[B] < 1) per_sm[B] = 1;
  }
  const int64_t maxb = (int64_t)per_sm[B] * c->sm_count;
  int grid = (int)(nrounds < maxb ? nrounds : maxb);
  if (grid < 1) grid = 1;
  void* args[] = {&a};
  if (grid == 1) {
    k_gmres<B><<<1, GT, 0, c->stream>>>(a);
  } else {
    RSIM_CUDA(cudaLaunchCooperativeKernel((void*)k_gmres<B>, grid, GT, args, 0, c->stream));
  }
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

}  // namespace

int launch_gmres(rsim_gpu_ctx* c, const rsim_solver_opts* o) {
  if (c->nA <= 0) return RSIM_OK;
  switch (c->b) {
    case 1: return launch_g<1>(c, o);
    case 2: return launch_g<2>(c, o);
    default: return launch_g<3>(c, o);
  }
}
