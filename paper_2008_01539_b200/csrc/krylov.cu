// krylov.cu — K3 (SpMV) + K5 (fused vector updates / dot products) inside ONE
// persistent BiCGSTAB kernel per linear solve.
//
// Replaces solve(J, F) with the north star's BiCGSTAB on
// the block-Jacobi-scaled system Â = D^{-1}J (unit block diagonal, never
// stored; block-Jacobi preconditioning is therefore built in).
//
// Why persistent: the active systems of the localized solver are small
// (SURVEY.md §7 H2), where one launch + one host sync per Krylov iteration
// would dominate.  The whole iteration loop runs on the device; phases are
// separated by grid-wide barriers (one __syncthreads when the grid is a
// single CTA), and every block redundantly reduces the chunk partials in the
// canonical order (blockops.h), so all blocks take the same branch and the
// result is bit-identical to the CPU oracle.
//
// Latency design: 1024-thread CTAs, each owning whole 2048-row chunks with 2
// rows per thread whose loads are issued together; per-row dot values are
// staged in shared memory and summed by 256 "canonical" threads, so the
// reduction order is the canonical one while the loads run 2048-wide.
//
// Element formulas (identical in oracle/oracle.cpp bicgstab()):
//   p = r + β (p − ω v);  s = r − α v;  x = (x + α p) + ω s;  r = s − ω t.
#include <cooperative_groups.h>

#include <cstdlib>

#include "ctx.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int KT = 1024;                   // threads per CTA
constexpr int RPT = RSIM_RED_CHUNK / KT;   // rows per thread per chunk (2)

struct KArgs {
  int32_t nA, nslot, maxit, fixed;
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
  double *x, *r, *r0, *p, *v, *s, *t;
  double* part;  // [4][pstride]
  int32_t pstride;
  DevScalars* dsc;
};

// 256 canonical threads (warps 0..7) hold the sums; all 1024 threads call it.
__device__ __forceinline__ double bsum(double s, double* sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (w < 8) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) s = s + __shfl_down_sync(0xffffffffu, s, off);
    if (lane == 0) sm[w] = s;
  }
  __syncthreads();
  if (w == 0) {
    double r = (lane < 8) ? sm[lane] : 0.0;
#pragma unroll
    for (int off = 4; off >= 1; off >>= 1) r = r + __shfl_down_sync(0xffffffffu, r, off);
    if (lane == 0) sm[8] = r;
  }
  __syncthreads();
  double out = sm[8];
  __syncthreads();
  return out;
}

// Canonical reduction of P partials (every CTA redundantly; identical bits).
__device__ __forceinline__ double reduce_parts(const double* part, int P, double* sm, double* lvl) {
  const int t = threadIdx.x;
  auto level = [&](const double* src, int m) {
    double s = 0.0;
    if (t < RSIM_RED_THREADS) {
#pragma unroll
      for (int k = 0; k < RSIM_RED_ITEMS; ++k) {
        int idx = t + RSIM_RED_THREADS * k;
        if (idx < m) s = s + src[idx];
      }
    }
    return bsum(s, sm);
  };
  if (P <= RSIM_RED_CHUNK) return level(part, P);
  const int P2 = (P + RSIM_RED_CHUNK - 1) / RSIM_RED_CHUNK;
  for (int g = 0; g < P2; ++g) {
    double r = level(part + g * RSIM_RED_CHUNK, min(RSIM_RED_CHUNK, P - g * RSIM_RED_CHUNK));
    if (t == 0) lvl[g] = r;
  }
  __syncthreads();
  return level(lvl, P2);
}

// Sum the staged per-row values of one chunk in canonical order -> partial.
template <int NV>
__device__ __forceinline__ void chunk_commit(const double* vals, int m, double* sm, double* const* P, int c) {
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    double s = 0.0;
    if (threadIdx.x < RSIM_RED_THREADS) {
#pragma unroll
      for (int k = 0; k < RSIM_RED_ITEMS; ++k) {
        int idx = threadIdx.x + RSIM_RED_THREADS * k;
        if (idx < m) s = s + vals[q * RSIM_RED_CHUNK + idx];
      }
    }
    double r = bsum(s, sm);
    if (threadIdx.x == 0) P[q][c] = r;
  }
}

// y = Â x for RPT rows of one thread (loads of all rows issued before use).
template <int B>
__device__ __forceinline__ void spmv_rows(const KArgs& a, int64_t base, int64_t nr, const double* __restrict__ xin,
                                          double* __restrict__ yout, double (*acc)[B]) {
  const int32_t* __restrict__ col = a.ell_col;
  const double* __restrict__ val = a.ell_val;
  int32_t cl[RPT][6];
  int64_t l[RPT];
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    l[j] = base + threadIdx.x + KT * j;
#pragma unroll
    for (int s = 0; s < 6; ++s) cl[j][s] = (l[j] < nr && s < a.nslot) ? __ldg(&col[s * a.cap + l[j]]) : -1;
  }
#pragma unroll
  for (int j = 0; j < RPT; ++j)
#pragma unroll
    for (int c = 0; c < B; ++c) acc[j][c] = l[j] < nr ? xin[l[j] * B + c] : 0.0;
#pragma unroll
  for (int s = 0; s < 6; ++s)
#pragma unroll
    for (int j = 0; j < RPT; ++j)
      if (cl[j][s] >= 0)
        rsim::blk::gemv_acc_flat<B>(&val[((int64_t)s * a.cap + l[j]) * B * B], &xin[(int64_t)cl[j][s] * B], acc[j]);
  if (a.has_nnc) {
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      if (l[j] >= nr) continue;
      int64_t i = a.act[l[j]];
      int32_t q0 = a.nptr[i], q1 = a.nptr[i + 1];
      for (int32_t q = q0; q < q1; ++q) {
        int32_t cc = a.nnc_lcol[q];
        if (cc >= 0) rsim::blk::gemv_acc_flat<B>(&a.nnc_val[(int64_t)q * B * B], &xin[(int64_t)cc * B], acc[j]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < RPT; ++j)
    if (l[j] < nr)
#pragma unroll
      for (int c = 0; c < B; ++c) yout[l[j] * B + c] = acc[j][c];
}

template <int B>
__global__ void __launch_bounds__(KT) k_bicgstab(const KArgs a) {
  __shared__ double vals[2 * RSIM_RED_CHUNK];
  __shared__ double sm[9];
  __shared__ double lvl[64];
  const bool single = gridDim.x == 1;
  auto sync = [&]() {
    if (single) __syncthreads();
    else cg::this_grid().sync();
  };
  const int64_t nr = a.nA;
  const int nch = (int)((nr + RSIM_RED_CHUNK - 1) / RSIM_RED_CHUNK);
  const int tid = threadIdx.x;
  double* P0 = a.part;
  double* P1 = a.part + a.pstride;
  double* P2 = a.part + 2 * a.pstride;
  double* P3 = a.part + 3 * a.pstride;
  double* const PP01[2] = {P0, P1};
  double* const PP23[2] = {P2, P3};
  double* const PP1[1] = {P1};

  // ---- init: r = r0 = rhs, x = 0;  partials (rhs, rhs) and (F, F)
  for (int c = blockIdx.x; c < nch; c += gridDim.x) {
    const int64_t base = (int64_t)c * RSIM_RED_CHUNK;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int idx = tid + KT * j;
      const int64_t l = base + idx;
      double v0 = 0.0, v1 = 0.0;
      if (l < nr) {
        double bv[B], fv[B];
#pragma unroll
        for (int e = 0; e < B; ++e) { bv[e] = a.rhs[l * B + e]; fv[e] = a.F_raw[l * B + e]; }
#pragma unroll
        for (int e = 0; e < B; ++e) { a.r[l * B + e] = bv[e]; a.r0[l * B + e] = bv[e]; a.x[l * B + e] = 0.0; }
        v0 = rsim::blk::rowdot<B>(bv, bv);
        v1 = rsim::blk::rowdot<B>(fv, fv);
      }
      vals[idx] = v0;
      vals[RSIM_RED_CHUNK + idx] = v1;
    }
    chunk_commit<2>(vals, (int)(nr - base < RSIM_RED_CHUNK ? nr - base : RSIM_RED_CHUNK), sm, PP01, c);
  }
  sync();
  const double bb = reduce_parts(P0, nch, sm, lvl);
  if (blockIdx.x == 0) {  // ‖F‖₂ of the assembly (canonical)
    double f2 = reduce_parts(P1, nch, sm, lvl);
    if (tid == 0) a.dsc->f2 = sqrt(f2);
  }
  const double bnorm = sqrt(bb);
  if (bnorm == 0.0) {
    if (blockIdx.x == 0 && tid == 0) { a.dsc->lin_iters = 0; a.dsc->lin_relres = 0.0; }
    return;
  }
  const bool fixed = a.fixed > 0;
  const int maxit = fixed ? a.fixed : a.maxit;
  const double tol = a.rtol * bnorm;
  double rho = 1.0, alpha = 1.0, omega = 1.0, rho_new = bb;
  int status = RSIM_ENOCONV;
  int it = 0;
  double relres = 0.0;
  for (it = 1; it <= maxit; ++it) {
    // ---- p update
    const double beta = (it == 1) ? 0.0 : (rho_new / rho) * (alpha / omega);
    for (int c = blockIdx.x; c < nch; c += gridDim.x) {
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int64_t l = (int64_t)c * RSIM_RED_CHUNK + tid + KT * j;
        if (l < nr) {
#pragma unroll
          for (int e = 0; e < B; ++e) {
            const int64_t q = l * B + e;
            a.p[q] = (it == 1) ? a.r[q] : a.r[q] + beta * (a.p[q] - omega * a.v[q]);
          }
        }
      }
    }
    sync();
    // ---- v = Â p ; (r0, v)
    for (int c = blockIdx.x; c < nch; c += gridDim.x) {
      const int64_t base = (int64_t)c * RSIM_RED_CHUNK;
      double acc[RPT][B];
      spmv_rows<B>(a, base, nr, a.p, a.v, acc);
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int idx = tid + KT * j;
        const int64_t l = base + idx;
        vals[idx] = (l < nr) ? rsim::blk::rowdot<B>(&a.r0[l * B], acc[j]) : 0.0;
      }
      chunk_commit<1>(vals, (int)(nr - base < RSIM_RED_CHUNK ? nr - base : RSIM_RED_CHUNK), sm, &P0, c);
    }
    sync();
    const double r0v = reduce_parts(P0, nch, sm, lvl);
    if (r0v == 0.0 || !isfinite(r0v)) { status = RSIM_ENUM; break; }
    alpha = rho_new / r0v;
    // ---- s = r − α v ; (s, s)
    for (int c = blockIdx.x; c < nch; c += gridDim.x) {
      const int64_t base = (int64_t)c * RSIM_RED_CHUNK;
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int idx = tid + KT * j;
        const int64_t l = base + idx;
        double v0 = 0.0;
        if (l < nr) {
          double sv[B];
#pragma unroll
          for (int e = 0; e < B; ++e) {
            const int64_t q = l * B + e;
            sv[e] = a.r[q] - alpha * a.v[q];
            a.s[q] = sv[e];
          }
          v0 = rsim::blk::rowdot<B>(sv, sv);
        }
        vals[idx] = v0;
      }
      chunk_commit<1>(vals, (int)(nr - base < RSIM_RED_CHUNK ? nr - base : RSIM_RED_CHUNK), sm, PP1, c);
    }
    sync();
    const double ss = reduce_parts(P1, nch, sm, lvl);
    if (!fixed && sqrt(ss) <= tol) {
      for (int c = blockIdx.x; c < nch; c += gridDim.x)
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
          const int64_t l = (int64_t)c * RSIM_RED_CHUNK + tid + KT * j;
          if (l < nr)
#pragma unroll
            for (int e = 0; e < B; ++e) a.x[l * B + e] = a.x[l * B + e] + alpha * a.p[l * B + e];
        }
      relres = sqrt(ss) / bnorm;
      status = RSIM_OK;
      break;
    }
    // ---- t = Â s ; (t, s), (t, t)
    for (int c = blockIdx.x; c < nch; c += gridDim.x) {
      const int64_t base = (int64_t)c * RSIM_RED_CHUNK;
      double acc[RPT][B];
      spmv_rows<B>(a, base, nr, a.s, a.t, acc);
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int idx = tid + KT * j;
        const int64_t l = base + idx;
        vals[idx] = (l < nr) ? rsim::blk::rowdot<B>(acc[j], &a.s[l * B]) : 0.0;
        vals[RSIM_RED_CHUNK + idx] = (l < nr) ? rsim::blk::rowdot<B>(acc[j], acc[j]) : 0.0;
      }
      chunk_commit<2>(vals, (int)(nr - base < RSIM_RED_CHUNK ? nr - base : RSIM_RED_CHUNK), sm, PP23, c);
    }
    sync();
    const double ts = reduce_parts(P2, nch, sm, lvl);
    const double tt = reduce_parts(P3, nch, sm, lvl);
    if (tt == 0.0 || !isfinite(tt)) { status = RSIM_ENUM; break; }
    omega = ts / tt;
    // ---- x, r update ; (r, r), (r0, r)
    for (int c = blockIdx.x; c < nch; c += gridDim.x) {
      const int64_t base = (int64_t)c * RSIM_RED_CHUNK;
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const int idx = tid + KT * j;
        const int64_t l = base + idx;
        double v0 = 0.0, v1 = 0.0;
        if (l < nr) {
          double rv[B], r0v_[B];
#pragma unroll
          for (int e = 0; e < B; ++e) {
            const int64_t q = l * B + e;
            const double sq = a.s[q];
            a.x[q] = (a.x[q] + alpha * a.p[q]) + omega * sq;
            rv[e] = sq - omega * a.t[q];
            a.r[q] = rv[e];
            r0v_[e] = a.r0[q];
          }
          v0 = rsim::blk::rowdot<B>(rv, rv);
          v1 = rsim::blk::rowdot<B>(r0v_, rv);
        }
        vals[idx] = v0;
        vals[RSIM_RED_CHUNK + idx] = v1;
      }
      chunk_commit<2>(vals, (int)(nr - base < RSIM_RED_CHUNK ? nr - base : RSIM_RED_CHUNK), sm, PP01, c);
    }
    sync();
    const double rr = reduce_parts(P0, nch, sm, lvl);
    rho = rho_new;
    rho_new = reduce_parts(P1, nch, sm, lvl);
    relres = sqrt(rr) / bnorm;
    if (!fixed && sqrt(rr) <= tol) { status = RSIM_OK; break; }
    if (omega == 0.0 || rho_new == 0.0 || !isfinite(rho_new)) { status = RSIM_ENUM; break; }
  }
  if (it > maxit) { it = maxit; status = fixed ? RSIM_OK : RSIM_ENOCONV; }
  if (blockIdx.x == 0 && tid == 0) {
    a.dsc->lin_iters = it;
    a.dsc->lin_relres = relres;
    if (status != RSIM_OK) a.dsc->status = status;
  }
}


int single_max_chunks() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("RSIM_KRYLOV_SINGLE_MAX");
    v = e ? std::atoi(e) : 2;
  }
  return v;
}

template <int B>
int launch_b(rsim_gpu_ctx* c, const rsim_solver_opts* o) {
  KArgs a;
  a.nA = c->nA;
  a.nslot = c->nslot;
  a.maxit = o->lin_maxit;
  a.fixed = o->fixed_lin_iters;
  a.cap = c->n;
  a.has_nnc = c->has_nnc;
  a.rtol = o->lin_rtol;
  a.ell_col = c->ell_col; a.ell_val = c->ell_val;
  a.act = c->act; a.nptr = c->nptr; a.nnc_lcol = c->nnc_lcol; a.nnc_val = c->nnc_val;
  a.rhs = c->rhs; a.F_raw = c->F_raw;
  a.x = c->x; a.r = c->r; a.r0 = c->r0; a.p = c->p; a.v = c->v; a.s = c->s; a.t = c->t;
  a.part = c->part;
  a.pstride = (int32_t)((c->n + RSIM_RED_CHUNK - 1) / RSIM_RED_CHUNK);
  a.dsc = c->dsc;
  const int nch = (c->nA + RSIM_RED_CHUNK - 1) / RSIM_RED_CHUNK;
  // small systems: one cluster with matrix + vectors in distributed smem
  {
    int r = launch_krylov_dsm(c, o);
    if (r != RSIM_ENOTAPPLICABLE) return r;
  }
  if (c->max_coop_blocks[B] == 0) {
    int per_sm = 0;
    RSIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bicgstab<B>, KT, 0));
    c->max_coop_blocks[B] = per_sm * c->sm_count;
    if (c->max_coop_blocks[B] < 1) c->max_coop_blocks[B] = 1;
  }
  int grid = nch < c->max_coop_blocks[B] ? nch : c->max_coop_blocks[B];
  if (nch <= single_max_chunks()) grid = 1;
  if (grid < 1) grid = 1;
  void* args[] = {&a};
  if (grid == 1) {
    k_bicgstab<B><<<1, KT, 0, c->stream>>>(a);
  } else {
    RSIM_CUDA(cudaLaunchCooperativeKernel((void*)k_bicgstab<B>, grid, KT, args, 0, c->stream));
  }
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

}  // namespace

int launch_krylov(rsim_gpu_ctx* c, const rsim_solver_opts* o) {
  if (c->nA <= 0) return RSIM_OK;
  switch (c->b) {
    case 1: return launch_b<1>(c, o);
    case 2: return launch_b<2>(c, o);
    default: return launch_b<3>(c, o);
  }
}
