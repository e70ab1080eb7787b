// krylov.cu — K3 (SpMV) + K5 (fused vector updates / dot products) inside ONE
// persistent cooperative BiCGSTAB kernel per linear solve.
//
// Replaces solve(J, F) with the north star's BiCGSTAB on
// the block-Jacobi-scaled system Â = D^{-1}J (unit block diagonal, never
// stored; block-Jacobi preconditioning is therefore built in).
//
// Why persistent: the active systems of the localized solver are small
// (SURVEY.md §7 H2 — c1 has ~10^2 active cells), where one launch + one host
// sync per Krylov iteration would dominate.  The whole iteration loop runs on
// the device; phases are separated by grid-wide barriers (one __syncthreads
// when the grid is a single CTA), and every block redundantly reduces the
// chunk partials in the canonical order (blockops.h), so all blocks take the
// same branch and the result is bit-identical to the CPU oracle.
//
// Element formulas (identical in oracle/oracle.cpp bicgstab()):
//   p = r + β (p − ω v);  s = r − α v;  x = (x + α p) + ω s;  r = s − ω t.
#include <cooperative_groups.h>

#include "ctx.cuh"

namespace cg = cooperative_groups;

namespace {

struct KArgs {
  int32_t nA, nslot, maxit, fixed;
  int64_t cap;
  bool has_nnc;
  double rtol;
  const int32_t* __restrict__ ell_col;
  const double* __restrict__ ell_val;
  const int32_t* __restrict__ act;
  const int32_t* __restrict__ nptr;
  const int32_t* __restrict__ nnc_lcol;
  const double* __restrict__ nnc_val;
  const double* __restrict__ rhs;
  const double* __restrict__ part_f2;
  double *x, *r, *r0, *p, *v, *s, *t;
  double* part;  // [4][pstride]
  int32_t pstride;
  DevScalars* dsc;
};

template <int B>
__device__ __forceinline__ void spmv_row(const KArgs& a, int64_t l, const double* __restrict__ xin,
                                         double* __restrict__ yout, double* acc) {
#pragma unroll
  for (int c = 0; c < B; ++c) acc[c] = xin[l * B + c];
#pragma unroll
  for (int s = 0; s < 6; ++s) {
    if (s >= a.nslot) break;
    int32_t cl = a.ell_col[s * a.cap + l];
    if (cl >= 0) rsim::blk::gemv_acc_flat<B>(&a.ell_val[((int64_t)s * a.cap + l) * B * B], &xin[(int64_t)cl * B], acc);
  }
  if (a.has_nnc) {
    int64_t i = a.act[l];
    int32_t q0 = a.nptr[i], q1 = a.nptr[i + 1];
    for (int32_t q = q0; q < q1; ++q) {
      int32_t cl = a.nnc_lcol[q];
      if (cl >= 0) rsim::blk::gemv_acc_flat<B>(&a.nnc_val[(int64_t)q * B * B], &xin[(int64_t)cl * B], acc);
    }
  }
#pragma unroll
  for (int c = 0; c < B; ++c) yout[l * B + c] = acc[c];
}

struct Sync {
  cg::grid_group g;
  bool single;
  __device__ void operator()() {
    if (single) __syncthreads();
    else g.sync();
  }
};

template <int B>
__global__ void __launch_bounds__(256) k_bicgstab(const KArgs a) {
  __shared__ double sm[9];
  __shared__ double lvl[64];
  Sync sync{cg::this_grid(), gridDim.x == 1};
  const int64_t nr = a.nA;
  const int nch = (int)((nr + RSIM_RED_CHUNK - 1) / RSIM_RED_CHUNK);
  const int tid = threadIdx.x;
  double* P0 = a.part;
  double* P1 = a.part + a.pstride;
  double* P2 = a.part + 2 * a.pstride;
  double* P3 = a.part + 3 * a.pstride;

#define CHUNK_LOOP_BEGIN                                               \
  for (int c = blockIdx.x; c < nch; c += gridDim.x) {                  \
    double acc0 = 0.0, acc1 = 0.0;                                     \
    (void)acc0; (void)acc1;                                            \
    for (int k = 0; k < RSIM_RED_ITEMS; ++k) {                         \
      const int64_t l = (int64_t)c * RSIM_RED_CHUNK + tid + RSIM_RED_THREADS * k; \
      if (l < nr) {
#define CHUNK_LOOP_END_1(PA)                                           \
      }                                                                \
    }                                                                  \
    double rr0 = block_sum_canon(acc0, sm);                            \
    if (tid == 0) PA[c] = rr0;                                         \
  }
#define CHUNK_LOOP_END_2(PA, PB)                                       \
      }                                                                \
    }                                                                  \
    double rr0 = block_sum_canon(acc0, sm);                            \
    double rr1 = block_sum_canon(acc1, sm);                            \
    if (tid == 0) { PA[c] = rr0; PB[c] = rr1; }                        \
  }

  // ---- init: r = r0 = rhs, x = 0;  bb = (r, r)
  CHUNK_LOOP_BEGIN
  for (int e = 0; e < B; ++e) {
    double b = a.rhs[l * B + e];
    a.r[l * B + e] = b;
    a.r0[l * B + e] = b;
    a.x[l * B + e] = 0.0;
  }
  acc0 = acc0 + rsim::blk::rowdot<B>(&a.rhs[l * B], &a.rhs[l * B]);
  CHUNK_LOOP_END_1(P0)
  sync();
  const double bb = reduce_partials_canon(P0, nch, sm, lvl);
  if (blockIdx.x == 0) {  // finalize the assembly's ‖F‖₂ (canonical)
    double f2 = reduce_partials_canon(a.part_f2, a.dsc->part_count, sm, lvl);
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
    CHUNK_LOOP_BEGIN
    for (int e = 0; e < B; ++e) {
      const int64_t q = l * B + e;
      a.p[q] = (it == 1) ? a.r[q] : a.r[q] + beta * (a.p[q] - omega * a.v[q]);
    }
    }}}
    sync();
    // ---- v = Â p ; (r0, v)
    CHUNK_LOOP_BEGIN
    double vv[B];
    spmv_row<B>(a, l, a.p, a.v, vv);
    acc0 = acc0 + rsim::blk::rowdot<B>(&a.r0[l * B], vv);
    CHUNK_LOOP_END_1(P0)
    sync();
    const double r0v = reduce_partials_canon(P0, nch, sm, lvl);
    if (r0v == 0.0 || !isfinite(r0v)) { status = RSIM_ENUM; break; }
    alpha = rho_new / r0v;
    // ---- s = r − α v ; (s, s)
    CHUNK_LOOP_BEGIN
    double sv[B];
    for (int e = 0; e < B; ++e) {
      const int64_t q = l * B + e;
      sv[e] = a.r[q] - alpha * a.v[q];
      a.s[q] = sv[e];
    }
    acc0 = acc0 + rsim::blk::rowdot<B>(sv, sv);
    CHUNK_LOOP_END_1(P1)
    sync();
    const double ss = reduce_partials_canon(P1, nch, sm, lvl);
    if (!fixed && sqrt(ss) <= tol) {
      CHUNK_LOOP_BEGIN
      for (int e = 0; e < B; ++e) {
        const int64_t q = l * B + e;
        a.x[q] = a.x[q] + alpha * a.p[q];
      }
      }}}
      relres = sqrt(ss) / bnorm;
      status = RSIM_OK;
      break;
    }
    // ---- t = Â s ; (t, s), (t, t)
    CHUNK_LOOP_BEGIN
    double tv[B];
    spmv_row<B>(a, l, a.s, a.t, tv);
    acc0 = acc0 + rsim::blk::rowdot<B>(tv, &a.s[l * B]);
    acc1 = acc1 + rsim::blk::rowdot<B>(tv, tv);
    CHUNK_LOOP_END_2(P2, P3)
    sync();
    const double ts = reduce_partials_canon(P2, nch, sm, lvl);
    const double tt = reduce_partials_canon(P3, nch, sm, lvl);
    if (tt == 0.0 || !isfinite(tt)) { status = RSIM_ENUM; break; }
    omega = ts / tt;
    // ---- x, r update ; (r, r), (r0, r)
    CHUNK_LOOP_BEGIN
    double rv[B];
    for (int e = 0; e < B; ++e) {
      const int64_t q = l * B + e;
      const double sq = a.s[q];
      a.x[q] = (a.x[q] + alpha * a.p[q]) + omega * sq;
      rv[e] = sq - omega * a.t[q];
      a.r[q] = rv[e];
    }
    acc0 = acc0 + rsim::blk::rowdot<B>(rv, rv);
    acc1 = acc1 + rsim::blk::rowdot<B>(&a.r0[l * B], rv);
    CHUNK_LOOP_END_2(P0, P1)
    sync();
    const double rr = reduce_partials_canon(P0, nch, sm, lvl);
    rho = rho_new;
    rho_new = reduce_partials_canon(P1, nch, sm, lvl);
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
#undef CHUNK_LOOP_BEGIN
#undef CHUNK_LOOP_END_1
#undef CHUNK_LOOP_END_2
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
  a.rhs = c->rhs; a.part_f2 = c->part_f2;
  a.x = c->x; a.r = c->r; a.r0 = c->r0; a.p = c->p; a.v = c->v; a.s = c->s; a.t = c->t;
  a.part = c->part;
  a.pstride = (int32_t)((c->n + RSIM_RED_CHUNK - 1) / RSIM_RED_CHUNK);
  a.dsc = c->dsc;
  const int nch = (c->nA + RSIM_RED_CHUNK - 1) / RSIM_RED_CHUNK;
  if (c->max_coop_blocks[B] == 0) {
    int per_sm = 0;
    RSIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bicgstab<B>, 256, 0));
    c->max_coop_blocks[B] = per_sm * c->sm_count;
    if (c->max_coop_blocks[B] < 1) c->max_coop_blocks[B] = 1;
  }
  int grid = nch < c->max_coop_blocks[B] ? nch : c->max_coop_blocks[B];
  if (grid < 1) grid = 1;
  void* args[] = {&a};
  if (grid == 1) {
    k_bicgstab<B><<<1, 256, 0, c->stream>>>(a);
  } else {
    RSIM_CUDA(cudaLaunchCooperativeKernel((void*)k_bicgstab<B>, grid, 256, args, 0, c->stream));
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
