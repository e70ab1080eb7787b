// direct.cu — exact solve of small active systems (
// SPEC.md:311-325 solve(J, F), the Krylov cross-check), opts.lin_method =
// RSIM_LIN_DIRECT, n_A·b ≤ RSIM_DIRECT_MAX unknowns.
//
// Dense LU with partial pivoting of Â = D⁻¹J, the operation sequence of
// oracle/oracle.cpp direct_solve() (pivot = first max |w_ik|, swap across all
// columns, l = w_ik / w_kk, w_ij −= l·w_kj with one product and one
// subtraction), so the factors and x are bit-identical to the oracle's.
//
// Layout: W column-major N×N in HBM (128 MB at N = 4096, allocated on first
// use).  k_direct_build scatters the unit diagonal, the ELL (or structural)
// slots and the NNC blocks, one thread per row block in the canonical entry
// order.  k_direct_lu is one cooperative kernel: column j is owned by CTA
// j mod G.  Step k reads column k from a double-buffered copy (colbuf[k&1],
// written by its owner at the end of step k−1), so every CTA finds the pivot
// and forms the multipliers redundantly in shared memory while the owners
// swap and update their own columns in place: ONE grid barrier per step.
// CTA 0 then does the permutation and both triangular solves (column-
// oriented: one __syncthreads per k) and the canonical (F,F) reduction.
#include <cooperative_groups.h>

#include "ctx.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int DT = 256;  // threads per CTA
constexpr int kMaxOwn = 64;  // columns per CTA at most (G >= N / 64)

struct DArgs {
  int32_t nA, nslot, b;
  int32_t nx, ny, nz;
  bool d3, implicit, has_nnc, f2_parts;
  int64_t cap, N;
  const int32_t *ell_col, *act, *nptr, *nnc_lcol;
  const double *ell_val, *nnc_val, *rhs, *F_raw, *part_f2;
  double* W;       // N×N column-major
  double* colbuf;  // [2][N]
  int32_t* piv;    // [N]
  double* x;
  DevScalars* dsc;
};

__global__ void k_direct_zero(double* W, int64_t nn, int64_t N) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nn; e += (int64_t)gridDim.x * blockDim.x)
    W[e] = (e / N == e % N) ? 1.0 : 0.0;
}

template <int B>
__global__ void k_direct_build(const DArgs a) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= a.nA) return;
  const int64_t N = a.N;
  auto add = [&](int64_t cl, const double* blk) {
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int c = 0; c < B; ++c) {
        double* w = &a.W[(cl * B + c) * N + l * B + r];
        *w = *w + blk[r * B + c];
      }
  };
  int32_t cl[6];
#pragma unroll
  for (int s = 0; s < 6; ++s) cl[s] = -1;
  if (a.implicit) {
    implicit_cols(a.nx, a.ny, a.nz, a.d3, l, cl);
  } else {
    for (int s = 0; s < a.nslot; ++s) cl[s] = a.ell_col[s * a.cap + l];
  }
  for (int s = 0; s < a.nslot; ++s)
    if (cl[s] >= 0) {
      double M[B * B];
      ell_load<B>(a.ell_val, a.cap, s, l, M);
      add(cl[s], M);
    }
  if (a.has_nnc) {
    const int64_t i = a.act[l];
    for (int32_t q = a.nptr[i]; q < a.nptr[i + 1]; ++q)
      if (a.nnc_lcol[q] >= 0) add(a.nnc_lcol[q], &a.nnc_val[(int64_t)q * B * B]);
  }
}

// (value, index) with "first maximal |value|" order; bad = a non-finite entry
struct Piv {
  double v;
  int64_t i;
  int bad;
};
__device__ __forceinline__ Piv piv_max(Piv a, Piv b) {
  Piv r;
  r.bad = a.bad | b.bad;
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) { r.v = b.v; r.i = b.i; }
  else { r.v = a.v; r.i = a.i; }
  return r;
}

template <int B>
__global__ void __launch_bounds__(DT) k_direct_lu(const DArgs a) {
  extern __shared__ double sc[];  // column k (rows k..N-1), then the multipliers
  __shared__ Piv sp[DT / 32];
  __shared__ int s_fail;
  __shared__ double s_wk[kMaxOwn], s_wp[kMaxOwn];  // w_kj, w_pj of the own columns (step k)
  auto grid = cg::this_grid();
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t N = a.N;
  const int G = gridDim.x;
  // the first column copy (step 0 reads column 0 as built)
  if (blockIdx.x == 0)
    for (int64_t i = t; i < N; i += DT) a.colbuf[i] = a.W[i];
  grid.sync();
  int fail = 0;
  for (int64_t k = 0; k < N; ++k) {
    const double* cb = a.colbuf + (k & 1) * N;
    // ---- pivot search, redundantly in every CTA
    Piv p{-1.0, k, 0};
    for (int64_t i = k + t; i < N; i += DT) {
      const double v = cb[i];
      sc[i - k] = v;
      if (!isfinite(v)) p.bad = 1;
      else if (fabs(v) > p.v) { p.v = fabs(v); p.i = i; }  // ascending i: first max per thread
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      Piv q;
      q.v = __shfl_down_sync(0xffffffffu, p.v, o);
      q.i = __shfl_down_sync(0xffffffffu, p.i, o);
      q.bad = __shfl_down_sync(0xffffffffu, p.bad, o);
      p = piv_max(p, q);
    }
    if (lane == 0) sp[w] = p;
    __syncthreads();
    if (t == 0) {
      Piv r = sp[0];
      for (int q = 1; q < DT / 32; ++q) r = piv_max(r, sp[q]);
      sp[0] = r;
      s_fail = (r.bad || r.v == 0.0) ? 1 : 0;
      if (s_fail && blockIdx.x == 0) atomicMin(&a.dsc->bad_cell, a.act[k / B]);  // the pivot column's cell
    }
    __syncthreads();
    if (s_fail) { fail = 1; break; }  // every CTA takes the same branch
    const int64_t pv = sp[0].i;
    // ---- swap in the shared copy, multipliers l_i = w_ik / w_kk (i > k)
    if (t == 0 && pv != k) {
      const double tmp = sc[0];
      sc[0] = sc[pv - k];
      sc[pv - k] = tmp;
    }
    __syncthreads();
    const double d = sc[0];
    for (int64_t i = k + 1 + t; i < N; i += DT) sc[i - k] = sc[i - k] / d;
    __syncthreads();
    if (blockIdx.x == 0 && t == 0) a.piv[k] = (int32_t)pv;
    // ---- own columns: swap rows k / pv (all columns), update j > k.
    // Phase 1 reads w_kj / w_pj of every own column into shared memory (one
    // barrier), so phase 2 writes without any per-column barrier: the owner
    // of row pv uses the old row-k value, thread 0 writes the swapped row k
    // (and row pv of the L columns, j < k), which nobody reads in phase 2.
    if (t < kMaxOwn) {  // own column c = blockIdx.x + c·G
      const int64_t j = blockIdx.x + (int64_t)t * G;
      if (j < N) { s_wk[t] = a.W[j * N + k]; s_wp[t] = a.W[j * N + pv]; }
    }
    __syncthreads();
    int c = 0;
    for (int64_t j = blockIdx.x; j < N; j += G, ++c) {
      double* cj = a.W + j * N;
      if (j == k) {  // column k: pivot and multipliers from the (swapped) shared copy
        for (int64_t i = k + t; i < N; i += DT) cj[i] = sc[i - k];
        continue;
      }
      const double wk = s_wk[c], wp = s_wp[c];
      if (t == 0) {
        cj[k] = wp;
        if (j < k && pv != k) cj[pv] = wk;
      }
      if (j > k) {
        int64_t i = k + 1 + t;
        for (; i + 3 * DT < N; i += 4 * DT) {  // 4 independent rows in flight per thread
          double w0 = cj[i], w1 = cj[i + DT], w2 = cj[i + 2 * DT], w3 = cj[i + 3 * DT];
          if (i == pv) w0 = wk;
          if (i + DT == pv) w1 = wk;
          if (i + 2 * DT == pv) w2 = wk;
          if (i + 3 * DT == pv) w3 = wk;
          cj[i] = w0 - sc[i - k] * wp;
          cj[i + DT] = w1 - sc[i + DT - k] * wp;
          cj[i + 2 * DT] = w2 - sc[i + 2 * DT - k] * wp;
          cj[i + 3 * DT] = w3 - sc[i + 3 * DT - k] * wp;
        }
        for (; i < N; i += DT) {
          const double wi = (i == pv) ? wk : cj[i];
          cj[i] = wi - sc[i - k] * wp;
        }
      }
    }
    if (k + 1 < N && (int)((k + 1) % G) == (int)blockIdx.x) {  // the next step's column copy
      __syncthreads();
      const double* cn = a.W + (k + 1) * N;
      double* nb = a.colbuf + ((k + 1) & 1) * N;
      for (int64_t i = k + 1 + t; i < N; i += DT) nb[i] = cn[i];
    }
    grid.sync();
  }
  if (blockIdx.x != 0) return;
  // ---- CTA 0: status, the canonical (F,F) reduction, permutation and solves
  __shared__ double ws[8];
  __shared__ double parts[256];
  {
    // chunk partials (256 rows each, canonical tree), then one more level
    const int64_t nch = ((int64_t)a.nA + 255) / 256;
    for (int64_t c0 = 0; c0 < nch; ++c0) {
      double v;
      if (a.f2_parts) {
        v = 0.0;
      } else {
        const int64_t l = c0 * 256 + t;
        v = 0.0;
        if (l < a.nA) {
          double f[B];
#pragma unroll
          for (int e = 0; e < B; ++e) f[e] = a.F_raw[l * B + e];
          v = rsim::blk::rowdot<B>(f, f);
        }
      }
      v = warp_tree(v);
      if (lane == 0) ws[w] = v;
      __syncthreads();
      if (t == 0) parts[c0] = a.f2_parts ? a.part_f2[c0] : tree8(ws);
      __syncthreads();
    }
    double f2;
    if (nch == 1) {
      f2 = parts[0];
    } else {
      double v = t < nch ? parts[t] : 0.0;
      v = warp_tree(v);
      if (lane == 0) ws[w] = v;
      __syncthreads();
      f2 = tree8(ws);
    }
    if (t == 0) {
      a.dsc->f2 = sqrt(f2);
      a.dsc->lin_iters = 1;
      a.dsc->lin_relres = 0.0;
      if (fail) a.dsc->status = RSIM_ENUM;
    }
  }
  if (fail) return;
  double* x = a.x;
  for (int64_t i = t; i < N; i += DT) x[i] = a.rhs[i];
  __syncthreads();
  if (t == 0)
    for (int64_t k = 0; k < N; ++k) {
      const int64_t pv = a.piv[k];
      if (pv != k) { const double tmp = x[k]; x[k] = x[pv]; x[pv] = tmp; }
    }
  __syncthreads();
  for (int64_t k = 0; k < N; ++k) {
    const double xk = x[k];
    const double* ck = a.W + k * N;
    for (int64_t i = k + 1 + t; i < N; i += DT) x[i] = x[i] - ck[i] * xk;
    __syncthreads();
  }
  __shared__ double s_xk;
  for (int64_t k = N - 1; k >= 0; --k) {
    const double* ck = a.W + k * N;
    if (t == 0) { s_xk = x[k] / ck[k]; x[k] = s_xk; }
    __syncthreads();
    const double xk = s_xk;
    for (int64_t i = t; i < k; i += DT) x[i] = x[i] - ck[i] * xk;
    __syncthreads();
  }
}

template <int B>
int launch_b(rsim_gpu_ctx* c) {
  const int64_t N = (int64_t)c->nA * B;
  if (N > RSIM_DIRECT_MAX) return RSIM_EARG;
  if (N > c->dn_cap) {  // grow on demand, all three buffers or none
    if (c->dn_W) cudaFree(c->dn_W);
    if (c->dn_colbuf) cudaFree(c->dn_colbuf);
    if (c->dn_piv) cudaFree(c->dn_piv);
    c->dn_W = nullptr; c->dn_colbuf = nullptr; c->dn_piv = nullptr; c->dn_cap = 0;
    const int64_t M = N < 512 ? 512 : N;
    cudaError_t e1 = cudaMalloc(&c->dn_W, sizeof(double) * M * M);
    cudaError_t e2 = cudaMalloc(&c->dn_colbuf, sizeof(double) * 2 * M);
    cudaError_t e3 = cudaMalloc(&c->dn_piv, sizeof(int32_t) * M);
    if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess) {
      if (c->dn_W) cudaFree(c->dn_W);
      if (c->dn_colbuf) cudaFree(c->dn_colbuf);
      if (c->dn_piv) cudaFree(c->dn_piv);
      c->dn_W = nullptr; c->dn_colbuf = nullptr; c->dn_piv = nullptr;
      cudaGetLastError();
      rsim_set_error("direct solve: workspace allocation failed");
      return RSIM_ECUDA;
    }
    c->dn_cap = M;
  }
  DArgs a;
  a.nA = c->nA; a.nslot = c->nslot; a.b = B;
  a.nx = c->nx; a.ny = c->ny; a.nz = c->nz;
  a.d3 = c->d3; a.implicit = c->cols_implicit; a.has_nnc = c->has_nnc; a.f2_parts = c->f2_parts;
  a.cap = c->ell_cap; a.N = N;
  a.ell_col = c->ell_col; a.act = c->act; a.nptr = c->nptr; a.nnc_lcol = c->nnc_lcol;
  a.ell_val = c->ell_val; a.nnc_val = c->nnc_val; a.rhs = c->rhs; a.F_raw = c->F_raw; a.part_f2 = c->part_f2;
  a.W = c->dn_W; a.colbuf = c->dn_colbuf; a.piv = c->dn_piv; a.x = c->x; a.dsc = c->dsc;
  const int64_t nn = N * N;
  const int zb = (int)((nn + 255) / 256 < 4 * c->sm_count ? (nn + 255) / 256 : 4 * c->sm_count);
  k_direct_zero<<<zb, 256, 0, c->stream>>>(a.W, nn, N);
  k_direct_build<B><<<(c->nA + 127) / 128, 128, 0, c->stream>>>(a);
  c->launches += 2;
  RSIM_CUDA(cudaGetLastError());
  // G: ~8+ columns per CTA, at most the co-resident CTAs
  const size_t smem = sizeof(double) * (size_t)N;
  int per_sm = 0;
  RSIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_direct_lu<B>, DT, smem));
  int gmax = per_sm * c->sm_count;
  int g = (int)((N + 7) / 8);
  if (g > gmax) g = gmax;
  if (g > c->sm_count) g = c->sm_count;
  if (g < 1) g = 1;
  if ((N + g - 1) / g > kMaxOwn) return RSIM_EARG;  // (never at N <= RSIM_DIRECT_MAX on 148 SMs)
  void* args[] = {&a};
  RSIM_CUDA(cudaLaunchCooperativeKernel((void*)k_direct_lu<B>, g, DT, args, smem, c->stream));
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

}  // namespace

int launch_direct(rsim_gpu_ctx* c, const rsim_solver_opts* /*o*/) {
  switch (c->b) {
    case 1: return launch_b<1>(c);
    case 2: return launch_b<2>(c);
    default: return launch_b<3>(c);
  }
}
