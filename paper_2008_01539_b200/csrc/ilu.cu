// ilu.cu — level-scheduled block ILU(0) of the block-Jacobi-scaled active
// system (north star: "BiCGSTAB/GMRES with block-Jacobi or level-scheduled
// ILU(0)"), restating oracle.cpp ilu0_factor():
//   rows in the local (natural) order, IKJ: for each lower entry k of row i
//   (ascending column) L_ik = A_ik D_k^{-1}, then A_ij -= L_ik U_kj over row
//   k's upper entries (ascending j) present in row i (j == i: diagonal).
// The schedule: row i's forward level is 1 + the max level of its lower
// neighbours (backward: of its upper neighbours); rows of one level are
// independent, each is computed by one thread with the oracle's operation
// order, so factors and triangular solves are bit-identical to the oracle.
// The sparsity pattern and the level schedule are integer bookkeeping done by
// the host per assembly (one D2H of the ELL columns); the factorisation and
// both triangular solves are GPU kernels (no CPU numerics).
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

#include "ctx.cuh"
#include "ilu.cuh"

namespace cg = cooperative_groups;

namespace {

template <int B>
__global__ void __launch_bounds__(256) k_ilu_factor(IluArgs f, const int32_t* __restrict__ src, int32_t nnz,
                                                    const double* __restrict__ ell_val, int64_t ell_cap,
                                                    const double* __restrict__ nnc_val, DevScalars* dsc) {
  constexpr int BB = B * B;
  auto grid = cg::this_grid();
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  double* val = const_cast<double*>(f.val);
  double* dinv = const_cast<double*>(f.dinv);
  if (gtid == 0) dsc->ilu_bad = 0;
  for (int64_t p = gtid; p < nnz; p += gstride) {  // gather the scaled blocks into CSR order
    const int32_t s = src[p];
    if (s >= 0) {  // s = slot · cap + local row (ELL value layout: ctx.cuh ell_at)
      const int32_t slot = s / (int32_t)ell_cap;
      const int64_t l = s - (int64_t)slot * ell_cap;
#pragma unroll
      for (int q = 0; q < BB; ++q) val[(int64_t)p * BB + q] = ell_val[ell_at(ell_cap, BB, slot, q, l)];
    } else {
      const double* from = &nnc_val[(int64_t)(-s - 1) * BB];
#pragma unroll
      for (int q = 0; q < BB; ++q) val[(int64_t)p * BB + q] = from[q];
    }
  }
  grid.sync();
  for (int lv = 0; lv < f.nf; ++lv) {
    for (int64_t k = f.foff[lv] + gtid; k < f.foff[lv + 1]; k += gstride) {
      const int32_t i = f.frows[k];
      double dg[BB];
#pragma unroll
      for (int q = 0; q < BB; ++q) dg[q] = (q % (B + 1) == 0) ? 1.0 : 0.0;
      for (int32_t p = f.ptr[i]; p < f.ptr[i + 1] && f.col[p] < i; ++p) {
        const int32_t kk = f.col[p];
        double L[BB];
        rsim::blk::gemm_flat<B>(&val[(int64_t)p * BB], &dinv[(int64_t)kk * BB], L);
#pragma unroll
        for (int q = 0; q < BB; ++q) val[(int64_t)p * BB + q] = L[q];
        for (int32_t r = f.ptr[kk]; r < f.ptr[kk + 1]; ++r) {
          const int32_t j = f.col[r];
          if (j <= kk) continue;
          if (j == i) {
            rsim::blk::gemm_sub_flat<B>(L, &val[(int64_t)r * BB], dg);
          } else {
            for (int32_t t = f.ptr[i]; t < f.ptr[i + 1]; ++t)
              if (f.col[t] == j) {
                rsim::blk::gemm_sub_flat<B>(L, &val[(int64_t)r * BB], &val[(int64_t)t * BB]);
                break;
              }
          }
        }
      }
      if (!rsim::blk::inv_flat<B>(dg, &dinv[(int64_t)i * BB])) atomicExch(&dsc->ilu_bad, 1);
    }
    grid.sync();
  }
}

template <class T>
int grow(T** p, int64_t& cap, int64_t need) {
  if (need <= cap) return RSIM_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  const int64_t n = need + need / 4 + 64;
  RSIM_CUDA(cudaMalloc((void**)p, sizeof(T) * n));
  cap = n;
  return RSIM_OK;
}

template <int B>
int factor_launch(rsim_gpu_ctx* c) {
  IluArgs f = ilu_args(c);
  static int per_sm = 0;
  if (per_sm == 0) {
    RSIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ilu_factor<B>, 256, 0));
    if (per_sm < 1) per_sm = 1;
  }
  const int64_t want = std::max<int64_t>((c->ilu.nnz + 255) / 256, (c->ilu.maxw + 255) / 256);
  const int64_t maxb = (int64_t)per_sm * c->sm_count;
  int grid = (int)std::max<int64_t>(1, std::min(want, maxb));
  int32_t nnz = c->ilu.nnz;
  const int32_t* src = c->ilu.src;
  const double* ev = c->ell_val;
  int64_t ecap = c->ell_cap;
  const double* nv = c->nnc_val;
  DevScalars* dsc = c->dsc;
  void* args[] = {&f, &src, &nnz, &ev, &ecap, &nv, &dsc};
  RSIM_CUDA(cudaLaunchCooperativeKernel((void*)k_ilu_factor<B>, grid, 256, args, 0, c->stream));
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

}  // namespace

int ilu_prepare(rsim_gpu_ctx* c) {
  const int32_t n = c->nA, b = c->b;
  if (n <= 0) return RSIM_OK;
  RSIM_TRY(launch_materialize_cols(c));
  // ---- pattern (host bookkeeping): ELL columns + active NNC columns, sorted per row
  std::vector<int32_t> ecol((size_t)c->nslot * n), act(n), nlcol(c->nnc_total);
  RSIM_CUDA(cudaStreamSynchronize(c->stream));
  for (int s = 0; s < c->nslot; ++s)
    RSIM_CUDA(cudaMemcpy(&ecol[(size_t)s * n], c->ell_col + (int64_t)s * c->ell_cap, sizeof(int32_t) * n,
                         cudaMemcpyDeviceToHost));
  if (c->has_nnc) {
    RSIM_CUDA(cudaMemcpy(act.data(), c->act, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    RSIM_CUDA(cudaMemcpy(nlcol.data(), c->nnc_lcol, sizeof(int32_t) * c->nnc_total, cudaMemcpyDeviceToHost));
  }
  std::vector<int32_t> ptr(n + 1, 0), col, src;
  col.reserve((size_t)n * c->nslot);
  src.reserve((size_t)n * c->nslot);
  std::vector<std::pair<int32_t, int32_t>> ent;
  for (int32_t l = 0; l < n; ++l) {
    ent.clear();
    for (int s = 0; s < c->nslot; ++s) {
      const int32_t cl = ecol[(size_t)s * n + l];
      if (cl >= 0) ent.emplace_back(cl, (int32_t)(s * c->ell_cap + l));  // ELL value index (slot-major)
    }
    if (c->has_nnc) {
      const int64_t i = act[l];
      for (int32_t q = c->h_nptr[i]; q < c->h_nptr[i + 1]; ++q)
        if (nlcol[q] >= 0) ent.emplace_back(nlcol[q], -(q + 1));
    }
    std::stable_sort(ent.begin(), ent.end(), [](auto& x, auto& y) { return x.first < y.first; });
    for (auto& e : ent) { col.push_back(e.first); src.push_back(e.second); }
    ptr[l + 1] = (int32_t)col.size();
  }
  // ---- level schedules
  std::vector<int32_t> flev(n, 0), blev(n, 0);
  int32_t nf = 0, nb = 0;
  for (int32_t i = 0; i < n; ++i) {
    int32_t lv = 0;
    for (int32_t p = ptr[i]; p < ptr[i + 1] && col[p] < i; ++p) lv = std::max(lv, flev[col[p]] + 1);
    flev[i] = lv;
    nf = std::max(nf, lv + 1);
  }
  for (int32_t i = n - 1; i >= 0; --i) {
    int32_t lv = 0;
    for (int32_t p = ptr[i]; p < ptr[i + 1]; ++p)
      if (col[p] > i) lv = std::max(lv, blev[col[p]] + 1);
    blev[i] = lv;
    nb = std::max(nb, lv + 1);
  }
  auto order = [&](const std::vector<int32_t>& lev, int32_t nl, std::vector<int32_t>& rows, std::vector<int32_t>& off) {
    off.assign(nl + 1, 0);
    for (int32_t i = 0; i < n; ++i) ++off[lev[i] + 1];
    for (int32_t k = 0; k < nl; ++k) off[k + 1] += off[k];
    rows.assign(n, 0);
    std::vector<int32_t> pos(off.begin(), off.end() - 1);
    for (int32_t i = 0; i < n; ++i) rows[pos[lev[i]]++] = i;
  };
  std::vector<int32_t> frows, foff, brows, boff;
  order(flev, nf, frows, foff);
  order(blev, nb, brows, boff);
  int32_t maxw = 0;
  for (int32_t k = 0; k < nf; ++k) maxw = std::max(maxw, foff[k + 1] - foff[k]);
  // ---- device buffers (grown on demand, one capacity per buffer)
  auto& I = c->ilu;
  const int64_t nnz = (int64_t)col.size(), nl = (int64_t)std::max(nf, nb) + 1;
  RSIM_TRY(grow(&I.col, I.cap[0], nnz));
  RSIM_TRY(grow(&I.src, I.cap[1], nnz));
  RSIM_TRY(grow(&I.val, I.cap[2], nnz * b * b));
  RSIM_TRY(grow(&I.ptr, I.cap[3], (int64_t)n + 1));
  RSIM_TRY(grow(&I.frows, I.cap[4], (int64_t)n));
  RSIM_TRY(grow(&I.brows, I.cap[5], (int64_t)n));
  RSIM_TRY(grow(&I.dinv, I.cap[6], (int64_t)n * b * b));
  RSIM_TRY(grow(&I.y, I.cap[7], (int64_t)n * b));
  RSIM_TRY(grow(&I.foff, I.cap[8], nl));
  RSIM_TRY(grow(&I.boff, I.cap[9], nl));
  I.nnz = (int32_t)nnz; I.nf = nf; I.nb = nb; I.maxw = maxw;
  auto up = [&](void* d, const void* h, size_t bytes) -> int {
    if (bytes) RSIM_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, c->stream));
    return RSIM_OK;
  };
  RSIM_TRY(up(I.ptr, ptr.data(), sizeof(int32_t) * (n + 1)));
  RSIM_TRY(up(I.col, col.data(), sizeof(int32_t) * nnz));
  RSIM_TRY(up(I.src, src.data(), sizeof(int32_t) * nnz));
  RSIM_TRY(up(I.frows, frows.data(), sizeof(int32_t) * n));
  RSIM_TRY(up(I.brows, brows.data(), sizeof(int32_t) * n));
  RSIM_TRY(up(I.foff, foff.data(), sizeof(int32_t) * (nf + 1)));
  RSIM_TRY(up(I.boff, boff.data(), sizeof(int32_t) * (nb + 1)));
  switch (b) {
    case 1: RSIM_TRY(factor_launch<1>(c)); break;
    case 2: RSIM_TRY(factor_launch<2>(c)); break;
    default: RSIM_TRY(factor_launch<3>(c)); break;
  }
  // the host vectors must outlive the async copies
  RSIM_CUDA(cudaStreamSynchronize(c->stream));
  return RSIM_OK;
}

void ilu_free(rsim_gpu_ctx* c) {
  auto& I = c->ilu;
  void* ps[] = {I.ptr, I.col, I.src, I.frows, I.foff, I.brows, I.boff, I.val, I.dinv, I.y};
  for (void* p : ps)
    if (p) cudaFree(p);
  I = rsim_gpu_ctx::Ilu{};
}
