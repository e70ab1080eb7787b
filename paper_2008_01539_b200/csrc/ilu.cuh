// ilu.cuh — device side of the level-scheduled block ILU(0) (ilu.cu): the
// argument block and the triangular-solve routine used inside the persistent
// Krylov kernels.  Each row's operations follow oracle.cpp ilu0_apply() in the
// same order, so the result does not depend on the schedule.
#pragma once
#include "ctx.cuh"

struct IluArgs {
  int32_t n;              // rows (n_A)
  const int32_t* ptr;     // [n+1] row entries, sorted by column, diagonal excluded
  const int32_t* col;     // [nnz]
  const double* val;      // [nnz][B*B]  L (col < row) / U (col > row)
  const double* dinv;     // [n][B*B]    inverse diagonal blocks of U
  const int32_t* frows;   // rows ordered by forward level, offsets foff[nf+1]
  const int32_t* foff;
  int32_t nf;
  const int32_t* brows;   // rows ordered by backward level, offsets boff[nb+1]
  const int32_t* boff;
  int32_t nb;
  double* y;              // [n][B] forward-solve result
};

// out = (LU)^{-1} z over the whole grid; `sync` is the grid barrier between levels
template <int B, class SYNC>
__device__ __forceinline__ void ilu_apply(const IluArgs& f, const double* z, double* out, SYNC&& sync) {
  constexpr int BB = B * B;
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x;
  for (int lv = 0; lv < f.nf; ++lv) {
    for (int64_t k = f.foff[lv] + gtid; k < f.foff[lv + 1]; k += gstride) {
      const int32_t i = f.frows[k];
      double t[B];
#pragma unroll
      for (int c = 0; c < B; ++c) t[c] = z[(int64_t)i * B + c];
      for (int32_t p = f.ptr[i]; p < f.ptr[i + 1] && f.col[p] < i; ++p)
        rsim::blk::gemv_sub_flat<B>(&f.val[(int64_t)p * BB], &f.y[(int64_t)f.col[p] * B], t);
#pragma unroll
      for (int c = 0; c < B; ++c) f.y[(int64_t)i * B + c] = t[c];
    }
    sync();
  }
  for (int lv = 0; lv < f.nb; ++lv) {
    for (int64_t k = f.boff[lv] + gtid; k < f.boff[lv + 1]; k += gstride) {
      const int32_t i = f.brows[k];
      double t[B];
#pragma unroll
      for (int c = 0; c < B; ++c) t[c] = f.y[(int64_t)i * B + c];
      for (int32_t p = f.ptr[i]; p < f.ptr[i + 1]; ++p)
        if (f.col[p] > i) rsim::blk::gemv_sub_flat<B>(&f.val[(int64_t)p * BB], &out[(int64_t)f.col[p] * B], t);
      rsim::blk::gemv_flat<B>(&f.dinv[(int64_t)i * BB], t, &out[(int64_t)i * B]);
    }
    sync();
  }
}

__host__ inline IluArgs ilu_args(const rsim_gpu_ctx* c) {
  IluArgs f;
  f.n = c->nA;
  f.ptr = c->ilu.ptr; f.col = c->ilu.col; f.val = c->ilu.val; f.dinv = c->ilu.dinv;
  f.frows = c->ilu.frows; f.foff = c->ilu.foff; f.nf = c->ilu.nf;
  f.brows = c->ilu.brows; f.boff = c->ilu.boff; f.nb = c->ilu.nb;
  f.y = c->ilu.y;
  return f;
}
