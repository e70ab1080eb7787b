// eos.cu — Peng-Robinson flash on the GPU:
// one thread per cell runs the two-sided Michelsen stability test and, when
// unstable, successive substitution with Rachford-Rice, all in registers
// (include/rsim/eos.h, shared with the CPU oracle for bit-identical results).
// Cell-parallel and compute-bound: per cell it reads p and z (8(1+nc) B) and
// writes status, ν_g, x, y, Z_o, Z_g (1 + 8(3+2nc) B) once; the work between
// is tens to hundreds of rlog / rexp evaluations, so there is no memory
// roofline to chase and no tensor-core shape.
#include <cuda_runtime.h>

#include <cstring>

#include "rsim/eos.h"
#include "rsim/gpu_abi.h"

namespace {

using rsim::eos::Terms;

template <int NC>
__global__ void __launch_bounds__(128) k_flash(const Terms t, int64_t n, const double* __restrict__ p,
                                               const double* __restrict__ z, uint8_t* __restrict__ status,
                                               double* __restrict__ nu_g, double* __restrict__ x,
                                               double* __restrict__ y, double* __restrict__ zfac,
                                               int32_t* __restrict__ iters) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double zi[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) zi[c] = z[i * NC + c];
  rsim::eos::Flash<NC> R;
  rsim::eos::flash<NC>(t, p[i], zi, R);
  status[i] = (uint8_t)R.status;
  nu_g[i] = R.nu_g;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    x[i * NC + c] = R.x[c];
    y[i * NC + c] = R.y[c];
  }
  zfac[2 * i] = R.Zo;
  zfac[2 * i + 1] = R.Zg;
  if (iters) iters[i] = R.iters;
}

bool valid(const rsim_eos_params* e, double T, int64_t n) {
  if (!e || !(T > 0.0) || n < 0 || e->nc < 1 || e->nc > RSIM_EOS_NCMAX) return false;
  for (int i = 0; i < e->nc; ++i)
    if (!(e->tc[i] > 0.0 && e->pc[i] > 0.0)) return false;
  return true;
}

}  // namespace

extern "C" {

int rsim_eos_case3(rsim_eos_params* o) {
  if (!o) return RSIM_EARG;
  std::memset(o, 0, sizeof(*o));
  o->nc = 2;
  o->tc[0] = 190.56; o->pc[0] = 4.599e6; o->omega[0] = 0.0115; o->mw[0] = 0.016043;  // C1
  o->tc[1] = 617.7;  o->pc[1] = 2.110e6; o->omega[1] = 0.4923; o->mw[1] = 0.142285;  // C10
  o->flash_tol = 1e-8;
  o->flash_maxit = 500;
  o->stab_maxit = 200;
  return RSIM_OK;
}

int rsim_eos_flash_dev(const rsim_eos_params* e, double T, int64_t n, const double* p, const double* z,
                       uint8_t* status, double* nu_g, double* x, double* y, double* zfac, int32_t* iters,
                       void* stream) {
  if (!valid(e, T, n) || (n > 0 && (!p || !z || !status || !nu_g || !x || !y || !zfac))) return RSIM_EARG;
  if (n == 0) return RSIM_OK;
  const Terms t = rsim::eos::terms(*e, T);
  const unsigned blocks = (unsigned)((n + 127) / 128);
  cudaStream_t s = (cudaStream_t)stream;
  switch (e->nc) {
    case 1: k_flash<1><<<blocks, 128, 0, s>>>(t, n, p, z, status, nu_g, x, y, zfac, iters); break;
    case 2: k_flash<2><<<blocks, 128, 0, s>>>(t, n, p, z, status, nu_g, x, y, zfac, iters); break;
    case 3: k_flash<3><<<blocks, 128, 0, s>>>(t, n, p, z, status, nu_g, x, y, zfac, iters); break;
    default: k_flash<4><<<blocks, 128, 0, s>>>(t, n, p, z, status, nu_g, x, y, zfac, iters); break;
  }
  return cudaGetLastError() == cudaSuccess ? RSIM_OK : RSIM_ECUDA;
}

int rsim_eos_flash(const rsim_eos_params* e, double T, int64_t n, const double* p, const double* z,
                   uint8_t* status, double* nu_g, double* x, double* y, double* zfac, int32_t* iters) {
  if (!valid(e, T, n) || (n > 0 && (!p || !z || !status || !nu_g || !x || !y || !zfac))) return RSIM_EARG;
  if (n == 0) return RSIM_OK;
  int dev = 0, cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt < 1) return RSIM_ECUDA;
  cudaDeviceProp pr;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaGetDeviceProperties(&pr, dev) != cudaSuccess || pr.major != 10)
    return RSIM_ECUDA;  // sm_100 only, no CPU fallback
  const int nc = e->nc;
  const size_t bp = n * 8, bz = n * nc * 8;
  char* d = nullptr;
  const size_t tot = bp + bz + bp + 2 * bz + 2 * bp + n * 4 + n;
  if (cudaMalloc(&d, tot) != cudaSuccess) return RSIM_ECUDA;
  size_t off = 0;
  double* dp = (double*)(d + off); off += bp;
  double* dz = (double*)(d + off); off += bz;
  double* dnu = (double*)(d + off); off += bp;
  double* dx = (double*)(d + off); off += bz;
  double* dy = (double*)(d + off); off += bz;
  double* dzf = (double*)(d + off); off += 2 * bp;
  int32_t* dit = (int32_t*)(d + off); off += n * 4;
  uint8_t* dst = (uint8_t*)(d + off);
  int rc = RSIM_OK;
  cudaStream_t s = nullptr;
  if (cudaMemcpyAsync(dp, p, bp, cudaMemcpyHostToDevice, s) != cudaSuccess ||
      cudaMemcpyAsync(dz, z, bz, cudaMemcpyHostToDevice, s) != cudaSuccess)
    rc = RSIM_ECUDA;
  if (rc == RSIM_OK) rc = rsim_eos_flash_dev(e, T, n, dp, dz, dst, dnu, dx, dy, dzf, dit, s);
  if (rc == RSIM_OK &&
      (cudaMemcpyAsync(status, dst, n, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
       cudaMemcpyAsync(nu_g, dnu, bp, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
       cudaMemcpyAsync(x, dx, bz, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
       cudaMemcpyAsync(y, dy, bz, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
       cudaMemcpyAsync(zfac, dzf, 2 * bp, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
       (iters && cudaMemcpyAsync(iters, dit, n * 4, cudaMemcpyDeviceToHost, s) != cudaSuccess) ||
       cudaStreamSynchronize(s) != cudaSuccess))
    rc = RSIM_ECUDA;
  cudaFree(d);
  return rc;
}

}  // extern "C"
