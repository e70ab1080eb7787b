// spmv_occ.cu — does the b = 3 ELL SpMV of the grid BiCGSTAB scale with
// occupancy?  Synthetic 3D 7-point system (6 slot-major ELL slots of 3x3 fp64
// blocks, like krylov.cu), y = x + Σ_s A_s x_col(s), one row per thread, all
// six gathers in flight vs one at a time; the occupancy is capped with dynamic
// shared memory.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a spmv_occ.cu -o spmv_occ
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

constexpr int B = 3;

template <int SG, int MINB>
__global__ void __launch_bounds__(256, MINB) k_spmv(int64_t n, int nx, int ny, int nz, int64_t cap, const int* __restrict__ col,
                                               const double* __restrict__ val, const double* __restrict__ x,
                                               double* __restrict__ y) {
  // persistent grid-stride over 256-row rounds (the krylov.cu scheme), MINB CTAs per SM
  for (int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; l < n + 255 - threadIdx.x; l += (int64_t)gridDim.x * blockDim.x) {
  if (l >= n) continue;
  double acc[B];
#pragma unroll
  for (int e = 0; e < B; ++e) acc[e] = x[l * B + e];
  int cl[6];
#pragma unroll
  for (int s = 0; s < 6; ++s) cl[s] = __ldg(&col[s * cap + l]);
#pragma unroll
  for (int s0 = 0; s0 < 6; s0 += SG) {
    double xv[SG][B];
#pragma unroll
    for (int k = 0; k < SG; ++k)
      if (cl[s0 + k] >= 0)
#pragma unroll
        for (int e = 0; e < B; ++e) xv[k][e] = __ldg(&x[(int64_t)cl[s0 + k] * B + e]);
#pragma unroll
    for (int k = 0; k < SG; ++k)
      if (cl[s0 + k] >= 0) {
        const double* M = &val[((int64_t)(s0 + k) * cap + l) * B * B];
#pragma unroll
        for (int r = 0; r < B; ++r) {
          double sr = M[r * B] * xv[k][0];
#pragma unroll
          for (int c = 1; c < B; ++c) sr = sr + M[r * B + c] * xv[k][c];
          acc[r] = acc[r] + sr;
        }
      }
    if (SG < 6) asm volatile("" ::: "memory");
  }
#pragma unroll
  for (int e = 0; e < B; ++e) y[l * B + e] = acc[e];
  }
}

int main(int argc, char** argv) {
  const int nx = 96, ny = 96, nz = 84;
  const int64_t n = (int64_t)nx * ny * nz, cap = n;
  std::vector<int> col(6 * n);
  for (int64_t i = 0; i < n; ++i) {
    const int ix = i % nx, iy = (i / nx) % ny, iz = i / (nx * ny);
    const int64_t nb[6] = {iz > 0 ? i - nx * ny : -1, iy > 0 ? i - nx : -1, ix > 0 ? i - 1 : -1,
                           ix < nx - 1 ? i + 1 : -1, iy < ny - 1 ? i + nx : -1, iz < nz - 1 ? i + nx * ny : -1};
    for (int s = 0; s < 6; ++s) col[s * n + i] = (int)nb[s];
  }
  std::vector<double> val(6 * n * 9), x(n * 3);
  for (size_t k = 0; k < val.size(); ++k) val[k] = 1e-3 * ((k * 2654435761u) % 1000);
  for (size_t k = 0; k < x.size(); ++k) x[k] = 1.0 + 1e-3 * (k % 997);
  int* dcol; double *dval, *dx, *dy;
  cudaMalloc(&dcol, col.size() * 4); cudaMalloc(&dval, val.size() * 8);
  cudaMalloc(&dx, x.size() * 8); cudaMalloc(&dy, x.size() * 8);
  cudaMemcpy(dcol, col.data(), col.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dval, val.data(), val.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dx, x.data(), x.size() * 8, cudaMemcpyHostToDevice);
  const double bytes = (double)n * (6 * (9 * 8 + 4) + 2 * 3 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto run = [&](auto kern, int sg, int minb) {
    cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 0);  // max L1
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, 0);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kern);
    const int grid = 148 * minb;
    for (int w = 0; w < 3; ++w) kern<<<grid, 256>>>(n, nx, ny, nz, cap, dcol, dval, dx, dy);
    cudaEventRecord(e0);
    const int reps = 20;
    for (int w = 0; w < reps; ++w) kern<<<grid, 256>>>(n, nx, ny, nz, cap, dcol, dval, dx, dy);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("SG=%d CTAs/SM=%d (occ %d, %d regs, %zu B local) %.3f ms %.0f GB/s\n", sg, minb, occ, fa.numRegs,
           fa.localSizeBytes, ms, bytes / ms / 1e6);
  };
  run(k_spmv<1, 1>, 1, 1); run(k_spmv<1, 2>, 1, 2); run(k_spmv<1, 4>, 1, 4); run(k_spmv<1, 8>, 1, 8);
  run(k_spmv<6, 1>, 6, 1); run(k_spmv<6, 2>, 6, 2); run(k_spmv<6, 4>, 6, 4); run(k_spmv<6, 8>, 6, 8);
  run(k_spmv<2, 4>, 2, 4); run(k_spmv<3, 4>, 3, 4);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return 0;
}
