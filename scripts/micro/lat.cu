// Micro-benchmark: dependent-chain latency of fp64 ops, shuffles and smem loads (cycles).
#include <cstdio>
__global__ void k(double* out, long long* t, double a, double b) {
  __shared__ double sm[64];
  sm[threadIdx.x & 63] = threadIdx.x;
  __syncthreads();
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < 256; ++i) { x = x + b; }
  long long t1 = clock64();
  for (int i = 0; i < 256; ++i) { x = x * b; }
  long long t2 = clock64();
  for (int i = 0; i < 256; ++i) { x = __fma_rn(x, b, a); }
  long long t3 = clock64();
  for (int i = 0; i < 256; ++i) { x = x + __shfl_down_sync(0xffffffffu, x, 1); }
  long long t4 = clock64();
  int idx = threadIdx.x & 7;
  for (int i = 0; i < 256; ++i) { double y = sm[idx]; idx = ((int)y + i) & 7; x += y; }
  long long t5 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { t[0] = t1 - t0; t[1] = t2 - t1; t[2] = t3 - t2; t[3] = t4 - t3; t[4] = t5 - t4; }
}
int main() {
  double* o; long long* t; cudaMalloc(&o, 1024 * 8); cudaMalloc(&t, 64);
  for (int rep = 0; rep < 2; ++rep) {
    k<<<1, 32>>>(o, t, 1.0, 1.0000001);
    long long h[5]; cudaMemcpy(h, t, 40, cudaMemcpyDeviceToHost);
    printf("per op cycles: dadd %.1f dmul %.1f dfma %.1f shfl+dadd %.1f lds+iadd+dadd %.1f\n", h[0] / 256.0, h[1] / 256.0, h[2] / 256.0, h[3] / 256.0, h[4] / 256.0);
  }
  return 0;
}
