// Micro-benchmark: the cluster Krylov kernel's reduction (warp trees -> smem ->
// relaxed cluster barrier -> warp q gathers canonical warp sums via DSMEM ->
// tree -> __syncthreads broadcast), isolated: cycles per reduction.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ double warp_tree_n(double v, int n) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) { if (off >= n) v = v + 0.0; else v = v + __shfl_down_sync(0xffffffffu, v, off); }
  return v;
}
__device__ __forceinline__ double tree8(const double* w) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = w[k];
#pragma unroll
  for (int off = 4; off >= 1; off >>= 1)
#pragma unroll
    for (int k = 0; k < off; ++k) a[k] = a[k] + a[k + off];
  return a[0];
}
template <int NQ, int MODE>
__global__ void k_red(int iters, long long* out, double* sink, int nr) {
  __shared__ double ws[2][5][32];
  __shared__ double res_s[5];
  cg::cluster_group cl = cg::this_cluster();
  const int G = cl.num_blocks();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int LWPC = __ffs(blockDim.x >> 5) - 1;
  const int nch = (nr + 255) / 256;
  const uint32_t ws_u32 = smem_u32(&ws[0][0][0]);
  int wbuf = 0;
  double acc = 0.0, val[NQ];
  for (int q = 0; q < NQ; ++q) val[q] = 1e-3 * (tid + q);
  cl.sync();
  long long t0 = clock64(), tsync = 0, tshfl = 0, tgather = 0, tfin = 0;
  for (int i = 0; i < iters; ++i) {
    long long tA = clock64();
    double v[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) v[q] = val[q] + acc;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
      for (int q = 0; q < NQ; ++q) v[q] = v[q] + __shfl_down_sync(0xffffffffu, v[q], off);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < NQ; ++q) ws[wbuf][q][w] = v[q];
    long long ta = clock64();
    tshfl += ta - tA;
    __syncthreads();
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
    long long tb = clock64();
    tsync += tb - ta;
    for (int q = w; q < NQ; q += (1 << LWPC)) {
      double cp[2] = {0.0, 0.0};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = lane + 32 * h;
        if (c < nch) {
          double w8[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int gw = (c << 3) | k;
            double x = 0.0;
            if (MODE == 0) {
              if ((gw << 5) < nr) {
                const uint32_t ad = mapa_u32(ws_u32, gw >> LWPC) + (uint32_t)(((wbuf * 5 + q) * 32 + (gw & ((1 << LWPC) - 1))) * 8);
                asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(x) : "r"(ad) : "memory");
              }
            } else {
              const double* rp = cl.map_shared_rank(&ws[wbuf][q][0], gw >> LWPC);
              x = ((gw << 5) < nr) ? rp[gw & ((1 << LWPC) - 1)] : 0.0;
            }
            w8[k] = x;
          }
          cp[h] = tree8(w8);
        }
      }
      double r;
      if (nch == 1) r = cp[0];
      else { double W[8] = {warp_tree_n(cp[0], nch), warp_tree_n(cp[1], nch - 32), 0, 0, 0, 0, 0, 0}; r = tree8(W); }
      if (lane == 0) res_s[q] = r;
    }
    long long tc = clock64();
    tgather += tc - tb;
    __syncthreads();
    double s = 0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) s += res_s[q];
    acc = s * 1e-30;
    tfin += clock64() - tc;
    wbuf ^= 1;
  }
  long long t1 = clock64();
  if (tid == 0 && cl.block_rank() == 0) { out[0] = (t1 - t0) / iters; out[1] = tsync / iters; out[2] = tshfl / iters; out[3] = tgather / iters; out[4] = tfin / iters; }
  sink[blockIdx.x * blockDim.x + tid] = acc;
  cl.sync();
}
__device__ __forceinline__ void mb_init(uint32_t bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c) : "memory"); }
__device__ __forceinline__ void mb_expect(uint32_t bar, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b) : "memory"); }
__device__ __forceinline__ void st_async(uint32_t ra, double v, uint32_t rb) { asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra), "l"(__double_as_longlong(v)), "r"(rb) : "memory"); }
__device__ __forceinline__ void mb_wait(uint32_t bar, uint32_t par) {
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}" ::"r"(bar), "r"(par) : "memory");
}
// push variant: every warp's lanes 0..G-1 st.async the warp's NQ sums into CTA
// k's table [q][global warp]; each CTA waits on its transaction barrier, then
// warp q finishes quantity q from LOCAL shared memory; __syncthreads broadcast.
template <int NQ>
__global__ void k_push(int iters, long long* out, double* sink, int nr) {
  __shared__ double tab[2][5][512];
  __shared__ double res_s[5];
  __shared__ __align__(8) uint64_t bar[2];
  cg::cluster_group cl = cg::this_cluster();
  const int G = cl.num_blocks(), rank = cl.block_rank();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, tid = threadIdx.x;
  const int WPC = blockDim.x >> 5;
  const int nch = (nr + 255) / 256;
  if (tid == 0) { mb_init(smem_u32(&bar[0]), 1); mb_init(smem_u32(&bar[1]), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  cl.sync();
  const uint32_t rt = mapa_u32(smem_u32(&tab[0][0][0]), lane < G ? lane : 0), rb = mapa_u32(smem_u32(&bar[0]), lane < G ? lane : 0);
  double acc = 0.0, val[NQ];
  for (int q = 0; q < NQ; ++q) val[q] = 1e-3 * (tid + q);
  long long t0 = clock64(), tsync = 0, tshfl = 0, tgather = 0, tfin = 0;
  for (int i = 0; i < iters; ++i) {
    long long tA = clock64();
    const int X = i & 1; const uint32_t par = (i >> 1) & 1;
    if (tid == 0) mb_expect(smem_u32(&bar[X]), (uint32_t)(G * WPC * NQ * 8));
    double v[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) v[q] = val[q] + acc;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
      for (int q = 0; q < NQ; ++q) v[q] = v[q] + __shfl_down_sync(0xffffffffu, v[q], off);
    double bv[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) bv[q] = __shfl_sync(0xffffffffu, v[q], 0);
    if (lane < G)
#pragma unroll
      for (int q = 0; q < NQ; ++q) st_async(rt + (uint32_t)(((X * 5 + q) * 512 + rank * WPC + w) * 8), bv[q], rb + X * 8);
    long long ta = clock64();
    tshfl += ta - tA;
    mb_wait(smem_u32(&bar[X]), par);
    long long tb = clock64();
    tsync += tb - ta;
    for (int q = w; q < NQ; q += WPC) {
      double cp[2] = {0.0, 0.0};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = lane + 32 * h;
        if (c < nch) {
          double w8[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) { const int gw = (c << 3) | k; w8[k] = ((gw << 5) < nr) ? tab[X][q][gw] : 0.0; }
          cp[h] = tree8(w8);
        }
      }
      double r;
      if (nch == 1) r = cp[0];
      else { double W[8] = {warp_tree_n(cp[0], nch), warp_tree_n(cp[1], nch - 32), 0, 0, 0, 0, 0, 0}; r = tree8(W); }
      if (lane == 0) res_s[q] = r;
    }
    long long tc = clock64();
    tgather += tc - tb;
    __syncthreads();
    double s = 0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) s += res_s[q];
    acc = s * 1e-30;
    tfin += clock64() - tc;
  }
  long long t1 = clock64();
  if (tid == 0 && rank == 0) { out[0] = (t1 - t0) / iters; out[1] = tsync / iters; out[2] = tshfl / iters; out[3] = tgather / iters; out[4] = tfin / iters; }
  sink[blockIdx.x * blockDim.x + tid] = acc;
  cl.sync();
}

template <class K>
void run(K k, int G, int T, int nr, const char* name) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G); cfg.blockDim = dim3(T);
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = G; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  long long* d; cudaMalloc(&d, 64); double* sink; cudaMalloc(&sink, 16 * 1024 * 8);
  int it = 2000;
  cudaLaunchKernelEx(&cfg, k, it, d, sink, nr);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[5]; cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
  printf("%-6s G=%2d T=%4d nr=%5d : %5lld cyc/red | shfl+sts %4lld | sync+cluster %4lld | gather+tree (warp0) %4lld | bcast %4lld %s\n", name, G, T, nr, h[0], h[2], h[1], h[3], h[4], e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d); cudaFree(sink);
}
int main() {
  for (int G : {4, 10, 16}) {
    run(k_red<2, 0>, G, 256, G * 256, "NQ=2");
    run(k_push<2>, G, 256, G * 256, "push2");
    run(k_red<5, 0>, G, 256, G * 256, "NQ=5");
    run(k_push<5>, G, 256, G * 256, "push5");
    run(k_red<5, 0>, G, 512, G * 512, "NQ=5");
    run(k_push<5>, G, 512, G * 512, "push5");
  }
  return 0;
}
