// Micro-benchmark: latency of cluster-wide exchange primitives (cycles/iter).
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int r) { uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o; }
__device__ __forceinline__ void mb_init(uint32_t bar, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(c) : "memory"); }
__device__ __forceinline__ void mb_expect(uint32_t bar, uint32_t b) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(b) : "memory"); }
__device__ __forceinline__ void st_async(uint32_t ra, double v, uint32_t rb) { asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra), "l"(__double_as_longlong(v)), "r"(rb) : "memory"); }
template <bool CL>
__device__ __forceinline__ void mb_wait(uint32_t bar, uint32_t par) {
  if (CL) asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}" ::"r"(bar), "r"(par) : "memory");
  else asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}" ::"r"(bar), "r"(par) : "memory");
}
__global__ void k_clsync(int iters, long long* out, double*) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = (t1 - t0) / iters;
}
__global__ void k_clsync_relaxed(int iters, long long* out, double*) {
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = (t1 - t0) / iters;
}
// all-to-all: MODE 0 = every warp sends 1 double to every CTA; 1 = syncthreads + warp 0 sends
template <int MODE, bool CL>
__global__ void k_a2a(int iters, long long* out, double* sink) {
  __shared__ double recv[2][512];
  __shared__ __align__(8) uint64_t bar[2];
  cg::cluster_group cl = cg::this_cluster();
  const int G = cl.num_blocks(), rank = cl.block_rank();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, WPC = blockDim.x >> 5;
  if (threadIdx.x == 0) { mb_init(smem_u32(&bar[0]), 1); mb_init(smem_u32(&bar[1]), 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  cl.sync();
  const uint32_t rr = mapa_u32(smem_u32(&recv[0][0]), lane < G ? lane : 0), rbb = mapa_u32(smem_u32(&bar[0]), lane < G ? lane : 0);
  double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    const int X = i & 1; const uint32_t par = (i >> 1) & 1;
    if (threadIdx.x == 0) mb_expect(smem_u32(&bar[X]), MODE == 0 ? G * WPC * 8 : G * 8);
    if (MODE == 0) {
      __syncwarp();
      if (lane < G) st_async(rr + (X * 512 + rank * WPC + w) * 8, acc + i, rbb + X * 8);
    } else {
      __syncthreads();
      if (w == 0 && lane < G) st_async(rr + (X * 512 + rank) * 8, acc + i, rbb + X * 8);
    }
    mb_wait<CL>(smem_u32(&bar[X]), par);
    acc += recv[X][lane];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) out[0] = (t1 - t0) / iters;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  cl.sync();
}
// DSMEM read latency chain
__global__ void k_dsmem_lat(int iters, long long* out, double* sink) {
  __shared__ double buf[256];
  cg::cluster_group cl = cg::this_cluster();
  buf[threadIdx.x] = threadIdx.x;
  cl.sync();
  const double* rem = cl.map_shared_rank(buf, (cl.block_rank() + 1) % cl.num_blocks());
  uint32_t ra = mapa_u32(smem_u32(buf), (cl.block_rank() + 1) % cl.num_blocks());
  double a = 0; int idx = threadIdx.x & 1;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) { double v; asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra + idx * 8) : "memory"); a += v; idx = (int)v & 1; }
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) { double v = rem[idx]; a += v; idx = (int)v & 1; }
  long long t2 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) { out[0] = (t1 - t0) / iters; out[1] = (t2 - t1) / iters; }
  sink[blockIdx.x * blockDim.x + threadIdx.x] = a;
  cl.sync();
}
template <class K>
long long run2(K k, int G, int T, int iters, double* sink, long long* h2 = nullptr) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G); cfg.blockDim = dim3(T);
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = G; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  long long* d; cudaMalloc(&d, 16); cudaMemset(d, 0, 16);
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, iters, d, sink);
  cudaError_t e2 = cudaDeviceSynchronize();
  long long h[2] = {0, 0}; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); cudaFree(d);
  if (e != cudaSuccess || e2 != cudaSuccess) { printf("err %s %s\n", cudaGetErrorString(e), cudaGetErrorString(e2)); return -1; }
  if (h2) *h2 = h[1];
  return h[0];
}
int main() {
  double* sink; cudaMalloc(&sink, 16 * 1024 * 8);
  const int it = 2000;
  for (int T : {128, 256, 512}) for (int G : {1, 2, 4, 8, 10, 16}) {
    printf("T=%4d G=%2d  cluster.sync %5lld  relaxed %5lld  a2a-warp %5lld  a2a-warp(acq.cta) %5lld  a2a-cta %5lld  a2a-cta(acq.cta) %5lld\n", T, G,
           run2(k_clsync, G, T, it, sink), run2(k_clsync_relaxed, G, T, it, sink), run2(k_a2a<0, true>, G, T, it, sink),
           run2(k_a2a<0, false>, G, T, it, sink), run2(k_a2a<1, true>, G, T, it, sink), run2(k_a2a<1, false>, G, T, it, sink));
  }
  for (int G : {2, 8, 16}) { long long b = 0; long long a = run2(k_dsmem_lat, G, 256, it, sink, &b); printf("G=%d dsmem load-use latency: ld.shared::cluster %lld  generic %lld\n", G, a, b); }
  return 0;
}
