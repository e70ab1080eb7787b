// krylov_dsm.cu — cluster-resident BiCGSTAB for small active systems.
//
// The localized solver's active systems are small (~10^2-10^4
// rows), so a Krylov iteration is bound by latency, not HBM.  This kernel runs
// the whole solve inside ONE thread-block cluster of G <= 16 CTAs:
//
//   * CTA g owns the contiguous local rows [g*RC, (g+1)*RC), RC = 64..1024
//     (RC/32 canonical warps, blockops.h); a reduction is warp shuffles into
//     shared memory, one cluster barrier, then a DSMEM gather of the canonical
//     warp sums and the canonical tree (identical in every CTA);
//   * the Krylov vectors and (when it fits) the ELL rows of each CTA live in
//     its shared memory for the whole solve — global traffic is the initial
//     load and the final store of x;
//   * every neighbour's tagged shared address (own CTA: ld.shared, peer CTA:
//     ld.shared::cluster) is resolved once per solve;
//   * the neighbours' p (via r = s − ω t) and s are recomputed at the gather
//     site (same formulas, same bits), and BiCGSTAB runs with two reductions
//     per iteration ((r0,v) with the lagged (r,r); (s,s), (t,s), (t,t),
//     (r0,s), (r0,t) with ρ = (r0,s) − ω (r0,t)): 2 cluster barriers per
//     iteration, 4 with the Neumann-1 preconditioner;
//   * cluster barriers are relaxed (no GPU-scope fence) after a __syncthreads
//     that drains the CTA's shared stores — see csync().
// Element formulas and reduction order are those of oracle/oracle.cpp
// bicgstab(); results are bit-identical to it and to krylov.cu.

#include <cooperative_groups.h>

#include <cstdlib>
#include <map>
#include <tuple>
#include <type_traits>

#include "ctx.cuh"

namespace cg = cooperative_groups;

namespace {

// ---- shared::cluster addressing (PTX; sm_90+)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, int r) {
  uint32_t o;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r));
  return o;
}
#ifndef RSIM_DSM_SG512
#define RSIM_DSM_SG512 1
#endif
#ifndef RSIM_DSM_PUSH
#define RSIM_DSM_PUSH 1
#endif
#ifndef RSIM_DSM_TRACE
#define RSIM_DSM_TRACE 0
#endif
constexpr bool kTrace = RSIM_DSM_TRACE != 0;
constexpr int GMAX = 16;
constexpr int NNCMAX = 256;             // NNC entries cached in smem per CTA
constexpr int NNC_GLOBAL = 0x40000000;  // flag in the range end: entries stay in global

struct DArgs {
  int32_t nA, nslot, maxit, fixed, LRC, nch, neu;
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
  double* x;
  DevScalars* dsc;
  unsigned long long* trace;  // optional [8] cycle accumulators (RSIM_KTRACE)
  // fused Newton update (K6, sets.cu k_update) in the epilogue, Newton loops only
  int32_t upd;
  double eps;
  rsim::phys::Fluid fl;
  double *u, *dp, *last_dp;
  uint8_t *st, *flags;
};

// Cluster loads of a row's B components (shared::cluster address; B = 3 is padded to 4).
__device__ __forceinline__ void mb_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mb_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// 8-byte store into a peer CTA's shared memory that completes bytes on the
// peer's transaction mbarrier (the completion has release semantics at
// cluster scope: the issuing warp's earlier shared-memory writes, ordered by
// __syncwarp / __syncthreads, are visible to the peer after its wait)
__device__ __forceinline__ void st_async_f64(uint32_t remote_addr, double v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(remote_addr),
               "l"(__double_as_longlong(v)), "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void mb_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// Row loads of B components through a generic pointer into this CTA's or a
// peer CTA's shared memory (the hardware routes a peer window to DSMEM).
// B = 3 rows are padded to 4 doubles, so every row starts 16-byte aligned.
template <int B>
__device__ __forceinline__ void ldg_row(const double* p, double* o) {
  if constexpr (B == 1) {
    o[0] = p[0];
  } else {
    const double2 v = *reinterpret_cast<const double2*>(p);
    o[0] = v.x;
    o[1] = v.y;
    if constexpr (B == 3) o[2] = p[2];
  }
}

template <int B, int NS, bool MS, int MAXT>
__global__ void __launch_bounds__(MAXT, 1) k_krylov_dsm(const DArgs a) {
  // Shared layout (identical in every CTA, so a neighbour row's cluster
  // address is mapa(base, owner) + row offset, computed once per solve):
  //   V[RC][11][BP]: per row r, p0, p1, v0, v1, ph, sh, s, t, r0, x (p, v
  //   double-buffered: neighbours read the previous iterate while the owner
  //   writes the new one; s, t feed the neighbours' recompute of r)
  //   mval[NS][RC][B*B] (MS), NNC ranges, NNC blocks + cluster addresses.
  // Own-row-only vectors r0, x, s, t live in registers.
  constexpr int BP = (B == 3) ? 4 : B;
  constexpr int ROWD = 11 * BP;
  constexpr uint32_t ROWB = ROWD * 8;
  constexpr int O_R = 0, O_P = 1, O_V = 3, O_PH = 5, O_SH = 6, O_S = 7, O_T = 8, O_R0 = 9, O_X = 10;
  extern __shared__ __align__(16) double dyn[];
  const int RC = 1 << a.LRC;
  double* V = dyn;
  double* mval = V + RC * ROWD;                                     // [NS][RC][B*B]  (MS)
  int2* nrng = (int2*)(mval + (MS ? NS * RC * B * B : 0));          // [RC] NNC ranges (has_nnc)
  double* nsv = (double*)(nrng + RC);                               // [NNCMAX][B*B] NNC blocks
  const double** nsa = (const double**)(nsv + NNCMAX * B * B);       // [NNCMAX] NNC row pointers
  __shared__ int nnc_cnt;
  __shared__ double ws[2][5][32];  // [buf][q][warp]: canonical warp sums of this CTA
  __shared__ double res_s[5];
#if RSIM_DSM_PUSH
  __shared__ double tab[2][5][64];            // [buf][q][chunk | warp] pushed by every CTA (st.async)
  __shared__ __align__(8) uint64_t mbar[2];   // one transaction barrier per tab buffer
#endif

  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int G = (int)cluster.num_blocks();
  const int tid = threadIdx.x;
  const int w = tid >> 5, lane = tid & 31;
  const int64_t nr = a.nA;
  const int nch = a.nch;
  const int LWPC = a.LRC - 5;  // log2(warps per CTA)
  const uint32_t ws_u32 = smem_u32(&ws[0][0][0]);
  const int LSH = a.LRC;  // log2(RC)
  const int RCM = RC - 1;
  const int64_t l = (int64_t)rank * RC + tid;
  const bool valid = l < nr;
  const int lam = tid;
  double* Vo = V + lam * ROWD;  // own row
  // generic pointer to local row j's vector block (own CTA or a peer's window)
  auto caddr = [&](int32_t j) -> const double* {
    const int g = j >> LSH;
    const double* base = g == rank ? V : cluster.map_shared_rank(V, g);
    return base + (size_t)(j & RCM) * ROWD;
  };
  int wbuf = 0;

  // Cluster-wide barrier after which every CTA's earlier shared-memory writes
  // are visible to DSMEM reads: __syncthreads drains this CTA's pending shared
  // stores, then a relaxed cluster barrier (no GPU-scope fence: nothing in the
  // solve loop writes global memory, and DSMEM reads are served by the owner
  // SM's shared memory, not a cache).  ~160 cycles against ~400 for
  // cluster.sync() with its MEMBAR.GPU (scripts/micro/xchg.cu).
  __shared__ unsigned long long tc[8];  // RSIM_KTRACE cycle accumulators (rank 0, thread 0)
  __shared__ unsigned long long tcr[8];  // per-CTA: [0,1] csync wait, [2,3] spmv, [4] reduce tail (warp 0 / last warp)
  // tracing is compiled in only with -DRSIM_DSM_TRACE (its registers cost the
  // 512-thread variant spills); RSIM_KTRACE=1 then enables it at run time
  const bool tr = kTrace && a.trace && rank == 0 && tid == 0;
  const int trw = (kTrace && a.trace && lane == 0) ? (w == 0 ? 1 : (w == (RC >> 5) - 1 ? 2 : 0)) : 0;
  if (kTrace && a.trace && tid < 8) tcr[tid] = 0;
  auto csync = [&]() {
    const long long tb = (kTrace && (tr || trw)) ? clock64() : 0;
    __syncthreads();
    if (G > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
    if (kTrace && tr) tc[6] += (unsigned long long)(clock64() - tb);
    if (kTrace && trw) tcr[trw - 1] += (unsigned long long)(clock64() - tb);
  };
#if RSIM_DSM_PUSH
  // Canonical reduction by PUSH: warp trees; with RC >= 256 (a CTA owns whole
  // 256-row chunks) warp 0 forms this CTA's chunk partials, otherwise every
  // warp ships its canonical warp sum; the values go with st.async straight
  // into every CTA's table, completing bytes on that CTA's transaction
  // mbarrier, so after its own wait a CTA reads everything from LOCAL shared
  // memory (no cluster barrier, no remote loads); warp q finishes quantity q,
  // one __syncthreads broadcasts.  Tables alternate; a CTA can run at most one
  // reduction ahead (its next contribution needs everyone's previous one).
  const bool chunk_mode = a.LRC >= 8;
  const int CPC = chunk_mode ? (1 << (a.LRC - 8)) : 0;  // chunks per CTA
  const int WPC = 1 << LWPC;
  const uint32_t tab_u32 = smem_u32(&tab[0][0][0]), bar_u32 = smem_u32(&mbar[0]);
  const uint32_t my_tab = mapa_u32(tab_u32, lane < G ? lane : 0);  // lane k talks to CTA k
  const uint32_t my_bar = mapa_u32(bar_u32, lane < G ? lane : 0);
  int kx = 0;
  auto reduce = [&](auto NQc, const double* val, double* out) {
    constexpr int NQ = decltype(NQc)::value;
    double v[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) v[q] = val[q];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
      for (int q = 0; q < NQ; ++q) v[q] = v[q] + __shfl_down_sync(0xffffffffu, v[q], off);
    const int X = kx & 1;
    const uint32_t par = (uint32_t)(kx >> 1) & 1u;
    ++kx;
    if (tid == 0) mb_arrive_expect_tx(bar_u32 + X * 8, chunk_mode ? (uint32_t)(nch * NQ * 8) : (uint32_t)(G * WPC * NQ * 8));
    if (chunk_mode) {
      if (lane == 0)
#pragma unroll
        for (int q = 0; q < NQ; ++q) ws[wbuf][q][w] = v[q];
      __syncthreads();
      if (w == 0)
        for (int pi = lane; pi < CPC * G; pi += 32) {
          const int j = pi / G, dst = pi - j * G;
          const int c = rank * CPC + j;
          if (c < nch) {
            const uint32_t rt = mapa_u32(tab_u32, dst), rb = mapa_u32(bar_u32, dst) + X * 8;
#pragma unroll
            for (int q = 0; q < NQ; ++q)
              st_async_f64(rt + (uint32_t)(((X * 5 + q) * 64 + c) * 8), tree8(&ws[wbuf][q][8 * j]), rb);
          }
        }
    } else {
      __syncwarp();
      double bq[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) bq[q] = __shfl_sync(0xffffffffu, v[q], 0);
      if (lane < G)
#pragma unroll
        for (int q = 0; q < NQ; ++q) st_async_f64(my_tab + (uint32_t)(((X * 5 + q) * 64 + rank * WPC + w) * 8), bq[q], my_bar + X * 8);
    }
    const long long tb = (kTrace && trw) ? clock64() : 0;
    mb_wait(bar_u32 + X * 8, par);
    if (kTrace && trw) tcr[trw - 1] += (unsigned long long)(clock64() - tb);
    for (int q = w; q < NQ; q += WPC) {  // warp q finishes quantity q from local shared memory
      double cp0 = 0.0, cp1 = 0.0;
      if (chunk_mode) {
        if (lane < nch) cp0 = tab[X][q][lane];
        if (lane + 32 < nch) cp1 = tab[X][q][lane + 32];
      } else if (lane < nch) {  // nch <= 8 here
        double w8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int gw = 8 * lane + k;
          w8[k] = (gw < G * WPC && ((int64_t)gw << 5) < nr) ? tab[X][q][gw] : 0.0;  // structural zero
        }
        cp0 = tree8(w8);
      }
      double r;
      if (nch == 1) {
        r = cp0;
      } else {
        // lanes >= n hold +0.0, so the shuffle tree of warp_tree_n is bit-identical
        double W[8] = {warp_tree_n(cp0, nch), nch > 32 ? warp_tree_n(cp1, nch - 32) : 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        r = tree8(W);
      }
      if (lane == 0) res_s[q] = r;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NQ; ++q) out[q] = res_s[q];
    wbuf ^= 1;
  };
#else
  // Canonical reduction of NQ per-row values (one per thread): warp trees into
  // shared memory, ONE cluster barrier, then warp q of every CTA gathers the 8
  // warp sums of each chunk via DSMEM and finishes the canonical tree (8-way
  // per chunk, then over the chunk partials); one __syncthreads broadcasts.
  auto reduce = [&](auto NQc, const double* val, double* out) {
    constexpr int NQ = decltype(NQc)::value;
    double v[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) v[q] = val[q];
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
      for (int q = 0; q < NQ; ++q) v[q] = v[q] + __shfl_down_sync(0xffffffffu, v[q], off);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < NQ; ++q) ws[wbuf][q][w] = v[q];
    csync();
    const long long t_tail = (kTrace && trw == 1) ? clock64() : 0;
    for (int q = w; q < NQ; q += (1 << LWPC)) {  // warp w finishes quantities w, w+WPC, ...
      double cp[2] = {0.0, 0.0};
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // lane c holds chunk c (and c + 32)
        const int c = lane + 32 * h;
        if (c < nch) {
          double w8[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {  // canonical warp 8c+k lives on CTA gw >> LWPC
            const int gw = (c << 3) | k;
            double x = 0.0;  // warp entirely past n_A: structural zero
            if (((int64_t)gw << 5) < nr) {
              const uint32_t ad = mapa_u32(ws_u32, gw >> LWPC) + (uint32_t)(((wbuf * 5 + q) * 32 + (gw & ((1 << LWPC) - 1))) * 8);
              asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(x) : "r"(ad) : "memory");
            }
            w8[k] = x;
          }
          cp[h] = tree8(w8);
        }
      }
      if (nch == 1) {
        if (lane == 0) res_s[q] = cp[0];
      } else {
        double W[8] = {warp_tree_n(cp[0], nch), warp_tree_n(cp[1], nch - 32), 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        if (lane == 0) res_s[q] = tree8(W);
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NQ; ++q) out[q] = res_s[q];
    if (kTrace && trw == 1) tcr[4] += (unsigned long long)(clock64() - t_tail);
    wbuf ^= 1;
  };
#endif
  auto xbar = [&]() { csync(); };

  // neighbour rows: cluster address per Cartesian slot (bit s of nmask = present)
  const double* na[NS];
  uint32_t nmask = 0;
#pragma unroll
  for (int s = 0; s < NS; ++s) na[s] = nullptr;

  // neighbour value of the vector being multiplied, recomputed at the gather site:
  //   mode 0: p_new_j = (s_j - omega t_j) + beta (p_old_j - omega v_old_j)   (it > 1)
  //   mode 1: p_new_j = r_j                                     (it == 1)
  //   mode 2: s_j     = r_j - alpha v_new_j
  //   mode 3: (M^-1 p)_j, mode 4: (M^-1 s)_j   (stored by the owner, Neumann-1)
  auto gather = [&](auto MODEc, const double* ad, int offo, double beta, double omega, double alpha, double* out) {
    constexpr int MODE = decltype(MODEc)::value;
    if constexpr (MODE == 3) {
      ldg_row<B>(ad + O_PH * BP, out);
    } else if constexpr (MODE == 4) {
      ldg_row<B>(ad + O_SH * BP, out);
    } else if constexpr (MODE == 1) {
      ldg_row<B>(ad + O_R * BP, out);
    } else if constexpr (MODE == 0) {  // r_j = s_j − ω t_j (previous iterate); offo: old p (v 2 vectors later)
      double S_[B], T_[B], P_[B], V_[B];
      ldg_row<B>(ad + O_S * BP, S_);
      ldg_row<B>(ad + O_T * BP, T_);
      ldg_row<B>(ad + offo, P_);
      ldg_row<B>(ad + offo + 2 * BP, V_);
#pragma unroll
      for (int e = 0; e < B; ++e) {
        const double rj = S_[e] - omega * T_[e];
        out[e] = rj + beta * (P_[e] - omega * V_[e]);
      }
    } else {  // offo: the current v
      double R_[B], V_[B];
      ldg_row<B>(ad + O_R * BP, R_);
      ldg_row<B>(ad + offo, V_);
#pragma unroll
      for (int e = 0; e < B; ++e) out[e] = R_[e] - alpha * V_[e];
    }
  };

  // y = xown + Σ_slots Â_s x_col (+ NNC), canonical order
  auto spmv = [&](auto MODEc, int offo, const double* xown, double beta, double omega, double alpha, double* y) {
    const long long t_sp = (kTrace && trw) ? clock64() : 0;
    // slots in groups of SG (all in flight within a group); the 512/1024-thread
    // variants (128/64 registers) use SG = 2 so the gathered rows do not spill.
    // The accumulation order (slots ascending) is unchanged.
    constexpr int SG = MAXT <= 256 ? NS : RSIM_DSM_SG512;
    double acc[B];
#pragma unroll
    for (int e = 0; e < B; ++e) acc[e] = xown[e];
#pragma unroll
    for (int s0 = 0; s0 < NS; s0 += SG) {
      double xv[SG][B];
#pragma unroll
      for (int k = 0; k < SG; ++k)
        if (s0 + k < NS && (nmask & (1u << (s0 + k)))) gather(MODEc, na[s0 + k], offo, beta, omega, alpha, xv[k]);
#pragma unroll
      for (int k = 0; k < SG; ++k) {
        const int s = s0 + k;
        if (s < NS && (nmask & (1u << s))) {
          if (MS) {
            rsim::blk::gemv_acc_flat<B>(&mval[((size_t)s * RC + lam) * B * B], xv[k], acc);
          } else if (ell_es(B * B) == 1) {
            rsim::blk::gemv_acc_flat<B>(&a.ell_val[ell_at(a.cap, B * B, s, 0, l)], xv[k], acc);
          } else {
            double M[B * B];
            ell_load<B>(a.ell_val, a.cap, s, l, M);
            rsim::blk::gemv_acc_flat<B>(M, xv[k], acc);
          }
        }
      }
      if (SG < NS) asm volatile("" ::: "memory");  // keep the next group's loads after this group's math
    }
    if (a.has_nnc) {
      const int2 rg = nrng[lam];
      if (rg.y & NNC_GLOBAL) {
        for (int32_t q = rg.x; q < (rg.y & ~NNC_GLOBAL); ++q) {
          const int32_t c2 = a.nnc_lcol[q];
          if (c2 >= 0) {
            double xn[B];
            gather(MODEc, caddr(c2), offo, beta, omega, alpha, xn);
            rsim::blk::gemv_acc_flat<B>(&a.nnc_val[(int64_t)q * B * B], xn, acc);
          }
        }
      } else {
        for (int32_t q = rg.x; q < rg.y; ++q) {
          double xn[B];
          gather(MODEc, nsa[q], offo, beta, omega, alpha, xn);
          rsim::blk::gemv_acc_flat<B>(&nsv[q * B * B], xn, acc);
        }
      }
    }
#pragma unroll
    for (int e = 0; e < B; ++e) y[e] = acc[e];
    if (kTrace && trw) tcr[1 + trw] += (unsigned long long)(clock64() - t_sp);
  };

  // own-row r0 and x live in shared memory (register pressure of the 512-thread variant)
  double* r0r = Vo + O_R0 * BP;
  double* xr = Vo + O_X * BP;
  double sr[B], tr_[B];
  double res[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int e = 0; e < B; ++e) { sr[e] = 0.0; tr_[e] = 0.0; }
  // ---- load: matrix rows (MS), neighbour addresses, rhs -> r, r0; x = 0; (b,b), (F,F)
  if (tid == 0) nnc_cnt = 0;
#if RSIM_DSM_PUSH
  if (tid == 0) {
    mb_init(bar_u32, 1);
    mb_init(bar_u32 + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster.sync();  // every CTA's barriers initialised before the first st.async
#else
  __syncthreads();
#endif
  {
    double val[3] = {0.0, 0.0, 0.0};
    if (valid) {
      double bv[B], fv[B];
#pragma unroll
      for (int e = 0; e < B; ++e) {
        bv[e] = a.rhs[l * B + e];
        fv[e] = a.F_raw[l * B + e];
        Vo[O_R * BP + e] = bv[e];
        r0r[e] = bv[e];
        xr[e] = 0.0;
        Vo[O_P * BP + e] = 0.0; Vo[(O_P + 1) * BP + e] = 0.0;
        Vo[O_V * BP + e] = 0.0; Vo[(O_V + 1) * BP + e] = 0.0;
      }
      val[0] = rsim::blk::rowdot<B>(bv, bv);
      val[1] = rsim::blk::rowdot<B>(fv, fv);
      if (a.has_nnc) {  // cache this row's active NNC blocks in smem (order preserved)
        const int64_t i = a.act[l];
        const int32_t q0 = a.nptr[i], q1 = a.nptr[i + 1];
        int k = 0;
        for (int32_t q = q0; q < q1; ++q) k += a.nnc_lcol[q] >= 0;
        const int base = k ? atomicAdd(&nnc_cnt, k) : 0;
        if (base + k <= NNCMAX) {
          int m = base;
          for (int32_t q = q0; q < q1; ++q) {
            const int32_t c2 = a.nnc_lcol[q];
            if (c2 < 0) continue;
            nsa[m] = caddr(c2);
#pragma unroll
            for (int e = 0; e < B * B; ++e) nsv[m * B * B + e] = a.nnc_val[(int64_t)q * B * B + e];
            ++m;
          }
          nrng[lam] = make_int2(base, base + k);
        } else {
          nrng[lam] = make_int2(q0, q1 | NNC_GLOBAL);
        }
      }
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const int32_t cl = a.ell_col[s * a.cap + l];
        if (cl >= 0) {
          nmask |= 1u << s;
          na[s] = caddr(cl);
          if (kTrace && a.trace && (cl >> LSH) != rank) atomicAdd(&tcr[5], 1ull);
          if (MS)
#pragma unroll
            for (int e = 0; e < B * B; ++e)
              mval[((size_t)s * RC + lam) * B * B + e] = a.ell_val[ell_at(a.cap, B * B, s, e, l)];
        }
      }
    }
    reduce(std::integral_constant<int, 2>{}, val, res);
  }
  const double bb = res[0];
  if (rank == 0 && tid == 0) a.dsc->f2 = sqrt(res[1]);
  const double bnorm = sqrt(bb);
  const bool fixed = a.fixed > 0;
  const int maxit = fixed ? a.fixed : a.maxit;
  const double tol = a.rtol * bnorm;
  double rho = 1.0, alpha = 1.0, omega = 1.0, rho_new = bb;
  int status = RSIM_OK;
  int it = 0;
  double relres = 0.0;
  int cur = 0;  // buffer holding the current iteration's p, v
  if (bnorm != 0.0) {
    status = RSIM_ENOCONV;
    if (tr)
      for (int k = 0; k < 8; ++k) tc[k] = 0;
    long long t0 = kTrace ? clock64() : 0;
#define KT_MARK(k) do { if (tr) { long long t1 = clock64(); tc[k] += (unsigned long long)(t1 - t0); t0 = t1; } } while (0)
    int it_total = 0;
    // attempt 0: as configured; attempt 1 (only after a Neumann-1 breakdown or
    // cap): block-Jacobi only, restarted from x0 = 0 (same rule as the oracle)
    for (int attempt = 0; attempt < (a.neu ? 2 : 1); ++attempt) {
    const bool neu = a.neu && attempt == 0;
    if (attempt) {
      if (valid)
#pragma unroll
        for (int e = 0; e < B; ++e) {
          Vo[O_R * BP + e] = a.rhs[l * B + e];
          xr[e] = 0.0;
        }
      rho = 1.0; alpha = 1.0; omega = 1.0; rho_new = bb;
      cur = 0;
      status = RSIM_ENOCONV;
      xbar();
    }
    for (it = 1; it <= maxit; ++it) {
      KT_MARK(7);
      const double beta = (it == 1) ? 0.0 : (rho_new / rho) * (alpha / omega);
      double* Pc = Vo + (O_P + cur) * BP;          // own p (this iteration)
      double* Vc = Vo + (O_V + cur) * BP;          // own v (this iteration)
      const double* Po = Vo + (O_P + (cur ^ 1)) * BP;
      const double* Vold = Vo + (O_V + (cur ^ 1)) * BP;
      const int off_po = (O_P + (cur ^ 1)) * BP;  // neighbours' old p
      const int off_vc = (O_V + cur) * BP;        // neighbours' current v
      // ---- p = r + β (p − ω v) (own; neighbours recompute r = s − ω t and p)
      //      BJ:  v = Â p;   Neumann-1: ph = p + (p − Â p), barrier, v = Â ph
      //      reduce (r0, v) and the lagged (r, r) of the previous iterate
      double phr[B];
      {
        double val[2] = {0.0, 0.0};
        double pown[B], y[B], rown[B];
        if (valid) {
#pragma unroll
          for (int e = 0; e < B; ++e) {
            rown[e] = Vo[O_R * BP + e];
            pown[e] = (it == 1) ? rown[e] : rown[e] + beta * (Po[e] - omega * Vold[e]);
            Pc[e] = pown[e];
          }
          if (it == 1) spmv(std::integral_constant<int, 1>{}, 0, pown, beta, omega, 0.0, y);
          else spmv(std::integral_constant<int, 0>{}, off_po, pown, beta, omega, 0.0, y);
        }
        if (neu) {
          if (valid)
#pragma unroll
            for (int e = 0; e < B; ++e) {
              phr[e] = pown[e] + (pown[e] - y[e]);
              Vo[O_PH * BP + e] = phr[e];
            }
          xbar();
          if (valid) spmv(std::integral_constant<int, 3>{}, 0, phr, 0.0, 0.0, 0.0, y);
        } else {
#pragma unroll
          for (int e = 0; e < B; ++e) phr[e] = pown[e];
        }
        if (valid) {
#pragma unroll
          for (int e = 0; e < B; ++e) Vc[e] = y[e];
          val[0] = rsim::blk::rowdot<B>(r0r, y);
          val[1] = rsim::blk::rowdot<B>(rown, rown);
        }
        KT_MARK(0);
        reduce(std::integral_constant<int, 2>{}, val, res);
        KT_MARK(1);
      }
      if (it > 1 && !fixed && sqrt(res[1]) <= tol) {  // previous iterate converged
        relres = sqrt(res[1]) / bnorm;
        status = RSIM_OK;
        --it;
        break;
      }
      const double r0v = res[0];
      if (r0v == 0.0 || !isfinite(r0v)) { status = RSIM_ENUM; break; }
      alpha = rho_new / r0v;
      // ---- s = r − α v (own + recomputed for neighbours; stored for the next r recompute)
      //      BJ: t = Â s;  Neumann-1: sh = s + (s − Â s), barrier, t = Â sh
      //      reduce (s,s), (t,s), (t,t), (r0,s), (r0,t)
      double shr[B];
      {
        double val[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        double y[B];
        if (valid) {
#pragma unroll
          for (int e = 0; e < B; ++e) {
            sr[e] = Vo[O_R * BP + e] - alpha * Vc[e];
            Vo[O_S * BP + e] = sr[e];
          }
          spmv(std::integral_constant<int, 2>{}, off_vc, sr, 0.0, 0.0, alpha, y);
        }
        if (neu) {
          if (valid)
#pragma unroll
            for (int e = 0; e < B; ++e) {
              shr[e] = sr[e] + (sr[e] - y[e]);
              Vo[O_SH * BP + e] = shr[e];
            }
          xbar();
          if (valid) spmv(std::integral_constant<int, 4>{}, 0, shr, 0.0, 0.0, 0.0, y);
        } else {
#pragma unroll
          for (int e = 0; e < B; ++e) shr[e] = sr[e];
        }
        if (valid) {
#pragma unroll
          for (int e = 0; e < B; ++e) {
            tr_[e] = y[e];
            Vo[O_T * BP + e] = y[e];
          }
          val[0] = rsim::blk::rowdot<B>(sr, sr);
          val[1] = rsim::blk::rowdot<B>(y, sr);
          val[2] = rsim::blk::rowdot<B>(y, y);
          val[3] = rsim::blk::rowdot<B>(r0r, sr);
          val[4] = rsim::blk::rowdot<B>(r0r, y);
        }
        KT_MARK(2);
        reduce(std::integral_constant<int, 5>{}, val, res);
        KT_MARK(3);
      }
      const double ssn = res[0], ts = res[1], tt = res[2], r0s = res[3], r0t = res[4];
      if (!fixed && sqrt(ssn) <= tol) {
        if (valid)
#pragma unroll
          for (int e = 0; e < B; ++e) xr[e] = xr[e] + alpha * phr[e];
        relres = sqrt(ssn) / bnorm;
        status = RSIM_OK;
        break;
      }
      if (tt == 0.0 || !isfinite(tt)) { status = RSIM_ENUM; break; }
      omega = ts / tt;
      // ---- x, r update (own rows; neighbours recompute r from s, t)
      if (valid)
#pragma unroll
        for (int e = 0; e < B; ++e) {
          xr[e] = (xr[e] + alpha * phr[e]) + omega * shr[e];
          Vo[O_R * BP + e] = sr[e] - omega * tr_[e];
        }
      KT_MARK(4);
      rho = rho_new;
      rho_new = r0s - omega * r0t;
      if (omega == 0.0 || rho_new == 0.0 || !isfinite(rho_new)) { status = RSIM_ENUM; break; }
      cur ^= 1;
    }
    if (it > maxit) {  // iteration cap: residual of the last iterate (one more reduction)
      it = maxit;
      double val[1] = {0.0};
      if (valid) {
        double rv[B];
#pragma unroll
        for (int e = 0; e < B; ++e) rv[e] = Vo[O_R * BP + e];
        val[0] = rsim::blk::rowdot<B>(rv, rv);
      }
      reduce(std::integral_constant<int, 1>{}, val, res);
      relres = sqrt(res[0]) / bnorm;
      status = (fixed || sqrt(res[0]) <= tol) ? RSIM_OK : RSIM_ENOCONV;
    }
    it_total += it;
    if (!(neu && (status == RSIM_ENUM || status == RSIM_ENOCONV))) break;
    }
    it = it_total;
    if (tr)
      for (int k = 0; k < 8; ++k) atomicAdd(&a.trace[k], tc[k]);
#undef KT_MARK
  }
  if (valid)
#pragma unroll
    for (int e = 0; e < B; ++e) a.x[l * B + e] = xr[e];
  if (a.upd) {  // K6 in the epilogue (same operations as k_update): u += δu, substitution, flags, ‖δp‖∞
    double aA = 0.0, aB = 0.0;
    bool bad = false;
    if (valid) {
      const int64_t i = a.act[l];
      double ui[B];
#pragma unroll
      for (int c = 0; c < B; ++c) ui[c] = a.u[i * B + c];
      uint8_t stv = a.st[i];
      const double d = rsim::phys::apply_update<B>(a.fl, ui, stv, xr);
#pragma unroll
      for (int c = 0; c < B; ++c) a.u[i * B + c] = ui[c];
      a.st[i] = stv;
      const double ad = fabs(d);
      bad = !isfinite(d);
      a.dp[i] = d;
      a.last_dp[i] = ad;
      uint8_t f = a.flags[i];
      if (ad >= a.eps) {
        f |= F_FLAG;
        if (f & F_B) f |= F_D0;
      }
      a.flags[i] = f;
      aA = ad;
      aB = (f & F_B) ? ad : 0.0;
    }
    if (bad) a.dsc->status = RSIM_ENUM;
    const double wa = warp_max(aA), wb = warp_max(aB);
    if (lane == 0) {
      if (wa > 0.0) atomic_max_bits(&a.dsc->maxA, wa);
      if (wb > 0.0) atomic_max_bits(&a.dsc->maxB, wb);
    }
  }
  if (kTrace && a.trace) {
    if (valid) atomicAdd(&tcr[6], 1ull);
    __syncthreads();
    if (tid < 8) atomicAdd(&a.trace[8 + rank * 8 + tid], tcr[tid]);
  }
  if (rank == 0 && tid == 0) {
    a.dsc->lin_iters = it;
    a.dsc->lin_relres = relres;
    if (status != RSIM_OK) a.dsc->status = status;
  }
  cluster.sync();  // keep every CTA's shared memory alive until all remote reads are done
}

size_t smem_bytes(int B, int NS, bool MS, int LRC) {
  const size_t R = (size_t)1 << LRC;
  const size_t BP = (B == 3) ? 4 : B;
  size_t b = 11 * R * BP * sizeof(double) + R * sizeof(int2) + NNCMAX * (B * B * sizeof(double) + sizeof(const double*));
  if (MS) b += NS * R * B * B * sizeof(double);
  return b;
}

template <int B, int NS, bool MS, int MAXT>
int launch_t(rsim_gpu_ctx* c, const DArgs& a, int G, int TPB, size_t smem, bool* ok) {
  static std::map<std::tuple<int, int, size_t>, bool> fits;
  auto key = std::make_tuple(G, TPB, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G, 1, 1);
  cfg.blockDim = dim3(TPB, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // the dynamic-smem attribute is a per-kernel maximum: only ever raise it
  static size_t attr_max = 0;
  auto ensure_attr = [&](size_t need) -> cudaError_t {
    if (need <= attr_max) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k_krylov_dsm<B, NS, MS, MAXT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)need);
    if (e == cudaSuccess) attr_max = need;
    return e;
  };
  auto itf = fits.find(key);
  if (itf == fits.end()) {
    bool f = ensure_attr(smem) == cudaSuccess;
    cudaFuncSetAttribute(k_krylov_dsm<B, NS, MS, MAXT>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int ncl = 0;
    f = f && cudaOccupancyMaxActiveClusters(&ncl, k_krylov_dsm<B, NS, MS, MAXT>, &cfg) == cudaSuccess && ncl >= 1;
    cudaGetLastError();
    itf = fits.emplace(key, f).first;
  }
  *ok = itf->second;
  if (!*ok) return RSIM_OK;
  RSIM_CUDA(ensure_attr(smem));
  RSIM_CUDA(cudaLaunchKernelEx(&cfg, k_krylov_dsm<B, NS, MS, MAXT>, a));
  return RSIM_OK;
}

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return (e && *e) ? std::atoi(e) : dflt;
}

template <int B, int NS>
int launch_bn(rsim_gpu_ctx* c, DArgs& a, int G, int TPB, bool* ok) {
  static const int tmin = env_int("RSIM_DSM_MINT", 0);  // experiments: smallest MAXT variant to use
  const int sel = TPB < tmin ? tmin : TPB;  // template variant (blockDim stays TPB)
  const size_t with_m = smem_bytes(B, NS, true, a.LRC), without = smem_bytes(B, NS, false, a.LRC);
  const size_t cap = 220 * 1024;
  if (with_m <= cap) {
    int r = sel <= 256   ? launch_t<B, NS, true, 256>(c, a, G, TPB, with_m, ok)
            : sel <= 512 ? launch_t<B, NS, true, 512>(c, a, G, TPB, with_m, ok)
                         : launch_t<B, NS, true, 1024>(c, a, G, TPB, with_m, ok);
    if (r != RSIM_OK || *ok) return r;
  }
  if (without <= cap)
    return sel <= 256   ? launch_t<B, NS, false, 256>(c, a, G, TPB, without, ok)
           : sel <= 512 ? launch_t<B, NS, false, 512>(c, a, G, TPB, without, ok)
                        : launch_t<B, NS, false, 1024>(c, a, G, TPB, without, ok);
  *ok = false;
  return RSIM_OK;
}

int dsm_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("RSIM_NO_CLUSTER");
    v = (e && *e == '1') ? 1 : 0;
  }
  return v;
}

}  // namespace

int launch_krylov_dsm(rsim_gpu_ctx* c, const rsim_solver_opts* o) {
  if (dsm_disabled() || c->nA <= 0 || c->cols_implicit || (c->f2_parts && !c->keep_F)) return RSIM_ENOTAPPLICABLE;
  const int nch = (c->nA + RSIM_RED_CHUNK - 1) / RSIM_RED_CHUNK;
  if (nch > 4 * GMAX) return RSIM_ENOTAPPLICABLE;
  DArgs a;
  a.nA = c->nA;
  a.nslot = c->nslot;
  a.maxit = o->lin_maxit;
  a.fixed = o->fixed_lin_iters;
  a.neu = o->precond == RSIM_PREC_NEUMANN1;
  a.nch = nch;
  a.cap = c->ell_cap;
  a.has_nnc = c->has_nnc;
  a.rtol = o->lin_rtol;
  a.ell_col = c->ell_col;
  a.ell_val = c->ell_val;
  a.act = c->act;
  a.nptr = c->nptr;
  a.nnc_lcol = c->nnc_lcol;
  a.nnc_val = c->nnc_val;
  a.rhs = c->rhs;
  a.F_raw = c->F_raw;
  a.x = c->x;
  a.trace = c->ktrace;
  a.upd = c->fuse_update ? 1 : 0;
  a.eps = c->fuse_eps;
  a.fl = rsim::phys::Fluid(c->fl);
  a.u = c->u; a.dp = c->dp; a.last_dp = c->last_dp; a.st = c->st; a.flags = c->flags;
  a.dsc = c->dsc;
  // one chunk per CTA when possible (G = nch <= 16), else 2 or 4 chunks per CTA
  // (powers of two, so the owner of a row is a shift)
  // rows per CTA: the smallest power of two >= 64 that fits the system in
  // <= 16 CTAs (more CTAs = shorter per-CTA critical path)
  static int minl = -1;
  if (minl < 0) {
    const char* e = std::getenv("RSIM_DSM_MINLRC");
    minl = e ? std::atoi(e) : 6;
  }
  for (int LRC = minl; LRC <= 10; ++LRC) {
    const int RC = 1 << LRC;
    const int G = (c->nA + RC - 1) / RC;
    if (G > GMAX) continue;
    a.LRC = LRC;
    const int TPB = RC;
    bool ok = false;
    int r;
    switch (c->b * 10 + c->nslot) {
      case 14: r = launch_bn<1, 4>(c, a, G, TPB, &ok); break;
      case 16: r = launch_bn<1, 6>(c, a, G, TPB, &ok); break;
      case 24: r = launch_bn<2, 4>(c, a, G, TPB, &ok); break;
      case 26: r = launch_bn<2, 6>(c, a, G, TPB, &ok); break;
      case 34: r = launch_bn<3, 4>(c, a, G, TPB, &ok); break;
      default: r = launch_bn<3, 6>(c, a, G, TPB, &ok); break;
    }
    if (r != RSIM_OK) return r;
    if (ok) {
      c->launches++;
      c->update_applied = c->fuse_update;
      RSIM_CUDA(cudaGetLastError());
      return RSIM_OK;
    }
  }
  return RSIM_ENOTAPPLICABLE;
}
