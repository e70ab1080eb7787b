// krylov.cu — K3 (SpMV) + K5 (fused vector updates / dot products) inside ONE
// persistent cooperative BiCGSTAB kernel per linear solve (large systems).
//
// Replaces solve(J, F) with the north star's BiCGSTAB on
// the block-Jacobi-scaled system Â = D^{-1}J (unit block diagonal, never
// stored; block-Jacobi preconditioning is therefore built in).
//
// The whole iteration loop runs on the device.  A CTA of 1024 threads owns 4
// consecutive 256-row canonical chunks per round (one row per thread), so a
// chunk partial is 8 warp shuffles + an 8-way tree inside the CTA; phases are
// separated by grid-wide barriers and every CTA reduces the chunk partials
// with the same canonical tree (blockops.h) — all CTAs take identical
// branches and the results are bit-identical to oracle/oracle.cpp.
// Small systems (<= 64 chunks) go to krylov_dsm.cu (one cluster, DSMEM).
//
// Per iteration 3 grid barriers: the p- and s-updates of neighbours are
// recomputed at the gather site (p, v double-buffered), (s,s) is reduced
// together with (t,s), (t,t).
// Element formulas (identical in oracle/oracle.cpp bicgstab()):
//   p = r + β (p − ω v);  s = r − α v;  x = (x + α p) + ω s;  r = s − ω t.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "ctx.cuh"
#include "ilu.cuh"

namespace cg = cooperative_groups;

namespace {

// Threads per CTA per block size (template parameter of the kernel; one CTA
// per SM, so KT fixes the register cap: 1024 -> 64, 512 -> 128).  Measured on
// the config-3 / config-4 first Newton systems (100 Neumann-1 iterations,
// scripts/krylov_c4.py): b = 2 66.2 -> 44.9 µs per iteration with 512 threads
// and one slot per gather group, b = 3 551 -> 454 µs with 512 threads (no spills)
// (768 threads: 440 µs on that system but 10.19 vs 9.63 s for the whole config-4
// run, whose smaller systems lose more to round imbalance; 768 for b = 2: 58.6 µs;
// b = 3 with 1024 threads: 461 µs and ~0.8 KB of local traffic per row-phase
// left, 256 threads for b = 2: 64-68 µs); b = 1 (config 5 at 1-100 %) keeps
// 1024 threads and all six slots in flight.
#ifndef RSIM_KT1
#define RSIM_KT1 1024
#endif
#ifndef RSIM_KT2
#define RSIM_KT2 512
#endif
#ifndef RSIM_KT3
#define RSIM_KT3 512
#endif
__host__ __device__ constexpr int kt_for(int B) { return B == 1 ? RSIM_KT1 : (B == 2 ? RSIM_KT2 : RSIM_KT3); }
#ifndef RSIM_SPMV_SG1
#define RSIM_SPMV_SG1 6
#endif
#ifndef RSIM_SPMV_SG2
#define RSIM_SPMV_SG2 1
#endif
#ifndef RSIM_SPMV_SG3
#define RSIM_SPMV_SG3 1
#endif
// Recompute fusion (neighbours' p and s formed at the gather sites, two grid barriers and the
// p / s store passes less per iteration) up to this many rows.  b = 1: 2^20 (config 5: above it the
// extra gather traffic costs more than the barriers).  b >= 2: always — the per-row matrix work
// dominates and the fused kernel wins at every size measured in round 2: config 3 standard Newton
// (2.1 M rows, b = 2) 3.38 -> 2.66 s per 2 steps, config 4 standard Newton (4.2 M rows, b = 3)
// 12.75 -> 11.90 s, config 4 adaptive DD (subdomain systems > 2^20 rows) 13.54 -> 12.97 s per run;
// below 2^20 rows the unfused kernel is 10-18 % slower on the config-4 localized run.
__host__ __device__ constexpr int64_t fuse_max_rows(int B) { return B == 1 ? ((int64_t)1 << 20) : ((int64_t)1 << 40); }

struct KArgs {
  int32_t nA, nslot, maxit, fixed;
  int32_t nx, ny, nz;
  bool d3, implicit;  // implicit: full set, structural ELL columns (not stored)
  int32_t stage;      // rounds staged per block-level commit (1..RSTAGE)
  int64_t cap;
  bool has_nnc;
  double rtol;
  const int32_t* ell_col;
  const double* ell_val;
  const uint8_t* ell_po;
  const int32_t* act;
  const int32_t* nptr;
  const int32_t* nnc_lcol;
  const double* nnc_val;
  const double* rhs;
  const double* F_raw;
  const double* part_f2;  // (F,F) chunk partials of the assembly (f2_parts)
  bool f2_parts;
  double *x, *r, *r0, *p, *v, *s, *t, *p2, *v2, *ph, *sh;
  int32_t neu, fuse, ilu;  // neu: Neumann-1; ilu: level-scheduled ILU(0) (never fused)
  int32_t fuse_s;          // unfused, block-Jacobi: s recomputed at the t-SpMV gather sites (no s pass)
  IluArgs fa;
  double* part;   // [5][pstride]  level-1 partials
  double* part2;  // [5][pstride2] level-2 partials (very large systems)
  int32_t pstride, pstride2;
  int32_t red_small_max;  // chunk partials reduced redundantly by every CTA up to this count
  int32_t stream;         // b = 1: matrix values through streaming (evict-first) loads
  int32_t kblk;           // consecutive rounds per CTA (blocked-cyclic distribution; 1 = round-robin)
  int32_t alt;            // sweep direction alternates between phases (L2 reuse of the previous sweep's tail)
  DevScalars* dsc;
};

#ifndef RSIM_RSTAGE
#define RSIM_RSTAGE 8
#endif
constexpr int RSTAGE = RSIM_RSTAGE;  // rounds whose warp sums are staged before one block-level commit
struct Red {
  double ws[5][32];  // warp sums of the current round (level-2 / small reductions)
  double lvl[5][64];
  double res[5];
  double wsr[RSTAGE][5][32];  // staged warp sums of up to RSTAGE rounds
  int64_t rid[RSTAGE];        // their round ids
};

// Stage the warp sums of one round (no block barrier); every RSTAGE rounds,
// and after the CTA's last round, one barrier pair turns them into level-1
// chunk partials (8-way trees, canonical).  Warps thus run ahead through up
// to RSTAGE rounds of loads instead of meeting at two barriers per round.
template <int CPR, int NQ>
__device__ __forceinline__ void stage_round(Red& R, const double* val, int slot, int64_t rd, bool flush,
                                            int nstaged, int64_t nch, double* part, int pstride) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef RSIM_DBG_NORED  // timing experiment only (wrong numerics): no warp trees
  if (lane == 0) for (int q = 0; q < NQ; ++q) R.wsr[slot][q][w] = val[q];
#else
  // the NQ warp trees level by level (each quantity: v + shfl_down(v, 16), 8, 4, 2, 1 as in
  // warp_tree, so the same bits): 5 dependent shuffle steps instead of 5·NQ
  double v[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) v[q] = val[q];
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1)
#pragma unroll
    for (int q = 0; q < NQ; ++q) v[q] = v[q] + __shfl_down_sync(0xffffffffu, v[q], off);
  if (lane == 0)
#pragma unroll
    for (int q = 0; q < NQ; ++q) R.wsr[slot][q][w] = v[q];
#endif
  if (threadIdx.x == 0) R.rid[slot] = rd;
  if (!flush) return;
  __syncthreads();
  for (int k = threadIdx.x; k < nstaged * CPR * NQ; k += blockDim.x) {
    const int sl = k / (CPR * NQ), rem = k - sl * CPR * NQ, q = rem / CPR, g = rem % CPR;
    const int64_t c = R.rid[sl] * CPR + g;
    if (c < nch) part[q * pstride + c] = tree8(&R.wsr[sl][q][8 * g]);
  }
  __syncthreads();
}

// Per-round commit: warp trees of up to 3 quantities -> 8-way trees -> level-1
// partials of the 4 chunks of this round.
template <int CPR>
__device__ __forceinline__ void commit_round(Red& R, int NQ, const double* val, int64_t chunk0, int64_t nch,
                                             double* part, int pstride) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int q = 0; q < NQ; ++q) {
    double v = warp_tree(val[q]);
    if (lane == 0) R.ws[q][w] = v;
  }
  __syncthreads();
  if ((int)threadIdx.x < CPR * NQ) {
    const int g = threadIdx.x % CPR, q = threadIdx.x / CPR;
    if (chunk0 + g < nch) part[q * pstride + chunk0 + g] = tree8(&R.ws[q][8 * g]);
  }
  __syncthreads();
}

// Canonical reduction of P partials (P <= 64*256) held in global memory, done
// by ONE CTA (all 1024 threads call it), for NQ quantities at once: one pass
// over the partials per 4 chunks for all of them (NQ-fold fewer dependent
// load + barrier steps).  src(q) gives quantity q's partials; results in
// R.res[q].  Per quantity: warp trees + 8-way trees over chunks of 256
// partials, then the same over the chunk results (blockops.h canonical tree).
template <int CPR, class SF>
__device__ __forceinline__ void reduce_small_multi(Red& R, int NQ, SF&& src, int P) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (P == 1) {
    if ((int)threadIdx.x < NQ) R.res[threadIdx.x] = src(threadIdx.x)[0];
    __syncthreads();
    return;
  }
  const int P2 = (P + 255) / 256;
  for (int c0 = 0; c0 < P2; c0 += CPR) {
    const int idx = c0 * 256 + threadIdx.x;
    double v[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) v[q] = (q < NQ && idx < P) ? src(q)[idx] : 0.0;  // all loads in flight
#pragma unroll
    for (int q = 0; q < 5; ++q)
      if (q < NQ) {
        const double t = warp_tree(v[q]);
        if (lane == 0) R.ws[q][w] = t;
      }
    __syncthreads();
    if ((int)threadIdx.x < CPR * NQ) {
      const int g = threadIdx.x % CPR, q = threadIdx.x / CPR;
      if (c0 + g < P2) R.lvl[q][c0 + g] = tree8(&R.ws[q][8 * g]);
    }
    __syncthreads();
  }
  if (P2 == 1) {
    if ((int)threadIdx.x < NQ) R.res[threadIdx.x] = R.lvl[threadIdx.x][0];
  } else {
#pragma unroll
    for (int q = 0; q < 5; ++q)
      if (q < NQ) {
        const double t = warp_tree(threadIdx.x < (unsigned)P2 ? R.lvl[q][threadIdx.x] : 0.0);
        if (lane == 0 && w < 8) R.ws[q][w] = t;
      }
    __syncthreads();
    if ((int)threadIdx.x < NQ) R.res[threadIdx.x] = tree8(&R.ws[threadIdx.x][0]);
  }
  __syncthreads();
}

// Vectors a gather may read (read-only in the current phase).
struct Vecs {
  const double *r, *po, *vo, *s, *t;
};

// Neighbour value of the vector being multiplied, recomputed from vectors
// that are read-only in the current phase (same formula as the owner, so the
// same bits):  mode 0: p_j = (s_j − ω t_j) + β (p_old_j − ω v_old_j), the
// previous iterate's r recomputed from its s, t;  mode 1: p_j = r_j;
// mode 2: s_j = r_j − α v_j (vo = current v);  mode 3: x_j read directly from `po`.
template <int B>
__device__ __forceinline__ void nbr_val(int mode, const Vecs& X, int64_t j, double beta, double omega, double alpha,
                                        double* out) {
#pragma unroll
  for (int e = 0; e < B; ++e) {
    const int64_t q = j * B + e;
    if (mode == 3) out[e] = X.po[q];
    else if (mode == 1) out[e] = X.r[q];
    else if (mode == 0) out[e] = (X.s[q] - omega * X.t[q]) + beta * (X.po[q] - omega * X.vo[q]);
    else out[e] = X.r[q] - alpha * X.vo[q];
  }
}

// b = 1: matrix row (columns + values) loaded one round ahead.  In the passes that end
// with a reduction a warp otherwise runs load -> wait -> math -> 5-step shuffle trees ->
// next round's loads, i.e. nothing in flight during the trees (measured on config 5 at
// 100 %: the trees cost 16 % of the v pass, 14 % of the t pass).  The next round's row is
// requested BEFORE the trees; its columns are then known when the round starts, so the
// gathers no longer wait for a column load either.
#ifndef RSIM_PRE1
#define RSIM_PRE1 1
#endif
#ifndef RSIM_LDCS  // experiment: matrix values through streaming (evict-first) loads so the vectors keep L2
#define RSIM_LDCS 0
#endif
#ifndef RSIM_EARLY_R0  // b = 1: r0 / r of a row requested before its product (see the v pass)
#define RSIM_EARLY_R0 1
#endif
#ifndef RSIM_EARLY_R0_BMAX  // ... for block sizes up to this one
#define RSIM_EARLY_R0_BMAX 1
#endif
#ifndef RSIM_XR_LOADFIRST  // b >= 2: x/r update pass loads all components before its first store
#define RSIM_XR_LOADFIRST 1    // (config 4 run 8.86 -> 8.73 s; early r0 / r for b = 3: 8.86 -> 9.01 s, so BMAX stays 1)
#endif
struct Pre1 {
  double m[6];
  int32_t c[6];
};
__device__ __forceinline__ void pre_load1(const KArgs& a, int64_t l, bool ok, Pre1& P) {
#pragma unroll
  for (int s = 0; s < 6; ++s) { P.c[s] = -1; P.m[s] = 0.0; }
  if (!ok) return;
  if (a.implicit) {
    implicit_cols(a.nx, a.ny, a.nz, a.d3, l, P.c);
#pragma unroll
    for (int s = 0; s < 6; ++s)
      if (P.c[s] >= 0) P.m[s] = (RSIM_LDCS || a.stream) ? __ldcs(&a.ell_val[(int64_t)s * a.cap + l]) : a.ell_val[(int64_t)s * a.cap + l];
  } else {  // columns not known yet: the value slot of an absent neighbour is loaded and ignored
#pragma unroll
    for (int s = 0; s < 6; ++s)
      if (s < a.nslot) {
        P.c[s] = __ldg(&a.ell_col[(int64_t)s * a.cap + l]);
        P.m[s] = (RSIM_LDCS || a.stream) ? __ldcs(&a.ell_val[(int64_t)s * a.cap + l]) : a.ell_val[(int64_t)s * a.cap + l];
      }
  }
}

// Columns (and the NNC row flag) of a warp's NEXT round, requested at the start of the
// current one (b = 2, partial sets).  Without it every round of every SpMV pass
// starts with two dependent DRAM round trips — the column load, then the block values
// (guarded by column >= 0) and the gathers — and the passes are latency-bound.
#ifndef RSIM_COLPRE
#define RSIM_COLPRE 1
#endif
struct ColPre {
  int32_t c[6];
  uint32_t f;
};
__device__ __forceinline__ void cols_load(const KArgs& a, int64_t l, bool ok, ColPre& C) {
#pragma unroll
  for (int s = 0; s < 6; ++s) C.c[s] = -1;
  C.f = 0u;
  if (!ok) return;
#pragma unroll
  for (int s = 0; s < 6; ++s)
    if (s < a.nslot) C.c[s] = __ldg(&a.ell_col[(int64_t)s * a.cap + l]);
  if (a.has_nnc) C.f = (uint32_t)__ldg(&a.ell_po[l]);
}

template <int B>
__device__ __forceinline__ void spmv_row(const KArgs& a, int64_t l, int mode, const Vecs& X, double beta,
                                         double omega, double alpha, const double* own, double* acc,
                                         const Pre1* pre = nullptr, const ColPre* cpre = nullptr) {
  const int32_t* __restrict__ col = a.ell_col;
  const double* __restrict__ val = a.ell_val;
  int32_t cl[6];
#pragma unroll
  for (int s = 0; s < 6; ++s) cl[s] = -1;
  if (B == 1 && pre) {
#pragma unroll
    for (int s = 0; s < 6; ++s) cl[s] = pre->c[s];
  } else if (cpre) {
#pragma unroll
    for (int s = 0; s < 6; ++s) cl[s] = cpre->c[s];
  } else if (a.implicit) {
    implicit_cols(a.nx, a.ny, a.nz, a.d3, l, cl);
  } else {
#pragma unroll
    for (int s = 0; s < 6; ++s)
      if (s < a.nslot) cl[s] = __ldg(&col[s * a.cap + l]);
  }
  // row flags (K1): is there any NNC block to multiply?  Loaded with the columns, so
  // the act -> nptr chain (two dependent gathers per row and pass that almost always
  // found an empty range: 7 % of the stall samples on a config-4 solve) is gone.
  const uint32_t rowf = cpre ? cpre->f : (a.has_nnc ? (uint32_t)__ldg(&a.ell_po[l]) : 0u);
  // Slots in groups of SG: all gathers of a group in flight, then its blocks.
  // Gathering all six neighbours first keeps 6·B doubles live and spills them
  // to local memory at 64 registers (b = 3: ~1 KB of local traffic per row and
  // SpMV, measured 1.4× the algorithmic DRAM bytes).  Accumulation order is
  // unchanged (slots ascending), so the bits are the same.
  // Pressure-only blocks (blockops.h col0_only, K1's ell_po bits) are NOT special-cased.
  // Measured on the whole config-3 / config-4 runs (round 2, scripts/ab_r02_s5.sh):
  // skipping their zero columns per lane (K1's ell_po bit) makes warps whose rows
  // disagree run both block shapes (avg 14 / 22 active lanes, 9.7 -> 13.0 s on
  // config 4); predicated loads + select 11.3 s; a warp-uniform choice 11.0 s.
  constexpr int SG = B == 1 ? RSIM_SPMV_SG1 : (B == 2 ? RSIM_SPMV_SG2 : RSIM_SPMV_SG3);
#pragma unroll
  for (int e = 0; e < B; ++e) acc[e] = own[e];
#pragma unroll
  for (int s0 = 0; s0 < 6; s0 += SG) {
    double xv[SG][B];
#pragma unroll
    for (int k = 0; k < SG; ++k)
#ifdef RSIM_DBG_NOGATHER  // timing experiment only (wrong numerics): neighbour := own row
      if (s0 + k < 6 && cl[s0 + k] >= 0) nbr_val<B>(mode, X, l, beta, omega, alpha, xv[k]);
#else
      if (s0 + k < 6 && cl[s0 + k] >= 0) nbr_val<B>(mode, X, cl[s0 + k], beta, omega, alpha, xv[k]);
#endif
#pragma unroll
    for (int k = 0; k < SG; ++k)
      if (s0 + k < 6 && cl[s0 + k] >= 0) {
        if (B == 1 && pre) {
          rsim::blk::gemv_acc_flat<B>(&pre->m[s0 + k], xv[k], acc);
        } else if (ell_es(B * B) == 1) {  // row-major blocks: the product reads them in place
          const double* __restrict__ Mp = &val[ell_at(a.cap, B * B, s0 + k, 0, l)];
#if RSIM_LDCS
#pragma unroll
          for (int r = 0; r < B; ++r) {  // gemv_acc_flat's expression order, streaming (evict-first) loads
            double sm = __ldcs(&Mp[r * B]) * xv[k][0];
#pragma unroll
            for (int c = 1; c < B; ++c) sm = sm + __ldcs(&Mp[r * B + c]) * xv[k][c];
            acc[r] = acc[r] + sm;
          }
#else
          rsim::blk::gemv_acc_flat<B>(Mp, xv[k], acc);
#endif
        } else {
          double M[B * B];
#if RSIM_LDCS
          const double* __restrict__ vp = val + ell_at(a.cap, B * B, s0 + k, 0, l);
#pragma unroll
          for (int e = 0; e < B * B; ++e) M[e] = __ldcs(&vp[e * ell_es(B * B)]);
#else
          ell_load<B>(val, a.cap, s0 + k, l, M);
#endif
          rsim::blk::gemv_acc_flat<B>(M, xv[k], acc);
        }
      }
    if (SG < 6) asm volatile("" ::: "memory");  // keep the next group's loads after this group's math
  }
  if (a.has_nnc && (rowf & ELL_ROW_NNC)) {  // rare: rows of fracture cells and the cells they cross
    const int64_t i = a.act[l];
    const int32_t q0 = a.nptr[i], q1 = a.nptr[i + 1];
    for (int32_t q = q0; q < q1; ++q) {
      const int32_t cc = a.nnc_lcol[q];
      if (cc >= 0) {
        double xn[B];
        nbr_val<B>(mode, X, cc, beta, omega, alpha, xn);
        rsim::blk::gemv_acc_flat<B>(&a.nnc_val[(int64_t)q * B * B], xn, acc);
      }
    }
  }
}

// L2 prefetch (prefetch.global.L2) of the matrix rows a warp will read in its NEXT round.
// Off.  History (round 2, config 5, 50 iterations, same box each): alone it gained 2.5-4 % on
// b = 1 partial sets (5 % 9.11 -> 8.89 ms, 20 % 28.1 -> 26.9, 50 % 64.6 -> 62.4); once the next
// round's row is requested into registers before the shuffle trees (Pre1 below) it is redundant
// and costs 6-7 % (20 %: 24.7 ms without vs 26.5 with, 50 %: 58.2 vs 62.2, 1 %: 2.30 vs 2.49).
// For b = 2 / 3 it was slower from the start (config 3 1.25 -> 1.31 s, config 4 9.7 -> 10.8 s).
#ifndef RSIM_PF
#define RSIM_PF 0
#endif
template <int B>
__device__ __forceinline__ void prefetch_rows(const KArgs& a, int64_t l) {
  const int lane = threadIdx.x & 31;
  const int64_t l0 = l - lane;
  if (l0 >= a.nA) return;
  constexpr int LPS = 2 * B * B;  // 128 B lines per slot and warp
  for (int idx = lane; idx < a.nslot * LPS; idx += 32) {
    const int sl = idx / LPS, ln = idx - sl * LPS;
    const double* q = a.ell_val + ell_at(a.cap, B * B, sl, 0, l0) + ln * 16;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
  }
  if (!a.implicit && lane < a.nslot) {
    const int32_t* q = a.ell_col + (int64_t)lane * a.cap + l0;
    asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
  }
}

// Per-pass wall time of one solve (debug builds, -DRSIM_KTIME=1; scripts/ab_krylov_build.sh):
// block 0 accumulates globaltimer deltas at the grid barriers that end each pass and prints
// them when the kernel ends.  Adds one barrier after the x/r pass; never on in the product.
#ifndef RSIM_KTIME
#define RSIM_KTIME 0
#endif
// FUSE is a template parameter: the two variants have different live state,
// and one kernel holding both spills heavily at 64 registers / thread.
template <int B, bool FUSE, bool ILU, int KT>
__global__ void __launch_bounds__(KT, 1) k_bicgstab(const KArgs a) {
  constexpr int CPR = KT / 256;  // canonical chunks per round
  __shared__ Red R;
  const bool single = gridDim.x == 1;
  auto sync = [&]() {
    if (single) __syncthreads();
    else cg::this_grid().sync();
  };
  const int64_t nr = a.nA;
  const int64_t nch = (nr + 255) / 256;
  const int64_t nrounds = (nch + CPR - 1) / CPR;
  const int tid = threadIdx.x;

  // global canonical reduction of NQ quantities whose level-1 partials are in
  // a.part (quantity 1 of the init may come from the assembly's part_f2)
  auto reduce = [&](int NQ, const double* src1 = nullptr) {
    sync();
    const int P1 = (int)nch;
    auto src = [&](int q) { return (q == 1 && src1) ? src1 : a.part + q * a.pstride; };
    if (P1 <= a.red_small_max) {
      reduce_small_multi<CPR>(R, NQ, src, P1);
    } else {
      // distributed level 2, one more barrier, then the (small) rest per CTA
      const int P2 = (P1 + 255) / 256;
      for (int64_t rr = blockIdx.x; rr * CPR < P2; rr += gridDim.x) {
        const int64_t c2 = rr * CPR + (tid >> 8);
        const int64_t idx = c2 * 256 + (tid & 255);
        double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (int q = 0; q < NQ; ++q) v[q] = idx < P1 ? src(q)[idx] : 0.0;
        commit_round<CPR>(R, NQ, v, rr * CPR, P2, a.part2, a.pstride2);
      }
      sync();
      reduce_small_multi<CPR>(R, NQ, [&](int q) { return (const double*)(a.part2 + q * a.pstride2); }, P2);
    }
  };

  // Sweep order: with a.alt every phase walks the rounds in the direction
  // opposite to the previous phase, so the rows it starts with are the ones the
  // previous phase touched last (still in L2).  Row results do not depend on the
  // order (reductions go through per-chunk partials), so the bits are unchanged.
  bool rev = false;
  // Blocked-cyclic rounds (a.kblk > 1): CTA b takes kblk consecutive rounds, then jumps
  // grid·kblk ahead, so the ±y neighbours of a round are rows the same SM has just read
  // (L1) while all CTAs still work inside one window of grid·kblk rounds (L2).  The ragged
  // tail past the last full window stays round-robin.  A bijection on the rounds, so the
  // bits are unchanged.
  const int64_t GK = (int64_t)gridDim.x * a.kblk, NF = (nrounds / GK) * GK;
  auto rmap = [&](int64_t rd0) {
    const int64_t v = rev ? nrounds - 1 - rd0 : rd0;
    if (a.kblk <= 1 || v >= NF) return v;
    const int64_t sb = v / GK, w = v - sb * GK;
    const int64_t jj = w / gridDim.x, b = w - jj * gridDim.x;
    return sb * GK + b * a.kblk + jj;
  };
  auto flip = [&]() { if (a.alt) rev = !rev; };
  unsigned long long kt_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, kt_last = 0;
  auto tick = [&](int ph) {
    if (RSIM_KTIME && blockIdx.x == 0 && tid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (ph >= 0) kt_acc[ph] += t - kt_last;
      kt_last = t;
    }
  };
  auto pf = [&](int64_t rd0) {  // matrix rows of this CTA's next round (SpMV passes)
    if (RSIM_PF && B == 1 && !a.implicit && rd0 + gridDim.x < nrounds) prefetch_rows<B>(a, rmap(rd0 + gridDim.x) * KT + tid);
  };
#define ROUNDS_BEGIN                                                         \
  {                                                                          \
  int rloc = 0;                                                              \
  for (int64_t rd0 = blockIdx.x; rd0 < nrounds; rd0 += gridDim.x, ++rloc) {  \
    const int64_t rd = rmap(rd0);                                            \
    const int64_t l = rd * KT + tid;                                         \
    const bool ok = l < nr;                                                  \
    double val[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
#define ROUNDS_END(NQ)                                                       \
    {                                                                        \
      const int slot = rloc % a.stage;                                       \
      const bool last = rd0 + gridDim.x >= nrounds;                          \
      stage_round<CPR, NQ>(R, val, slot, rd, slot == a.stage - 1 || last, slot + 1, nch, a.part, a.pstride); \
    }                                                                        \
  }                                                                          \
  flip();                                                                    \
  }

  constexpr bool PRE = B == 1 && RSIM_PRE1;
  Pre1 P1;
  const Pre1* pre = PRE ? &P1 : nullptr;
  auto pre_first = [&]() {  // before a reducing SpMV pass: this CTA's first round
    if (PRE) {
      const int64_t l = rmap(blockIdx.x) * KT + tid;
      pre_load1(a, l, (int64_t)blockIdx.x < nrounds && l < nr, P1);
    }
  };
  auto pre_next = [&](int64_t rd0) {  // at the end of a round, before its shuffle trees
    if (PRE) {
      const bool more = rd0 + gridDim.x < nrounds;
      const int64_t l = more ? rmap(rd0 + gridDim.x) * KT + tid : 0;
      pre_load1(a, l, more && l < nr, P1);
    }
  };
  // generic column preload (partial sets; b = 1 uses Pre1 in the reducing passes instead)
  ColPre Ccur, Cnx;
  // b = 2 only (measured on whole runs, same box: config 3 1.358 -> 1.290 s; for b = 3 the 14
  // extra live registers cost more than the round trip saves, config 4 8.85 -> 9.79 s, and the
  // b = 1 kernel, which needs it only in the Neumann passes, slows down by 3-5 % on config 5)
  const bool use_cp = RSIM_COLPRE && B == 2 && !a.implicit;
  auto cp_first = [&](bool skip) {
    if (use_cp && !skip) {
      const int64_t l = rmap(blockIdx.x) * KT + tid;
      cols_load(a, l, (int64_t)blockIdx.x < nrounds && l < nr, Ccur);
    }
  };
  auto cp_next = [&](int64_t rd0, bool skip) {  // at the START of a round: the next round's columns
    if (use_cp && !skip) {
      const bool more = rd0 + gridDim.x < nrounds;
      const int64_t l = more ? rmap(rd0 + gridDim.x) * KT + tid : 0;
      cols_load(a, l, more && l < nr, Cnx);
    }
  };
  auto cp_adv = [&](bool skip) { if (use_cp && !skip) Ccur = Cnx; };
  const ColPre* cpa = use_cp ? &Ccur : nullptr;           // passes without a reduction
  const ColPre* cpr = (use_cp && !PRE) ? &Ccur : nullptr;  // reducing passes (b = 1: Pre1 instead)
  // ---- init: r = r0 = rhs, x = 0;  (rhs, rhs), (F, F) (the latter from the
  //      assembly's canonical chunk partials when it left them)
  ROUNDS_BEGIN
  if (ok) {
    double bv[B];
#pragma unroll
    for (int e = 0; e < B; ++e) bv[e] = a.rhs[l * B + e];
#pragma unroll
    for (int e = 0; e < B; ++e) { a.r[l * B + e] = bv[e]; a.r0[l * B + e] = bv[e]; a.x[l * B + e] = 0.0; }
    val[0] = rsim::blk::rowdot<B>(bv, bv);
    if (!a.f2_parts) {
      double fv[B];
#pragma unroll
      for (int e = 0; e < B; ++e) fv[e] = a.F_raw[l * B + e];
      val[1] = rsim::blk::rowdot<B>(fv, fv);
    }
  }
  ROUNDS_END(2)  // (F,F) staged as zeros when the assembly left its chunk partials
  reduce(2, a.f2_parts ? a.part_f2 : nullptr);
  tick(-1);
  const double bb = R.res[0];
  if (blockIdx.x == 0 && tid == 0) a.dsc->f2 = sqrt(R.res[1]);
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
  int cur = 0;  // which (p, v) buffer pair holds the current iterate
  bool p_ready = false;  // unfused: the next p was stored by the x/r update pass
  // (fused: riding the x/r update of iteration k on the first pass of iteration k+1 was
  // measured and rejected in round 2: config 3 run 1.27 -> 1.39 s, config 4 11.1 -> 11.3 s)
  // fuse: neighbours' p and s are recomputed at the gather site (fewer grid
  // barriers, latency regime); !fuse: owners store p and s, then a barrier,
  // then plain gathers (less memory traffic, bandwidth regime).
  constexpr bool fuse = FUSE;
  int it_total = 0;
  // attempt 0: as configured; attempt 1 (only after a Neumann-1 breakdown or
  // cap): block-Jacobi only, restarted from x0 = 0 (same rule as the oracle)
  // ILU is a template parameter: the level-scheduled solves would otherwise
  // change the register allocation (and speed) of the common variants
  const bool ilu_bad = ILU && a.dsc->ilu_bad;
  for (int attempt = 0; attempt < ((a.neu || ILU) ? 2 : 1); ++attempt) {
  const bool neu = a.neu && attempt == 0;
  const bool ilu = ILU && attempt == 0;
  const bool prec = neu || ilu;  // ph = M^{-1} p, sh = M^{-1} s are stored
  if (ilu && ilu_bad) { status = RSIM_ENUM; it = 0; continue; }  // singular pivot: block-Jacobi only
  if (attempt) {
    for (int64_t rd0 = blockIdx.x; rd0 < nrounds; rd0 += gridDim.x) {
      const int64_t l = rmap(rd0) * KT + tid;
      if (l < nr)
#pragma unroll
        for (int e = 0; e < B; ++e) {
          a.r[l * B + e] = a.rhs[l * B + e];
          a.x[l * B + e] = 0.0;
        }
    }
    rho = 1.0; alpha = 1.0; omega = 1.0; rho_new = bb;
    cur = 0;
    p_ready = false;
    status = RSIM_ENOCONV;
    sync();
  }
  for (it = 1; it <= maxit; ++it) {
    const double beta = (it == 1) ? 0.0 : (rho_new / rho) * (alpha / omega);
    double* pc = cur ? a.p2 : a.p;
    double* vc = cur ? a.v2 : a.v;
    const double* po = cur ? a.p : a.p2;
    const double* vo = cur ? a.v : a.v2;
    const int pmode = it == 1 ? 1 : 0;
    const Vecs V0{a.r, po, vo, a.s, a.t};  // p_j = (s_j − ω t_j) + β (p_old_j − ω v_old_j)
    if (!fuse) {  // p = r + β (p − ω v), stored, then visible to all
      if (!p_ready)  // (else already stored by the previous x/r update pass)
      for (int64_t rd0 = blockIdx.x; rd0 < nrounds; rd0 += gridDim.x) {
        const int64_t l = rmap(rd0) * KT + tid;
        if (l < nr) {
          double pown[B];
          nbr_val<B>(pmode, V0, l, beta, omega, 0.0, pown);
#pragma unroll
          for (int e = 0; e < B; ++e) pc[l * B + e] = pown[e];
        }
      }
      sync();
      flip();
      tick(0);
    }
    if (neu) {  // ph = p + (p − Â p), stored, barrier
      cp_first(false);
      for (int64_t rd0 = blockIdx.x; rd0 < nrounds; rd0 += gridDim.x) {
        const int64_t l = rmap(rd0) * KT + tid;
        pf(rd0);
        cp_next(rd0, false);
        if (l < nr) {
          double pown[B], y[B];
          if (fuse) {
            nbr_val<B>(pmode, V0, l, beta, omega, 0.0, pown);
            spmv_row<B>(a, l, pmode, V0, beta, omega, 0.0, pown, y, nullptr, cpa);
#pragma unroll
            for (int e = 0; e < B; ++e) pc[l * B + e] = pown[e];
          } else {
#pragma unroll
            for (int e = 0; e < B; ++e) pown[e] = pc[l * B + e];
            spmv_row<B>(a, l, 3, Vecs{a.r, pc, vo, a.s, a.t}, 0.0, 0.0, 0.0, pown, y, nullptr, cpa);
          }
#pragma unroll
          for (int e = 0; e < B; ++e) a.ph[l * B + e] = pown[e] + (pown[e] - y[e]);
        }
        cp_adv(false);
      }
      sync();
      flip();
      tick(1);
    }
    if (ilu) ilu_apply<B>(a.fa, pc, a.ph, sync);  // ph = (LU)^{-1} p (p stored: unfused)
    // ---- v = Â p (BJ) or v = Â ph (Neumann-1, ILU(0)); (r0, v) and the lagged (r, r)
    pre_first();
    cp_first(PRE);
    ROUNDS_BEGIN
    pf(rd0);
    cp_next(rd0, PRE);
    if (ok) {
      double y[B];
      // b = 1: r0 and r of the row are requested before the product.  After it they sit
      // behind the store of v (the vectors may alias as far as the compiler knows), i.e. one
      // more exposed DRAM round trip per round (11 % of the stall samples at 100 % of config 5).
      // b >= 2 keeps the late loads: 2·b more live doubles would spill at the 128-register cap.
      double r0e[B], re[B];
      if (B <= RSIM_EARLY_R0_BMAX && RSIM_EARLY_R0) {
#pragma unroll
        for (int e = 0; e < B; ++e) { r0e[e] = a.r0[l * B + e]; re[e] = a.r[l * B + e]; }
      }
      if (prec) {
        spmv_row<B>(a, l, 3, Vecs{a.r, a.ph, vo, a.s, a.t}, 0.0, 0.0, 0.0, &a.ph[l * B], y, pre, cpr);
      } else if (fuse) {
        double pown[B];
        nbr_val<B>(pmode, V0, l, beta, omega, 0.0, pown);
#pragma unroll
        for (int e = 0; e < B; ++e) pc[l * B + e] = pown[e];
        spmv_row<B>(a, l, pmode, V0, beta, omega, 0.0, pown, y, pre, cpr);
      } else {
        spmv_row<B>(a, l, 3, Vecs{a.r, pc, vo, a.s, a.t}, 0.0, 0.0, 0.0, &pc[l * B], y, pre, cpr);
      }
#pragma unroll
      for (int e = 0; e < B; ++e) vc[l * B + e] = y[e];
      if (!(B <= RSIM_EARLY_R0_BMAX && RSIM_EARLY_R0)) {
#pragma unroll
        for (int e = 0; e < B; ++e) { r0e[e] = a.r0[l * B + e]; re[e] = a.r[l * B + e]; }
      }
      val[0] = rsim::blk::rowdot<B>(r0e, y);
      val[1] = rsim::blk::rowdot<B>(re, re);
    }
    cp_adv(PRE);
    pre_next(rd0);
    ROUNDS_END(2)
    reduce(2);
    tick(2);
    if (it > 1 && !fixed && sqrt(R.res[1]) <= tol) {  // previous iterate converged
      relres = sqrt(R.res[1]) / bnorm;
      status = RSIM_OK;
      --it;
      break;
    }
    const double r0v = R.res[0];
    if (r0v == 0.0 || !isfinite(r0v)) { status = RSIM_ENUM; break; }
    alpha = rho_new / r0v;
    const Vecs V2{a.r, po, vc, a.s, a.t};  // s_j = r_j − α v_j
    const bool fs = fuse || (!prec && a.fuse_s);  // s recomputed where gathered, stored by its owner
    if (!fs) {  // s = r − α v, stored, barrier
      for (int64_t rd0 = blockIdx.x; rd0 < nrounds; rd0 += gridDim.x) {
        const int64_t l = rmap(rd0) * KT + tid;
        if (l < nr)
#pragma unroll
          for (int e = 0; e < B; ++e) a.s[l * B + e] = a.r[l * B + e] - alpha * vc[l * B + e];
      }
      sync();
      flip();
      tick(3);
    }
    if (neu) {  // sh = s + (s − Â s), stored, barrier
      cp_first(false);
      for (int64_t rd0 = blockIdx.x; rd0 < nrounds; rd0 += gridDim.x) {
        const int64_t l = rmap(rd0) * KT + tid;
        pf(rd0);
        cp_next(rd0, false);
        if (l < nr) {
          double sv[B], y[B];
          if (fuse) {
            nbr_val<B>(2, V2, l, 0.0, 0.0, alpha, sv);
            spmv_row<B>(a, l, 2, V2, 0.0, 0.0, alpha, sv, y, nullptr, cpa);
          } else {
#pragma unroll
            for (int e = 0; e < B; ++e) sv[e] = a.s[l * B + e];
            spmv_row<B>(a, l, 3, Vecs{a.r, a.s, vc, a.s, a.t}, 0.0, 0.0, 0.0, sv, y, nullptr, cpa);
          }
#pragma unroll
          for (int e = 0; e < B; ++e) a.sh[l * B + e] = sv[e] + (sv[e] - y[e]);
        }
        cp_adv(false);
      }
      sync();
      flip();
      tick(4);
    }
    if (ilu) ilu_apply<B>(a.fa, a.s, a.sh, sync);  // sh = (LU)^{-1} s
    // ---- t = Â s (BJ) or t = Â sh (Neumann-1, ILU(0)); (s,s), (t,s), (t,t), (r0,s), (r0,t)
    pre_first();
    cp_first(PRE);
    ROUNDS_BEGIN
    pf(rd0);
    cp_next(rd0, PRE);
    if (ok) {
      double sv[B], y[B], r0e[B];
      if (B <= RSIM_EARLY_R0_BMAX && RSIM_EARLY_R0) {  // as in the v pass: r0 before the product, not behind the stores of s and t
#pragma unroll
        for (int e = 0; e < B; ++e) r0e[e] = a.r0[l * B + e];
      }
      if (prec) {
        if (fuse) nbr_val<B>(2, V2, l, 0.0, 0.0, alpha, sv);
        else
#pragma unroll
          for (int e = 0; e < B; ++e) sv[e] = a.s[l * B + e];
        spmv_row<B>(a, l, 3, Vecs{a.r, a.sh, vc, a.s, a.t}, 0.0, 0.0, 0.0, &a.sh[l * B], y, pre, cpr);
      } else if (fs) {
        nbr_val<B>(2, V2, l, 0.0, 0.0, alpha, sv);
        spmv_row<B>(a, l, 2, V2, 0.0, 0.0, alpha, sv, y, pre, cpr);
      } else {
#pragma unroll
        for (int e = 0; e < B; ++e) sv[e] = a.s[l * B + e];
        spmv_row<B>(a, l, 3, Vecs{a.r, a.s, vc, a.s, a.t}, 0.0, 0.0, 0.0, sv, y, pre, cpr);
      }
      if (fs)
#pragma unroll
        for (int e = 0; e < B; ++e) a.s[l * B + e] = sv[e];
#pragma unroll
      for (int e = 0; e < B; ++e) a.t[l * B + e] = y[e];
      val[0] = rsim::blk::rowdot<B>(sv, sv);
      val[1] = rsim::blk::rowdot<B>(y, sv);
      val[2] = rsim::blk::rowdot<B>(y, y);
      if (!(B <= RSIM_EARLY_R0_BMAX && RSIM_EARLY_R0)) {
#pragma unroll
        for (int e = 0; e < B; ++e) r0e[e] = a.r0[l * B + e];
      }
      val[3] = rsim::blk::rowdot<B>(r0e, sv);
      val[4] = rsim::blk::rowdot<B>(r0e, y);
    }
    cp_adv(PRE);
    pre_next(rd0);
    ROUNDS_END(5)
    reduce(5);
    tick(5);
    const double ss = R.res[0], ts = R.res[1], tt = R.res[2], r0s = R.res[3], r0t = R.res[4];
    const double* phv = prec ? a.ph : pc;
    const double* shv = prec ? a.sh : a.s;
    if (!fixed && sqrt(ss) <= tol) {
      for (int64_t rd0 = blockIdx.x; rd0 < nrounds; rd0 += gridDim.x) {
        const int64_t l = rmap(rd0) * KT + tid;
        if (l < nr)
#pragma unroll
          for (int e = 0; e < B; ++e) a.x[l * B + e] = a.x[l * B + e] + alpha * phv[l * B + e];
      }
      relres = sqrt(ss) / bnorm;
      status = RSIM_OK;
      break;
    }
    if (tt == 0.0 || !isfinite(tt)) { status = RSIM_ENUM; break; }
    omega = ts / tt;
    // ---- x, r update (own rows, no barrier — so it keeps the sweep direction of
    //      the phase that follows it (same rows per CTA) — neighbours recompute r from s, t
    //      until the next reduction, and the next p-pass reads only its own r).
    //      Unfused: the next iterate's p = r + β' (p − ω v) is formed here from
    //      the same registers (own row only; β' needs only this iteration's
    //      reductions), so the separate p pass and its re-read of s, t, p
    //      disappear.  Same expressions as nbr_val mode 0 -> same bits.
    const double rho_next = r0s - omega * r0t;
    const bool more = !(omega == 0.0 || rho_next == 0.0 || !isfinite(rho_next)) && it < maxit;
    const bool pfuse = !fuse && more;
    const double beta_next = pfuse ? (rho_next / rho_new) * (alpha / omega) : 0.0;
    double* pn = cur ? a.p : a.p2;  // the next iterate's p buffer
    // (two rounds of loads in flight per thread in this pass and in the s pass were
    //  measured on config 5 and are slower: 20 %: 28.1 -> 29.1 ms, 100 %: 115.7 -> 118.4 ms)
    for (int64_t rd0 = blockIdx.x; rd0 < nrounds; rd0 += gridDim.x) {
      const int64_t l = rmap(rd0) * KT + tid;
      if (l < nr) {
        if (B > 1 && RSIM_XR_LOADFIRST) {
          // b >= 2: all b components' loads before the first store — component by component, the
          // stores of x and r (which may alias the other vectors as far as the compiler knows)
          // fence the next component's loads: b dependent DRAM round trips per row
          double xx[B], pp[B], hh[B], sq[B], tq[B], pq[B], vq[B];
#pragma unroll
          for (int e = 0; e < B; ++e) {
            const int64_t q = l * B + e;
            xx[e] = a.x[q]; pp[e] = phv[q]; hh[e] = shv[q];
            sq[e] = prec ? a.s[q] : hh[e];
            tq[e] = a.t[q];
            if (pfuse) { pq[e] = prec ? pc[q] : pp[e]; vq[e] = vc[q]; }
          }
#pragma unroll
          for (int e = 0; e < B; ++e) {
            const int64_t q = l * B + e;
            a.x[q] = (xx[e] + alpha * pp[e]) + omega * hh[e];
            const double rq = sq[e] - omega * tq[e];
            a.r[q] = rq;
            if (pfuse) pn[q] = rq + beta_next * (pq[e] - omega * vq[e]);
          }
        } else {
#pragma unroll
          for (int e = 0; e < B; ++e) {
            const int64_t q = l * B + e;
            a.x[q] = (a.x[q] + alpha * phv[q]) + omega * shv[q];
            const double rq = a.s[q] - omega * a.t[q];
            a.r[q] = rq;
            if (pfuse) pn[q] = rq + beta_next * (pc[q] - omega * vc[q]);
          }
        }
      }
    }
    if (RSIM_KTIME) { sync(); tick(6); }
    p_ready = pfuse;
    rho = rho_new;
    rho_new = rho_next;
    if (omega == 0.0 || rho_new == 0.0 || !isfinite(rho_new)) { status = RSIM_ENUM; break; }
    cur ^= 1;
  }
  if (it > maxit) {  // iteration cap: residual of the last iterate (one more reduction)
    it = maxit;
    ROUNDS_BEGIN
    if (ok) val[0] = rsim::blk::rowdot<B>(&a.r[l * B], &a.r[l * B]);
    ROUNDS_END(1)
    reduce(1);
    relres = sqrt(R.res[0]) / bnorm;
    status = (fixed || sqrt(R.res[0]) <= tol) ? RSIM_OK : RSIM_ENOCONV;
  }
  it_total += it;
  if (!(prec && (status == RSIM_ENUM || status == RSIM_ENOCONV))) break;
  }
  it = it_total;
  if (RSIM_KTIME && blockIdx.x == 0 && tid == 0)
    printf("KTIME rows %d its %d us: p %.1f ph %.1f v+red %.1f s %.1f sh %.1f t+red %.1f xr %.1f\n", a.nA, it,
           kt_acc[0] * 1e-3, kt_acc[1] * 1e-3, kt_acc[2] * 1e-3, kt_acc[3] * 1e-3, kt_acc[4] * 1e-3,
           kt_acc[5] * 1e-3, kt_acc[6] * 1e-3);
  if (blockIdx.x == 0 && tid == 0) {
    a.dsc->lin_iters = it;
    a.dsc->lin_relres = relres;
    if (status != RSIM_OK) a.dsc->status = status;
  }
#undef ROUNDS_BEGIN
#undef ROUNDS_END
}

template <int B>
int launch_b(rsim_gpu_ctx* c, const rsim_solver_opts* o) {
  KArgs a;
  a.nA = c->nA;
  a.nslot = c->nslot;
  a.maxit = o->lin_maxit;
  a.fixed = o->fixed_lin_iters;
  a.nx = c->nx; a.ny = c->ny; a.nz = c->nz;
  a.d3 = c->d3;
  a.implicit = c->cols_implicit;
  // staging lets warps drift apart by several rounds (more loads in flight):
  // best for the regular full-grid sweep and long passes; short passes over
  // scattered partial sets prefer warps kept close (L1 reuse of the gathers)
  static const int stage_env = [] {  // env override: tuning only
    const char* e = std::getenv("RSIM_KSTAGE");
    return (e && *e) ? std::atoi(e) : 0;
  }();
  a.stage = 1;  // set below from the rounds per CTA
  a.cap = c->ell_cap;
  a.has_nnc = c->has_nnc;
  a.rtol = o->lin_rtol;
  a.ell_col = c->ell_col; a.ell_val = c->ell_val; a.ell_po = c->ell_po;
  a.act = c->act; a.nptr = c->nptr; a.nnc_lcol = c->nnc_lcol; a.nnc_val = c->nnc_val;
  a.rhs = c->rhs; a.F_raw = c->F_raw;
  a.part_f2 = c->part_f2;
  a.f2_parts = c->f2_parts;
  a.x = c->x; a.r = c->r; a.r0 = c->r0; a.p = c->p; a.v = c->v; a.s = c->s; a.t = c->t;
  a.p2 = c->p2; a.v2 = c->v2; a.ph = c->ph; a.sh = c->sh;
  a.neu = o->precond == RSIM_PREC_NEUMANN1;
  a.ilu = o->precond == RSIM_PREC_ILU0;
  a.fa = ilu_args(c);
  static const int64_t fuse_max = [] {  // env override: tuning only
    const char* e = std::getenv("RSIM_FUSE_MAX_ROWS");
    return (e && *e) ? (int64_t)std::atoll(e) : (int64_t)-1;
  }();
  a.fuse = (c->nA <= (fuse_max >= 0 ? fuse_max : fuse_max_rows(B)) && !a.ilu) ? 1 : 0;
  // s recompute at the gather sites (unfused block-Jacobi: no s pass, one grid barrier less), at
  // every size.  Round 1 measured a loss above 4 M rows (config 5 at 100 %: 114.5 -> 119.1 ms per 50
  // iterations) and capped it at 2^22; with the row preload and the early r0 / r loads of round 2
  // it wins everywhere: 20 % (6.7 M rows) 24.85 -> 23.60 ms, 50 % 57.0 -> 56.6, 100 % 109.9 -> 108.2.
  static const int64_t fuse_s_max = [] {  // env override: tuning only
    const char* e = std::getenv("RSIM_FUSE_S_MAX_ROWS");
    return (e && *e) ? (int64_t)std::atoll(e) : (int64_t)1 << 40;
  }();
  a.fuse_s = c->nA <= fuse_s_max ? 1 : 0;
  static const int32_t red_small = [] {  // env override: tuning only
    const char* e = std::getenv("RSIM_RED_SMALL_MAX");
    // measured on config 5 at 5 % (6 559 chunks): every CTA scanning all chunk
    // partials costs ~5 µs more per iteration than the distributed level 2 +
    // one extra grid barrier (9.89 -> 9.65 ms per 50 iterations)
    return (e && *e) ? (int32_t)std::atoi(e) : 2048;
  }();
  a.red_small_max = red_small < 64 * 256 ? red_small : 64 * 256;
  // Alternating sweep direction: every pass starts on the rows the previous pass
  // touched last, which are still in L2.  It pays when the solve's working set (matrix
  // + 11 vectors) is larger than L2, and costs a little when everything fits.  Whole
  // runs, round 2, same box: config 4 (b = 3, 0.2-0.8 M rows, 150-600 MB) 9.71 -> 9.03 s;
  // config 3 (b = 2, 150 k rows, 60 MB) 1.25 -> 1.31 s; config 5 at 20-100 % -0.2..-0.8 %.
  static const int alt_env = [] {  // env override: tuning only
    const char* e = std::getenv("RSIM_KALT");
    return (e && *e) ? std::atoi(e) : -1;
  }();
  {
    const int64_t row_bytes = (int64_t)c->nslot * (8 * B * B + 4) + 11 * 8 * B;
    a.alt = alt_env >= 0 ? alt_env : ((int64_t)c->nA * row_bytes > (int64_t)100e6 ? 1 : 0);
    // b = 1, working set beyond L2: the matrix values (read once per pass) go through
    // ld.global.cs so the gathered vectors keep L2 (config 5 at 100 %: 110.0 -> 107.4 ms per 50
    // iterations, 20 %: 24.5 -> 24.3).  Not for b >= 2: config 3, whose matrix fits in L2,
    // 1.28 -> 1.51 s per run; config 4 8.72 -> 8.77 s.
    a.stream = (B == 1 && (int64_t)c->nA * row_bytes > (int64_t)100e6) ? 1 : 0;
  }
  static const int kblk_env = [] {  // env override: tuning only
    const char* e = std::getenv("RSIM_KBLK");
    return (e && *e) ? std::atoi(e) : 0;
  }();
  a.kblk = kblk_env > 0 ? kblk_env : 1;
  a.pstride = (int32_t)((c->n + 255) / 256);
  a.pstride2 = (a.pstride + 255) / 256;
  a.part = c->part;
  a.part2 = c->part + 5 * (int64_t)a.pstride;
  a.dsc = c->dsc;
  constexpr int KT = kt_for(B), CPR = KT / 256;
  const int64_t nrounds = ((c->nA + 255) / 256 + CPR - 1) / CPR;
  auto kern = a.ilu ? k_bicgstab<B, false, true, KT>
                    : (a.fuse ? k_bicgstab<B, true, false, KT> : k_bicgstab<B, false, false, KT>);
  if (c->max_coop_blocks[B] == 0) {
    int per_sm = 0, per_sm2 = 0, per_sm3 = 0;
    RSIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bicgstab<B, true, false, KT>, KT, 0));
    RSIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_bicgstab<B, false, false, KT>, KT, 0));
    RSIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm3, k_bicgstab<B, false, true, KT>, KT, 0));
    if (per_sm2 < per_sm) per_sm = per_sm2;
    if (per_sm3 < per_sm) per_sm = per_sm3;
    c->max_coop_blocks[B] = per_sm * c->sm_count;
    if (c->max_coop_blocks[B] < 1) c->max_coop_blocks[B] = 1;
  }
  int grid = nrounds < c->max_coop_blocks[B] ? (int)nrounds : c->max_coop_blocks[B];
  if (grid < 1) grid = 1;
  {
    // measured on config 5 (50 iterations, rounds per CTA at 5 / 20 / 50 % =
    // 11 / 44 / 110): stage 1 -> 2 -> 4 -> 8 gives 9.35 / 9.15 / 9.31 / 10.07 ms
    // at 5 %, 30.7 / 29.1 / 28.4 / 28.4 at 20 %, 72.3 / 68.2 / 65.8 / 64.9 at 50 %
    const int64_t rpc = (nrounds + grid - 1) / grid;
    const int st = c->cols_implicit ? RSTAGE : (rpc < 24 ? 2 : (rpc < 96 ? 4 : 8));
    a.stage = stage_env > 0 ? stage_env : st;
    if (a.stage > RSTAGE) a.stage = RSTAGE;
  }
  void* args[] = {&a};
  if (grid == 1) {
    kern<<<1, KT, 0, c->stream>>>(a);
  } else {
    RSIM_CUDA(cudaLaunchCooperativeKernel((void*)kern, grid, KT, args, 0, c->stream));
  }
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

}  // namespace

int launch_krylov(rsim_gpu_ctx* c, const rsim_solver_opts* o) {
  if (c->nA <= 0) return RSIM_OK;
  // exact dense LU (direct.cu) up to RSIM_DIRECT_MAX unknowns; larger active
  // sets fall back to BiCGSTAB (the oracle applies the same rule)
  if (o->lin_method == RSIM_LIN_DIRECT && (int64_t)c->nA * c->b <= RSIM_DIRECT_MAX) return launch_direct(c, o);
  const bool ilu = o->precond == RSIM_PREC_ILU0;
  if (ilu) RSIM_TRY(ilu_prepare(c));
  if (o->lin_method == RSIM_LIN_GMRES) return launch_gmres(c, o);
  if (!ilu) {  // small systems: one cluster with matrix + vectors in distributed smem
    int r = launch_krylov_dsm(c, o);
    if (r != RSIM_ENOTAPPLICABLE) return r;
  }
  switch (c->b) {
    case 1: return launch_b<1>(c, o);
    case 2: return launch_b<2>(c, o);
    default: return launch_b<3>(c, o);
  }
}
