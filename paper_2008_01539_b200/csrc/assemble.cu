// assemble.cu — K1: fused cell-property evaluation + TPFA/PPU residual and
// block-Jacobi-scaled Jacobian over the active rows (+ the K2 pattern).
//
// Restates assemble(target_set) (Eq. 16 PAPER.md:252-256;
// Appendix A): rows only for V_A; a connection to a cell
// outside V_A uses that cell's current (frozen) state in the residual and the
// diagonal, with no column.
//
// Layout (DESIGN.md §HBM layout):
//   one thread per active row (‖F‖₂ is reduced canonically by the Krylov
//   kernel's init phase, which reads F anyway);
//   ELL column/value arrays slot-major [slot][cap] so warp stores coalesce;
//   NNC blocks indexed by the global NNC CSR slot (no scan needed);
//   no atomics except the ‖F‖∞ / singular-cell reductions.
// Block-Jacobi scaling is fused: the row is multiplied by D_ii^{-1} before it
// is stored, so the Krylov kernel sees a unit block diagonal (never stored).
#include <cstdlib>

#include "ctx.cuh"

namespace {

struct AsmArgs {
  rsim::phys::Fluid fl;
  double dt, inv_dt, bhp;
  int32_t nx, ny, nz, nslot, nA;
  int64_t cap;
  bool d3, has_nnc;
  const double *__restrict__ tx, *__restrict__ ty, *__restrict__ tz, *__restrict__ pv, *__restrict__ wi;
  const int32_t *__restrict__ nptr, *__restrict__ nnbr;
  const double* __restrict__ nt;
  const double *__restrict__ u, *__restrict__ mold;
  const uint8_t* __restrict__ st;
  const int32_t *__restrict__ act, *__restrict__ g2l;
  int32_t* ell_col;
  double* ell_val;
  uint8_t* ell_po;
  int32_t* nnc_lcol;
  double* nnc_val;
  double *F_raw, *rhs, *part_f2;
  bool keep_F;  // row kernel: store the raw residual (debug downloads only)
  DevScalars* dsc;
};

// Cartesian neighbour of slot s (ascending column order -z,-y,-x,+x,+y,+z;
// 2D: -y,-x,+x,+y).  Returns false when the slot falls off the grid.
__device__ __forceinline__ bool cart_nbr(const AsmArgs& a, int64_t i, int64_t ix, int64_t iy, int64_t iz, int s,
                                         int64_t& j, double& T) {
  const int64_t nxy = (int64_t)a.nx * a.ny;
  int k = a.d3 ? s : s + 1;  // 2D skips the -z slot
  switch (k) {
    case 0: if (iz == 0) return false; j = i - nxy; T = __ldg(&a.tz[j]); return true;
    case 1: if (iy == 0) return false; j = i - a.nx; T = __ldg(&a.ty[j]); return true;
    case 2: if (ix == 0) return false; j = i - 1; T = __ldg(&a.tx[j]); return true;
    case 3: if (ix == a.nx - 1) return false; j = i + 1; T = __ldg(&a.tx[i]); return true;
    case 4: if (iy == a.ny - 1) return false; j = i + a.nx; T = __ldg(&a.ty[i]); return true;
    default: if (iz == a.nz - 1) return false; j = i + nxy; T = __ldg(&a.tz[i]); return true;
  }
}

template <int B>
__device__ __forceinline__ void load_u(const AsmArgs& a, int64_t j, double* uj) {
#pragma unroll
  for (int c = 0; c < B; ++c) uj[c] = __ldg(&a.u[j * B + c]);
}

// Flux block of connection (i,j): adds to R/D, returns the raw off-diagonal O.
template <int B>
__device__ __forceinline__ void conn(const AsmArgs& a, const double* ui, const rsim::phys::Props<B>& Pi, int64_t j,
                                     double T, double* R, double (*D)[B], double (*O)[B]) {
  double uj[B];
  load_u<B>(a, j, uj);
  double dp = ui[0] - uj[0];
  bool up_i = !(dp < 0.0);
  if (up_i) {
    rsim::phys::flux_conn<B>(T, dp, true, Pi, R, D, O);
  } else {
    rsim::phys::Props<B> Pj;
    rsim::phys::props(a.fl, uj, B == 3 ? __ldg(&a.st[j]) : (uint8_t)0, Pj);
    rsim::phys::flux_conn<B>(T, dp, false, Pj, R, D, O);
  }
}

template <int B>
__device__ __forceinline__ void store_scaled(double* dst, const double (*Di)[B], const double (*O)[B]) {
  double S[B][B];
  rsim::blk::gemm<B>(Di, O, S);
#pragma unroll
  for (int r = 0; r < B; ++r)
#pragma unroll
    for (int c = 0; c < B; ++c) dst[r * B + c] = S[r][c];
}

// Scaled block D_ii^{-1}·O of (slot s, row l) into the ELL values (ctx.cuh ell_at);
// returns whether it is pressure-only (blockops.h col0_only).
template <int B, bool STREAM>
__device__ __forceinline__ bool store_scaled_ell(const AsmArgs& a, int s, int64_t l, const double (*Di)[B],
                                                 const double (*O)[B]) {
  double S[B][B];
  rsim::blk::gemm<B>(Di, O, S);
  double* dst = a.ell_val + ell_at(a.cap, B * B, s, 0, l);
#pragma unroll
  for (int r = 0; r < B; ++r)
#pragma unroll
    for (int c = 0; c < B; ++c) {
      if (STREAM) __stcs(&dst[(r * B + c) * ell_es(B * B)], S[r][c]);
      else dst[(r * B + c) * ell_es(B * B)] = S[r][c];
    }
  return rsim::blk::col0_only<B>(&S[0][0]);
}

// 8 lanes per active row: lanes 0..nslot-1 evaluate one Cartesian connection
// each (neighbour properties, PPU terms, raw off-diagonal block), lane 7 owns
// the row: accumulation, the connection terms added in canonical slot order,
// NNC connections, the well, D^{-1}; then every lane stores its scaled block.
// The terms are computed by physics.h flux_terms() and added in the same order
// as flux_conn() in the oracle, so rows are bit-identical.
#ifndef RSIM_K1ROW_MINB
#define RSIM_K1ROW_MINB 4  // b = 1 row kernel: blocks per SM (register cap 64)
#endif
constexpr int LPR = 8;
constexpr int RPB = 256 / LPR;
constexpr int64_t kRowKernelMin = 148 * 2048;  // rows: switch to one thread per row

template <int B>
__global__ void __launch_bounds__(256) k_assemble(const AsmArgs a) {
  __shared__ double sRc[RPB][6][B];
  __shared__ double sDc[RPB][6][B * B];
  __shared__ double sDi[RPB][B * B];
  __shared__ unsigned char sHas[RPB][6];
  const int rg = threadIdx.x / LPR, q = threadIdx.x % LPR;
  const int64_t l = (int64_t)blockIdx.x * RPB + rg;
  const bool valid = l < a.nA;
  double finf = 0.0;
  int64_t i = 0, ix = 0, iy = 0, iz = 0;
  double ui[B];
  rsim::phys::Props<B> Pi;
  if (valid) {
    i = a.act[l];
    const int64_t nxy = (int64_t)a.nx * a.ny;
    ix = i % a.nx; iy = (i / a.nx) % a.ny; iz = i / nxy;
    load_u<B>(a, i, ui);
    rsim::phys::props(a.fl, ui, B == 3 ? a.st[i] : (uint8_t)0, Pi);
  }
  double O[B][B];
  int32_t lcol = -1;
  bool nnc_act = false;  // owner lane: the row has an NNC block with an active column
  if (valid && q < a.nslot) {
    int64_t j;
    double T;
    bool has = false;
    if (cart_nbr(a, i, ix, iy, iz, q, j, T)) {
      double uj[B];
      load_u<B>(a, j, uj);
      const double dp = ui[0] - uj[0];
      const bool up_i = !(dp < 0.0);
      double Rc[B], Dc[B][B];
      if (up_i) {
        rsim::phys::flux_terms<B>(T, dp, true, Pi, Rc, Dc, O);
      } else {
        rsim::phys::Props<B> Pj;
        rsim::phys::props(a.fl, uj, B == 3 ? __ldg(&a.st[j]) : (uint8_t)0, Pj);
        rsim::phys::flux_terms<B>(T, dp, false, Pj, Rc, Dc, O);
      }
#pragma unroll
      for (int e = 0; e < B; ++e) {
        sRc[rg][q][e] = Rc[e];
#pragma unroll
        for (int v = 0; v < B; ++v) sDc[rg][q][e * B + v] = Dc[e][v];
      }
      lcol = __ldg(&a.g2l[j]);
      has = true;
    }
    sHas[rg][q] = has;
    a.ell_col[q * a.cap + l] = lcol;
  }
  __syncwarp();
  if (valid && q == LPR - 1) {
    double R[B], D[B][B], Mo[B];
#pragma unroll
    for (int c = 0; c < B; ++c) Mo[c] = __ldg(&a.mold[i * B + c]);
    rsim::phys::accum_row<B>(a.fl, __ldg(&a.pv[i]), ui[0], Pi, Mo, a.inv_dt, R, D);
    for (int s = 0; s < a.nslot; ++s)
      if (sHas[rg][s]) {
#pragma unroll
        for (int e = 0; e < B; ++e) {
          R[e] = R[e] + sRc[rg][s][e];
#pragma unroll
          for (int v = 0; v < B; ++v) D[e][v] = D[e][v] + sDc[rg][s][e * B + v];
        }
      }
    int32_t q0 = 0, q1 = 0;
    if (a.has_nnc) {
      q0 = __ldg(&a.nptr[i]);
      q1 = __ldg(&a.nptr[i + 1]);
      for (int32_t qq = q0; qq < q1; ++qq) {
        const int64_t j = __ldg(&a.nnbr[qq]);
        double On[B][B];
        conn<B>(a, ui, Pi, j, __ldg(&a.nt[qq]), R, D, On);
        const int32_t lc = __ldg(&a.g2l[j]);
        a.nnc_lcol[qq] = lc;
        nnc_act = nnc_act || lc >= 0;
      }
    }
    rsim::phys::well_row<B>(__ldg(&a.wi[i]), ui[0], a.bhp, Pi, R, D);
    double Di[B][B];
    if (!rsim::blk::inv(D, Di)) {
      atomicMin(&a.dsc->bad_cell, (int32_t)i);
      a.dsc->status = RSIM_ENUM;
#pragma unroll
      for (int r = 0; r < B; ++r)
#pragma unroll
        for (int c = 0; c < B; ++c) Di[r][c] = 0.0;
    }
    double y[B];
    rsim::blk::gemv<B>(Di, R, y);
#pragma unroll
    for (int e = 0; e < B; ++e) {
      a.F_raw[l * B + e] = R[e];
      a.rhs[l * B + e] = -y[e];
      finf = fmax(finf, fabs(R[e]));
    }
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int c = 0; c < B; ++c) sDi[rg][r * B + c] = Di[r][c];
    for (int32_t qq = q0; qq < q1; ++qq) {  // NNC blocks (rare): recompute + scale
      const int64_t j = __ldg(&a.nnbr[qq]);
      if (__ldg(&a.g2l[j]) < 0) continue;
      double On[B][B], Rd[B], Dd[B][B];
#pragma unroll
      for (int e = 0; e < B; ++e) {
        Rd[e] = 0.0;
#pragma unroll
        for (int v = 0; v < B; ++v) Dd[e][v] = 0.0;
      }
      conn<B>(a, ui, Pi, j, __ldg(&a.nt[qq]), Rd, Dd, On);
      store_scaled<B>(&a.nnc_val[(int64_t)qq * B * B], Di, On);
    }
  }
  __syncwarp();
  bool po = false;
  if (valid && q < a.nslot && lcol >= 0) {
    double Di[B][B];
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int c = 0; c < B; ++c) Di[r][c] = sDi[rg][r * B + c];
    po = store_scaled_ell<B, false>(a, q, l, Di, O);
  }
  if (B > 1 || a.has_nnc) {  // lane q of the row group holds slot q's bit, its owner lane the NNC bit
    const unsigned bal = __ballot_sync(0xffffffffu, po);
    const unsigned stored = __ballot_sync(0xffffffffu, valid && q < a.nslot && lcol >= 0);
    const unsigned nnb = __ballot_sync(0xffffffffu, nnc_act);
    const int base = threadIdx.x & 24;
    if (valid && q == 0)
      a.ell_po[l] = (uint8_t)(((bal >> base) & 0x3fu) | (((nnb >> (base + LPR - 1)) & 1u) ? ELL_ROW_NNC : 0u));
    if (B > 1 && (threadIdx.x & 31) == 0 && stored) {
      atomicAdd(&a.dsc->nblk, (unsigned long long)__popc(stored));
      if (bal) atomicAdd(&a.dsc->npo, (unsigned long long)__popc(bal));
    }
  }
  const double wm = warp_max(finf);
  if ((threadIdx.x & 31) == 0 && wm > 0.0) atomic_max_bits(&a.dsc->finf, wm);
}

// One thread per active row (large active sets: memory-bound, the 8-lane
// variant's redundant property evaluations cost more than they hide).
// Every neighbour load (face Υ, u_j, g2l_j, status_j) is issued before any
// arithmetic so a thread keeps ~4·nslot loads in flight; the ELL / residual
// stores are streaming (st.global.cs) so they do not evict the neighbour
// working set from L2.  b = 1 keeps the raw off-diagonal blocks in registers;
// b > 1 recomputes them in a second pass (same physics.h calls => same bits).
// FULL (V_A = all cells): act is the identity, every in-grid neighbour is
// active with local index = global index, so neither act / g2l are read nor
// the structural ELL columns stored (consumers use implicit_col()).
template <int B, bool FULL>
__global__ void __launch_bounds__(256, B == 1 ? RSIM_K1ROW_MINB : 1) k_assemble_row(const AsmArgs a) {
  constexpr bool KEEP = (B == 1);
  __shared__ double wsf[8];
  double finf = 0.0, ff = 0.0;
  uint32_t nblk = 0, npo = 0;
  const int64_t l = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (l < a.nA) {
    const int64_t i = FULL ? l : (int64_t)a.act[l];
    // 32-bit coordinates (n < 2^31, checked at create)
    const uint32_t nxy = (uint32_t)a.nx * (uint32_t)a.ny;
    const uint32_t iz = (uint32_t)i / nxy;
    const uint32_t rem = (uint32_t)i - iz * nxy;
    const uint32_t iy = rem / (uint32_t)a.nx, ix = rem - iy * (uint32_t)a.nx;
    // ---- neighbour indices and all loads up front
    int64_t jn[6];
    bool has[6];
    double Tn[6], un[6][B];
    int32_t gn[6];
    uint8_t sn[6];
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      has[s] = false;
      jn[s] = i;
      Tn[s] = 0.0;
      gn[s] = -1;
      sn[s] = 0;
      if (s >= a.nslot) continue;
      const int k = a.d3 ? s : s + 1;  // 2D skips the -z slot
      switch (k) {
        case 0: has[s] = iz > 0; jn[s] = i - nxy; break;
        case 1: has[s] = iy > 0; jn[s] = i - a.nx; break;
        case 2: has[s] = ix > 0; jn[s] = i - 1; break;
        case 3: has[s] = ix < (uint32_t)a.nx - 1; jn[s] = i + 1; break;
        case 4: has[s] = iy < (uint32_t)a.ny - 1; jn[s] = i + a.nx; break;
        default: has[s] = iz < (uint32_t)a.nz - 1; jn[s] = i + nxy; break;
      }
    }
#pragma unroll
    for (int s = 0; s < 6; ++s)
      if (has[s]) {
        const int k = a.d3 ? s : s + 1;
        const double* tf = (k == 0 || k == 5) ? a.tz : ((k == 1 || k == 4) ? a.ty : a.tx);
        Tn[s] = __ldg(&tf[k < 3 ? jn[s] : i]);  // face Υ stored at the lower cell
        load_u<B>(a, jn[s], un[s]);
        gn[s] = FULL ? (int32_t)jn[s] : __ldg(&a.g2l[jn[s]]);
        if (B == 3) sn[s] = __ldg(&a.st[jn[s]]);
      }
    double ui[B], Mo[B];
    load_u<B>(a, i, ui);
#pragma unroll
    for (int c = 0; c < B; ++c) Mo[c] = __ldg(&a.mold[i * B + c]);
    const double pv = __ldg(&a.pv[i]), wi = __ldg(&a.wi[i]);
    const uint8_t sti = B == 3 ? a.st[i] : (uint8_t)0;
    // ---- arithmetic (canonical order: accumulation, slots ascending, NNC, well)
    rsim::phys::Props<B> Pi;
    rsim::phys::props(a.fl, ui, sti, Pi);
    double R[B], D[B][B];
    rsim::phys::accum_row<B>(a.fl, pv, ui[0], Pi, Mo, a.inv_dt, R, D);
    double Okeep[6][B][B];
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      if (!has[s]) continue;
      double O[B][B];
      const double dp = ui[0] - un[s][0];
      if (!(dp < 0.0)) {
        rsim::phys::flux_conn<B>(Tn[s], dp, true, Pi, R, D, O);
      } else {
        rsim::phys::Props<B> Pj;
        rsim::phys::props(a.fl, un[s], sn[s], Pj);
        rsim::phys::flux_conn<B>(Tn[s], dp, false, Pj, R, D, O);
      }
      if (KEEP)
#pragma unroll
        for (int r = 0; r < B; ++r)
#pragma unroll
          for (int c = 0; c < B; ++c) Okeep[s][r][c] = O[r][c];
    }
    if (!FULL)
#pragma unroll
      for (int s = 0; s < 6; ++s)
        if (s < a.nslot) __stcs(&a.ell_col[s * a.cap + l], has[s] ? gn[s] : -1);
    int32_t q0 = 0, q1 = 0;
    bool nnc_act = false;  // the row has an NNC block with an active column
    if (a.has_nnc) {
      q0 = __ldg(&a.nptr[i]);
      q1 = __ldg(&a.nptr[i + 1]);
      for (int32_t q = q0; q < q1; ++q) {
        const int64_t j = __ldg(&a.nnbr[q]);
        double O[B][B];
        conn<B>(a, ui, Pi, j, __ldg(&a.nt[q]), R, D, O);
        const int32_t lc = __ldg(&a.g2l[j]);
        a.nnc_lcol[q] = lc;
        nnc_act = nnc_act || lc >= 0;
      }
    }
    rsim::phys::well_row<B>(wi, ui[0], a.bhp, Pi, R, D);
    double Di[B][B];
    if (!rsim::blk::inv(D, Di)) {
      atomicMin(&a.dsc->bad_cell, (int32_t)i);
      a.dsc->status = RSIM_ENUM;
#pragma unroll
      for (int r = 0; r < B; ++r)
#pragma unroll
        for (int c = 0; c < B; ++c) Di[r][c] = 0.0;
    }
    double y[B];
    rsim::blk::gemv<B>(Di, R, y);
#pragma unroll
    for (int e = 0; e < B; ++e) {
      if (a.keep_F) __stcs(&a.F_raw[l * B + e], R[e]);
      __stcs(&a.rhs[l * B + e], -y[e]);
      finf = fmax(finf, fabs(R[e]));
    }
    ff = rsim::blk::rowdot<B>(R, R);
    uint32_t pom = 0;
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      if (!has[s] || gn[s] < 0) continue;
      double O[B][B];
      if (KEEP) {
#pragma unroll
        for (int r = 0; r < B; ++r)
#pragma unroll
          for (int c = 0; c < B; ++c) O[r][c] = Okeep[s][r][c];
      } else {
        double Rd[B], Dd[B][B];
#pragma unroll
        for (int e = 0; e < B; ++e) {
          Rd[e] = 0.0;
#pragma unroll
          for (int v = 0; v < B; ++v) Dd[e][v] = 0.0;
        }
        const double dp = ui[0] - un[s][0];
        if (!(dp < 0.0)) {
          rsim::phys::flux_conn<B>(Tn[s], dp, true, Pi, Rd, Dd, O);
        } else {
          rsim::phys::Props<B> Pj;
          rsim::phys::props(a.fl, un[s], sn[s], Pj);
          rsim::phys::flux_conn<B>(Tn[s], dp, false, Pj, Rd, Dd, O);
        }
      }
      ++nblk;
      if (store_scaled_ell<B, true>(a, s, l, Di, O)) pom |= 1u << s;
    }
    if (B > 1 || a.has_nnc) __stcs(&a.ell_po[l], (uint8_t)(pom | (nnc_act ? ELL_ROW_NNC : 0u)));
    npo = __popc(pom);
    for (int32_t q = q0; q < q1; ++q) {
      const int64_t j = __ldg(&a.nnbr[q]);
      if (__ldg(&a.g2l[j]) < 0) continue;
      double O[B][B], Rd[B], Dd[B][B];
#pragma unroll
      for (int e = 0; e < B; ++e) {
        Rd[e] = 0.0;
#pragma unroll
        for (int v = 0; v < B; ++v) Dd[e][v] = 0.0;
      }
      conn<B>(a, ui, Pi, j, __ldg(&a.nt[q]), Rd, Dd, O);
      store_scaled<B>(&a.nnc_val[(int64_t)q * B * B], Di, O);
    }
  }
  const double wm = warp_max(finf);
  if ((threadIdx.x & 31) == 0 && wm > 0.0) atomic_max_bits(&a.dsc->finf, wm);
  if (B > 1) {
    const uint32_t wb = __reduce_add_sync(0xffffffffu, nblk), wp = __reduce_add_sync(0xffffffffu, npo);
    if ((threadIdx.x & 31) == 0 && wb) {
      atomicAdd(&a.dsc->nblk, (unsigned long long)wb);
      if (wp) atomicAdd(&a.dsc->npo, (unsigned long long)wp);
    }
  }
  // canonical chunk partial of (F, F): this block IS local chunk blockIdx.x
  // (256 rows; rows past n_A hold +0.0) — the Krylov init reduces these
  // instead of re-reading F
  const double wsum = warp_tree(ff);
  if ((threadIdx.x & 31) == 0) wsf[threadIdx.x >> 5] = wsum;
  __syncthreads();
  if (threadIdx.x == 0) a.part_f2[blockIdx.x] = tree8(wsf);
}

// FULL set, b = 1, no NNC, nx % 256 == 0, ny % FRY == 0 (config 5, standard
// Newton on single-phase grids): one 256-thread block per tile of 256 (x) ×
// FRY (y) cells of one plane.  The properties of every tile cell and of a
// one-cell halo are evaluated ONCE into shared memory (each needs an exp),
// instead of once per referencing row as in the row kernel (up to 7 per row,
// and warps pay for divergent upwind choices); the ±z neighbours are
// evaluated as in the row kernel.  Same physics.h calls and the same
// canonical order per row => the same bits.  Each tile row is one canonical
// 256-row chunk, so the (F,F) chunk partials come out as in the row kernel.
constexpr int FRY = 4;
template <bool D3>
__global__ void __launch_bounds__(256) k_assemble_full1(const AsmArgs a) {
  // p and ρ per tile/halo cell; dρ/dp = c·ρ and λρ = ρ·(1/μ) are re-formed
  // with the same multiplications props<1> uses (same bits).  Slots are
  // compile-time (no dynamically indexed arrays: nothing goes to local memory).
  __shared__ double su[FRY + 2][258], sA[FRY + 2][258];
  __shared__ double wsf[FRY][8];
  using rsim::phys::Props;
  const int t = threadIdx.x, lane = t & 31;
  const int x0 = blockIdx.x * 256, y0 = blockIdx.y * FRY, z = blockIdx.z;
  const int64_t nxy = (int64_t)a.nx * a.ny;
  const double cf = a.fl.c_f[1], imu = a.fl.inv_mu[1];
  auto rho_of = [&](double p) {
    double ui[1] = {p};
    Props<1> P;
    rsim::phys::props(a.fl, ui, (uint8_t)0, P);
    return P.A[0];
  };
  {
    double pr[FRY + 2];
#pragma unroll
    for (int r = 0; r < FRY + 2; ++r) {  // tile rows + halo rows, thread t = column x0 + t
      const int y = y0 - 1 + r;
      pr[r] = (y >= 0 && y < a.ny) ? __ldg(&a.u[(int64_t)z * nxy + (int64_t)y * a.nx + x0 + t]) : 0.0;
    }
    double ph = 0.0;
    int hr = -1, hc = 0;
    if (t < 2 * (FRY + 2)) {  // x halo columns x0-1 / x0+256
      const int r = t >> 1, y = y0 - 1 + r, x = (t & 1) ? x0 + 256 : x0 - 1;
      if (y >= 0 && y < a.ny && x >= 0 && x < a.nx) {
        hr = r; hc = (t & 1) ? 257 : 0;
        ph = __ldg(&a.u[(int64_t)z * nxy + (int64_t)y * a.nx + x]);
      }
    }
#pragma unroll
    for (int r = 0; r < FRY + 2; ++r) {
      const int y = y0 - 1 + r;
      if (y >= 0 && y < a.ny) { su[r][t + 1] = pr[r]; sA[r][t + 1] = rho_of(pr[r]); }
    }
    if (hr >= 0) { su[hr][hc] = ph; sA[hr][hc] = rho_of(ph); }
  }
  __syncthreads();
  const int x = x0 + t, c = t + 1;
  double finf = 0.0;
  double ty_prev = (y0 > 0) ? __ldg(&a.ty[(int64_t)z * nxy + (int64_t)(y0 - 1) * a.nx + x]) : 0.0;
#pragma unroll 1
  for (int ry = 0; ry < FRY; ++ry) {
    const int y = y0 + ry, r = ry + 1;
    const int64_t i = (int64_t)z * nxy + (int64_t)y * a.nx + x;  // = local row l (full set)
    const bool h0 = D3 && z > 0, h5 = D3 && z < a.nz - 1;
    const double txi = __ldg(&a.tx[i]), tyi = __ldg(&a.ty[i]);
    const double tzi = h5 ? __ldg(&a.tz[i]) : 0.0, tzm = h0 ? __ldg(&a.tz[i - nxy]) : 0.0;
    const double pzm = h0 ? __ldg(&a.u[i - nxy]) : 0.0, pzp = h5 ? __ldg(&a.u[i + nxy]) : 0.0;
    double txl = __shfl_up_sync(0xffffffffu, txi, 1);
    if (lane == 0) txl = x > 0 ? __ldg(&a.tx[i - 1]) : 0.0;
    const double pi = su[r][c], Ai = sA[r][c];
    Props<1> Pi;
    Pi.A[0] = Ai; Pi.dA[0][0] = cf * Ai; Pi.L[0] = Ai * imu; Pi.dL[0][0] = (cf * Ai) * imu;
    double R[1], D[1][1], Mo[1] = {__ldg(&a.mold[i])};
    rsim::phys::accum_row<1>(a.fl, __ldg(&a.pv[i]), pi, Pi, Mo, a.inv_dt, R, D);
    auto cn = [&](double T, double pj, double Aj) -> double {  // neighbour with known ρ
      double Oo[1][1];
      const double dp = pi - pj;
      if (!(dp < 0.0)) {
        rsim::phys::flux_conn<1>(T, dp, true, Pi, R, D, Oo);
      } else {
        Props<1> Pj;
        Pj.A[0] = Aj; Pj.dA[0][0] = cf * Aj; Pj.L[0] = Aj * imu; Pj.dL[0][0] = (cf * Aj) * imu;
        rsim::phys::flux_conn<1>(T, dp, false, Pj, R, D, Oo);
      }
      return Oo[0][0];
    };
    auto cz = [&](double T, double pj) -> double {  // ±z neighbour: ρ evaluated only when it is upwind
      double Oo[1][1];
      const double dp = pi - pj;
      if (!(dp < 0.0)) {
        rsim::phys::flux_conn<1>(T, dp, true, Pi, R, D, Oo);
      } else {
        double uj[1] = {pj};
        Props<1> Pj;
        rsim::phys::props(a.fl, uj, (uint8_t)0, Pj);
        rsim::phys::flux_conn<1>(T, dp, false, Pj, R, D, Oo);
      }
      return Oo[0][0];
    };
    // canonical slot order -z, -y, -x, +x, +y, +z (2D: no z slots)
    double O0 = 0.0, O1 = 0.0, O2 = 0.0, O3 = 0.0, O4 = 0.0, O5 = 0.0;
    const bool h1 = y > 0, h2 = x > 0, h3 = x < a.nx - 1, h4 = y < a.ny - 1;
    if (h0) O0 = cz(tzm, pzm);
    if (h1) O1 = cn(ty_prev, su[r - 1][c], sA[r - 1][c]);
    if (h2) O2 = cn(txl, su[r][c - 1], sA[r][c - 1]);
    if (h3) O3 = cn(txi, su[r][c + 1], sA[r][c + 1]);
    if (h4) O4 = cn(tyi, su[r + 1][c], sA[r + 1][c]);
    if (h5) O5 = cz(tzi, pzp);
    rsim::phys::well_row<1>(__ldg(&a.wi[i]), pi, a.bhp, Pi, R, D);
    double Di[1][1];
    if (!rsim::blk::inv(D, Di)) {
      atomicMin(&a.dsc->bad_cell, (int32_t)i);
      a.dsc->status = RSIM_ENUM;
      Di[0][0] = 0.0;
    }
    double yv[1];
    rsim::blk::gemv<1>(Di, R, yv);
    if (a.keep_F) __stcs(&a.F_raw[i], R[0]);
    __stcs(&a.rhs[i], -yv[0]);
    finf = fmax(finf, fabs(R[0]));
    auto st = [&](int q, bool h, double O) {
      if (!h) return;
      double Oq[1][1] = {{O}}, S[1][1];
      rsim::blk::gemm<1>(Di, Oq, S);
      __stcs(&a.ell_val[(int64_t)q * a.cap + i], S[0][0]);
    };
    if (D3) {
      st(0, h0, O0); st(1, h1, O1); st(2, h2, O2); st(3, h3, O3); st(4, h4, O4); st(5, h5, O5);
    } else {
      st(0, h1, O1); st(1, h2, O2); st(2, h3, O3); st(3, h4, O4);
    }
    const double ws = warp_tree(rsim::blk::rowdot<1>(R, R));
    if (lane == 0) wsf[ry][t >> 5] = ws;
    ty_prev = tyi;
  }
  const double wm = warp_max(finf);
  if (lane == 0 && wm > 0.0) atomic_max_bits(&a.dsc->finf, wm);
  __syncthreads();
  if (t < FRY) {  // canonical chunk partial of each tile row (256 consecutive rows)
    const int64_t row0 = (int64_t)z * nxy + (int64_t)(y0 + t) * a.nx + x0;
    a.part_f2[row0 >> 8] = tree8(wsf[t]);
  }
}

// Old-time accumulation M^n = pv φ(p) A(u) for every cell (set_state / Δt change).
template <int B>
__global__ void k_mold(rsim::phys::Fluid fl, int64_t n, const double* __restrict__ u, const uint8_t* __restrict__ st,
                       const double* __restrict__ pv, double* __restrict__ mold) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double ui[B];
#pragma unroll
  for (int c = 0; c < B; ++c) ui[c] = u[i * B + c];
  rsim::phys::Props<B> P;
  rsim::phys::props(fl, ui, st[i], P);
  double M[B];
  rsim::phys::mass<B>(fl, pv[i], ui[0], P, M);
#pragma unroll
  for (int c = 0; c < B; ++c) mold[i * B + c] = M[c];
}

// debug download of an implicit-column assembly: write the structural columns
__global__ void k_materialize_cols(int32_t nx, int32_t ny, int32_t nz, bool d3, int nslot, int64_t n, int64_t cap,
                                   int32_t* __restrict__ ell_col) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int32_t cl[6];
  implicit_cols(nx, ny, nz, d3, i, cl);
  for (int s = 0; s < nslot; ++s) ell_col[s * cap + i] = cl[s];
}

}  // namespace

int launch_materialize_cols(rsim_gpu_ctx* c) {
  if (!c->cols_implicit) return RSIM_OK;
  k_materialize_cols<<<(c->n + 255) / 256, 256, 0, c->stream>>>(c->nx, c->ny, c->nz, c->d3, c->nslot, c->n,
                                                                c->ell_cap, c->ell_col);
  c->launches++;
  c->cols_implicit = false;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

static bool tile_full1_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("RSIM_NO_TILE_K1");
    v = (e && *e == '1') ? 0 : 1;
  }
  return v == 1;
}

int launch_assemble(rsim_gpu_ctx* c) {
  if (c->nA <= 0) return RSIM_OK;
  AsmArgs a;
  a.fl = rsim::phys::Fluid(c->fl);
  a.dt = c->dt;
  a.inv_dt = 1.0 / c->dt;
  a.bhp = c->bhp;
  a.nx = c->nx; a.ny = c->ny; a.nz = c->nz;
  a.nslot = c->nslot;
  a.nA = c->nA;
  // compact slot stride: the slot slabs of the current system are adjacent
  // (one contiguous ~nslot·n_A·b²·8 B region instead of slabs n apart)
  c->ell_cap = ((c->nA + 31) / 32) * 32;
  a.cap = c->ell_cap;
  a.d3 = c->d3;
  a.has_nnc = c->has_nnc;
  a.tx = c->tx; a.ty = c->ty; a.tz = c->tz; a.pv = c->pv; a.wi = c->wi;
  a.nptr = c->nptr; a.nnbr = c->nnbr; a.nt = c->nt;
  a.u = c->u; a.mold = c->mold; a.st = c->st;
  a.act = c->act; a.g2l = c->g2l;
  a.ell_col = c->ell_col; a.ell_val = c->ell_val; a.ell_po = c->ell_po;
  a.nnc_lcol = c->nnc_lcol; a.nnc_val = c->nnc_val;
  a.F_raw = c->F_raw; a.rhs = c->rhs; a.part_f2 = c->part_f2;
  a.keep_F = c->keep_F;
  a.dsc = c->dsc;
  // small active sets: 8 lanes per row (latency); large: one thread per row (bandwidth)
  c->cols_implicit = false;
  c->f2_parts = c->nA >= kRowKernelMin;  // row kernel: (F,F) as canonical chunk partials
  if (c->nA < kRowKernelMin) {
    const int64_t nblocks = (c->nA + RPB - 1) / RPB;
    switch (c->b) {
      case 1: k_assemble<1><<<nblocks, 256, 0, c->stream>>>(a); break;
      case 2: k_assemble<2><<<nblocks, 256, 0, c->stream>>>(a); break;
      default: k_assemble<3><<<nblocks, 256, 0, c->stream>>>(a); break;
    }
  } else {
    const int64_t nblocks = (c->nA + 255) / 256;
    const bool full = c->nA == c->n;
    c->cols_implicit = full;
    if (full && c->b == 1 && !c->has_nnc && c->nx % 256 == 0 && c->ny % FRY == 0 && tile_full1_enabled()) {
      if (c->d3) k_assemble_full1<true><<<dim3(c->nx / 256, c->ny / FRY, c->nz), 256, 0, c->stream>>>(a);
      else k_assemble_full1<false><<<dim3(c->nx / 256, c->ny / FRY, c->nz), 256, 0, c->stream>>>(a);
      c->launches++;
      RSIM_CUDA(cudaGetLastError());
      return RSIM_OK;
    }
    switch (c->b * 2 + (full ? 1 : 0)) {
      case 2: k_assemble_row<1, false><<<nblocks, 256, 0, c->stream>>>(a); break;
      case 3: k_assemble_row<1, true><<<nblocks, 256, 0, c->stream>>>(a); break;
      case 4: k_assemble_row<2, false><<<nblocks, 256, 0, c->stream>>>(a); break;
      case 5: k_assemble_row<2, true><<<nblocks, 256, 0, c->stream>>>(a); break;
      case 6: k_assemble_row<3, false><<<nblocks, 256, 0, c->stream>>>(a); break;
      default: k_assemble_row<3, true><<<nblocks, 256, 0, c->stream>>>(a); break;
    }
  }
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

int launch_mold(rsim_gpu_ctx* c) {
  const int th = 256;
  const int64_t blocks = (c->n + th - 1) / th;
  switch (c->b) {
    case 1: k_mold<1><<<blocks, th, 0, c->stream>>>(rsim::phys::Fluid(c->fl), c->n, c->u, c->st, c->pv, c->mold); break;
    case 2: k_mold<2><<<blocks, th, 0, c->stream>>>(rsim::phys::Fluid(c->fl), c->n, c->u, c->st, c->pv, c->mold); break;
    default: k_mold<3><<<blocks, th, 0, c->stream>>>(rsim::phys::Fluid(c->fl), c->n, c->u, c->st, c->pv, c->mold); break;
  }
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}
