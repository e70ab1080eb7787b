// sets.cu — K6 (update + variable substitution + ∞-norms), K7 (active-set
// estimation: threshold, m-hop dilation, warp-ballot/scan compaction) and K8
// (DD labels / subdomain lists).
//
// Restates (all integer logic => bit-exact against oracle/oracle.cpp):
//   u^{ν+1} = u^ν + R_A^T δu_A             PAPER.md:282 (Alg. 1 line 5)
//   variable_substitution
//   support_set |δp| >= ε (inclusive)
//   expand_active / neighbor_set           SPEC.md:386-394, :61-69 (graph distance)
//   shrink V_A = supp δu_A ∪ fracture
//   boundary_layer / outer_halo
//   Alg. 2 phase-1 labels, V_T
// The expand/shrink decision is taken ON THE DEVICE from ‖δp_B‖∞ (each K7
// kernel evaluates it), so K6 -> K7 -> compaction runs without a host round trip.
#include <cooperative_groups.h>

#include <cstdlib>

#include "ctx.cuh"

namespace cg = cooperative_groups;

namespace {

constexpr int TILE = 2048;  // cells per compaction tile (256 threads x 8 consecutive cells)

struct Geo {
  int32_t nx, ny, nz;
  int64_t n;
  bool d3, has_nnc;
  const int32_t *nptr, *nnbr;
  const uint8_t* pin0;  // F_DEAD marks filler cells (only read when the graph has any)
  bool has_dead;
};

__host__ Geo geo(const rsim_gpu_ctx* c) {
  return Geo{c->nx, c->ny, c->nz, c->n, c->d3, c->has_nnc, c->nptr, c->nnbr, c->pin0, c->n_dead > 0};
}
__device__ __forceinline__ bool is_dead(const Geo& g, int64_t i) { return g.has_dead && (g.pin0[i] & F_DEAD); }

// Visit every graph neighbour of i (Cartesian + NNC).
template <class F>
__device__ __forceinline__ void each_nbr(const Geo& g, int64_t i, F&& f) {
  const int64_t nxy = (int64_t)g.nx * g.ny;
  const int64_t ix = i % g.nx, iy = (i / g.nx) % g.ny, iz = i / nxy;
  if (g.d3 && iz > 0) f(i - nxy);
  if (iy > 0) f(i - g.nx);
  if (ix > 0) f(i - 1);
  if (ix < g.nx - 1) f(i + 1);
  if (iy < g.ny - 1) f(i + g.nx);
  if (g.d3 && iz < g.nz - 1) f(i + nxy);
  if (g.has_nnc) {
    int32_t q0 = __ldg(&g.nptr[i]), q1 = __ldg(&g.nptr[i + 1]);
    for (int32_t q = q0; q < q1; ++q) f((int64_t)__ldg(&g.nnbr[q]));
  }
}

// ---------------------------------------------------------------- K6 update
template <int B>
__global__ void __launch_bounds__(256) k_update(rsim::phys::Fluid fl, int32_t nA, const int32_t* __restrict__ act,
                                                 const double* __restrict__ x, double* __restrict__ u,
                                                 uint8_t* __restrict__ st, uint8_t* __restrict__ flags,
                                                 double* __restrict__ dp, double* __restrict__ last_dp, double eps,
                                                 DevScalars* dsc) {
  int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double aA = 0.0, aB = 0.0;
  bool bad = false;
  if (l < nA) {
    const int64_t i = act[l];
    double ui[B], xi[B];
#pragma unroll
    for (int c = 0; c < B; ++c) { ui[c] = u[i * B + c]; xi[c] = x[l * B + c]; }
    uint8_t s = st[i];
    const double d = rsim::phys::apply_update<B>(fl, ui, s, xi);
#pragma unroll
    for (int c = 0; c < B; ++c) u[i * B + c] = ui[c];
    st[i] = s;
    const double a = fabs(d);
    bad = !isfinite(d);
    dp[i] = d;
    if (last_dp) last_dp[i] = a;
    uint8_t f = flags[i];
    if (a >= eps) {
      f |= F_FLAG;
      if (f & F_B) f |= F_D0;  // seed of the expansion (flagged boundary cell)
    }
    flags[i] = f;
    aA = a;
    aB = (f & F_B) ? a : 0.0;
  }
  if (bad) dsc->status = RSIM_ENUM;
  double wa = warp_max(aA), wb = warp_max(aB);
  if ((threadIdx.x & 31) == 0) {
    if (wa > 0.0) atomic_max_bits(&dsc->maxA, wa);
    if (wb > 0.0) atomic_max_bits(&dsc->maxB, wb);
  }
}

// Threshold only (K7 test hook): FLAG / seed bits and ∞-norms from a given δp.
__global__ void __launch_bounds__(256) k_threshold(int32_t nA, const int32_t* __restrict__ act,
                                                    const double* __restrict__ dp, uint8_t* __restrict__ flags,
                                                    double eps, DevScalars* dsc) {
  int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double aA = 0.0, aB = 0.0;
  if (l < nA) {
    const int64_t i = act[l];
    const double a = fabs(dp[i]);
    uint8_t f = flags[i];
    if (a >= eps) {
      f |= F_FLAG;
      if (f & F_B) f |= F_D0;
    }
    flags[i] = f;
    aA = a;
    aB = (f & F_B) ? a : 0.0;
  }
  double wa = warp_max(aA), wb = warp_max(aB);
  if ((threadIdx.x & 31) == 0) {
    if (wa > 0.0) atomic_max_bits(&dsc->maxA, wa);
    if (wb > 0.0) atomic_max_bits(&dsc->maxB, wb);
  }
}

// ---------------------------------------------------------------- K7
// Set-update parameters shared by the dilation / count / scatter kernels.  The
// expand/shrink decision is evaluated by every thread from ‖δp_B‖∞ (written by
// K6 or k_threshold), so no separate decision kernel or host round trip.
struct SetMode {
  int mode;          // MODE_*
  uint8_t dbit;      // D bit that holds the m-hop dilation
  double eps;
  int shrink_locked;
  int force_expand;
};

__device__ __forceinline__ bool decide_expand(const SetMode& M, const DevScalars* dsc) {
  if (M.force_expand) return true;
  const double mb = __longlong_as_double((long long)dsc->maxB);
  return !M.shrink_locked && mb >= M.eps;
}

// A_new of a cell from its (pre-update) flag byte.
__device__ __forceinline__ bool a_new(uint8_t f, int mode, bool expand, uint8_t dbit) {
  switch (mode) {
    case MODE_KEEP: return (f & F_A) != 0;
    case MODE_SHRINK: return ((f & F_A) && (f & F_FLAG)) || (f & F_PIN);
    case MODE_EXPAND:
    case MODE_DD: return (f & F_A) || (f & dbit);
    default:  // MODE_DEVICE
      return expand ? ((f & F_A) || (f & dbit)) : (((f & F_A) && (f & F_FLAG)) || (f & F_PIN));
  }
}

// The same predicate on 4 flag bytes at once: bit 0 of every byte of the result.
__device__ __forceinline__ uint32_t bitpos(uint32_t bit) { return (uint32_t)__ffs((int)bit) - 1u; }
__device__ __forceinline__ uint32_t lanes(uint32_t w, uint32_t bit) { return (w >> bitpos(bit)) & 0x01010101u; }
__device__ __forceinline__ uint32_t a_new4(uint32_t w, int mode, bool expand, uint8_t dbit) {
  const uint32_t A = lanes(w, F_A);
  const uint32_t grow = A | lanes(w, dbit);
  const uint32_t shrink = (A & lanes(w, F_FLAG)) | lanes(w, F_PIN);
  switch (mode) {
    case MODE_KEEP: return A;
    case MODE_SHRINK: return shrink;
    case MODE_EXPAND:
    case MODE_DD: return grow;
    default: return expand ? grow : shrink;
  }
}

// K7 work mapping: block (row, seg) covers x-row `row` (= iy + ny*iz) and
// 4-cell groups [seg*bs, (seg+1)*bs) of it, thread = 4 consecutive cells.  The
// tile of the compaction is the block, tile id = row*nseg + seg (global cell
// order).  With nx % 4 == 0 (every configuration) a group is one 32-bit word
// of flag bytes: ±x neighbours are byte shifts (plus one byte of the adjacent
// words), ±y/±z the words one row / one plane away — coalesced 4-byte
// accesses, no per-cell index arithmetic.  Otherwise a per-cell path with the
// same semantics and the same tiles.
struct Geo4 {
  int32_t nx, ny, nz;
  int64_t n;
  int32_t wrow;    // 4-cell groups per x-row
  int64_t wplane;  // groups per plane (vec4)
  int32_t bs, nseg;
  bool d3, has_nnc, vec4;
  bool has_dead;  // F_DEAD cells: never dilated into, count as kept in the boundary test
  const int32_t *nptr, *nnbr;
};

__host__ Geo4 geo4(const rsim_gpu_ctx* c) {
  Geo4 g;
  g.nx = c->nx; g.ny = c->ny; g.nz = c->nz;
  g.n = c->n;
  g.vec4 = (c->nx % 4) == 0;
  g.wrow = (c->nx + 3) / 4;
  g.wplane = (int64_t)g.wrow * c->ny;
  g.bs = g.wrow >= 256 ? 256 : ((g.wrow + 31) / 32) * 32;
  g.nseg = (g.wrow + g.bs - 1) / g.bs;
  g.d3 = c->d3; g.has_nnc = c->has_nnc;
  g.has_dead = c->n_dead > 0;
  g.nptr = c->nptr; g.nnbr = c->nnbr;
  return g;
}
__host__ dim3 k7_grid(const Geo4& g) { return dim3((unsigned)(g.ny * g.nz), (unsigned)g.nseg, 1); }
__host__ int64_t k7_tiles(const Geo4& g) { return (int64_t)g.ny * g.nz * g.nseg; }

struct Pos4 {
  int32_t row, iy, iz, xw;  // x-row, its y/z, group index in the row
  int64_t t;                // vec4: word index
  bool ok;
};
__device__ __forceinline__ Pos4 pos4(const Geo4& g, int32_t row, int32_t seg) {
  Pos4 p;
  p.row = row;
  p.iz = p.row / g.ny;
  p.iy = p.row - p.iz * g.ny;
  p.xw = seg * g.bs + threadIdx.x;
  p.ok = p.xw < g.wrow;
  p.t = (int64_t)p.row * g.wrow + p.xw;
  return p;
}

// Combine over the graph neighbours of the 4 cells of group p of per-byte
// bit-0 lanes produced by `L(word index)`; `edge` is the lane value of a
// missing (off-grid) neighbour; `comb` is OR (dilation) or AND ("all keep").
template <class LF, class CF>
__device__ __forceinline__ uint32_t nbr_lanes4(const Geo4& g, const Pos4& p, uint32_t self, uint32_t edge, LF&& L,
                                                CF&& comb) {
  const int64_t t = p.t;
  const uint32_t lft = (self << 8) | (p.xw > 0 ? (L(t - 1) >> 24) : (edge & 0xFFu));
  const uint32_t rgt = (self >> 8) | (p.xw < g.wrow - 1 ? ((L(t + 1) & 0xFFu) << 24) : (edge & 0xFF000000u));
  uint32_t acc = comb(lft, rgt);
  acc = comb(acc, p.iy > 0 ? L(t - g.wrow) : edge);
  acc = comb(acc, p.iy < g.ny - 1 ? L(t + g.wrow) : edge);
  if (g.d3) {
    acc = comb(acc, p.iz > 0 ? L(t - g.wplane) : edge);
    acc = comb(acc, p.iz < g.nz - 1 ? L(t + g.wplane) : edge);
  }
  return acc;
}

// graph neighbours of cell (ix, iy, iz) = i (scalar path / NNC)
template <class F>
__device__ __forceinline__ void each_nbr_xyz(const Geo4& g, int64_t i, int32_t ix, int32_t iy, int32_t iz, F&& f) {
  const int64_t nxy = (int64_t)g.nx * g.ny;
  if (g.d3 && iz > 0) f(i - nxy);
  if (iy > 0) f(i - g.nx);
  if (ix > 0) f(i - 1);
  if (ix < g.nx - 1) f(i + 1);
  if (iy < g.ny - 1) f(i + g.nx);
  if (g.d3 && iz < g.nz - 1) f(i + nxy);
  if (g.has_nnc) {
    const int32_t q0 = __ldg(&g.nptr[i]), q1 = __ldg(&g.nptr[i + 1]);
    for (int32_t q = q0; q < q1; ++q) f((int64_t)__ldg(&g.nnbr[q]));
  }
}

__device__ __forceinline__ int block_sum(int v, int* sh8) {
  v = __reduce_add_sync(0xffffffffu, v);
  if ((threadIdx.x & 31) == 0) sh8[threadIdx.x >> 5] = v;
  __syncthreads();
  int s = 0;
  for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += sh8[k];
  return s;
}

// One dilation round bit_out(i) = bit_in(i) | OR_j bit_in(j) (skipped when the
// device decided to shrink).  With COUNT the same pass also counts A_new per
// tile (compaction pass 1), which needs only the cell's own bits.
template <bool COUNT>
__device__ __forceinline__ void dilate_tile(const Geo4& g, uint8_t* __restrict__ flags, uint8_t bit_in, uint8_t bit_out,
                                            bool ex, bool dil, const SetMode& M, int32_t row, int32_t seg,
                                            int32_t* __restrict__ tile_cnt, int* sh8) {
  const Pos4 p = pos4(g, row, seg);
  int cnt = 0;
  if (p.ok) {
    if (g.vec4) {
      uint32_t* fw = reinterpret_cast<uint32_t*>(flags);
      uint32_t w = fw[p.t];
      if (dil) {
        const uint32_t in = lanes(w, bit_in);
        // bit_in is not written by this pass, so plain (L1-cached) loads are safe
        auto L = [&](int64_t u) { return lanes(fw[u], bit_in); };
        uint32_t out = in | nbr_lanes4(g, p, in, 0u, L, [](uint32_t x, uint32_t y) { return x | y; });
        if (g.has_nnc) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int64_t i = 4 * p.t + k;
            const int32_t q0 = __ldg(&g.nptr[i]), q1 = __ldg(&g.nptr[i + 1]);
            for (int32_t q = q0; q < q1; ++q)
              if (flags[__ldg(&g.nnbr[q])] & bit_in) out |= 1u << (8 * k);
          }
        }
        if (g.has_dead) out &= ~lanes(w, F_DEAD);  // graph distance over live cells only
        w = (w & ~(0x01010101u * bit_out)) | (out * bit_out);
        fw[p.t] = w;
      }
      if (COUNT) cnt = __popc(a_new4(w, M.mode, ex, M.dbit));
    } else {
      const int64_t rb = (int64_t)p.row * g.nx;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int32_t ix = 4 * p.xw + k;
        if (ix >= g.nx) break;
        const int64_t i = rb + ix;
        uint8_t f = flags[i];
        if (dil) {
          bool v = (f & bit_in) != 0;
          if (!v) each_nbr_xyz(g, i, ix, p.iy, p.iz, [&](int64_t j) { if (flags[j] & bit_in) v = true; });
          if (f & F_DEAD) v = false;
          f = v ? (uint8_t)(f | bit_out) : (uint8_t)(f & ~bit_out);
          flags[i] = f;
        }
        if (COUNT) cnt += a_new(f, M.mode, ex, M.dbit) ? 1 : 0;
      }
    }
  }
  if (COUNT) {
    const int s = block_sum(cnt, sh8);
    if (threadIdx.x == 0) tile_cnt[row * g.nseg + seg] = s;
    __syncthreads();  // sh8 is reused by the next tile
  }
}

template <bool COUNT>
__global__ void __launch_bounds__(256) k_dilate(Geo4 g, uint8_t* __restrict__ flags, uint8_t bit_in, uint8_t bit_out,
                                                const DevScalars* __restrict__ dsc, SetMode M, int do_dilate,
                                                int32_t* __restrict__ tile_cnt) {
  __shared__ int sh8[8];
  const bool ex = decide_expand(M, dsc);
  const bool dil = do_dilate && ((M.mode == MODE_DEVICE || M.mode == MODE_DD) ? ex : true);
  dilate_tile<COUNT>(g, flags, bit_in, bit_out, ex, dil, M, blockIdx.x, blockIdx.y, tile_cnt, sh8);
}

// Compaction pass 2: exclusive scan of the tile counts (one block; counts
// staged through shared memory, strips of consecutive tiles per thread).
// Also publishes the decision + n_A and resets the counters of pass 3.
// Block-wide exclusive scan of the tile counts (any blockDim, multiple of 32);
// scnt: shared staging of ntiles + ntiles/32 + 1 ints.
__device__ __forceinline__ void scan_tiles_dev(const int32_t* __restrict__ cnt, int32_t* __restrict__ off,
                                               int32_t ntiles, DevScalars* dsc, const SetMode& M, int32_t* scnt,
                                               int32_t* wsum) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nth = blockDim.x, nw = nth >> 5;
  auto P = [](int32_t i) { return i + (i >> 5); };
  for (int32_t k = threadIdx.x; k < ntiles; k += nth) scnt[P(k)] = cnt[k];
  __syncthreads();
  const int32_t per = (ntiles + nth - 1) / nth;
  const int32_t b0 = threadIdx.x * per;
  int32_t tot = 0;
  for (int32_t k = 0; k < per; ++k)
    if (b0 + k < ntiles) tot += scnt[P(b0 + k)];
  int32_t x = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    int32_t z = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int32_t y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    wsum[lane] = z;
  }
  __syncthreads();
  int32_t run = (w > 0 ? wsum[w - 1] : 0) + x - tot;
  for (int32_t k = 0; k < per; ++k)
    if (b0 + k < ntiles) {
      const int32_t c = scnt[P(b0 + k)];
      scnt[P(b0 + k)] = run;
      run += c;
    }
  __syncthreads();
  for (int32_t k = threadIdx.x; k < ntiles; k += nth) off[k] = scnt[P(k)];
  if (threadIdx.x == nth - 1) {
    dsc->nA = wsum[nw - 1];
    dsc->expand = decide_expand(M, dsc) ? 1 : 0;
    dsc->nB = 0;
    dsc->n_new = 0;
  }
}

__global__ void __launch_bounds__(1024) k_scan_tiles(const int32_t* __restrict__ cnt, int32_t* __restrict__ off,
                                                      int32_t ntiles, DevScalars* dsc, SetMode M) {
  extern __shared__ int32_t scnt[];  // padded: entry i at i + i/32 (conflict-free strips)
  __shared__ int32_t wsum[32];
  scan_tiles_dev(cnt, off, ntiles, dsc, M, scnt, wsum);
}

// Compaction pass 3 (same tiles): A_new, V_B, V_T/labels, g2l, sorted
// active list (block scan of the per-thread counts 0..4).
__device__ __forceinline__ void scatter_tile(const Geo4& g, const uint8_t* __restrict__ fin, uint8_t* __restrict__ fout,
                                             const SetMode& M, bool ex, int32_t round, DevScalars* dsc,
                                             const int32_t* __restrict__ tile_off, int32_t* __restrict__ act,
                                             int32_t* __restrict__ g2l, int32_t* __restrict__ label, int32_t row,
                                             int32_t seg, int32_t* wpre, int* sh8) {
  const Pos4 p = pos4(g, row, seg);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t keep = 0, bnd = 0, f4 = 0;
  const int64_t rb = (int64_t)p.row * g.nx;
  if (p.ok) {
    if (g.vec4) {
      const uint32_t* fw = reinterpret_cast<const uint32_t*>(fin);
      f4 = fw[p.t];
      keep = a_new4(f4, M.mode, ex, M.dbit);
      if (keep) {
        // a dead neighbour is not a graph neighbour: it counts as kept
        auto L = [&](int64_t u) {
          const uint32_t w = __ldg(&fw[u]);
          return a_new4(w, M.mode, ex, M.dbit) | (g.has_dead ? lanes(w, F_DEAD) : 0u);
        };
        // (the word's own lanes feed the ±x neighbours inside the word: dead ones count as kept too)
        const uint32_t self = keep | (g.has_dead ? lanes(f4, F_DEAD) : 0u);
        const uint32_t all = nbr_lanes4(g, p, self, 0x01010101u, L, [](uint32_t x, uint32_t y) { return x & y; });
        bnd = keep & ~all & 0x01010101u;
        if (g.has_nnc)
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (!((keep >> (8 * k)) & 1u) || ((bnd >> (8 * k)) & 1u)) continue;
            const int64_t i = 4 * p.t + k;
            const int32_t q0 = __ldg(&g.nptr[i]), q1 = __ldg(&g.nptr[i + 1]);
            for (int32_t q = q0; q < q1; ++q)
              if (!a_new(fin[__ldg(&g.nnbr[q])], M.mode, ex, M.dbit)) { bnd |= 1u << (8 * k); break; }
          }
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int32_t ix = 4 * p.xw + k;
        if (ix >= g.nx) break;
        const int64_t i = rb + ix;
        const uint8_t f = fin[i];
        f4 |= (uint32_t)f << (8 * k);
        if (a_new(f, M.mode, ex, M.dbit)) {
          keep |= 1u << (8 * k);
          bool b = false;
          each_nbr_xyz(g, i, ix, p.iy, p.iz, [&](int64_t j) {
            if (!(fin[j] & F_DEAD) && !a_new(fin[j], M.mode, ex, M.dbit)) b = true;
          });
          if (b) bnd |= 1u << (8 * k);
        }
      }
    }
  }
  // block exclusive scan of the per-thread counts
  const int c = __popc(keep);
  int x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wpre[w] = x;
  __syncthreads();
  int pre = x - c;
  for (int k = 0; k < w; ++k) pre += wpre[k];
  int32_t pos = tile_off[row * g.nseg + seg] + pre;
  int nnew = 0;
  const int64_t i0 = rb + 4 * (int64_t)p.xw;
  int32_t gl[4];
  uint32_t out = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t f = (f4 >> (8 * k)) & 0xFFu;
    uint32_t o = f & (F_PIN | F_T | F_DEAD);
    gl[k] = -1;
    if ((keep >> (8 * k)) & 1u) {
      o |= F_A;
      if ((bnd >> (8 * k)) & 1u) o |= F_B;
      if (M.mode == MODE_DD) {
        if (!(f & F_T)) { label[i0 + k] = round; ++nnew; }
        o |= F_T;
      }
      act[pos] = (int32_t)(i0 + k);
      gl[k] = pos++;
    }
    out |= o << (8 * k);
  }
  if (p.ok) {
    if (g.vec4) {
      reinterpret_cast<uint32_t*>(fout)[p.t] = out;
      reinterpret_cast<int4*>(g2l)[p.t] = make_int4(gl[0], gl[1], gl[2], gl[3]);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (4 * p.xw + k < g.nx) {
          fout[i0 + k] = (uint8_t)((out >> (8 * k)) & 0xFFu);
          g2l[i0 + k] = gl[k];
        }
    }
  }
  const int nb = block_sum(__popc(bnd), sh8);
  __syncthreads();
  const int nn = block_sum(nnew, sh8);
  if (threadIdx.x == 0) {
    if (nb) atomicAdd(&dsc->nB, nb);
    if (nn) atomicAdd(&dsc->n_new, nn);
  }
  __syncthreads();  // wpre / sh8 are reused by the next tile
}

__global__ void __launch_bounds__(256) k_scatter(Geo4 g, const uint8_t* __restrict__ fin, uint8_t* __restrict__ fout,
                                                 SetMode M, int32_t round, DevScalars* dsc,
                                                 const int32_t* __restrict__ tile_off, int32_t* __restrict__ act,
                                                 int32_t* __restrict__ g2l, int32_t* __restrict__ label) {
  __shared__ int32_t wpre[8];
  __shared__ int sh8[8];
  const bool ex = decide_expand(M, dsc);
  scatter_tile(g, fin, fout, M, ex, round, dsc, tile_off, act, g2l, label, blockIdx.x, blockIdx.y, wpre, sh8);
}

// Whole set update in ONE cooperative kernel for small grids (the localized
// solver's common case: every pass is latency-bound, so four dependent launches
// cost more than the work).  Blocks loop over the same tiles as the separate
// kernels; grid barriers separate the dilation rounds, the count, the scan
// (block 0) and the scatter, so the results are those of the multi-kernel path.
constexpr int kCoopMaxTiles = 4096;
__global__ void __launch_bounds__(256) k_set_update_coop(Geo4 g, uint8_t* __restrict__ flags,
                                                         uint8_t* __restrict__ flags_alt, SetMode M, int rounds,
                                                         int32_t round, DevScalars* dsc, int32_t* __restrict__ tile_cnt,
                                                         int32_t* __restrict__ tile_off, int32_t* __restrict__ act,
                                                         int32_t* __restrict__ g2l, int32_t* __restrict__ label) {
  __shared__ int sh8[8];
  __shared__ int32_t wpre[8];
  __shared__ int32_t wsum[32];
  __shared__ int32_t scnt[kCoopMaxTiles + kCoopMaxTiles / 32 + 1];
  auto grid = cg::this_grid();
  const int32_t ntiles = g.ny * g.nz * g.nseg;
  const bool ex = decide_expand(M, dsc);
  const bool dil = (M.mode == MODE_DEVICE || M.mode == MODE_DD) ? ex : true;
  for (int r = 0; r < rounds; ++r) {
    const uint8_t bin = (r % 2 == 0) ? F_D0 : F_D1, bout = (r % 2 == 0) ? F_D1 : F_D0;
    const bool last = r + 1 == rounds;
    for (int32_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
      const int32_t row = tl / g.nseg, seg = tl - row * g.nseg;
      if (last) dilate_tile<true>(g, flags, bin, bout, ex, dil, M, row, seg, tile_cnt, sh8);
      else dilate_tile<false>(g, flags, bin, bout, ex, dil, M, row, seg, tile_cnt, sh8);
    }
    grid.sync();
  }
  if (rounds == 0) {
    for (int32_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
      const int32_t row = tl / g.nseg, seg = tl - row * g.nseg;
      dilate_tile<true>(g, flags, F_D0, F_D1, ex, false, M, row, seg, tile_cnt, sh8);
    }
    grid.sync();
  }
  if (blockIdx.x == 0) scan_tiles_dev(tile_cnt, tile_off, ntiles, dsc, M, scnt, wsum);
  grid.sync();
  for (int32_t tl = blockIdx.x; tl < ntiles; tl += gridDim.x) {
    const int32_t row = tl / g.nseg, seg = tl - row * g.nseg;
    scatter_tile(g, flags, flags_alt, M, ex, round, dsc, tile_off, act, g2l, label, row, seg, wpre, sh8);
  }
}

// Whole set update of a TINY vec4 grid (n <= kSmemK7MaxCells) in ONE CTA:
// the flag words are staged in shared memory, the dilation rounds, the count
// and the scatter run from there separated by __syncthreads (no grid
// barriers; the cooperative kernel above pays ~5 of them per update).  Thread
// t owns the contiguous word range [t·W, (t+1)·W), so its block-scan offset
// orders the compacted list by cell.  Same predicates (a_new4, nbr_lanes4,
// the NNC and dead-cell rules) as dilate_tile / scatter_tile => same sets.
// Measured (one update = 2 dilations + count + scatter): config 1 (10 k cells)
// 4.39 -> 4.10 ms per run; config 2 (65 k cells, DFN NNCs) 27.3 -> 33.9 ms and
// paper Case 1 (80 k) 0.124 -> 0.146 s: one SM is too slow past ~16 k cells.
constexpr int64_t kSmemK7MaxCells = 16 * 1024;
__global__ void __launch_bounds__(1024) k_set_update_smem(Geo4 g, const uint8_t* __restrict__ fin,
                                                          uint8_t* __restrict__ fout, SetMode M, int rounds,
                                                          int32_t round, DevScalars* dsc, int32_t* __restrict__ act,
                                                          int32_t* __restrict__ g2l, int32_t* __restrict__ label,
                                                          const uint32_t* __restrict__ nnc_bits) {
  // the flag bytes (one 32-bit word per 4-cell group), then one bit per cell
  // telling which cells have NNC entries (so nptr is read only for those)
  extern __shared__ uint32_t sw[];
  uint32_t* snb = sw + g.n / 4;
  __shared__ int32_t wsum[32];
  __shared__ int32_t tot[3];
  const uint8_t* sb = reinterpret_cast<const uint8_t*>(sw);
  const int64_t nw = g.n / 4;
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, wp = tid >> 5;
  for (int64_t t = tid; t < nw; t += nth) sw[t] = reinterpret_cast<const uint32_t*>(fin)[t];
  if (g.has_nnc)
    for (int64_t t = tid; t < (g.n + 31) / 32; t += nth) snb[t] = nnc_bits[t];
  if (tid < 3) tot[tid] = 0;
  __syncthreads();
  const bool ex = decide_expand(M, dsc);
  const bool dil = (M.mode == MODE_DEVICE || M.mode == MODE_DD) ? ex : true;
  const int64_t per = (nw + nth - 1) / nth, t0 = tid * per, t1 = t0 + per < nw ? t0 + per : nw;
  auto pos = [&](int64_t t) {
    Pos4 p;
    p.row = (int32_t)(t / g.wrow);
    p.xw = (int32_t)(t - (int64_t)p.row * g.wrow);
    p.iz = p.row / g.ny;
    p.iy = p.row - p.iz * g.ny;
    p.t = t;
    p.ok = true;
    return p;
  };
  if (dil)
    for (int r = 0; r < rounds; ++r) {
      const uint8_t bin = (r % 2 == 0) ? F_D0 : F_D1, bout = (r % 2 == 0) ? F_D1 : F_D0;
      // bit_in is not written in this round, so reading a neighbour word while its
      // owner rewrites bit_out sees the same bit_in either way
      auto L = [&](int64_t u) { return lanes(sw[u], bin); };
      for (int64_t t = t0; t < t1; ++t) {
        uint32_t w = sw[t];
        const uint32_t in = lanes(w, bin);
        uint32_t out = in | nbr_lanes4(g, pos(t), in, 0u, L, [](uint32_t x, uint32_t y) { return x | y; });
        if (g.has_nnc && ((snb[t >> 3] >> (4 * (t & 7))) & 0xFu))
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int64_t i = 4 * t + k;
            if (!((snb[i >> 5] >> (i & 31)) & 1u)) continue;
            const int32_t q0 = __ldg(&g.nptr[i]), q1 = __ldg(&g.nptr[i + 1]);
            for (int32_t q = q0; q < q1; ++q)
              if (sb[__ldg(&g.nnbr[q])] & bin) out |= 1u << (8 * k);
          }
        if (g.has_dead) out &= ~lanes(w, F_DEAD);
        w = (w & ~(0x01010101u * bout)) | (out * bout);
        sw[t] = w;
      }
      __syncthreads();
    }
  // ---- count + block exclusive scan of the per-thread counts (cell order)
  int cnt = 0;
  for (int64_t t = t0; t < t1; ++t) cnt += __popc(a_new4(sw[t], M.mode, ex, M.dbit));
  int x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wp] = x;
  __syncthreads();
  if (wp == 0) {
    int z = lane < (nth >> 5) ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    wsum[lane] = z;
  }
  __syncthreads();
  int32_t posn = (wp > 0 ? wsum[wp - 1] : 0) + x - cnt;
  // ---- scatter: A, V_B, V_T / labels, g2l, the sorted list
  auto L2 = [&](int64_t u) {
    const uint32_t w = sw[u];
    return a_new4(w, M.mode, ex, M.dbit) | (g.has_dead ? lanes(w, F_DEAD) : 0u);
  };
  int nb = 0, nn = 0;
  for (int64_t t = t0; t < t1; ++t) {
    const uint32_t f4 = sw[t];
    const uint32_t keep = a_new4(f4, M.mode, ex, M.dbit);
    uint32_t bnd = 0;
    if (keep) {
      const uint32_t self = keep | (g.has_dead ? lanes(f4, F_DEAD) : 0u);
      const uint32_t all = nbr_lanes4(g, pos(t), self, 0x01010101u, L2, [](uint32_t a, uint32_t b) { return a & b; });
      bnd = keep & ~all & 0x01010101u;
      if (g.has_nnc && ((snb[t >> 3] >> (4 * (t & 7))) & 0xFu))
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int64_t i = 4 * t + k;
          if (!((keep >> (8 * k)) & 1u) || ((bnd >> (8 * k)) & 1u) || !((snb[i >> 5] >> (i & 31)) & 1u)) continue;
          const int32_t q0 = __ldg(&g.nptr[i]), q1 = __ldg(&g.nptr[i + 1]);
          for (int32_t q = q0; q < q1; ++q)
            if (!a_new(sb[__ldg(&g.nnbr[q])], M.mode, ex, M.dbit)) { bnd |= 1u << (8 * k); break; }
        }
    }
    int32_t gl[4];
    uint32_t out = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t f = (f4 >> (8 * k)) & 0xFFu;
      uint32_t o = f & (F_PIN | F_T | F_DEAD);
      gl[k] = -1;
      if ((keep >> (8 * k)) & 1u) {
        o |= F_A;
        if ((bnd >> (8 * k)) & 1u) o |= F_B;
        if (M.mode == MODE_DD) {
          if (!(f & F_T)) { label[4 * t + k] = round; ++nn; }
          o |= F_T;
        }
        act[posn] = (int32_t)(4 * t + k);
        gl[k] = posn++;
      }
      out |= o << (8 * k);
    }
    nb += __popc(bnd);
    reinterpret_cast<uint32_t*>(fout)[t] = out;
    reinterpret_cast<int4*>(g2l)[t] = make_int4(gl[0], gl[1], gl[2], gl[3]);
  }
  nb = __reduce_add_sync(0xffffffffu, nb);
  nn = __reduce_add_sync(0xffffffffu, nn);
  if (lane == 0) {
    if (nb) atomicAdd(&tot[0], nb);
    if (nn) atomicAdd(&tot[1], nn);
  }
  __syncthreads();
  if (tid == 0) {
    dsc->nA = wsum[(nth >> 5) - 1];
    dsc->expand = ex ? 1 : 0;
    dsc->nB = tot[0];
    dsc->n_new = tot[1];
  }
}

// ---- row-group variants (vec4 grids): a thread owns the same 4-cell group in
// RG consecutive x-rows of one plane.  The ±y neighbour words of the group
// column are loaded once and reused by the RG rows, the ±x neighbours come
// from the adjacent lanes by warp shuffles (a load only at warp edges), the
// ±z neighbours are loads.  Tiles are unchanged (one per x-row segment), so a
// block produces RG tile counts / scans.
constexpr int RG = 4;

struct PosRG {
  int32_t iz, iy0, xw, nrow;  // plane, first row, group in row, rows in this group (<= RG)
  int64_t t0;                 // word index of (iy0, xw)
  bool ok;
};
__device__ __forceinline__ PosRG pos_rg(const Geo4& g) {
  PosRG p;
  const int32_t gpp = (g.ny + RG - 1) / RG;  // row groups per plane
  p.iz = blockIdx.x / gpp;
  p.iy0 = (blockIdx.x - p.iz * gpp) * RG;
  p.nrow = g.ny - p.iy0 < RG ? g.ny - p.iy0 : RG;
  p.xw = blockIdx.y * g.bs + threadIdx.x;
  p.ok = p.xw < g.wrow;
  p.t0 = ((int64_t)p.iz * g.ny + p.iy0) * g.wrow + p.xw;
  return p;
}
__host__ dim3 rg_grid(const Geo4& g) { return dim3((unsigned)(((g.ny + RG - 1) / RG) * g.nz), (unsigned)g.nseg, 1); }

// per-byte lanes of the x-neighbours of `in` (row word of this lane): the lanes
// of the left / right word come from lane-1 / lane+1, or a load at warp edges.
template <class LF>
__device__ __forceinline__ uint32_t xnbr_lanes(const Geo4& g, const PosRG& p, int64_t t, bool valid, uint32_t in,
                                               uint32_t edge, bool or_mode, LF&& L) {
  const int lane = threadIdx.x & 31;
  uint32_t lw = __shfl_up_sync(0xffffffffu, in, 1);
  uint32_t rw = __shfl_down_sync(0xffffffffu, in, 1);
  if (lane == 0) lw = (valid && p.xw > 0) ? L(t - 1) : 0u;
  if (lane == 31) rw = (valid && p.xw < g.wrow - 1) ? L(t + 1) : 0u;
  const uint32_t lft = (in << 8) | (p.xw > 0 ? (lw >> 24) : (edge & 0xFFu));
  const uint32_t rgt = (in >> 8) | (p.xw < g.wrow - 1 ? ((rw & 0xFFu) << 24) : (edge & 0xFF000000u));
  return or_mode ? (lft | rgt) : (lft & rgt);
}

template <bool COUNT>
__global__ void __launch_bounds__(256) k_dilate_rg(Geo4 g, uint8_t* __restrict__ flags, uint8_t bit_in,
                                                   uint8_t bit_out, const DevScalars* __restrict__ dsc, SetMode M,
                                                   int do_dilate, int32_t* __restrict__ tile_cnt) {
  __shared__ int sh[8][RG];
  const bool ex = decide_expand(M, dsc);
  const bool dil = do_dilate && ((M.mode == MODE_DEVICE || M.mode == MODE_DD) ? ex : true);
  const PosRG p = pos_rg(g);
  uint32_t* fw = reinterpret_cast<uint32_t*>(flags);
  auto L = [&](int64_t u) { return lanes(fw[u], bit_in); };  // bit_in is not written by this pass
  uint32_t col[RG + 2];
  uint32_t own[RG];
#pragma unroll
  for (int j = 0; j < RG + 2; ++j) {
    const int32_t iy = p.iy0 - 1 + j;
    const bool in_rows = iy >= 0 && iy < g.ny && (j == 0 || j == RG + 1 || j - 1 < p.nrow);
    uint32_t wv = 0;
    if (p.ok && in_rows) wv = fw[p.t0 + (int64_t)(j - 1) * g.wrow];
    if (j >= 1 && j <= RG) own[j - 1] = wv;
    col[j] = lanes(wv, bit_in);
  }
  int cnt[RG];
#pragma unroll
  for (int k = 0; k < RG; ++k) {
    cnt[k] = 0;
    const int64_t t = p.t0 + (int64_t)k * g.wrow;
    uint32_t w = own[k];
    if (dil) {
      const uint32_t in = col[k + 1];
      uint32_t out = in | xnbr_lanes(g, p, t, p.ok && k < p.nrow, in, 0u, true, L) | col[k] | col[k + 2];
      if (p.ok && k < p.nrow) {
        if (g.d3) {
          if (p.iz > 0) out |= L(t - g.wplane);
          if (p.iz < g.nz - 1) out |= L(t + g.wplane);
        }
        if (g.has_nnc) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int64_t i = 4 * t + e;
            const int32_t q0 = __ldg(&g.nptr[i]), q1 = __ldg(&g.nptr[i + 1]);
            for (int32_t q = q0; q < q1; ++q)
              if (flags[__ldg(&g.nnbr[q])] & bit_in) out |= 1u << (8 * e);
          }
        }
        w = (w & ~(0x01010101u * bit_out)) | (out * bit_out);
        fw[t] = w;
      }
    }
    if (COUNT && p.ok && k < p.nrow) cnt[k] = __popc(a_new4(w, M.mode, ex, M.dbit));
  }
  if (COUNT) {
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < RG; ++k) {
      const int v = __reduce_add_sync(0xffffffffu, cnt[k]);
      if (lane == 0) sh[wi][k] = v;
    }
    __syncthreads();
    if (threadIdx.x < p.nrow) {
      int s = 0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s += sh[q][threadIdx.x];
      const int32_t row = p.iz * g.ny + p.iy0 + threadIdx.x;
      tile_cnt[row * g.nseg + blockIdx.y] = s;
    }
  }
}

// BT (block tiles, one segment per x-row): the offsets are per block (its RG
// rows), the rows' offsets inside the block come from the block's own counts.
template <bool BT>
__global__ void __launch_bounds__(256) k_scatter_rg(Geo4 g, const uint8_t* __restrict__ fin,
                                                    uint8_t* __restrict__ fout, SetMode M, int32_t round,
                                                    DevScalars* dsc, const int32_t* __restrict__ tile_off,
                                                    int32_t* __restrict__ act, int32_t* __restrict__ g2l,
                                                    int32_t* __restrict__ label) {
  __shared__ unsigned long long wpre[8];
  __shared__ int sh8[8];
  const bool ex = decide_expand(M, dsc);
  const PosRG p = pos_rg(g);
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const uint32_t* fw = reinterpret_cast<const uint32_t*>(fin);
  auto K = [&](int64_t u) { return a_new4(__ldg(&fw[u]), M.mode, ex, M.dbit); };
  uint32_t kc[RG + 2], own[RG];
#pragma unroll
  for (int j = 0; j < RG + 2; ++j) {
    const int32_t iy = p.iy0 - 1 + j;
    const bool row_ok = iy >= 0 && iy < g.ny && (j == 0 || j == RG + 1 || j - 1 < p.nrow);
    uint32_t wv = 0;
    if (p.ok && row_ok) wv = __ldg(&fw[p.t0 + (int64_t)(j - 1) * g.wrow]);
    if (j >= 1 && j <= RG) own[j - 1] = wv;
    // off-grid rows count as "keep" for the boundary test (no neighbour there)
    kc[j] = (iy >= 0 && iy < g.ny) ? a_new4(wv, M.mode, ex, M.dbit) : 0x01010101u;
  }
  uint32_t keep[RG], bnd[RG];
  unsigned long long packed = 0;  // 16-bit per-row counts
#pragma unroll
  for (int k = 0; k < RG; ++k) {
    const int64_t t = p.t0 + (int64_t)k * g.wrow;
    const bool rok = p.ok && k < p.nrow;
    keep[k] = rok ? kc[k + 1] : 0u;
    const uint32_t xa = xnbr_lanes(g, p, t, rok, keep[k], 0x01010101u, false, K);
    bnd[k] = 0;
    if (keep[k]) {
      uint32_t all = xa & kc[k] & kc[k + 2];
      if (g.d3) {
        all &= p.iz > 0 ? K(t - g.wplane) : 0x01010101u;
        all &= p.iz < g.nz - 1 ? K(t + g.wplane) : 0x01010101u;
      }
      bnd[k] = keep[k] & ~all & 0x01010101u;
      if (g.has_nnc)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (!((keep[k] >> (8 * e)) & 1u) || ((bnd[k] >> (8 * e)) & 1u)) continue;
          const int64_t i = 4 * t + e;
          const int32_t q0 = __ldg(&g.nptr[i]), q1 = __ldg(&g.nptr[i + 1]);
          for (int32_t q = q0; q < q1; ++q)
            if (!a_new(fin[__ldg(&g.nnbr[q])], M.mode, ex, M.dbit)) { bnd[k] |= 1u << (8 * e); break; }
        }
    }
    packed |= (unsigned long long)__popc(keep[k]) << (16 * k);
  }
  // block exclusive scan of the packed per-row counts (row sums <= 4*256 < 2^16)
  unsigned long long x = packed;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wpre[wi] = x;
  __syncthreads();
  unsigned long long pre = x - packed;
  for (int q = 0; q < wi; ++q) pre += wpre[q];
  unsigned long long rowoff = 0;  // BT: exclusive prefix of the row totals inside the block
  int32_t boff = 0;
  if (BT) {
    unsigned long long tot = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) tot += wpre[q];
#pragma unroll
    for (int k = 1; k < RG; ++k) rowoff += ((tot >> (16 * (k - 1))) & 0xFFFFu) << (16 * k);
    rowoff += (rowoff << 16) + (rowoff << 32) + (rowoff << 48);  // running sums (fields < 2^16)
    boff = tile_off[blockIdx.x];
  }
  int nb = 0, nnew = 0;
#pragma unroll
  for (int k = 0; k < RG; ++k) {
    if (!(p.ok && k < p.nrow)) continue;
    const int64_t t = p.t0 + (int64_t)k * g.wrow;
    const int32_t row = p.iz * g.ny + p.iy0 + k;
    int32_t pos = (BT ? boff + (int32_t)((rowoff >> (16 * k)) & 0xFFFFu) : tile_off[row * g.nseg + blockIdx.y]) +
                  (int32_t)((pre >> (16 * k)) & 0xFFFFu);
    const int64_t i0 = 4 * t;
    int32_t gl[4];
    uint32_t out = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t f = (own[k] >> (8 * e)) & 0xFFu;
      uint32_t o = f & (F_PIN | F_T | F_DEAD);
      gl[e] = -1;
      if ((keep[k] >> (8 * e)) & 1u) {
        o |= F_A;
        if ((bnd[k] >> (8 * e)) & 1u) o |= F_B;
        if (M.mode == MODE_DD) {
          if (!(f & F_T)) { label[i0 + e] = round; ++nnew; }
          o |= F_T;
        }
        act[pos] = (int32_t)(i0 + e);
        gl[e] = pos++;
      }
      out |= o << (8 * e);
    }
    reinterpret_cast<uint32_t*>(fout)[t] = out;
    reinterpret_cast<int4*>(g2l)[t] = make_int4(gl[0], gl[1], gl[2], gl[3]);
    nb += __popc(bnd[k]);
  }
  const int nbs = block_sum(nb, sh8);
  __syncthreads();
  const int nns = block_sum(nnew, sh8);
  if (threadIdx.x == 0) {
    if (nbs) atomicAdd(&dsc->nB, nbs);
    if (nns) atomicAdd(&dsc->n_new, nns);
  }
}

// Pinned-cell mask (fracture or perforated), computed once per context.
__global__ void k_pin_mask(int64_t n, const uint8_t* __restrict__ kind, const double* __restrict__ wi,
                           uint8_t* __restrict__ pin0) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool pin = kind[i] == RSIM_KIND_FRACTURE || wi[i] > 0.0;
  pin0[i] = kind[i] == RSIM_KIND_DEAD ? (uint8_t)F_DEAD : (pin ? (uint8_t)(F_PIN | F_A) : (uint8_t)0);
}

// Reset flags to the pinned set (A|PIN), or to all-active: 16 cells per
// thread (uint4), scalar tail.
__global__ void k_set_reset(int64_t n, const uint8_t* __restrict__ pin0, uint8_t* __restrict__ flags,
                            int all_active) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n16 = n / 16;
  if (t < n16) {
    uint4 v = reinterpret_cast<const uint4*>(pin0)[t];
    if (all_active) {  // every live cell (dead filler cells stay out)
      auto a = [](uint32_t w) { return (0x01010101u & ~((w >> 7) & 0x01010101u)) * F_A; };
      v.x |= a(v.x); v.y |= a(v.y); v.z |= a(v.z); v.w |= a(v.w);
    }
    reinterpret_cast<uint4*>(flags)[t] = v;
  } else if (t == n16) {
    for (int64_t i = 16 * n16; i < n; ++i)
      flags[i] = (uint8_t)(pin0[i] | (all_active && !(pin0[i] & F_DEAD) ? F_A : 0));
  }
}

// Support-set seed for an externally given δp (config 5):
// flags = pinned set | D0 where |δp| >= ε  (reset + seed in one pass, 4 cells
// per thread: one flag word, two double2 loads).
// With `bits` (n % 32 == 0) the seed is also written as a bitmap (bit i%32 of
// word i/32), the input of the bitmap dilation: 8 lanes' nibbles per word.
__global__ void k_reset_seed(int64_t n, const uint8_t* __restrict__ pin0, const double* __restrict__ dp, double eps,
                             uint8_t* __restrict__ flags, uint32_t* __restrict__ bits) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n4 = n / 4;
  if (bits) {  // n % 32 == 0: whole 8-lane groups are in range together
    uint32_t nib = 0;
    if (t < n4) {
      uint32_t w = reinterpret_cast<const uint32_t*>(pin0)[t];
      const double2 a = __ldcs(reinterpret_cast<const double2*>(dp) + 2 * t);
      const double2 b = __ldcs(reinterpret_cast<const double2*>(dp) + 2 * t + 1);
      nib = (fabs(a.x) >= eps ? 1u : 0u) | (fabs(a.y) >= eps ? 2u : 0u) | (fabs(b.x) >= eps ? 4u : 0u) |
            (fabs(b.y) >= eps ? 8u : 0u);
      w |= ((nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21)) * (uint32_t)F_D0;
      reinterpret_cast<uint32_t*>(flags)[t] = w;
    }
    uint32_t x = nib << (4 * (threadIdx.x & 7));
    x |= __shfl_xor_sync(0xffffffffu, x, 1);
    x |= __shfl_xor_sync(0xffffffffu, x, 2);
    x |= __shfl_xor_sync(0xffffffffu, x, 4);
    if ((threadIdx.x & 7) == 0 && t < n4) bits[t >> 3] = x;
    return;
  }
  if (t < n4) {
    uint32_t w = reinterpret_cast<const uint32_t*>(pin0)[t];
    const double2 a = reinterpret_cast<const double2*>(dp)[2 * t];
    const double2 b = reinterpret_cast<const double2*>(dp)[2 * t + 1];
    if (fabs(a.x) >= eps) w |= (uint32_t)F_D0;
    if (fabs(a.y) >= eps) w |= (uint32_t)F_D0 << 8;
    if (fabs(b.x) >= eps) w |= (uint32_t)F_D0 << 16;
    if (fabs(b.y) >= eps) w |= (uint32_t)F_D0 << 24;
    reinterpret_cast<uint32_t*>(flags)[t] = w;
  } else if (t == n4) {
    for (int64_t i = 4 * n4; i < n; ++i) flags[i] = (uint8_t)(pin0[i] | (fabs(dp[i]) >= eps ? F_D0 : 0));
  }
}

__global__ void k_set_list(const int32_t* __restrict__ list, int32_t n, uint8_t* __restrict__ flags) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) flags[list[k]] |= F_A;
}

// D0 := PIN (first-step initial set = pinned + m-halo).
__global__ void k_seed_pinned(int64_t n, uint8_t* __restrict__ flags) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint8_t f = flags[i];
  flags[i] = (f & F_PIN) ? (uint8_t)(f | F_D0) : (uint8_t)(f & ~(F_D0 | F_D1));
}

// A := {|p - p_prev| >= eps} ∪ PIN (support of the last timestep).
template <int B>
__global__ void k_initial_support(int64_t n, const double* __restrict__ u, const double* __restrict__ p_prev,
                                  double eps, uint8_t* __restrict__ flags) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint8_t f = flags[i];
  if (fabs(u[i * B] - p_prev[i]) >= eps) f |= F_A;
  flags[i] = f;
}

// ---------------------------------------------------------------- K8 / DD
__global__ void k_dd_begin(int64_t n, uint8_t* __restrict__ flags, int32_t* __restrict__ label,
                           double* __restrict__ last_dp) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint8_t f = flags[i];
  if (f & F_A) { f |= F_T; label[i] = 0; } else { f &= ~F_T; label[i] = -1; }
  flags[i] = f;
  last_dp[i] = 0.0;
}

// predicate compaction over labels: sel=0 -> label==k ; sel=1 -> halo of k
__device__ __forceinline__ bool dd_pred(const Geo& g, const int32_t* __restrict__ label, int64_t i, int k, int sel) {
  int32_t li = label[i];
  if (sel == 0) return li == k;
  if (li == k || is_dead(g, i)) return false;
  bool h = false;
  each_nbr(g, i, [&](int64_t j) { if (label[j] == k) h = true; });
  return h;
}

// Sizes of every subdomain list and halo list in one pass: cell i counts for
// its own label (sub) and once for every distinct neighbour label k != label(i)
// (halo of k) — integer sums, order-independent.  hist: [2][n_sub] in global.
__global__ void __launch_bounds__(256) k_dd_hist(Geo g, const int32_t* __restrict__ label, int n_sub,
                                                 int32_t* __restrict__ hist) {
  extern __shared__ int32_t sh[];  // [2][n_sub]
  for (int k = threadIdx.x; k < 2 * n_sub; k += blockDim.x) sh[k] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * TILE + threadIdx.x * 8;
  for (int q = 0; q < 8; ++q) {
    const int64_t i = base + q;
    if (i >= g.n) break;
    const int32_t li = label[i];
    if (li >= 0 && li < n_sub) atomicAdd(&sh[li], 1);
    if (is_dead(g, i)) continue;
    // each distinct neighbour label counts once: the j-th neighbour counts
    // unless an earlier neighbour (enumeration order) carries the same label
    int idx = 0;
    each_nbr(g, i, [&](int64_t j) {
      const int32_t lj = label[j];
      const int me = idx++;
      if (lj < 0 || lj >= n_sub || lj == li) return;
      int k2 = 0;
      bool dup = false;
      each_nbr(g, i, [&](int64_t j2) {
        if (k2++ < me && label[j2] == lj) dup = true;
      });
      if (!dup) atomicAdd(&sh[n_sub + lj], 1);
    });
  }
  __syncthreads();
  for (int k = threadIdx.x; k < 2 * n_sub; k += blockDim.x)
    if (sh[k]) atomicAdd(&hist[k], sh[k]);
}

__global__ void __launch_bounds__(256) k_dd_count(Geo g, const int32_t* __restrict__ label, int k, int sel,
                                                  int32_t* __restrict__ tile_cnt) {
  __shared__ int32_t wsum[8];
  const int64_t base = (int64_t)blockIdx.x * TILE + threadIdx.x * 8;
  int cnt = 0;
  for (int q = 0; q < 8; ++q) {
    int64_t i = base + q;
    if (i < g.n && dd_pred(g, label, i, k, sel)) ++cnt;
  }
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) cnt += __shfl_down_sync(0xffffffffu, cnt, off);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < 8; ++w) s += wsum[w];
    tile_cnt[blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(256) k_dd_scatter(Geo g, const int32_t* __restrict__ label, int k, int sel,
                                                    const int32_t* __restrict__ tile_off, int32_t* __restrict__ out) {
  __shared__ int32_t wsum[8];
  const int64_t base = (int64_t)blockIdx.x * TILE + threadIdx.x * 8;
  uint8_t keep[8];
  int cnt = 0;
  for (int q = 0; q < 8; ++q) {
    int64_t i = base + q;
    keep[q] = (i < g.n && dd_pred(g, label, i, k, sel)) ? 1 : 0;
    cnt += keep[q];
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  int wpre = 0;
  for (int q = 0; q < w; ++q) wpre += wsum[q];
  int pos = tile_off[blockIdx.x] + wpre + x - cnt;
  for (int q = 0; q < 8; ++q)
    if (keep[q]) out[pos++] = (int32_t)(base + q);
}

__global__ void k_g2l_scatter(const int32_t* __restrict__ list, int32_t n, int32_t* __restrict__ g2l, int clear) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) g2l[list[k]] = clear ? -1 : (int32_t)k;
}

__global__ void k_halo_max(const int32_t* __restrict__ list, int64_t n, const double* __restrict__ last_dp,
                           DevScalars* dsc) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double a = k < n ? last_dp[list[k]] : 0.0;
  double w = warp_max(a);
  if ((threadIdx.x & 31) == 0 && w > 0.0) atomic_max_bits(&dsc->halo, w);
}

__global__ void k_zero_list(const int32_t* __restrict__ list, int32_t n, double* __restrict__ last_dp) {
  int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) last_dp[list[k]] = 0.0;
}

// Fig. 8 categories: 0 inactive, 1 active, 2 boundary, 3 active+update, 4 boundary+update.
__global__ void k_categories(int64_t n, const uint8_t* __restrict__ flags, const double* __restrict__ dp, double eps,
                             uint8_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint8_t f = flags[i];
  uint8_t c = 0;
  if (f & F_A) {
    bool upd = fabs(dp[i]) >= eps;
    c = (f & F_B) ? (upd ? 4 : 2) : (upd ? 3 : 1);
  }
  out[i] = c;
}

// D0 := {|δp| >= eps} over all cells (c5 synthetic update).
__global__ void k_seed_support(int64_t n, const double* __restrict__ dp, double eps, uint8_t* __restrict__ flags) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint8_t f = flags[i] & (uint8_t)~(F_D0 | F_D1);
  if (fabs(dp[i]) >= eps) f |= F_D0;
  flags[i] = f;
}

template <int B>
__global__ void k_state_from_dp(int64_t n, const double* __restrict__ dp, double p_hi, double scale,
                                double* __restrict__ u) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) u[i * B] = p_hi - scale * dp[i];
}

inline int64_t nblk(int64_t n, int th) { return (n + th - 1) / th; }

}  // namespace

// ---- bitmap dilation (large vec4 grids with nx % 32 == 0 and no NNC): the
// m hop rounds run on a 1-bit-per-cell map (n/8 bytes, L2-resident) with 32
// cells per thread instead of on the flag bytes; the count pass merges the
// final map into the flag byte's D bit, so the count / scan / scatter passes
// and their results are those of the byte path.
struct GeoB {
  int64_t nbw;      // bit words
  int32_t brow;     // bit words per x-row
  int64_t bplane;   // bit words per plane
  int32_t ny, nz;
  bool d3;
};
__host__ GeoB geob(const rsim_gpu_ctx* c) {
  GeoB g;
  g.nbw = c->n / 32;
  g.brow = c->nx / 32;
  g.bplane = (int64_t)g.brow * c->ny;
  g.ny = c->ny; g.nz = c->nz;
  g.d3 = c->d3;
  return g;
}

// bitmap of flag bit `bit` (32 cells per thread: two 16-byte loads)
__global__ void k_pack_bits(int64_t nbw, const uint8_t* __restrict__ flags, uint8_t bit, uint32_t* __restrict__ bits) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nbw) return;
  const uint4* f = reinterpret_cast<const uint4*>(flags) + 2 * t;
  const uint4 a = f[0], b = f[1];
  const uint32_t ws[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
  const uint32_t sh = bitpos(bit);
  uint32_t x = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t l = (ws[k] >> sh) & 0x01010101u;  // byte lanes -> 4 bits
    x |= ((l & 1u) | ((l >> 7) & 2u) | ((l >> 14) & 4u) | ((l >> 21) & 8u)) << (4 * k);
  }
  bits[t] = x;
}

// one hop: out(i) = in(i) | OR over the 6 Cartesian neighbours
__global__ void k_dilate_bits(GeoB g, const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                              const DevScalars* __restrict__ dsc, SetMode M) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= g.nbw) return;
  const bool ex = decide_expand(M, dsc);
  if ((M.mode == MODE_DEVICE || M.mode == MODE_DD) && !ex) return;  // no dilation this update
  const int64_t row = t / g.brow;
  const int32_t xw = (int32_t)(t - row * g.brow);
  const int32_t iz = (int32_t)(row / g.ny), iy = (int32_t)(row - (int64_t)iz * g.ny);
  const uint32_t v = in[t];
  uint32_t o = v | (v << 1) | (v >> 1);
  if (xw > 0) o |= in[t - 1] >> 31;
  if (xw < g.brow - 1) o |= in[t + 1] << 31;
  if (iy > 0) o |= in[t - g.brow];
  if (iy < g.ny - 1) o |= in[t + g.brow];
  if (g.d3) {
    if (iz > 0) o |= in[t - g.bplane];
    if (iz < g.nz - 1) o |= in[t + g.bplane];
  }
  out[t] = o;
}

// count pass of the bitmap path (row groups as k_dilate_rg<true>): the final
// map goes into the D bit of the flag words, then A_new is counted per tile
__global__ void __launch_bounds__(256) k_count_merge_rg(Geo4 g, uint8_t* __restrict__ flags,
                                                         const uint32_t* __restrict__ bits,
                                                         const DevScalars* __restrict__ dsc, SetMode M,
                                                         int32_t* __restrict__ tile_cnt, bool bt) {
  __shared__ int sh[8][RG];
  const bool ex = decide_expand(M, dsc);
  const bool dil = (M.mode == MODE_DEVICE || M.mode == MODE_DD) ? ex : true;
  const PosRG p = pos_rg(g);
  uint32_t* fw = reinterpret_cast<uint32_t*>(flags);
  int cnt[RG];
#pragma unroll
  for (int k = 0; k < RG; ++k) {
    cnt[k] = 0;
    if (!(p.ok && k < p.nrow)) continue;
    const int64_t t = p.t0 + (int64_t)k * g.wrow;
    uint32_t w = fw[t];
    if (dil) {
      const uint32_t nib = (__ldg(&bits[t >> 3]) >> (4 * (t & 7))) & 0xFu;
      const uint32_t l = (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
      w = (w & ~(0x01010101u * M.dbit)) | (l * M.dbit);
      fw[t] = w;
    }
    cnt[k] = __popc(a_new4(w, M.mode, ex, M.dbit));
  }
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < RG; ++k) {
    const int v = __reduce_add_sync(0xffffffffu, cnt[k]);
    if (lane == 0) sh[wi][k] = v;
  }
  __syncthreads();
  if (bt) {  // one count per block (its RG rows)
    if (threadIdx.x == 0) {
      int s = 0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q)
        for (int k = 0; k < RG; ++k) s += sh[q][k];
      tile_cnt[blockIdx.x] = s;
    }
  } else if (threadIdx.x < p.nrow) {
    int s = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s += sh[q][threadIdx.x];
    const int32_t row = p.iz * g.ny + p.iy0 + threadIdx.x;
    tile_cnt[row * g.nseg + blockIdx.y] = s;
  }
}

// Keep pass of the bitmap path with block tiles (one x-row segment): A_new of
// every cell from its flag byte with the final dilation bit merged in, as a
// keep bitmap (1 bit per cell) + one count per block.  The flag bytes are not
// rewritten: the scatter takes A_new of a cell and of its neighbours from the
// keep bitmap (L1/L2-resident) and only the cell's own byte from the flags.
__device__ __forceinline__ uint32_t nib_to_lanes(uint32_t nib) {
  return (nib & 1u) | ((nib & 2u) << 7) | ((nib & 4u) << 14) | ((nib & 8u) << 21);
}
__device__ __forceinline__ uint32_t lanes_to_nib(uint32_t l) {
  return (l & 1u) | ((l >> 7) & 2u) | ((l >> 14) & 4u) | ((l >> 21) & 8u);
}
__global__ void __launch_bounds__(256) k_keep_rg(Geo4 g, const uint8_t* __restrict__ flags,
                                                 const uint32_t* __restrict__ bits, uint32_t* __restrict__ keepbits,
                                                 const DevScalars* __restrict__ dsc, SetMode M,
                                                 int32_t* __restrict__ blk_cnt) {
  // the block's cells (RG consecutive x-rows of one plane, as in the scatter)
  // are the contiguous flag words [w0, w0 + nrow·wrow): 4 words (16 cells,
  // one uint4) per thread, half a keep-bitmap word
  __shared__ int sh[8];
  const bool ex = decide_expand(M, dsc);
  const bool dil = (M.mode == MODE_DEVICE || M.mode == MODE_DD) ? ex : true;
  const int32_t gpp = (g.ny + RG - 1) / RG;
  const int32_t iz = blockIdx.x / gpp, iy0 = (blockIdx.x - iz * gpp) * RG;
  const int32_t nrow = g.ny - iy0 < RG ? g.ny - iy0 : RG;
  const int64_t w0 = ((int64_t)iz * g.ny + iy0) * g.wrow;
  const int64_t nq = (int64_t)nrow * g.wrow / 4;
  const int lane = threadIdx.x & 31;
  const uint4* f4 = reinterpret_cast<const uint4*>(flags) + w0 / 4;
  int cnt = 0;
  for (int64_t q0 = 0; q0 < nq; q0 += blockDim.x) {  // warp-uniform trip count
    const int64_t q = q0 + threadIdx.x;
    uint32_t nib16 = 0;
    if (q < nq) {
      const uint4 v = __ldcs(&f4[q]);
      uint32_t ws[4] = {v.x, v.y, v.z, v.w};
      uint32_t dm = 0;
      if (dil) dm = (__ldg(&bits[(w0 + 4 * q) >> 3]) >> (16 * (q & 1))) & 0xFFFFu;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        uint32_t w = ws[e];
        if (dil) w = (w & ~(0x01010101u * M.dbit)) | (nib_to_lanes((dm >> (4 * e)) & 0xFu) * M.dbit);
        nib16 |= lanes_to_nib(a_new4(w, M.mode, ex, M.dbit)) << (4 * e);
      }
      cnt += __popc(nib16);
    }
    const uint32_t other = __shfl_xor_sync(0xffffffffu, nib16, 1);
    if (q < nq && (q & 1) == 0) keepbits[(w0 + 4 * q) >> 3] = nib16 | (other << 16);
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  if (lane == 0) sh[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) s += sh[q];
    blk_cnt[blockIdx.x] = s;
  }
}

// Scatter of the bitmap path (block tiles): A_new lanes of a word and of its
// neighbours from the keep bitmap, the cell's own byte for PIN / T.
__global__ void __launch_bounds__(256) k_scatter_kb(Geo4 g, const uint8_t* __restrict__ fin,
                                                    const uint32_t* __restrict__ keepbits,
                                                    uint8_t* __restrict__ fout, SetMode M, int32_t round,
                                                    DevScalars* dsc, const int32_t* __restrict__ blk_off,
                                                    int32_t* __restrict__ act, int32_t* __restrict__ g2l,
                                                    int32_t* __restrict__ label) {
  __shared__ unsigned long long wpre[8];
  __shared__ int sh8[8];
  const PosRG p = pos_rg(g);
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  const uint32_t* fw = reinterpret_cast<const uint32_t*>(fin);
  const int32_t boff = blk_off[blockIdx.x];
  auto K = [&](int64_t u) { return nib_to_lanes((__ldg(&keepbits[u >> 3]) >> (4 * (u & 7))) & 0xFu); };
  uint32_t kc[RG + 2], own[RG];
#pragma unroll
  for (int j = 0; j < RG + 2; ++j) {
    const int32_t iy = p.iy0 - 1 + j;
    const bool row_ok = iy >= 0 && iy < g.ny && (j == 0 || j == RG + 1 || j - 1 < p.nrow);
    const int64_t t = p.t0 + (int64_t)(j - 1) * g.wrow;
    if (j >= 1 && j <= RG) own[j - 1] = (p.ok && row_ok) ? __ldcs(&fw[t]) : 0u;
    // off-grid rows count as "keep" for the boundary test (no neighbour there)
    kc[j] = (iy >= 0 && iy < g.ny) ? ((p.ok && row_ok) ? K(t) : 0u) : 0x01010101u;
  }
  uint32_t keep[RG], bnd[RG];
  unsigned long long packed = 0;  // 16-bit per-row counts
#pragma unroll
  for (int k = 0; k < RG; ++k) {
    const int64_t t = p.t0 + (int64_t)k * g.wrow;
    const bool rok = p.ok && k < p.nrow;
    keep[k] = rok ? kc[k + 1] : 0u;
    const uint32_t xa = xnbr_lanes(g, p, t, rok, keep[k], 0x01010101u, false, K);
    bnd[k] = 0;
    if (keep[k]) {
      uint32_t all = xa & kc[k] & kc[k + 2];
      if (g.d3) {
        all &= p.iz > 0 ? K(t - g.wplane) : 0x01010101u;
        all &= p.iz < g.nz - 1 ? K(t + g.wplane) : 0x01010101u;
      }
      bnd[k] = keep[k] & ~all & 0x01010101u;
    }
    packed |= (unsigned long long)__popc(keep[k]) << (16 * k);
  }
  unsigned long long x = packed;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wpre[wi] = x;
  __syncthreads();
  unsigned long long pre = x - packed, tot = 0;
  for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
    if (q < wi) pre += wpre[q];
    tot += wpre[q];
  }
  unsigned long long rowoff = 0;  // exclusive prefix of the row totals inside the block
#pragma unroll
  for (int k = 1; k < RG; ++k) rowoff += ((tot >> (16 * (k - 1))) & 0xFFFFu) << (16 * k);
  rowoff += (rowoff << 16) + (rowoff << 32) + (rowoff << 48);  // running sums (fields < 2^16)
  int nb = 0, nnew = 0;
#pragma unroll
  for (int k = 0; k < RG; ++k) {
    if (!(p.ok && k < p.nrow)) continue;
    const int64_t t = p.t0 + (int64_t)k * g.wrow;
    int32_t pos = boff + (int32_t)((rowoff >> (16 * k)) & 0xFFFFu) + (int32_t)((pre >> (16 * k)) & 0xFFFFu);
    const int64_t i0 = 4 * t;
    int32_t gl[4];
    uint32_t out = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t f = (own[k] >> (8 * e)) & 0xFFu;
      uint32_t o = f & (F_PIN | F_T | F_DEAD);
      gl[e] = -1;
      if ((keep[k] >> (8 * e)) & 1u) {
        o |= F_A;
        if ((bnd[k] >> (8 * e)) & 1u) o |= F_B;
        if (M.mode == MODE_DD) {
          if (!(f & F_T)) { label[i0 + e] = round; ++nnew; }
          o |= F_T;
        }
        act[pos] = (int32_t)(i0 + e);
        gl[e] = pos++;
      }
      out |= o << (8 * e);
    }
    reinterpret_cast<uint32_t*>(fout)[t] = out;
    reinterpret_cast<int4*>(g2l)[t] = make_int4(gl[0], gl[1], gl[2], gl[3]);
    nb += __popc(bnd[k]);
  }
  const int nbs = block_sum(nb, sh8);
  __syncthreads();
  const int nns = block_sum(nnew, sh8);
  if (threadIdx.x == 0) {
    if (nbs) atomicAdd(&dsc->nB, nbs);
    if (nns) atomicAdd(&dsc->n_new, nns);
  }
}

// ============================================================== launchers
int launch_update(rsim_gpu_ctx* c, double eps) {
  if (c->nA <= 0) return RSIM_OK;
  RSIM_CUDA(cudaMemsetAsync(&c->dsc->maxA, 0, 2 * sizeof(unsigned long long), c->stream));
  const int64_t g = nblk(c->nA, 256);
  switch (c->b) {
    case 1: k_update<1><<<g, 256, 0, c->stream>>>(rsim::phys::Fluid(c->fl), c->nA, c->act, c->x, c->u, c->st, c->flags, c->dp, c->last_dp, eps, c->dsc); break;
    case 2: k_update<2><<<g, 256, 0, c->stream>>>(rsim::phys::Fluid(c->fl), c->nA, c->act, c->x, c->u, c->st, c->flags, c->dp, c->last_dp, eps, c->dsc); break;
    default: k_update<3><<<g, 256, 0, c->stream>>>(rsim::phys::Fluid(c->fl), c->nA, c->act, c->x, c->u, c->st, c->flags, c->dp, c->last_dp, eps, c->dsc); break;
  }
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

int launch_threshold(rsim_gpu_ctx* c, double eps) {
  RSIM_CUDA(cudaMemsetAsync(&c->dsc->maxA, 0, 2 * sizeof(unsigned long long), c->stream));
  if (c->nA > 0) {
    k_threshold<<<nblk(c->nA, 256), 256, 0, c->stream>>>(c->nA, c->act, c->dp, c->flags, eps, c->dsc);
    c->launches++;
  }
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

// Full set update: [m-1 dilation rounds] + [round m fused with the tile count]
// + scan + scatter.  4 launches for m = 2, no host round trip.
// bitmap dilation: large grids (row-group path), whole bit words per x-row, no NNC
static bool bits_path_possible(const rsim_gpu_ctx* c) {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("RSIM_NO_BITS_K7");
    v = (e && *e == '1') ? 0 : 1;
  }
  if (!v || c->has_nnc || c->nx % 32 != 0 || !c->bits[0]) return false;
  const Geo4 g = geo4(c);
  const dim3 grg = rg_grid(g);
  return g.vec4 && (int64_t)grg.x * grg.y >= 16 * 148;
}

static bool keepbits_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("RSIM_NO_KEEPBITS_K7");
    v = (e && *e == '1') ? 0 : 1;
  }
  return v == 1;
}

static bool smem_set_update_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("RSIM_NO_SMEM_K7");
    v = (e && *e == '1') ? 0 : 1;
  }
  return v == 1;
}

static bool coop_set_update_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = std::getenv("RSIM_NO_COOP_K7");
    v = (e && *e == '1') ? 0 : 1;
  }
  return v == 1;
}

// single-block tile scan (counts staged in dynamic shared memory)
static int launch_scan_tiles(rsim_gpu_ctx* c, int64_t ntiles, const SetMode& M) {
  const size_t smem = (size_t)(ntiles + ntiles / 32 + 1) * sizeof(int32_t);
  if (smem > 220 * 1024) {
    rsim_set_error("set update: grid too large for the single-block tile scan");
    return RSIM_EARG;
  }
  static size_t attr = 48 * 1024;
  if (smem > attr) {
    RSIM_CUDA(cudaFuncSetAttribute(k_scan_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
    attr = 220 * 1024;
  }
  k_scan_tiles<<<1, 1024, smem, c->stream>>>(c->tile_cnt, c->tile_off, (int32_t)ntiles, c->dsc, M);
  c->launches++;
  return RSIM_OK;
}

int launch_set_update(rsim_gpu_ctx* c, int mode, int round, double eps, int m, int shrink_locked, int force_expand,
                      int do_dilate) {
  const Geo4 g = geo4(c);
  const dim3 grid = k7_grid(g);
  SetMode M;
  M.mode = mode;
  M.dbit = (m % 2 == 0) ? F_D0 : F_D1;
  M.eps = eps;
  M.shrink_locked = shrink_locked;
  M.force_expand = force_expand;
  const int64_t ntiles = k7_tiles(g);
  const int rounds = do_dilate ? m : 0;
  const dim3 grg = rg_grid(g);
  // row groups reuse the ±y words RG-fold but give RG-fold fewer blocks: only
  // for grids large enough to fill the GPU many times over
  const bool use_rg = g.vec4 && !g.has_dead && (int64_t)grg.x * grg.y >= 16 * 148;
  if (g.vec4 && c->n <= kSmemK7MaxCells && smem_set_update_enabled()) {  // small grid: one CTA, flags in smem
    const size_t smem = (size_t)(c->n / 4 + (c->n + 31) / 32) * sizeof(uint32_t);
    static size_t attr = 0;
    if (smem > 48 * 1024 && attr < 220 * 1024) {
      RSIM_CUDA(cudaFuncSetAttribute(k_set_update_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
      attr = 220 * 1024;
    }
    k_set_update_smem<<<1, 1024, smem, c->stream>>>(g, c->flags, c->flags_alt, M, rounds, round, c->dsc, c->act_buf,
                                                     c->g2l, c->label, c->nnc_bits);
    c->launches++;
    RSIM_CUDA(cudaGetLastError());
    std::swap(c->flags, c->flags_alt);
    c->act = c->act_buf;
    return RSIM_OK;
  }
  if (!use_rg && ntiles <= kCoopMaxTiles && coop_set_update_enabled()) {
    static int per_sm = 0;
    if (per_sm == 0) {
      RSIM_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_set_update_coop, g.bs, 0));
      if (per_sm < 1) per_sm = 1;
    }
    static const int gmax = [] {
      const char* e = std::getenv("RSIM_K7_COOP_GRID");
      return (e && *e) ? std::atoi(e) : 1 << 30;
    }();
    int64_t maxb = (int64_t)per_sm * c->sm_count;
    if (maxb > gmax) maxb = gmax;
    int grid = (int)(ntiles < maxb ? ntiles : maxb);
    int32_t* tc = c->tile_cnt;
    int32_t* to = c->tile_off;
    int32_t* ab = c->act_buf;
    int32_t* gl = c->g2l;
    int32_t* lb = c->label;
    uint8_t* f0 = c->flags;
    uint8_t* f1 = c->flags_alt;
    DevScalars* ds = c->dsc;
    Geo4 gg = g;
    SetMode MM = M;
    int rr = rounds;
    int32_t rd = round;
    void* args[] = {&gg, &f0, &f1, &MM, &rr, &rd, &ds, &tc, &to, &ab, &gl, &lb};
    RSIM_CUDA(cudaLaunchCooperativeKernel((void*)k_set_update_coop, grid, g.bs, args, 0, c->stream));
    c->launches++;
    RSIM_CUDA(cudaGetLastError());
    std::swap(c->flags, c->flags_alt);
    c->act = c->act_buf;
    return RSIM_OK;
  }
  bool bt = false;
  const bool seeded = c->seed_bits_ready;
  c->seed_bits_ready = false;
  if (use_rg && rounds > 0 && bits_path_possible(c)) {
    const GeoB gb = geob(c);
    const int64_t nb = nblk(gb.nbw, 256);
    if (!seeded) {
      k_pack_bits<<<nb, 256, 0, c->stream>>>(gb.nbw, c->flags, F_D0, c->bits[0]);
      c->launches++;
    }
    for (int r = 0; r < rounds; ++r) {
      k_dilate_bits<<<nb, 256, 0, c->stream>>>(gb, c->bits[r & 1], c->bits[(r + 1) & 1], c->dsc, M);
      c->launches++;
    }
    bt = g.nseg == 1;  // block tiles: RG-fold fewer offsets to scan
    if (bt && keepbits_enabled()) {
      uint32_t* kb = c->bits[(rounds + 1) & 1];  // the buffer the final map is not in
      k_keep_rg<<<grg, g.bs, 0, c->stream>>>(g, c->flags, c->bits[rounds & 1], kb, c->dsc, M, c->tile_cnt);
      c->launches++;
      { const int r = launch_scan_tiles(c, (int64_t)grg.x, M); if (r != RSIM_OK) return r; }
      k_scatter_kb<<<grg, g.bs, 0, c->stream>>>(g, c->flags, kb, c->flags_alt, M, round, c->dsc, c->tile_off,
                                                c->act_buf, c->g2l, c->label);
      c->launches++;
      RSIM_CUDA(cudaGetLastError());
      std::swap(c->flags, c->flags_alt);
      c->act = c->act_buf;
      return RSIM_OK;
    }
    k_count_merge_rg<<<grg, g.bs, 0, c->stream>>>(g, c->flags, c->bits[rounds & 1], c->dsc, M, c->tile_cnt, bt);
    c->launches++;
  } else {
  for (int r = 0; r + 1 < rounds; ++r) {
    uint8_t bin = (r % 2 == 0) ? F_D0 : F_D1, bout = (r % 2 == 0) ? F_D1 : F_D0;
    if (use_rg) k_dilate_rg<false><<<grg, g.bs, 0, c->stream>>>(g, c->flags, bin, bout, c->dsc, M, 1, c->tile_cnt);
    else k_dilate<false><<<grid, g.bs, 0, c->stream>>>(g, c->flags, bin, bout, c->dsc, M, 1, c->tile_cnt);
    c->launches++;
  }
  {
    const int r = rounds - 1;
    uint8_t bin = (r % 2 == 0) ? F_D0 : F_D1, bout = (r % 2 == 0) ? F_D1 : F_D0;
    if (use_rg)
      k_dilate_rg<true><<<grg, g.bs, 0, c->stream>>>(g, c->flags, bin, bout, c->dsc, M, rounds > 0 ? 1 : 0,
                                                     c->tile_cnt);
    else
      k_dilate<true><<<grid, g.bs, 0, c->stream>>>(g, c->flags, bin, bout, c->dsc, M, rounds > 0 ? 1 : 0,
                                                   c->tile_cnt);
    c->launches++;
  }
  }
  { const int r = launch_scan_tiles(c, bt ? (int64_t)grg.x : ntiles, M); if (r != RSIM_OK) return r; }
  if (use_rg && bt)
    k_scatter_rg<true><<<grg, g.bs, 0, c->stream>>>(g, c->flags, c->flags_alt, M, round, c->dsc, c->tile_off,
                                                    c->act_buf, c->g2l, c->label);
  else if (use_rg)
    k_scatter_rg<false><<<grg, g.bs, 0, c->stream>>>(g, c->flags, c->flags_alt, M, round, c->dsc, c->tile_off, c->act_buf,
                                              c->g2l, c->label);
  else
    k_scatter<<<grid, g.bs, 0, c->stream>>>(g, c->flags, c->flags_alt, M, round, c->dsc, c->tile_off, c->act_buf,
                                            c->g2l, c->label);
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  std::swap(c->flags, c->flags_alt);
  c->act = c->act_buf;
  return RSIM_OK;
}

static int ensure_pin0(rsim_gpu_ctx* c) {
  if (!c->pin0) {
    RSIM_CUDA(cudaMalloc(&c->pin0, c->n + 16));
    k_pin_mask<<<nblk(c->n, 256), 256, 0, c->stream>>>(c->n, c->kind, c->wi, c->pin0);
    c->launches++;
  }
  return RSIM_OK;
}
#define TRY_K7(x) do { const int r_ = (x); if (r_ != RSIM_OK) return r_; } while (0)

int launch_set_reset(rsim_gpu_ctx* c, int all_active) {
  TRY_K7(ensure_pin0(c));
  k_set_reset<<<nblk(c->n / 16 + 1, 256), 256, 0, c->stream>>>(c->n, c->pin0, c->flags, all_active);
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

int launch_set_list(rsim_gpu_ctx* c, const int32_t* list, int32_t n) {
  if (n <= 0) return RSIM_OK;
  k_set_list<<<nblk(n, 256), 256, 0, c->stream>>>(list, n, c->flags);
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

int launch_seed_pinned(rsim_gpu_ctx* c) {
  k_seed_pinned<<<nblk(c->n, 256), 256, 0, c->stream>>>(c->n, c->flags);
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

int launch_initial_support(rsim_gpu_ctx* c, double eps) {
  const int64_t g = nblk(c->n, 256);
  switch (c->b) {
    case 1: k_initial_support<1><<<g, 256, 0, c->stream>>>(c->n, c->u, c->p_prev, eps, c->flags); break;
    case 2: k_initial_support<2><<<g, 256, 0, c->stream>>>(c->n, c->u, c->p_prev, eps, c->flags); break;
    default: k_initial_support<3><<<g, 256, 0, c->stream>>>(c->n, c->u, c->p_prev, eps, c->flags); break;
  }
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

int launch_dd_begin(rsim_gpu_ctx* c) {
  k_dd_begin<<<nblk(c->n, 256), 256, 0, c->stream>>>(c->n, c->flags, c->label, c->last_dp);
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

// Build sorted per-subdomain cell lists and their outer halos.
int launch_dd_partition(rsim_gpu_ctx* c, int32_t n_sub, int32_t* sizes) {
  Geo g = geo(c);
  const int64_t ntiles = nblk(c->n, TILE);
  DDLists& d = c->dd;
  d.n_sub = n_sub;
  d.sub_off.assign(n_sub + 1, 0);
  d.halo_off.assign(n_sub + 1, 0);
  d.selected = -1;
  std::vector<int32_t> cnt_sub(n_sub), cnt_halo(n_sub);
  // all list sizes in one pass and one sync (Phase-2 setup happens once per timestep)
  {
    std::vector<int32_t> h(2 * (size_t)n_sub, 0);
    if (2 * (int64_t)n_sub > d.hist_cap) {
      if (d.hist) cudaFree(d.hist);
      d.hist_cap = 2 * (int64_t)n_sub + 64;
      RSIM_CUDA(cudaMalloc(&d.hist, sizeof(int32_t) * d.hist_cap));
    }
    int32_t* dh = d.hist;
    RSIM_CUDA(cudaMemsetAsync(dh, 0, sizeof(int32_t) * 2 * n_sub, c->stream));
    k_dd_hist<<<ntiles, 256, sizeof(int32_t) * 2 * n_sub, c->stream>>>(g, c->label, n_sub, dh);
    c->launches++;
    RSIM_CUDA(cudaMemcpyAsync(h.data(), dh, sizeof(int32_t) * 2 * n_sub, cudaMemcpyDeviceToHost, c->stream));
    RSIM_CUDA(cudaStreamSynchronize(c->stream));
    for (int k = 0; k < n_sub; ++k) { cnt_sub[k] = h[k]; cnt_halo[k] = h[n_sub + k]; }
  }
  for (int k = 0; k < n_sub; ++k) {
    d.sub_off[k + 1] = d.sub_off[k] + cnt_sub[k];
    d.halo_off[k + 1] = d.halo_off[k] + cnt_halo[k];
    if (sizes) sizes[k] = cnt_sub[k];
  }
  if (d.sub_off[n_sub] > d.sub_cap) {
    if (d.sub_cells) cudaFree(d.sub_cells);
    d.sub_cap = d.sub_off[n_sub];
    RSIM_CUDA(cudaMalloc(&d.sub_cells, sizeof(int32_t) * d.sub_cap));
  }
  if (d.halo_off[n_sub] > d.halo_cap) {
    if (d.halo_cells) cudaFree(d.halo_cells);
    d.halo_cap = d.halo_off[n_sub];
    RSIM_CUDA(cudaMalloc(&d.halo_cells, sizeof(int32_t) * d.halo_cap));
  }
  for (int sel = 0; sel < 2; ++sel)
    for (int k = 0; k < n_sub; ++k) {
      int32_t* out = sel ? d.halo_cells + d.halo_off[k] : d.sub_cells + d.sub_off[k];
      k_dd_count<<<ntiles, 256, 0, c->stream>>>(g, c->label, k, sel, c->tile_cnt);
      { const int r = launch_scan_tiles(c, ntiles, SetMode{MODE_KEEP, 0, 0.0, 1, 0}); if (r != RSIM_OK) return r; }
      k_dd_scatter<<<ntiles, 256, 0, c->stream>>>(g, c->label, k, sel, c->tile_off, out);
      c->launches += 2;
    }
  // clear the localized g2l (every cell -1) before per-subdomain selection
  RSIM_CUDA(cudaMemsetAsync(c->g2l, 0xff, sizeof(int32_t) * c->n, c->stream));
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

int launch_dd_select(rsim_gpu_ctx* c, int32_t k) {
  DDLists& d = c->dd;
  if (d.selected >= 0) {
    int32_t ps = d.selected;
    int32_t np = (int32_t)(d.sub_off[ps + 1] - d.sub_off[ps]);
    if (np > 0) {
      k_g2l_scatter<<<nblk(np, 256), 256, 0, c->stream>>>(d.sub_cells + d.sub_off[ps], np, c->g2l, 1);
      c->launches++;
    }
  }
  int32_t nk = (int32_t)(d.sub_off[k + 1] - d.sub_off[k]);
  int64_t nh = d.halo_off[k + 1] - d.halo_off[k];
  if (nk > 0) {
    k_g2l_scatter<<<nblk(nk, 256), 256, 0, c->stream>>>(d.sub_cells + d.sub_off[k], nk, c->g2l, 0);
    c->launches++;
  }
  RSIM_CUDA(cudaMemsetAsync(&c->dsc->halo, 0, sizeof(unsigned long long), c->stream));
  if (nh > 0) {
    k_halo_max<<<nblk(nh, 256), 256, 0, c->stream>>>(d.halo_cells + d.halo_off[k], nh, c->last_dp, c->dsc);
    c->launches++;
  }
  c->act = d.sub_cells + d.sub_off[k];
  c->nA = nk;
  d.selected = k;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

int launch_dd_skip(rsim_gpu_ctx* c, int32_t k) {
  DDLists& d = c->dd;
  int32_t nk = (int32_t)(d.sub_off[k + 1] - d.sub_off[k]);
  if (nk > 0) {
    k_zero_list<<<nblk(nk, 256), 256, 0, c->stream>>>(d.sub_cells + d.sub_off[k], nk, c->last_dp);
    c->launches++;
  }
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

// flags := pinned | D0 where |δp| >= ε  (set reset + support seed, one pass)
int launch_reset_seed(rsim_gpu_ctx* c, double eps) {
  TRY_K7(ensure_pin0(c));
  uint32_t* bits = bits_path_possible(c) ? c->bits[0] : nullptr;
  k_reset_seed<<<nblk(c->n / 4 + 1, 256), 256, 0, c->stream>>>(c->n, c->pin0, c->dp, eps, c->flags, bits);
  c->seed_bits_ready = bits != nullptr;  // consumed by the next set update
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

int launch_seed_support(rsim_gpu_ctx* c, double eps) {
  k_seed_support<<<nblk(c->n, 256), 256, 0, c->stream>>>(c->n, c->dp, eps, c->flags);
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

int launch_state_from_dp(rsim_gpu_ctx* c, double p_hi, double scale) {
  const int64_t g = nblk(c->n, 256);
  switch (c->b) {
    case 1: k_state_from_dp<1><<<g, 256, 0, c->stream>>>(c->n, c->dp, p_hi, scale, c->u); break;
    case 2: k_state_from_dp<2><<<g, 256, 0, c->stream>>>(c->n, c->dp, p_hi, scale, c->u); break;
    default: k_state_from_dp<3><<<g, 256, 0, c->stream>>>(c->n, c->dp, p_hi, scale, c->u); break;
  }
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}

int launch_categories(rsim_gpu_ctx* c, uint8_t* out) {
  k_categories<<<nblk(c->n, 256), 256, 0, c->stream>>>(c->n, c->flags, c->dp, c->last_eps, out);
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}
