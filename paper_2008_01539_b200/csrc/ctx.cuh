// ctx.cuh — device context, flag bits and device-side helpers shared by the
// sm_100a kernels (assemble.cu, krylov.cu, sets.cu) and the C-ABI (abi.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "rsim/blockops.h"
#include "rsim/gpu_abi.h"
#include "rsim/physics.h"

// ---- per-cell flag bits (u8) -------------------------------------------------
enum : uint8_t {
  F_A = 1,     // in V_A (active)
  F_B = 2,     // in V_B (boundary layer of V_A)
  F_FLAG = 4,  // |δp| >= ε after the last update (support set, Eq. 14)
  F_PIN = 8,   // fracture or perforated cell: always active
  F_T = 16,    // in V_T (DD total active set)
  F_D0 = 32,   // dilation ping-pong bits
  F_D1 = 64,
  F_DEAD = 128,  // filler position of an EDFM fracture plane (RSIM_KIND_DEAD): no connections, never active
};

// Set-update modes of the final compaction pass.
enum { MODE_DEVICE = 0, MODE_SHRINK = 1, MODE_KEEP = 2, MODE_EXPAND = 3, MODE_DD = 4 };

// Device-resident scalars, one struct per ctx (D2H once per Newton iteration).
struct DevScalars {
  int32_t status;
  int32_t bad_cell;
  int32_t lin_iters;
  int32_t nA;
  int32_t nB;
  int32_t expand;
  int32_t n_new;
  int32_t pad0;
  double lin_relres;
  double f2;
  unsigned long long finf;  // bits of a non-negative double (atomicMax)
  unsigned long long maxA;
  unsigned long long maxB;
  unsigned long long halo;
  int32_t part_count;       // number of K1 F-norm partials
  int32_t ilu_bad;          // ILU(0) factorisation hit a singular pivot (=> block-Jacobi fallback)
  unsigned long long nblk;  // b > 1: ELL blocks the last assembly stored (active Cartesian neighbours)
  unsigned long long npo;   // ... of which pressure-only (bench: bytes the Krylov kernels actually need)
};

struct DDLists {
  int32_t n_sub = 0;
  std::vector<int64_t> sub_off, halo_off;  // host offsets (n_sub + 1)
  int32_t* sub_cells = nullptr;            // device, concatenated sorted lists
  int32_t* halo_cells = nullptr;
  int64_t sub_cap = 0, halo_cap = 0;
  int32_t* hist = nullptr;                 // device [2][n_sub] list sizes
  int64_t hist_cap = 0;
  int32_t selected = -1;
};

struct rsim_gpu_ctx {
  int b = 1;
  int32_t nx = 0, ny = 0, nz = 0;
  int64_t n = 0;
  int64_t n_dead = 0;
  // per-Newton-iteration hook (case runner --trace-flags): called by the host
  // solvers after each local solve + update, before the set update
  int (*iter_hook)(void* user, int32_t iter, int32_t subdomain) = nullptr;
  void* iter_user = nullptr;  // RSIM_KIND_DEAD cells (excluded from every set and from M_A's n)
  bool d3 = false;
  int nslot = 4;
  bool has_nnc = false;
  bool cols_implicit = false;  // last assembly: V_A = all cells, ELL columns not stored (structural)
  bool f2_parts = false;       // last assembly left (F,F) chunk partials in part_f2 (F_raw only if keep_F)
  bool keep_F = false;         // debug: the row kernel also stores the raw residual
  bool fuse_update = false;    // Newton loops: the cluster Krylov kernel also applies K6 (eps below)
  double fuse_eps = 0.0;
  bool update_applied = false; // the last Krylov launch already applied the update
  double* gm_V = nullptr;      // GMRES basis (RSIM_GMRES_M + 1 vectors), allocated on first use
  double* gm_part = nullptr;   // GMRES reduction partials
  double* dn_W = nullptr;      // direct solve: dense N×N (N ≤ RSIM_DIRECT_MAX), grown on demand
  int64_t dn_cap = 0;          // direct solve: N the three dn_* buffers are sized for
  double* dn_colbuf = nullptr; // direct solve: double-buffered pivot column
  int32_t* dn_piv = nullptr;   // direct solve: row interchanges
  struct Ilu {                 // level-scheduled block ILU(0) (ilu.cu)
    int32_t *ptr = nullptr, *col = nullptr, *src = nullptr, *frows = nullptr, *foff = nullptr, *brows = nullptr,
            *boff = nullptr;
    double *val = nullptr, *dinv = nullptr, *y = nullptr;
    int64_t cap[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};  // element capacities, one per buffer
    int32_t nnz = 0, nf = 0, nb = 0, maxw = 0;
  } ilu;
  int64_t nnc_total = 0;
  rsim_fluid_params fl{};
  double bhp = 0.0;
  double dt = 1.0;
  cudaStream_t stream = nullptr;
  int sm_count = 0;
  int max_coop_blocks[4] = {0, 0, 0, 0};  // per b (1..3)

  // graph (immutable)
  double *tx = nullptr, *ty = nullptr, *tz = nullptr, *pv = nullptr, *wi = nullptr;
  uint8_t* kind = nullptr;
  int32_t *nptr = nullptr, *nnbr = nullptr;
  double* nt = nullptr;

  // state
  double *u = nullptr, *u_start = nullptr, *mold = nullptr, *p_prev = nullptr;
  uint8_t *st = nullptr, *st_start = nullptr;

  // sets
  uint8_t *flags = nullptr, *flags_alt = nullptr;
  int32_t *act_buf = nullptr, *g2l = nullptr, *label = nullptr;
  int32_t* act = nullptr;  // current active list (act_buf or a DD sub-list)
  int32_t nA = 0;
  double *dp = nullptr, *last_dp = nullptr;
  int32_t *tile_cnt = nullptr, *tile_off = nullptr;
  int32_t* list_buf = nullptr;  // uploaded lists

  // local system (ELL + global-NNC-slot values).  Columns [slot][cap]; values in the
  // per-block-size layout of ell_at() below; ell_po marks the pressure-only blocks
  // (blockops.h col0_only, one bit per slot) for the cluster kernel's product select
  // and the bench's block counters.
  int32_t* ell_col = nullptr;
  int64_t ell_cap = 0;  // ELL slot stride of the current assembly: n_A rounded up to 32
  double* ell_val = nullptr;
  uint8_t* ell_po = nullptr;  // [cap] bit s: the block of slot s is pressure-only (b > 1)
  int32_t* nnc_lcol = nullptr;
  double* nnc_val = nullptr;
  double *F_raw = nullptr, *rhs = nullptr;
  double* part_f2 = nullptr;

  // Krylov
  double *x = nullptr, *r = nullptr, *r0 = nullptr, *p = nullptr, *v = nullptr, *s = nullptr, *t = nullptr;
  double *p2 = nullptr, *v2 = nullptr;  // second buffers of p, v (fused Krylov)
  double *ph = nullptr, *sh = nullptr;  // M^-1 p, M^-1 s (Neumann-1 preconditioner)
  double* part = nullptr;  // [4][nchunks_max]

  DevScalars* dsc = nullptr;   // device
  DevScalars* hsc = nullptr;   // pinned host mirror

  DDLists dd;

  // timing
  bool timing = false;
  struct Ev { cudaEvent_t a, b; int phase; };
  std::vector<Ev> ev_pool, ev_live;
  double ms[4] = {0, 0, 0, 0};
  double last_eps = 0.0;
  bool pending_nA = false;
  std::vector<int32_t> h_nptr, h_nnbr;
  int32_t launches = 0;
  cudaEvent_t marks[64] = {};
  double* u_ckpt = nullptr;
  uint8_t* st_ckpt = nullptr;
  void* l2_scratch = nullptr;
  int64_t counters[7] = {0, 0, 0, 0, 0, 0, 0};  // [5], [6]: Σ its · stored / pressure-only ELL blocks (b > 1)
  uint8_t* pin0 = nullptr;  // F_PIN|F_A for pinned cells, 0 elsewhere (reset source)
  unsigned long long* ktrace = nullptr;  // Krylov phase cycle counters (debug, RSIM_KTRACE=1)
  uint32_t* nnc_bits = nullptr;  // bit i: cell i has NNC entries (small-grid K7: skips the nptr reads)
  uint32_t* bits[2] = {nullptr, nullptr};  // K7 bitmap dilation ping-pong (n/32 words each; nx % 32 == 0)
  bool seed_bits_ready = false;            // bits[0] holds the D0 seed (written by the fused reset + seed)
};

// ---- error plumbing (abi.cu) -------------------------------------------------
void rsim_set_error(const std::string& msg);
int rsim_cuda_fail(cudaError_t e, const char* what);
#define RSIM_TRY(x)                    \
  do {                                 \
    const int rsim_r_ = (x);           \
    if (rsim_r_ != RSIM_OK) return rsim_r_; \
  } while (0)
#define RSIM_CUDA(call)                                   \
  do {                                                    \
    cudaError_t _e = (call);                              \
    if (_e != cudaSuccess) return rsim_cuda_fail(_e, #call); \
  } while (0)

// Phase timers (abi.cu): wrap kernel sequences of one phase.
void rsim_phase_begin(rsim_gpu_ctx* c, int phase);
void rsim_phase_end(rsim_gpu_ctx* c);

// ---- launchers implemented in the .cu files ---------------------------------
int launch_assemble(rsim_gpu_ctx* c);
int launch_krylov(rsim_gpu_ctx* c, const rsim_solver_opts* o);
// returns RSIM_ENOTAPPLICABLE when the system does not fit one cluster
constexpr int RSIM_ENOTAPPLICABLE = 100;
int launch_krylov_dsm(rsim_gpu_ctx* c, const rsim_solver_opts* o);
int launch_update(rsim_gpu_ctx* c, double eps);
int launch_mold(rsim_gpu_ctx* c);
int launch_set_reset(rsim_gpu_ctx* c, int all_active);
int launch_set_list(rsim_gpu_ctx* c, const int32_t* dev_list, int32_t n);
int launch_set_update(rsim_gpu_ctx* c, int mode, int round, double eps, int m, int shrink_locked, int force_expand,
                      int do_dilate);
int launch_threshold(rsim_gpu_ctx* c, double eps);
int launch_initial_support(rsim_gpu_ctx* c, double eps);
int launch_seed_pinned(rsim_gpu_ctx* c);
int launch_dd_begin(rsim_gpu_ctx* c);
int launch_dd_partition(rsim_gpu_ctx* c, int32_t n_sub, int32_t* sizes);
int launch_dd_select(rsim_gpu_ctx* c, int32_t k);
int launch_dd_skip(rsim_gpu_ctx* c, int32_t k);
int launch_categories(rsim_gpu_ctx* c, uint8_t* dev_out);
int launch_seed_support(rsim_gpu_ctx* c, double eps);
int launch_reset_seed(rsim_gpu_ctx* c, double eps);
int launch_materialize_cols(rsim_gpu_ctx* c);
int launch_gmres(rsim_gpu_ctx* c, const rsim_solver_opts* o);
int launch_direct(rsim_gpu_ctx* c, const rsim_solver_opts* o);
int ilu_prepare(rsim_gpu_ctx* c);  // pattern, level schedules, factorisation (precond == ILU0)
void ilu_free(rsim_gpu_ctx* c);
int launch_state_from_dp(rsim_gpu_ctx* c, double p_hi, double scale);

// ---- device helpers ------------------------------------------------------------
#ifdef __CUDACC__

__device__ __forceinline__ unsigned long long dbits(double a) {
  return (unsigned long long)__double_as_longlong(a);
}

// Canonical reduction helpers (blockops.h): a 256-row chunk is 8 warps; each
// warp shuffles 16..1 (lane 0 holds the warp sum), then the 8 warp sums are
// combined with offsets 4,2,1.
// Full active set (V_A = all cells, local == global index): the ELL columns
// of cell i are structural — the Cartesian neighbours in slot order, -1 off-grid.
__device__ __forceinline__ void implicit_cols(int32_t nx, int32_t ny, int32_t nz, bool d3, int64_t i, int32_t* cl) {
  const uint32_t nxy = (uint32_t)nx * (uint32_t)ny;
  uint32_t ix, iy, iz;
#ifndef RSIM_NO_POW2  // A/B switch
  if ((((uint32_t)nx & ((uint32_t)nx - 1u)) | ((uint32_t)ny & ((uint32_t)ny - 1u))) == 0u) {
    // power-of-two nx, ny (configs 2-5): shifts and masks instead of two integer divisions
    const int sx = 31 - __clz(nx), sy = 31 - __clz(ny);
    ix = (uint32_t)i & ((uint32_t)nx - 1u);
    iy = ((uint32_t)i >> sx) & ((uint32_t)ny - 1u);
    iz = (uint32_t)i >> (sx + sy);
  } else
#endif
  {
    iz = (uint32_t)i / nxy;
    const uint32_t rem = (uint32_t)i - iz * nxy;
    iy = rem / (uint32_t)nx;
    ix = rem - iy * (uint32_t)nx;
  }
  const int32_t ii = (int32_t)i;
  // constant indices only: a runtime slot counter would force cl[] (and the
  // caller's gathers) into local memory
  const int32_t ym = iy > 0 ? ii - nx : -1, xm = ix > 0 ? ii - 1 : -1;
  const int32_t xp = ix + 1 < (uint32_t)nx ? ii + 1 : -1, yp = iy + 1 < (uint32_t)ny ? ii + nx : -1;
  if (d3) {
    cl[0] = iz > 0 ? ii - (int32_t)nxy : -1;
    cl[1] = ym; cl[2] = xm; cl[3] = xp; cl[4] = yp;
    cl[5] = iz + 1 < (uint32_t)nz ? ii + (int32_t)nxy : -1;
  } else {
    cl[0] = ym; cl[1] = xm; cl[2] = xp; cl[3] = yp;
  }
}

// ELL block values of (slot s, local row l), element e = r·b + c.
//  * b <= 2: warp-tiled planar, [slot][l / 32][e][l % 32] (cap is a multiple of 32):
//    a warp's load of one element is one contiguous 256 B run and the b² runs of its
//    32 rows are adjacent, so a slot is ONE address stream.  Whole config-3 run (b = 2,
//    round 2, same box): 1.33 s with row-major blocks, 1.23 s tiled.
//  * b = 3: row-major blocks, [slot][l][e] (72 B per row).  Measured on the whole
//    config-4 run: row-major 9.7-9.9 s, fully planar [slot][e][cap] 12.7-13.4 s (54
//    address streams), warp-tiled 12.4 s (nine loads per block held in registers
//    before the product: the b = 3 kernel then spills at its 128-register cap).
// ell_es(b²) is the distance between consecutive elements of one block.
// ell_po[l]: bits 0..5 pressure-only block per slot (b > 1); bit 7 (ELL_ROW_NNC): the
// row has at least one NNC block with an active column (written when the graph has
// NNCs), so the Krylov kernels walk act -> nptr -> nnc_lcol only for such rows.
constexpr unsigned ELL_ROW_NNC = 0x80u;
__host__ __device__ constexpr int ell_es(int bb) { return bb > 4 ? 1 : 32; }
__host__ __device__ __forceinline__ int64_t ell_at(int64_t cap, int bb, int s, int e, int64_t l) {
  if (bb > 4) return ((int64_t)s * cap + l) * bb + e;
  return ((((int64_t)s * (cap >> 5) + (l >> 5)) * bb + e) << 5) + (l & 31);
}
// The whole block of (slot s, row l) as a flat row-major b×b array.
template <int B>
__device__ __forceinline__ void ell_load(const double* __restrict__ val, int64_t cap, int s, int64_t l, double* M) {
  const double* __restrict__ vp = val + ell_at(cap, B * B, s, 0, l);
#pragma unroll
  for (int e = 0; e < B * B; ++e) M[e] = vp[e * ell_es(B * B)];
}

__device__ __forceinline__ double warp_tree(double v) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) v = v + __shfl_down_sync(0xffffffffu, v, off);
  return v;
}
// warp_tree for a warp whose lanes >= n hold structural +0.0 (n warp-uniform):
// the additions of a structural zero are done locally (v + 0.0, same bits as
// adding the shuffled +0.0), only the offsets that can reach data shuffle.
__device__ __forceinline__ double warp_tree_n(double v, int n) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    if (off >= n) v = v + 0.0;
    else v = v + __shfl_down_sync(0xffffffffu, v, off);
  }
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

__device__ __forceinline__ void atomic_max_bits(unsigned long long* addr, double nonneg) {
  atomicMax(addr, dbits(nonneg));
}

// warp max of a non-negative double, lane 0 gets the result
__device__ __forceinline__ double warp_max(double a) {
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) a = fmax(a, __shfl_down_sync(0xffffffffu, a, off));
  return a;
}

#endif  // __CUDACC__
