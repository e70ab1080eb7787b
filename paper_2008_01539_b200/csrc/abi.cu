// abi.cu — implementation of the extern "C" boundary (include/rsim/gpu_abi.h):
// context lifetime, HBM layout, data movement, the active-set entry points
// and debug/parity downloads.  No CPU fallback anywhere: without an sm_100
// device rsim_gpu_create fails with RSIM_ECUDA.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <string>

#include "ctx.cuh"

static thread_local std::string g_err;

void rsim_set_error(const std::string& msg) { g_err = msg; }
int rsim_cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return RSIM_ECUDA;
}

void rsim_phase_begin(rsim_gpu_ctx* c, int phase) {
  if (!c->timing) return;
  rsim_gpu_ctx::Ev e;
  if (!c->ev_pool.empty()) { e = c->ev_pool.back(); c->ev_pool.pop_back(); }
  else { cudaEventCreate(&e.a); cudaEventCreate(&e.b); }
  e.phase = phase;
  cudaEventRecord(e.a, c->stream);
  c->ev_live.push_back(e);
}
void rsim_phase_end(rsim_gpu_ctx* c) {
  if (!c->timing || c->ev_live.empty()) return;
  cudaEventRecord(c->ev_live.back().b, c->stream);
}
static void harvest_timers(rsim_gpu_ctx* c) {
  for (auto& e : c->ev_live) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, e.a, e.b) == cudaSuccess) c->ms[e.phase] += ms;
    c->ev_pool.push_back(e);
  }
  c->ev_live.clear();
}

namespace {

template <class T>
int dalloc(T** p, int64_t count) {
  if (count <= 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, sizeof(T) * (size_t)count);
  if (e != cudaSuccess) return rsim_cuda_fail(e, "cudaMalloc");
  return RSIM_OK;
}
template <class T>
int h2d(rsim_gpu_ctx* c, T* dst, const T* src, int64_t count) {
  if (count <= 0) return RSIM_OK;
  RSIM_CUDA(cudaMemcpyAsync(dst, src, sizeof(T) * (size_t)count, cudaMemcpyHostToDevice, c->stream));
  return RSIM_OK;
}

#define TRY(x)                    \
  do {                            \
    int _r = (x);                 \
    if (_r != RSIM_OK) return _r; \
  } while (0)

int sync_stats(rsim_gpu_ctx* c) {
  RSIM_CUDA(cudaMemcpyAsync(c->hsc, c->dsc, sizeof(DevScalars), cudaMemcpyDeviceToHost, c->stream));
  RSIM_CUDA(cudaStreamSynchronize(c->stream));
  if (c->timing) harvest_timers(c);
  if (c->pending_nA) { c->nA = c->hsc->nA; c->pending_nA = false; }
  return RSIM_OK;
}

void fill_stats(rsim_gpu_ctx* c, rsim_gpu_stats* st) {
  if (!st) return;
  const DevScalars& h = *c->hsc;
  auto bd = [](unsigned long long b) { double d; std::memcpy(&d, &b, 8); return d; };
  st->status = h.status;
  st->bad_cell = h.bad_cell == INT_MAX ? -1 : h.bad_cell;
  st->lin_iters = h.lin_iters;
  st->n_active = c->nA;
  st->n_boundary = h.nB;
  st->expand = h.expand;
  st->n_new = h.n_new;
  st->pad = 0;
  st->lin_relres = h.lin_relres;
  st->f_norm2 = h.f2;
  st->f_norminf = bd(h.finf);
  st->dp_inf_A = bd(h.maxA);
  st->dp_inf_B = bd(h.maxB);
  st->halo_max = bd(h.halo);
}

__global__ void k_reset_scalars(DevScalars* d) {
  d->status = 0;
  d->bad_cell = INT_MAX;
  d->lin_iters = 0;
  d->lin_relres = 0.0;
  d->f2 = 0.0;
  d->finf = 0ull;
  d->maxA = 0ull;  // ‖δp‖∞ of the coming update (a fused update has no memset of its own)
  d->maxB = 0ull;
  d->nblk = 0ull;
  d->npo = 0ull;
}

// p component of the interleaved state: dst[i] = u[i*b]
__global__ void k_extract_p(int64_t n, int b, const double* __restrict__ u, double* __restrict__ dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = u[i * b];
}

int begin_step(rsim_gpu_ctx* c, double dt) {
  c->dt = dt;
  RSIM_CUDA(cudaMemcpyAsync(c->u_start, c->u, sizeof(double) * c->n * c->b, cudaMemcpyDeviceToDevice, c->stream));
  RSIM_CUDA(cudaMemcpyAsync(c->st_start, c->st, c->n, cudaMemcpyDeviceToDevice, c->stream));
  return launch_mold(c);
}

}  // namespace

// Internal helpers used by solvers.cpp (declared there).
int rsim_internal_begin_step(rsim_gpu_ctx* c, double dt) { return begin_step(c, dt); }
int rsim_internal_commit_step(rsim_gpu_ctx* c) {
  k_extract_p<<<(c->n + 255) / 256, 256, 0, c->stream>>>(c->n, c->b, c->u_start, c->p_prev);
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}
int rsim_internal_reset_scalars(rsim_gpu_ctx* c) {
  k_reset_scalars<<<1, 1, 0, c->stream>>>(c->dsc);
  c->launches++;
  RSIM_CUDA(cudaGetLastError());
  return RSIM_OK;
}
int rsim_internal_dd_begin(rsim_gpu_ctx* c) { return launch_dd_begin(c); }
void rsim_internal_set_iter_hook(rsim_gpu_ctx* c, int (*fn)(void*, int32_t, int32_t), void* user) {
  c->iter_hook = fn;
  c->iter_user = user;
}
double rsim_internal_dt(const rsim_gpu_ctx* c) { return c->dt; }
int rsim_internal_iter_hook(rsim_gpu_ctx* c, int32_t iter, int32_t subdomain) {
  return c->iter_hook ? c->iter_hook(c->iter_user, iter, subdomain) : RSIM_OK;
}
// cells of the graph for M_A = Σ n_A / n (dead filler cells are not cells of the model)
int64_t rsim_internal_n(const rsim_gpu_ctx* c) { return c->n - c->n_dead; }
int rsim_internal_b(const rsim_gpu_ctx* c) { return c->b; }
int32_t rsim_internal_nA(const rsim_gpu_ctx* c) { return c->nA; }

extern "C" {

const char* rsim_gpu_last_error(void) { return g_err.c_str(); }

int rsim_gpu_device_info(char* name, int32_t cap, int32_t* sm_count, int32_t* major, int32_t* minor) {
  int dev = 0, cnt = 0;
  RSIM_CUDA(cudaGetDeviceCount(&cnt));
  if (cnt < 1) { rsim_set_error("no CUDA device"); return RSIM_ECUDA; }
  RSIM_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp p;
  RSIM_CUDA(cudaGetDeviceProperties(&p, dev));
  if (name && cap > 0) { std::strncpy(name, p.name, cap - 1); name[cap - 1] = 0; }
  if (sm_count) *sm_count = p.multiProcessorCount;
  if (major) *major = p.major;
  if (minor) *minor = p.minor;
  return RSIM_OK;
}

int rsim_gpu_set_device(int32_t device) {
  RSIM_CUDA(cudaSetDevice(device));
  return RSIM_OK;
}

int rsim_gpu_counters(rsim_gpu_ctx* c, int64_t* out5, int32_t reset) {
  if (out5)
    for (int k = 0; k < 5; ++k) out5[k] = c->counters[k];
  if (reset)
    for (int k = 0; k < 5; ++k) c->counters[k] = 0;
  return RSIM_OK;
}

int rsim_gpu_block_counters(rsim_gpu_ctx* c, int64_t* out2, int32_t reset) {
  if (out2) { out2[0] = c->counters[5]; out2[1] = c->counters[6]; }
  if (reset) c->counters[5] = c->counters[6] = 0;
  return RSIM_OK;
}

int rsim_gpu_create(rsim_gpu_ctx** out, const rsim_graph_desc* g, const rsim_fluid_params* f) {
  if (!out || !g || !f || f->kind < 1 || f->kind > 3 || g->nx < 1 || g->ny < 1 || g->nz < 1 ||
      (int64_t)g->nx * g->ny * g->nz >= ((int64_t)1 << 31)) {  // cell ids are int32 (CSR, act, g2l)
    rsim_set_error("rsim_gpu_create: bad argument");
    return RSIM_EARG;
  }
  int32_t sms = 0, major = 0, minor = 0;
  TRY(rsim_gpu_device_info(nullptr, 0, &sms, &major, &minor));
  if (major != 10) {
    rsim_set_error("rsim_gpu_create: this build targets sm_100a (B200); device is sm_" + std::to_string(major) +
                   std::to_string(minor));
    return RSIM_ECUDA;
  }
  rsim_gpu_ctx* c = new rsim_gpu_ctx();
  *out = c;
  c->b = f->kind;
  c->fl = *f;
  c->nx = g->nx; c->ny = g->ny; c->nz = g->nz;
  c->n = (int64_t)g->nx * g->ny * g->nz;
  c->d3 = g->nz > 1;
  c->nslot = c->d3 ? 6 : 4;
  c->bhp = g->bhp;
  c->sm_count = sms;
  c->nnc_total = g->nnc_ptr ? g->nnc_ptr[c->n] : 0;
  for (int64_t i = 0; i < c->n; ++i) c->n_dead += g->kind[i] == RSIM_KIND_DEAD;
  c->has_nnc = c->nnc_total > 0;
  const int64_t n = c->n, b = c->b;
  const int64_t nchunks = (n + RSIM_RED_CHUNK - 1) / RSIM_RED_CHUNK;
  RSIM_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  TRY(dalloc(&c->tx, n)); TRY(dalloc(&c->ty, n)); TRY(dalloc(&c->tz, n));
  TRY(dalloc(&c->pv, n)); TRY(dalloc(&c->wi, n)); TRY(dalloc(&c->kind, n));
  TRY(dalloc(&c->nptr, n + 1));
  TRY(dalloc(&c->nnbr, c->nnc_total)); TRY(dalloc(&c->nt, c->nnc_total));
  TRY(dalloc(&c->u, n * b)); TRY(dalloc(&c->u_start, n * b)); TRY(dalloc(&c->mold, n * b));
  TRY(dalloc(&c->p_prev, n));
  TRY(dalloc(&c->st, n)); TRY(dalloc(&c->st_start, n));
  TRY(dalloc(&c->flags, n)); TRY(dalloc(&c->flags_alt, n));
  TRY(dalloc(&c->act_buf, n)); TRY(dalloc(&c->g2l, n)); TRY(dalloc(&c->label, n));
  TRY(dalloc(&c->list_buf, n));
  TRY(dalloc(&c->dp, n)); TRY(dalloc(&c->last_dp, n));
  if (g->nx % 32 == 0) { TRY(dalloc(&c->bits[0], n / 32 + 1)); TRY(dalloc(&c->bits[1], n / 32 + 1)); }
  {  // compaction tiles: K7 uses one tile per (x-row, 1024-cell segment), K8 one per 2048 cells
    const int64_t wrow = (g->nx + 3) / 4, bs = wrow >= 256 ? 256 : ((wrow + 31) / 32) * 32;
    const int64_t k7 = (int64_t)g->ny * g->nz * ((wrow + bs - 1) / bs);
    const int64_t nt = (k7 > nchunks ? k7 : nchunks) + 1;
    TRY(dalloc(&c->tile_cnt, nt)); TRY(dalloc(&c->tile_off, nt));
  }
  {  // slot stride = n_A rounded up to the 32-row tiles of the value layout (ctx.cuh ell_at)
    const int64_t ncap = ((n + 31) / 32) * 32;
    TRY(dalloc(&c->ell_col, c->nslot * ncap)); TRY(dalloc(&c->ell_val, c->nslot * ncap * b * b));
  }
  TRY(dalloc(&c->ell_po, n));
  c->ell_cap = n;
  TRY(dalloc(&c->nnc_lcol, c->nnc_total)); TRY(dalloc(&c->nnc_val, c->nnc_total * b * b));
  TRY(dalloc(&c->F_raw, n * b)); TRY(dalloc(&c->rhs, n * b));
  TRY(dalloc(&c->part_f2, nchunks));
  TRY(dalloc(&c->x, n * b)); TRY(dalloc(&c->r, n * b)); TRY(dalloc(&c->r0, n * b));
  TRY(dalloc(&c->p, n * b)); TRY(dalloc(&c->v, n * b)); TRY(dalloc(&c->s, n * b)); TRY(dalloc(&c->t, n * b));
  TRY(dalloc(&c->p2, n * b)); TRY(dalloc(&c->v2, n * b));
  TRY(dalloc(&c->ph, n * b)); TRY(dalloc(&c->sh, n * b));
  TRY(dalloc(&c->part, 6 * nchunks + 64));  // 5 level-1 + 5 level-2 partial rows
  TRY(dalloc(&c->dsc, 1));
  RSIM_CUDA(cudaMallocHost((void**)&c->hsc, sizeof(DevScalars)));
  std::memset(c->hsc, 0, sizeof(DevScalars));
  TRY(h2d(c, c->tx, g->tx, n)); TRY(h2d(c, c->ty, g->ty, n)); TRY(h2d(c, c->tz, g->tz, n));
  TRY(h2d(c, c->pv, g->pv, n)); TRY(h2d(c, c->wi, g->well_wi, n)); TRY(h2d(c, c->kind, g->kind, n));
  if (c->has_nnc) {
    TRY(h2d(c, c->nptr, g->nnc_ptr, n + 1));
    TRY(h2d(c, c->nnbr, g->nnc_nbr, c->nnc_total));
    TRY(h2d(c, c->nt, g->nnc_t, c->nnc_total));
    c->h_nptr.assign(g->nnc_ptr, g->nnc_ptr + n + 1);
    c->h_nnbr.assign(g->nnc_nbr, g->nnc_nbr + c->nnc_total);
    std::vector<uint32_t> nb((size_t)(n + 31) / 32, 0u);
    for (int64_t i = 0; i < n; ++i)
      if (g->nnc_ptr[i + 1] > g->nnc_ptr[i]) nb[(size_t)(i >> 5)] |= 1u << (i & 31);
    TRY(dalloc(&c->nnc_bits, (int64_t)nb.size()));
    TRY(h2d(c, c->nnc_bits, nb.data(), (int64_t)nb.size()));
  } else {
    RSIM_CUDA(cudaMemsetAsync(c->nptr, 0, sizeof(int32_t) * (n + 1), c->stream));
  }
  RSIM_CUDA(cudaMemsetAsync(c->dsc, 0, sizeof(DevScalars), c->stream));
  RSIM_CUDA(cudaMemsetAsync(c->g2l, 0xff, sizeof(int32_t) * n, c->stream));
  RSIM_CUDA(cudaMemsetAsync(c->dp, 0, sizeof(double) * n, c->stream));
  RSIM_CUDA(cudaMemsetAsync(c->last_dp, 0, sizeof(double) * n, c->stream));
  RSIM_CUDA(cudaMemsetAsync(c->flags, 0, n, c->stream));
  RSIM_CUDA(cudaMemsetAsync(c->label, 0xff, sizeof(int32_t) * n, c->stream));
  RSIM_CUDA(cudaStreamSynchronize(c->stream));
  c->act = c->act_buf;
  c->nA = 0;
  if (const char* e = std::getenv("RSIM_KTRACE"); e && *e == '1') {
    TRY(dalloc(&c->ktrace, RSIM_KTRACE_N));
    RSIM_CUDA(cudaMemset(c->ktrace, 0, RSIM_KTRACE_N * sizeof(unsigned long long)));
  }
  return RSIM_OK;
}

int rsim_gpu_set_debug(rsim_gpu_ctx* c, int32_t flags) {
  if (!c) return RSIM_EARG;
  c->keep_F = (flags & 1) != 0;
  return RSIM_OK;
}

int rsim_gpu_ktrace(rsim_gpu_ctx* c, unsigned long long* out) {
  if (!c->ktrace) return RSIM_EARG;
  RSIM_CUDA(cudaMemcpy(out, c->ktrace, RSIM_KTRACE_N * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  RSIM_CUDA(cudaMemset(c->ktrace, 0, RSIM_KTRACE_N * sizeof(unsigned long long)));
  return RSIM_OK;
}

int rsim_gpu_destroy(rsim_gpu_ctx* c) {
  if (!c) return RSIM_OK;
  cudaStreamSynchronize(c->stream);
  void* ptrs[] = {c->tx, c->ty, c->tz, c->pv, c->wi, c->kind, c->nptr, c->nnbr, c->nt, c->u, c->u_start,
                  c->mold, c->p_prev, c->st, c->st_start, c->flags, c->flags_alt, c->act_buf, c->g2l, c->label,
                  c->list_buf, c->dp, c->last_dp, c->tile_cnt, c->tile_off, c->ell_col, c->ell_val, c->ell_po, c->nnc_lcol,
                  c->nnc_val, c->F_raw, c->rhs, c->part_f2, c->x, c->r, c->r0, c->p, c->v, c->s, c->t, c->p2, c->v2, c->ph, c->sh, c->part,
                  c->dsc, c->dd.sub_cells, c->dd.halo_cells, c->u_ckpt, c->st_ckpt, c->l2_scratch, c->pin0, c->ktrace, c->nnc_bits,
                  c->gm_V, c->gm_part, c->dd.hist, c->bits[0], c->bits[1], c->dn_W, c->dn_colbuf, c->dn_piv};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  ilu_free(c);
  if (c->hsc) cudaFreeHost(c->hsc);
  for (auto& e : c->marks)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->ev_pool) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
  for (auto& e : c->ev_live) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return RSIM_OK;
}

int rsim_gpu_set_state(rsim_gpu_ctx* c, const double* u, const uint8_t* status, double dt) {
  if (!c || !u || !status || !(dt > 0)) { rsim_set_error("set_state: bad argument"); return RSIM_EARG; }
  TRY(h2d(c, c->u, u, c->n * c->b));
  TRY(h2d(c, c->st, status, c->n));
  TRY(begin_step(c, dt));
  RSIM_CUDA(cudaStreamSynchronize(c->stream));
  return RSIM_OK;
}

int rsim_gpu_set_dt(rsim_gpu_ctx* c, double dt) {
  if (!c || !(dt > 0)) return RSIM_EARG;
  c->dt = dt;
  return RSIM_OK;
}

int rsim_gpu_get_state(rsim_gpu_ctx* c, double* u, uint8_t* status) {
  if (!c || !u || !status) return RSIM_EARG;
  RSIM_CUDA(cudaMemcpyAsync(u, c->u, sizeof(double) * c->n * c->b, cudaMemcpyDeviceToHost, c->stream));
  RSIM_CUDA(cudaMemcpyAsync(status, c->st, c->n, cudaMemcpyDeviceToHost, c->stream));
  RSIM_CUDA(cudaStreamSynchronize(c->stream));
  return RSIM_OK;
}

int rsim_gpu_restore_state(rsim_gpu_ctx* c) {
  RSIM_CUDA(cudaMemcpyAsync(c->u, c->u_start, sizeof(double) * c->n * c->b, cudaMemcpyDeviceToDevice, c->stream));
  RSIM_CUDA(cudaMemcpyAsync(c->st, c->st_start, c->n, cudaMemcpyDeviceToDevice, c->stream));
  return RSIM_OK;
}

int rsim_gpu_set_active(rsim_gpu_ctx* c, const int32_t* sorted, int32_t n, rsim_gpu_stats* st) {
  if (!c || (n > 0 && !sorted) || n > c->n) return RSIM_EARG;
  rsim_phase_begin(c, 0);
  if (n < 0) {
    TRY(launch_set_reset(c, 1));
  } else {
    TRY(launch_set_reset(c, 0));
    TRY(h2d(c, c->list_buf, sorted, n));
    TRY(launch_set_list(c, c->list_buf, n));
  }
  TRY(launch_set_update(c, MODE_KEEP, 0, 0.0, 0, 1, 0, 0));
  rsim_phase_end(c);
  c->pending_nA = true;
  TRY(sync_stats(c));
  fill_stats(c, st);
  return RSIM_OK;
}

int rsim_gpu_initial_active(rsim_gpu_ctx* c, int32_t first_step, double eps, int32_t m, rsim_gpu_stats* st) {
  rsim_phase_begin(c, 0);
  TRY(launch_set_reset(c, 0));
  if (first_step) {
    TRY(launch_seed_pinned(c));
    TRY(launch_set_update(c, MODE_EXPAND, 0, eps, m, 0, 1, 1));
  } else {
    TRY(launch_initial_support(c, eps));
    TRY(launch_set_update(c, MODE_KEEP, 0, eps, 0, 1, 0, 0));
  }
  rsim_phase_end(c);
  c->pending_nA = true;
  TRY(sync_stats(c));
  fill_stats(c, st);
  return RSIM_OK;
}

int rsim_gpu_estimate_active(rsim_gpu_ctx* c, double eps, int32_t m, int32_t shrink_locked, rsim_gpu_stats* st) {
  rsim_phase_begin(c, 0);
  TRY(launch_set_update(c, MODE_DEVICE, 0, eps, m, shrink_locked, 0, 1));
  c->counters[4] += 1;
  rsim_phase_end(c);
  c->pending_nA = true;
  if (st) {
    TRY(sync_stats(c));
    fill_stats(c, st);
  }
  return RSIM_OK;
}

int rsim_gpu_assemble(rsim_gpu_ctx* c) {
  rsim_phase_begin(c, 1);
  c->counters[0] += c->nA;
  TRY(rsim_internal_reset_scalars(c));
  TRY(launch_assemble(c));
  rsim_phase_end(c);
  return RSIM_OK;
}

// C-linkage setter for the host-only translation units (simulate.cpp)
void rsim_set_error_c(const char* msg) { rsim_set_error(msg); }

int rsim_gpu_linear_solve(rsim_gpu_ctx* c, const rsim_solver_opts* o) {
  if (!c || !o) return RSIM_EARG;
  if (o->lin_method < RSIM_LIN_BICGSTAB || o->lin_method > RSIM_LIN_DIRECT || o->precond < RSIM_PREC_BJACOBI ||
      o->precond > RSIM_PREC_NEUMANN1) {
    rsim_set_error("rsim_gpu_linear_solve: lin_method / precond out of range");
    return RSIM_EARG;
  }
  rsim_phase_begin(c, 2);
  c->counters[2] += 1;
  c->counters[3] += c->nA;
  TRY(launch_krylov(c, o));
  rsim_phase_end(c);
  return RSIM_OK;
}

int rsim_gpu_update(rsim_gpu_ctx* c, double eps) {
  c->last_eps = eps;
  if (c->update_applied) {  // fused into the preceding cluster Krylov launch (Newton loops only)
    c->update_applied = false;
    return RSIM_OK;
  }
  rsim_phase_begin(c, 3);
  TRY(launch_update(c, eps));
  rsim_phase_end(c);
  return RSIM_OK;
}

// Newton loops: solve + update, with the update fused into the Krylov kernel
// when the cluster path runs (the public linear_solve never fuses).
int rsim_internal_solve_update(rsim_gpu_ctx* c, const rsim_solver_opts* o, double eps) {
  c->fuse_update = true;
  c->fuse_eps = eps;
  c->update_applied = false;
  const int r = rsim_gpu_linear_solve(c, o);
  c->fuse_update = false;
  if (r != RSIM_OK) return r;
  return rsim_gpu_update(c, eps);
}

int rsim_gpu_threshold(rsim_gpu_ctx* c, double eps) {
  c->last_eps = eps;
  return launch_threshold(c, eps);
}

int rsim_gpu_stats_get(rsim_gpu_ctx* c, rsim_gpu_stats* st) {
  TRY(sync_stats(c));
  fill_stats(c, st);
  return RSIM_OK;
}

int rsim_internal_add_row_iters(rsim_gpu_ctx* c, int64_t nA, int64_t its) {  // after the stats sync of the solve
  c->counters[1] += nA * its;
  c->counters[5] += (int64_t)c->hsc->nblk * its;
  c->counters[6] += (int64_t)c->hsc->npo * its;
  return RSIM_OK;
}

int rsim_gpu_dd_expand(rsim_gpu_ctx* c, double eps, int32_t m, int32_t round, rsim_gpu_stats* st) {
  rsim_phase_begin(c, 0);
  TRY(launch_set_update(c, MODE_DD, round, eps, m, 0, 0, 1));
  rsim_phase_end(c);
  c->pending_nA = true;
  TRY(sync_stats(c));
  fill_stats(c, st);
  return RSIM_OK;
}

int rsim_gpu_dd_partition(rsim_gpu_ctx* c, int32_t n_sub, int32_t* sizes_out) {
  if (n_sub < 1) return RSIM_EARG;
  rsim_phase_begin(c, 0);
  int r = launch_dd_partition(c, n_sub, sizes_out);
  rsim_phase_end(c);
  return r;
}

int rsim_gpu_dd_select(rsim_gpu_ctx* c, int32_t k, rsim_gpu_stats* st) {
  if (k < 0 || k >= c->dd.n_sub) return RSIM_EARG;
  rsim_phase_begin(c, 0);
  TRY(launch_dd_select(c, k));
  rsim_phase_end(c);
  if (st) {
    TRY(sync_stats(c));
    fill_stats(c, st);
  }
  return RSIM_OK;
}

int rsim_gpu_dd_skip(rsim_gpu_ctx* c, int32_t k) {
  if (k < 0 || k >= c->dd.n_sub) return RSIM_EARG;
  return launch_dd_skip(c, k);
}

int rsim_gpu_download_labels(rsim_gpu_ctx* c, int32_t* labels) {
  RSIM_CUDA(cudaMemcpyAsync(labels, c->label, sizeof(int32_t) * c->n, cudaMemcpyDeviceToHost, c->stream));
  RSIM_CUDA(cudaStreamSynchronize(c->stream));
  return RSIM_OK;
}

int rsim_gpu_download_active(rsim_gpu_ctx* c, int32_t* act, int32_t* n) {
  RSIM_CUDA(cudaStreamSynchronize(c->stream));
  if (n) *n = c->nA;
  if (act && c->nA > 0)
    RSIM_CUDA(cudaMemcpy(act, c->act, sizeof(int32_t) * c->nA, cudaMemcpyDeviceToHost));
  return RSIM_OK;
}

int rsim_gpu_download_flags(rsim_gpu_ctx* c, uint8_t* out) {
  uint8_t* tmp = nullptr;
  TRY(dalloc(&tmp, c->n));
  int r = launch_categories(c, tmp);
  if (r == RSIM_OK) {
    cudaMemcpyAsync(out, tmp, c->n, cudaMemcpyDeviceToHost, c->stream);
    cudaStreamSynchronize(c->stream);
  }
  cudaFree(tmp);
  return r;
}

int rsim_gpu_download_boundary(rsim_gpu_ctx* c, int32_t* vb, int32_t* n) {
  std::vector<uint8_t> f(c->n);
  RSIM_CUDA(cudaMemcpyAsync(f.data(), c->flags, c->n, cudaMemcpyDeviceToHost, c->stream));
  RSIM_CUDA(cudaStreamSynchronize(c->stream));
  int32_t k = 0;
  for (int64_t i = 0; i < c->n; ++i)
    if ((f[i] & F_A) && (f[i] & F_B)) { if (vb) vb[k] = (int32_t)i; ++k; }
  if (n) *n = k;
  return RSIM_OK;
}

int64_t rsim_gpu_download_system(rsim_gpu_ctx* c, double* F_raw, double* rhs, int32_t* rowptr, int32_t* col,
                                 double* val, int64_t cap_nnzb) {
  const int64_t nA = c->nA, b = c->b, bb = b * b, cap = c->ell_cap;
  TRY(launch_materialize_cols(c));
  RSIM_CUDA(cudaStreamSynchronize(c->stream));
  std::vector<int32_t> ecol(c->nslot * nA), act(nA);
  std::vector<double> eval(c->nslot * nA * bb);
  for (int s = 0; s < c->nslot; ++s) {
    RSIM_CUDA(cudaMemcpy(&ecol[s * nA], c->ell_col + s * cap, sizeof(int32_t) * nA, cudaMemcpyDeviceToHost));
  }
  {  // device layout (ctx.cuh ell_at) -> [slot][row][element] for the CSR copy below
    std::vector<double> dev((size_t)c->nslot * cap * bb);
    RSIM_CUDA(cudaMemcpy(dev.data(), c->ell_val, sizeof(double) * dev.size(), cudaMemcpyDeviceToHost));
    for (int s = 0; s < c->nslot; ++s)
      for (int64_t l = 0; l < nA; ++l)
        for (int e = 0; e < bb; ++e) eval[(s * nA + l) * bb + e] = dev[ell_at(cap, (int)bb, s, e, l)];
  }
  RSIM_CUDA(cudaMemcpy(act.data(), c->act, sizeof(int32_t) * nA, cudaMemcpyDeviceToHost));
  std::vector<int32_t> nlcol(c->nnc_total);
  std::vector<double> nval(c->nnc_total * bb);
  if (c->has_nnc) {
    RSIM_CUDA(cudaMemcpy(nlcol.data(), c->nnc_lcol, sizeof(int32_t) * c->nnc_total, cudaMemcpyDeviceToHost));
    RSIM_CUDA(cudaMemcpy(nval.data(), c->nnc_val, sizeof(double) * c->nnc_total * bb, cudaMemcpyDeviceToHost));
  }
  if (F_raw) {
    if (c->f2_parts && !c->keep_F) {
      rsim_set_error("download_system: raw residual not stored (large assembly; enable rsim_gpu_set_debug bit 0)");
      return -RSIM_EARG;
    }
    RSIM_CUDA(cudaMemcpy(F_raw, c->F_raw, sizeof(double) * nA * b, cudaMemcpyDeviceToHost));
  }
  if (rhs) RSIM_CUDA(cudaMemcpy(rhs, c->rhs, sizeof(double) * nA * b, cudaMemcpyDeviceToHost));
  int64_t nnz = 0;
  for (int64_t l = 0; l < nA; ++l) {
    if (rowptr) rowptr[l] = (int32_t)nnz;
    auto put = [&](int32_t cl, const double* v) {
      if (col && val && nnz < cap_nnzb) {
        col[nnz] = cl;
        std::memcpy(&val[nnz * bb], v, sizeof(double) * bb);
      }
      ++nnz;
    };
    for (int s = 0; s < c->nslot; ++s)
      if (ecol[s * nA + l] >= 0) put(ecol[s * nA + l], &eval[(s * nA + l) * bb]);
    if (c->has_nnc) {
      int64_t i = act[l];
      for (int32_t q = c->h_nptr[i]; q < c->h_nptr[i + 1]; ++q)
        if (nlcol[q] >= 0) put(nlcol[q], &nval[q * bb]);
    }
  }
  if (rowptr) rowptr[nA] = (int32_t)nnz;
  return nnz;
}

int rsim_gpu_download_solution(rsim_gpu_ctx* c, double* x) {
  RSIM_CUDA(cudaStreamSynchronize(c->stream));
  if (c->nA > 0) RSIM_CUDA(cudaMemcpy(x, c->x, sizeof(double) * c->nA * c->b, cudaMemcpyDeviceToHost));
  return RSIM_OK;
}

int rsim_gpu_upload_dp(rsim_gpu_ctx* c, const double* dp) {
  TRY(h2d(c, c->dp, dp, c->n));
  RSIM_CUDA(cudaStreamSynchronize(c->stream));
  return RSIM_OK;
}

int rsim_gpu_download_dp(rsim_gpu_ctx* c, double* dp) {
  RSIM_CUDA(cudaMemcpyAsync(dp, c->dp, sizeof(double) * c->n, cudaMemcpyDeviceToHost, c->stream));
  RSIM_CUDA(cudaStreamSynchronize(c->stream));
  return RSIM_OK;
}

int rsim_gpu_timers(rsim_gpu_ctx* c, int32_t enable, double* ms4, int32_t* launches) {
  RSIM_CUDA(cudaStreamSynchronize(c->stream));
  harvest_timers(c);
  if (ms4)
    for (int k = 0; k < 4; ++k) ms4[k] = c->ms[k];
  if (launches) *launches = c->launches;
  if (enable >= 0) {
    c->timing = enable != 0;
    for (int k = 0; k < 4; ++k) c->ms[k] = 0.0;
    c->launches = 0;
  }
  return RSIM_OK;
}

int rsim_gpu_mark(rsim_gpu_ctx* c, int32_t slot) {
  if (slot < 0 || slot >= 64) return RSIM_EARG;
  if (!c->marks[slot]) RSIM_CUDA(cudaEventCreate(&c->marks[slot]));
  RSIM_CUDA(cudaEventRecord(c->marks[slot], c->stream));
  return RSIM_OK;
}

int rsim_gpu_elapsed(rsim_gpu_ctx* c, int32_t a, int32_t b, double* ms) {
  if (a < 0 || a >= 64 || b < 0 || b >= 64 || !c->marks[a] || !c->marks[b]) return RSIM_EARG;
  RSIM_CUDA(cudaEventSynchronize(c->marks[b]));
  float f = 0.f;
  RSIM_CUDA(cudaEventElapsedTime(&f, c->marks[a], c->marks[b]));
  *ms = f;
  return RSIM_OK;
}

int rsim_gpu_flush_l2(rsim_gpu_ctx* c) {
  const size_t bytes = 512ull << 20;
  if (!c->l2_scratch) RSIM_CUDA(cudaMalloc(&c->l2_scratch, bytes));
  RSIM_CUDA(cudaMemsetAsync(c->l2_scratch, c->launches & 0xff, bytes, c->stream));
  return RSIM_OK;
}

int rsim_gpu_checkpoint(rsim_gpu_ctx* c, int32_t restore) {
  if (!c->u_ckpt) {
    TRY(dalloc(&c->u_ckpt, c->n * c->b));
    TRY(dalloc(&c->st_ckpt, c->n));
  }
  if (restore) {
    RSIM_CUDA(cudaMemcpyAsync(c->u, c->u_ckpt, sizeof(double) * c->n * c->b, cudaMemcpyDeviceToDevice, c->stream));
    RSIM_CUDA(cudaMemcpyAsync(c->st, c->st_ckpt, c->n, cudaMemcpyDeviceToDevice, c->stream));
  } else {
    RSIM_CUDA(cudaMemcpyAsync(c->u_ckpt, c->u, sizeof(double) * c->n * c->b, cudaMemcpyDeviceToDevice, c->stream));
    RSIM_CUDA(cudaMemcpyAsync(c->st_ckpt, c->st, c->n, cudaMemcpyDeviceToDevice, c->stream));
  }
  return RSIM_OK;
}

int rsim_gpu_support_active(rsim_gpu_ctx* c, double eps, int32_t m, rsim_gpu_stats* st) {
  c->last_eps = eps;
  rsim_phase_begin(c, 0);
  TRY(launch_reset_seed(c, eps));
  TRY(launch_set_update(c, MODE_EXPAND, 0, eps, m, 0, 1, 1));
  rsim_phase_end(c);
  c->pending_nA = true;
  if (st) {
    TRY(sync_stats(c));
    fill_stats(c, st);
  }
  return RSIM_OK;
}

int rsim_gpu_state_from_dp(rsim_gpu_ctx* c, double p_hi, double scale) {
  TRY(launch_state_from_dp(c, p_hi, scale));
  return begin_step(c, c->dt);
}

}  // extern "C"
