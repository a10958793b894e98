// C-ABI entry points (include/fitsne_b200.h).  Argument validation mirrors the
// reference's ValueError / FloatingPointError conditions; every call is
// stream-ordered on the caller's stream.
#include <cstring>
#include <string>
#include <algorithm>

#include "common.cuh"
#include "internal.h"
#include "fft.cuh"

namespace fitsne {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int ensure(DevBuf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return FITSNE_OK;
  if (b.ptr) {
    cudaFree(b.ptr);
    b.ptr = nullptr;
    b.cap = 0;
  }
  size_t want = bytes + bytes / 4;  // headroom for a growing embedding span
  cudaError_t e = cudaMalloc(&b.ptr, want);
  if (e != cudaSuccess) {
    cudaGetLastError();
    e = cudaMalloc(&b.ptr, bytes);
    want = bytes;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    b.ptr = nullptr;
    set_error(std::string("device allocation of ") + std::to_string(bytes) + " bytes failed");
    return FITSNE_ENOMEM;
  }
  b.cap = want;
  return FITSNE_OK;
}

static void release(DevBuf& b) {
  if (b.ptr) cudaFree(b.ptr);
  b.ptr = nullptr;
  b.cap = 0;
}

}  // namespace fitsne

using namespace fitsne;

#define CTX_CHECK(ctx)                                    \
  FITSNE_RANGE(__func__);                                 \
  do {                                                    \
    if (!(ctx)) {                                         \
      set_error("null context");                          \
      return FITSNE_EINVAL;                               \
    }                                                     \
    FITSNE_CUDA(cudaSetDevice((ctx)->device));            \
  } while (0)

static inline cudaStream_t S_(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static int check_interp(int p, int min_int, double ipi) {
  if (p < 2 || p > kMaxP) {
    set_error("points_per_interval must be in [2, 8]");
    return FITSNE_EINVAL;
  }
  if (min_int < 1) {
    set_error("min_intervals must be >= 1");
    return FITSNE_EINVAL;
  }
  if (!(ipi > 0)) {
    set_error("intervals_per_integer must be positive");
    return FITSNE_EINVAL;
  }
  return FITSNE_OK;
}

extern "C" {

const char* fitsne_last_error(void) { return g_last_error.c_str(); }
int fitsne_abi_version(void) { return FITSNE_ABI_VERSION; }

int fitsne_create(fitsne_ctx** out, int device, int dims, int dtype, int points_per_interval,
                  int min_intervals, double intervals_per_integer) {
  if (!out) { set_error("null output"); return FITSNE_EINVAL; }
  *out = nullptr;
  if (dims != 1 && dims != 2) { set_error("embedding dims must be 1 or 2"); return FITSNE_EINVAL; }
  if (dtype != FITSNE_F32 && dtype != FITSNE_F64) { set_error("dtype must be f32 or f64"); return FITSNE_EINVAL; }
  FITSNE_TRY(check_interp(points_per_interval, min_intervals, intervals_per_integer));
  FITSNE_CUDA(cudaSetDevice(device));
  fitsne_ctx* c = new fitsne_ctx();
  c->device = device;
  c->dims = dims;
  c->dtype = dtype;
  c->p = points_per_interval;
  c->min_intervals = min_intervals;
  c->intervals_per_integer = intervals_per_integer;
  int sms = 148;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) == cudaSuccess) c->num_sms = sms;
  cudaError_t e = cudaMallocHost(&c->h_grid, sizeof(fitsne_grid));
  if (e == cudaSuccess) e = cudaMallocHost(&c->h_scal, 64 * sizeof(double));
  // pinned pages are recycled between contexts and come back dirty: the
  // bounding-box sequence word polled in h_scal[15] must not hold an old
  // context's value
  if (e == cudaSuccess) std::memset(c->h_scal, 0, 64 * sizeof(double));
  if (e == cudaSuccess) e = cudaMallocHost(&c->h_status, 16 * sizeof(int32_t));
  if (e != cudaSuccess) {
    set_error(std::string("pinned allocation failed: ") + cudaGetErrorString(e));
    delete c;
    return FITSNE_ECUDA;
  }
  int rc = ensure(c->scal, 64 * sizeof(double));
  if (rc == FITSNE_OK) rc = ensure(c->counter, 64 * sizeof(int));
  if (rc != FITSNE_OK) { fitsne_destroy(c); return rc; }
  *out = c;
  return FITSNE_OK;
}

int fitsne_destroy(fitsne_ctx* c) {
  if (!c) return FITSNE_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  DevBuf* bufs[] = {&c->accum, &c->fbuf, &c->sbuf, &c->pot, &c->tw, &c->zpart, &c->bbox_part,
                    &c->scal, &c->counter, &c->forces, &c->gtmp, &c->part, &c->gen, &c->sortbuf,
                    &c->hy, &c->hg, &c->big, &c->bigtw, &c->y64, &c->r64, &c->dgrid,
                    &c->plan_table};
  for (DevBuf* b : bufs) release(*b);
  if (c->shadow) fitsne_destroy(c->shadow);
  if (c->h_dgrid) cudaFreeHost(c->h_dgrid);
  comm_free(c);
  free_tiled(c);
  if (c->ev_in) cudaEventDestroy(c->ev_in);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  if (c->ev_bbox) cudaEventDestroy(c->ev_bbox);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->spec) cudaStreamDestroy(c->spec);
  if (c->ev_spec_in) cudaEventDestroy(c->ev_spec_in);
  if (c->ev_spec) cudaEventDestroy(c->ev_spec);
  for (cudaEvent_t e : c->ev_piece)
    if (e) cudaEventDestroy(e);
  if (c->ev_out) cudaEventDestroy(c->ev_out);
  if (c->out) cudaStreamDestroy(c->out);
  if (c->hp) cudaStreamDestroy(c->hp);
  if (c->h_grid) cudaFreeHost(c->h_grid);
  if (c->h_scal) cudaFreeHost(c->h_scal);
  if (c->h_status) cudaFreeHost(c->h_status);
  delete c;
  return FITSNE_OK;
}

int fitsne_set_interp(fitsne_ctx* ctx, int p, int min_int, double ipi) {
  CTX_CHECK(ctx);
  FITSNE_TRY(check_interp(p, min_int, ipi));
  ctx->p = p;
  ctx->min_intervals = min_int;
  ctx->intervals_per_integer = ipi;
  ctx->grid_valid = false;
  return FITSNE_OK;
}

int fitsne_set_option(fitsne_ctx* ctx, int option, int value) {
  CTX_CHECK(ctx);
  if (option == FITSNE_OPT_SORTED_SPREAD) {
    if (value < 0 || value > 3) { set_error("spread mode must be 0, 1, 2 or 3"); return FITSNE_EINVAL; }
    ctx->sorted_spread = value;
    return FITSNE_OK;
  }
  if (option == FITSNE_OPT_OVERLAP) {
    if (value < 0 || value > 4) { set_error("overlap mode must be 0 .. 4"); return FITSNE_EINVAL; }
    if (ctx->side && value != ctx->overlap) {  // priority is fixed at creation
      cudaStreamSynchronize(ctx->side);
      cudaStreamDestroy(ctx->side);
      ctx->side = nullptr;
      if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
      if (ctx->ev_done) cudaEventDestroy(ctx->ev_done);
      ctx->ev_in = ctx->ev_done = nullptr;
    }
    ctx->overlap = value;
    return FITSNE_OK;
  }
  if (option == FITSNE_OPT_SPREAD_REPLICAS) {
    if (value < 1 || value > 16 || (value & (value - 1))) {
      set_error("spread replicas must be a power of two in [1, 16]");
      return FITSNE_EINVAL;
    }
    if (value != ctx->spread_replicas) {
      ctx->spread_replicas = value;
      ctx->accum_clean = false;   // re-zero the (possibly larger) accumulator
    }
    return FITSNE_OK;
  }
  if (option == FITSNE_OPT_SPMV_BLOCKS_PER_SM) {
    if (value < 0 || value > 32) { set_error("SpMV blocks per SM must be in [0, 32]"); return FITSNE_EINVAL; }
    ctx->spmv_blocks_per_sm = value;
    return FITSNE_OK;
  }
  if (option == FITSNE_OPT_TILED_SPMV) {
    if (value < 0 || value > 2) { set_error("tiled SpMV mode must be 0, 1 or 2"); return FITSNE_EINVAL; }
    ctx->tiled_spmv = value;
    return FITSNE_OK;
  }
  if (option == FITSNE_OPT_TILE_ROWS || option == FITSNE_OPT_TILE_COLS) {
    if (value < 2 || value > 16384 || (value & 1)) {
      set_error("tile rows / cols must be even and in [2, 16384]");
      return FITSNE_EINVAL;
    }
    const int R = option == FITSNE_OPT_TILE_ROWS ? value : ctx->tile_rows;
    const int C = option == FITSNE_OPT_TILE_COLS ? value : ctx->tile_cols;
    ctx->tile_rows = R;
    ctx->tile_cols = C;
    return FITSNE_OK;
  }
  if (option == FITSNE_OPT_FFT_PATH) {
    if (value < 0 || value > 2) { set_error("FFT path must be 0, 1 or 2"); return FITSNE_EINVAL; }
    ctx->fft_path = value;
    if (ctx->shadow) ctx->shadow->fft_path = value;
    return FITSNE_OK;
  }
  if (option == FITSNE_OPT_DEVICE_GRID) {
    if (value < 0 || value > 1) { set_error("device grid mode must be 0 or 1"); return FITSNE_EINVAL; }
    ctx->devgrid = value;
    return FITSNE_OK;
  }
  if (option == FITSNE_OPT_RELABEL) {
    if (value < 0 || value > 2) { set_error("relabel mode must be 0, 1 or 2"); return FITSNE_EINVAL; }
    ctx->relabel = value;
    return FITSNE_OK;
  }
  if (option == FITSNE_OPT_GRID_F64) {
    if (value < 0 || value > 2) { set_error("fp64 grid mode must be 0, 1 or 2"); return FITSNE_EINVAL; }
    ctx->grid_f64 = value;
    ctx->grid_valid = false;  // re-derive the pipeline with the next grid
    return FITSNE_OK;
  }
  if (option == FITSNE_OPT_FFT_COLS) {
    if (value != 1 && value != 2 && value != 4) { set_error("FFT columns per block must be 1, 2 or 4"); return FITSNE_EINVAL; }
    ctx->cols_per_block = value;
    return FITSNE_OK;
  }
  if (option == FITSNE_OPT_HOST_PIECES) {
    if (value < 0 || value > 2) { set_error("host schedule must be 0, 1 or 2"); return FITSNE_EINVAL; }
    ctx->host_pieces = value;
    return FITSNE_OK;
  }
  if (option == FITSNE_OPT_TILED_BANK_ORDER) {
    if (value < 0 || value > 2) { set_error("bank order must be 0, 1 or 2"); return FITSNE_EINVAL; }
    ctx->tiled_bank_order = value;
    return FITSNE_OK;
  }
  if (option == FITSNE_OPT_SPMV_JOIN) {
    if (value < 0 || value > 1) { set_error("spmv join must be 0 or 1"); return FITSNE_EINVAL; }
    ctx->spmv_join = value;
    return FITSNE_OK;
  }
  if (option == FITSNE_OPT_SPEC_AHEAD) {
    if (value < 0 || value > 1) { set_error("spectrum ahead must be 0 or 1"); return FITSNE_EINVAL; }
    ctx->spec_opt = value;
    return FITSNE_OK;
  }
  if (option == FITSNE_OPT_SIDE_GATHER) {
    if (value < 0 || value > 1) { set_error("side gather must be 0 or 1"); return FITSNE_EINVAL; }
    ctx->side_gather = value;
    return FITSNE_OK;
  }
  if (option == FITSNE_OPT_TILED_CTAS) {
    if (value < 0 || value > 65536) { set_error("tiled CTAs must be in [0, 65536]"); return FITSNE_EINVAL; }
    ctx->tiled_ctas = value;
    return FITSNE_OK;
  }
  set_error("unknown option");
  return FITSNE_EINVAL;
}

int fitsne_tiled_stats(fitsne_ctx* ctx, const void* Y, int64_t* out, void* stream) {
  CTX_CHECK(ctx);
  if (!out) { set_error("null output"); return FITSNE_EINVAL; }
  return tiled_stats(ctx, Y, out, S_(stream));
}

int fitsne_make_grid(fitsne_ctx* ctx, const void* Y, int64_t n, fitsne_grid* grid_host, void* stream) {
  CTX_CHECK(ctx);
  if (n < 1) { set_error("points must be a non-empty (N,) or (N, dims) array"); return FITSNE_EINVAL; }
  FITSNE_TRY(make_grid(ctx, Y, n, S_(stream)));
  if (grid_host) *grid_host = ctx->grid;
  return FITSNE_OK;
}

int fitsne_bbox(fitsne_ctx* ctx, const void* Y, int64_t n, double* bbox_host, void* stream) {
  CTX_CHECK(ctx);
  if (n < 1) {
    for (int d = 0; d < ctx->dims; ++d) { bbox_host[d] = INFINITY; bbox_host[ctx->dims + d] = -INFINITY; }
    return FITSNE_OK;
  }
  return compute_bbox(ctx, Y, n, bbox_host, S_(stream));
}

__global__ void k_bbox_empty(double* out, int S) {
  for (int d = 0; d < S; ++d) { out[d] = INFINITY; out[S + d] = INFINITY; }  // -max = +inf
  out[2 * S] = 0.0;
}

int fitsne_bbox_device(fitsne_ctx* ctx, const void* Y, int64_t n, double* bbox_dev, void* stream) {
  CTX_CHECK(ctx);
  if (!bbox_dev) { set_error("null bbox buffer"); return FITSNE_EINVAL; }
  if (n < 1) {
    k_bbox_empty<<<1, 1, 0, S_(stream)>>>(bbox_dev, ctx->dims);
    FITSNE_CHECK_LAUNCH();
    return FITSNE_OK;
  }
  return bbox_device(ctx, Y, n, bbox_dev, S_(stream));
}

int fitsne_grid_from_bbox(fitsne_ctx* ctx, const double* bbox_host, fitsne_grid* grid_host) {
  CTX_CHECK(ctx);
  fitsne_grid g;
  FITSNE_TRY(grid_from_bbox(ctx, bbox_host, &g));
  // no stream argument: the twiddle table is rebuilt (on the legacy stream)
  // only when the FFT length changes; wait for it only then, so the sharded
  // step has no host synchronisation here
  const int gen0 = ctx->tw_gen;
  FITSNE_TRY(install_grid(ctx, g, 0));
  if (ctx->tw_gen != gen0) FITSNE_CUDA(cudaStreamSynchronize(0));
  if (grid_host) *grid_host = g;
  return FITSNE_OK;
}

int fitsne_set_grid(fitsne_ctx* ctx, const fitsne_grid* gh) {
  CTX_CHECK(ctx);
  if (!gh) { set_error("null grid"); return FITSNE_EINVAL; }
  fitsne_grid g = *gh;
  if (g.dims != ctx->dims) { set_error("grid dims do not match the context"); return FITSNE_EINVAL; }
  if (g.n_intervals < 1) { set_error("n_intervals must be >= 1"); return FITSNE_EINVAL; }
  if (g.points_per_interval < 2 || g.points_per_interval > kMaxP) {
    set_error("points_per_interval must be in [2, 8]");
    return FITSNE_EINVAL;
  }
  for (int d = 0; d < g.dims; ++d)
    if (!(g.hi[d] > g.lo[d])) { set_error("grid bounds must satisfy hi > lo"); return FITSNE_EINVAL; }
  g.nodes_per_dim = g.n_intervals * g.points_per_interval;
  for (int d = 0; d < g.dims; ++d) g.spacing[d] = (g.hi[d] - g.lo[d]) / (double)g.nodes_per_dim;
  g.fft_len = smooth23_at_least(2 * g.nodes_per_dim - 1);
  g.status = 0;
  const int gen0 = ctx->tw_gen;
  FITSNE_TRY(install_grid(ctx, g, 0));
  if (ctx->tw_gen != gen0) FITSNE_CUDA(cudaStreamSynchronize(0));
  return FITSNE_OK;
}

int fitsne_point_interp(fitsne_ctx* ctx, const void* Y, int64_t n, int64_t* node_index, void* weights,
                        void* stream) {
  CTX_CHECK(ctx);
  return point_interp(ctx, Y, n, node_index, weights, S_(stream));
}

int fitsne_spread(fitsne_ctx* ctx, const void* Y, int64_t n, const void* charges, int ncharge,
                  void* coeffs, void* stream) {
  CTX_CHECK(ctx);
  if (ncharge < 1) { set_error("need at least one charge column"); return FITSNE_EINVAL; }
  return spread_general(ctx, Y, n, charges, ncharge, coeffs, S_(stream));
}

int fitsne_kernel_matvec(fitsne_ctx* ctx, int kernel, const void* coeffs, int ncol, void* out,
                         void* stream) {
  CTX_CHECK(ctx);
  return matvec_general(ctx, kernel, coeffs, ncol, out, S_(stream));
}

int fitsne_gather(fitsne_ctx* ctx, const void* Y, int64_t n, const void* values, int ncol, void* out,
                  void* stream) {
  CTX_CHECK(ctx);
  return gather_general(ctx, Y, n, values, ncol, out, S_(stream));
}

int fitsne_evaluate_nbody(fitsne_ctx* ctx, const void* Y, int64_t n, const void* charges, int ncharge,
                          int kernel, int include_self, void* out, void* stream) {
  CTX_CHECK(ctx);
  cudaStream_t st = S_(stream);
  if (n < 1) { set_error("points must be a non-empty (N,) or (N, dims) array"); return FITSNE_EINVAL; }
  FITSNE_TRY(make_grid(ctx, Y, n, st));
  size_t G = 1;
  for (int d = 0; d < ctx->dims; ++d) G *= (size_t)ctx->grid.nodes_per_dim;
  size_t es = dsize(ctx->dtype);
  FITSNE_TRY(ensure(ctx->gen, 2 * G * (size_t)ncharge * es));
  char* coeffs = (char*)ctx->gen.ptr;
  char* vals = coeffs + G * ncharge * es;
  FITSNE_TRY(spread_general(ctx, Y, n, charges, ncharge, coeffs, st));
  FITSNE_TRY(matvec_general(ctx, kernel, coeffs, ncharge, vals, st));
  FITSNE_TRY(gather_general(ctx, Y, n, vals, ncharge, out, st));
  if (!include_self) FITSNE_TRY(sub_inplace(ctx, out, charges, n * ncharge, st));
  return FITSNE_OK;
}

int fitsne_repulsive(fitsne_ctx* ctx, const void* Y, int64_t n, void* forces, double* z_host, void* k1,
                     void* k2, void* stream) {
  CTX_CHECK(ctx);
  cudaStream_t st = S_(stream);
  if (n < 2) { set_error("repulsion needs at least two points"); return FITSNE_EINVAL; }
  FITSNE_TRY(make_grid(ctx, Y, n, st));
  FITSNE_TRY(spread_tsne(ctx, Y, n, nullptr, st));
  FITSNE_TRY(fft_tsne(ctx, nullptr, n, k1 != nullptr, st));
  FITSNE_TRY(gather_tsne(ctx, Y, n, forces, k1, k2, st));
  FITSNE_TRY(read_scalars(ctx, 1, st));
  double z = ctx->h_scal[0];
  if (z_host) *z_host = z;
  if (!(z > 0)) { set_error("normalization Z must be positive"); return FITSNE_EZ; }
  return FITSNE_OK;
}

int fitsne_repulsive_exact(fitsne_ctx* ctx, const void* Y, int64_t n, void* forces, double* z_host,
                           void* k1, void* k2, void* stream) {
  CTX_CHECK(ctx);
  cudaStream_t st = S_(stream);
  if (n < 2) { set_error("repulsion needs at least two points"); return FITSNE_EINVAL; }
  if (!k1 || !k2) { set_error("exact repulsion needs k1 and k2 buffers"); return FITSNE_EINVAL; }
  FITSNE_TRY(exact_sums(ctx, Y, n, k1, k2, st));
  FITSNE_TRY(forces_from_sums(ctx, Y, n, k2, forces, st));
  FITSNE_TRY(read_scalars(ctx, 1, st));
  double z = ctx->h_scal[0];
  if (z_host) *z_host = z;
  if (!(z > 0)) { set_error("normalization Z must be positive"); return FITSNE_EZ; }
  return FITSNE_OK;
}

int fitsne_set_affinities(fitsne_ctx* ctx, const int64_t* rowptr, const int32_t* col, const void* val,
                          int64_t n_rows, int64_t row_begin, int64_t n_total, int64_t nnz) {
  CTX_CHECK(ctx);
  if (n_rows < 0 || row_begin < 0 || row_begin + n_rows > n_total || nnz < 0) {
    set_error("invalid affinity row range");
    return FITSNE_EINVAL;
  }
  if (n_total > 0x7fffffffLL) { set_error("more than 2^31-1 points"); return FITSNE_EINVAL; }
  ctx->rowptr = rowptr;
  ctx->col = col;
  ctx->val = val;
  ctx->n_rows = n_rows;
  ctx->row_begin = row_begin;
  ctx->n_total = n_total;
  ctx->nnz = nnz;
  ctx->plogp_valid = false;
  free_tiled(ctx);  // contents may have changed: re-tile on next use
  return FITSNE_OK;
}

int fitsne_attractive(fitsne_ctx* ctx, const void* Y_full, void* out, void* stream) {
  CTX_CHECK(ctx);
  return attractive(ctx, Y_full, nullptr, 1.0, out, 0, false, S_(stream));
}

int fitsne_gradient(fitsne_ctx* ctx, const void* Y, double alpha, void* grad, double* z_host,
                    void* stream) {
  CTX_CHECK(ctx);
  cudaStream_t st = S_(stream);
  if (!ctx->rowptr) { set_error("no affinities registered"); return FITSNE_EINVAL; }
  if (ctx->row_begin != 0 || ctx->n_rows != ctx->n_total) {
    set_error("fitsne_gradient needs all rows registered (use the sharded stages)");
    return FITSNE_EINVAL;
  }
  if (!(alpha >= 1.0)) { set_error("exaggeration alpha must be >= 1"); return FITSNE_EINVAL; }
  const int64_t n = ctx->n_total;
  if (n < 2) { set_error("repulsion needs at least two points"); return FITSNE_EINVAL; }
  // attractive SpMV on a side stream overlapping grid + spread + FFT, then a
  // thread-per-point gather-and-combine (attract.cu: gradient_overlapped)
  FITSNE_TRY(gradient_overlapped(ctx, Y, alpha, grad, st));
  if (z_host) {
    FITSNE_TRY(read_scalars(ctx, 1, st));
    *z_host = ctx->h_scal[0];
  }
  return FITSNE_OK;
}

int fitsne_gradient_host(fitsne_ctx* ctx, const void* Y_host, double alpha, void* grad_host,
                         void* stream) {
  CTX_CHECK(ctx);
  cudaStream_t st = S_(stream);
  if (!ctx->rowptr) { set_error("no affinities registered"); return FITSNE_EINVAL; }
  if (ctx->row_begin != 0 || ctx->n_rows != ctx->n_total) {
    set_error("fitsne_gradient_host needs all rows registered (use the sharded stages)");
    return FITSNE_EINVAL;
  }
  if (!Y_host || !grad_host) { set_error("null buffer"); return FITSNE_EINVAL; }
  if (!(alpha >= 1.0)) { set_error("exaggeration alpha must be >= 1"); return FITSNE_EINVAL; }
  if (ctx->n_total < 2) { set_error("repulsion needs at least two points"); return FITSNE_EINVAL; }
  return gradient_host(ctx, Y_host, alpha, grad_host, st);
}

int fitsne_kl(fitsne_ctx* ctx, const void* Y_full, double z, double* kl_host, void* stream) {
  CTX_CHECK(ctx);
  cudaStream_t st = S_(stream);
  if (!ctx->rowptr) { set_error("no affinities registered"); return FITSNE_EINVAL; }
  if (!ctx->plogp_valid) FITSNE_TRY(compute_plogp(ctx, st));
  FITSNE_TRY(kl_sum(ctx, Y_full, st));
  FITSNE_TRY(read_scalars(ctx, 2, st));
  // sum over stored entries of these rows (both triangles)
  *kl_host = ctx->plogp + ctx->h_scal[1] + ctx->psum * std::log(z);
  return FITSNE_OK;
}

int fitsne_step(fitsne_ctx* ctx, void* Y, const void* grad, void* velocity, void* gains, int64_t n,
                double momentum, double learning_rate, void* stream) {
  CTX_CHECK(ctx);
  return step_update(ctx, Y, grad, velocity, gains, n, momentum, learning_rate, S_(stream));
}

int fitsne_iterate(fitsne_ctx* ctx, const void* Y, void* Y_out, void* velocity, void* gains,
                   double alpha, double momentum, double learning_rate, double* kl_dev,
                   int32_t* status_dev, void* stream) {
  CTX_CHECK(ctx);
  if (!ctx->rowptr) { set_error("no affinities registered"); return FITSNE_EINVAL; }
  if (ctx->row_begin != 0 || ctx->n_rows != ctx->n_total) {
    set_error("fitsne_iterate needs all rows registered");
    return FITSNE_EINVAL;
  }
  if (ctx->n_total < 2) { set_error("repulsion needs at least two points"); return FITSNE_EINVAL; }
  return iterate_fused(ctx, Y, Y_out, velocity, gains, alpha, momentum, learning_rate, kl_dev,
                       status_dev, S_(stream));
}

int64_t fitsne_grid_accum_len(fitsne_ctx* ctx) {
  if (!ctx || !ctx->grid_valid) return 0;
  int64_t G = 1;
  for (int d = 0; d < ctx->dims; ++d) G *= ctx->grid.nodes_per_dim;
  return G * kNodeSlots;
}

int fitsne_grid_accum_dtype(fitsne_ctx* ctx) {
  if (!ctx) return FITSNE_F32;
  return ctx->wide ? FITSNE_F64 : ctx->dtype;
}

int fitsne_spread_tsne(fitsne_ctx* ctx, const void* Y_local, int64_t n_local, void* accum, void* stream) {
  CTX_CHECK(ctx);
  if (!accum) { set_error("null accumulator"); return FITSNE_EINVAL; }
  return spread_tsne(ctx, Y_local, n_local, accum, S_(stream));
}

int fitsne_fft_tsne(fitsne_ctx* ctx, void* accum, int64_t n_total, int with_k1, double* z_host,
                    void* stream) {
  CTX_CHECK(ctx);
  cudaStream_t st = S_(stream);
  FITSNE_TRY(fft_tsne(ctx, accum, n_total, with_k1 != 0, st));
  if (z_host) {
    FITSNE_TRY(read_scalars(ctx, 1, st));
    *z_host = ctx->h_scal[0];
    if (!(*z_host > 0)) { set_error("normalization Z must be positive"); return FITSNE_EZ; }
  }
  return FITSNE_OK;
}

int fitsne_gather_tsne(fitsne_ctx* ctx, const void* Y_local, int64_t n_local, void* forces, void* k1,
                       void* k2, void* stream) {
  CTX_CHECK(ctx);
  return gather_tsne(ctx, Y_local, n_local, forces, k1, k2, S_(stream));
}

int fitsne_gradient_rows(fitsne_ctx* ctx, const void* Y_full, const void* forces_local, double alpha,
                         void* grad_local, void* stream) {
  CTX_CHECK(ctx);
  return attractive(ctx, Y_full, forces_local, alpha, grad_local, 1, false, S_(stream));
}

int fitsne_combine_rows(fitsne_ctx* ctx, const void* attr, const void* frep, int64_t n, double alpha,
                        void* grad, void* stream) {
  CTX_CHECK(ctx);
  if (!(alpha >= 1.0)) { set_error("exaggeration alpha must be >= 1"); return FITSNE_EINVAL; }
  return combine_rows(ctx, attr, frep, n, alpha, grad, S_(stream));
}

int fitsne_read_z(fitsne_ctx* ctx, double* z_dst, void* stream) {
  CTX_CHECK(ctx);
  if (!z_dst) { set_error("null destination"); return FITSNE_EINVAL; }
  FITSNE_TRY(ensure(ctx->scal, 64 * sizeof(double)));
  FITSNE_CUDA(cudaMemcpyAsync(z_dst, ctx->scal.ptr, sizeof(double), cudaMemcpyDefault, S_(stream)));
  return FITSNE_OK;
}

int fitsne_exact_nbody(fitsne_ctx* ctx, const void* Y, int64_t n, const void* charges, int ncharge,
                       int kernel, int include_self, void* out, void* stream) {
  CTX_CHECK(ctx);
  return exact_nbody(ctx, Y, n, charges, ncharge, kernel, include_self, out, S_(stream));
}

}  // extern "C"
