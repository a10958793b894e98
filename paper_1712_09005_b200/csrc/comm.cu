// Sharded gradient over NCCL inside the C-ABI (SURVEY 8(b) fitsne_comm_init,
// 8(e)): a non-Python host runs the multi-GPU path with one context per rank
// and three library calls (fitsne_nccl_unique_id on rank 0, fitsne_comm_init,
// fitsne_gradient_sharded).  The step is the one parallel.py orchestrates
// with torch.distributed:
//
//   rank r owns points [N r / R, N (r+1) / R) and the CSR rows of them;
//   1. local bounding box {min, -max, -nonfinite} on the device, one MIN
//      all-reduce, one 40-byte readback -> the same grid on every rank
//      (nbody.py:131-143);
//   2. all-gather of Y into a padded layout (rank r's rows at [r m, r m +
//      count_r), m the largest shard; the CSR columns are remapped to it once);
//   3. the local rows' attractive SpMV on a side stream (optimizer.py:150-166);
//   4. private spread -> SUM all-reduce of the grid accumulator -> replicated
//      FFT stage + Parseval Z -> gather of F_rep for the local points;
//   5. grad = 4 (alpha F_attr - F_rep) for the local rows (optimizer.py:262).
//
// NCCL is resolved at run time (dlopen; the copy already loaded into the
// process -- e.g. torch's -- is preferred), so the library has no link-time
// NCCL dependency and never mixes two NCCL builds in one process.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "common.cuh"
#include "internal.h"

namespace fitsne {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

static NcclApi* nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
    api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
    api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
    api.all_reduce = (decltype(api.all_reduce))dlsym(h, "ncclAllReduce");
    api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
    api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce &&
             api.all_gather && api.error_string;
  });
  return api.ok ? &api : nullptr;
}

#define FITSNE_NCCL(expr)                                                                   \
  do {                                                                                      \
    ncclResult_t _r = (expr);                                                               \
    if (_r != ncclSuccess) {                                                                \
      ::fitsne::set_error(std::string("NCCL error: ") + nccl()->error_string(_r) + " at " \
                          __FILE__ ":" + std::to_string(__LINE__));                         \
      return FITSNE_ENCCL;                                                                  \
    }                                                                                       \
  } while (0)

static inline int64_t shard_lo(int64_t n, int r, int R) { return n * r / R; }

struct Comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  int64_t n = 0;        // points over all ranks
  int64_t m = 0;        // largest shard (padded layout stride)
  bool ragged = false;
  // what the padded-column CSR copy was made from
  const int32_t* col_src = nullptr;
  int64_t nnz_src = -1;
  DevBuf colmap, ypad, yfull, bbox, acc, fattr, frep, zh;
  cudaEvent_t ev_y = nullptr, ev_attr = nullptr, ev_z = nullptr;
  double* h_bbox = nullptr;
  double* h_z = nullptr;
};

int comm_free(fitsne_ctx* ctx) {
  Comm* c = ctx->comm;
  if (!c) return FITSNE_OK;
  if (c->comm && nccl()) nccl()->comm_destroy(c->comm);
  for (DevBuf* b : {&c->colmap, &c->ypad, &c->yfull, &c->bbox, &c->acc, &c->fattr, &c->frep, &c->zh})
    if (b->ptr) cudaFree(b->ptr);
  for (cudaEvent_t e : {c->ev_y, c->ev_attr, c->ev_z})
    if (e) cudaEventDestroy(e);
  if (c->h_bbox) cudaFreeHost(c->h_bbox);
  if (c->h_z) cudaFreeHost(c->h_z);
  delete c;
  ctx->comm = nullptr;
  return FITSNE_OK;
}

// col -> padded index: rank(col) m + (col - shard_lo(rank))
__global__ void k_pad_cols(const int32_t* __restrict__ col, int64_t nnz, int64_t n, int R, int64_t m,
                           int32_t* __restrict__ out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = col[k];
    int r = (int)((c * R) / n);  // shard_lo(r) <= c < shard_lo(r + 1), corrected below
    while (r > 0 && c < n * r / R) --r;
    while (r + 1 < R && c >= n * (r + 1) / R) ++r;
    out[k] = (int32_t)(r * m + (c - n * r / R));
  }
}

}  // namespace fitsne

using namespace fitsne;

extern "C" int fitsne_nccl_unique_id(void* id_out) {
  if (!id_out) { set_error("null output"); return FITSNE_EINVAL; }
  if (!nccl()) { set_error("NCCL (libnccl.so.2) could not be loaded"); return FITSNE_ENCCL; }
  ncclUniqueId id;
  FITSNE_NCCL(nccl()->get_unique_id(&id));
  std::memcpy(id_out, &id, sizeof(id));
  return FITSNE_OK;
}

extern "C" int fitsne_comm_init(fitsne_ctx* ctx, const void* unique_id, int rank, int nranks, int64_t n_total) {
  if (!ctx || !unique_id) { set_error("null argument"); return FITSNE_EINVAL; }
  FITSNE_RANGE("fitsne_comm_init");
  if (nranks < 1 || rank < 0 || rank >= nranks || n_total < nranks || n_total > 0x7fffffffLL) {
    set_error("invalid rank / world size / point count");
    return FITSNE_EINVAL;
  }
  if (!nccl()) { set_error("NCCL (libnccl.so.2) could not be loaded"); return FITSNE_ENCCL; }
  FITSNE_CUDA(cudaSetDevice(ctx->device));
  comm_free(ctx);
  Comm* c = new Comm();
  ctx->comm = c;
  c->rank = rank;
  c->nranks = nranks;
  c->n = n_total;
  for (int r = 0; r < nranks; ++r)
    c->m = std::max<int64_t>(c->m, shard_lo(n_total, r + 1, nranks) - shard_lo(n_total, r, nranks));
  c->ragged = c->m * nranks != n_total;
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  FITSNE_NCCL(nccl()->comm_init_rank(&c->comm, nranks, id, rank));
  FITSNE_CUDA(cudaEventCreateWithFlags(&c->ev_y, cudaEventDisableTiming));
  FITSNE_CUDA(cudaEventCreateWithFlags(&c->ev_attr, cudaEventDisableTiming));
  FITSNE_CUDA(cudaEventCreateWithFlags(&c->ev_z, cudaEventDisableTiming));
  FITSNE_CUDA(cudaMallocHost(&c->h_bbox, 8 * sizeof(double)));
  FITSNE_CUDA(cudaMallocHost(&c->h_z, sizeof(double)));
  return FITSNE_OK;
}

extern "C" int fitsne_comm_destroy(fitsne_ctx* ctx) {
  if (!ctx) return FITSNE_OK;
  return comm_free(ctx);
}

// One sharded evaluation for this rank's rows.  Y_local (n_local, s) and
// grad_local (n_local, s) in the context dtype; z_host optional.
static int gradient_sharded(fitsne_ctx* ctx, const void* Y_local, double alpha, void* grad_local,
                            double* z_host, cudaStream_t st) {
  Comm* c = ctx->comm;
  const int S = ctx->dims, R = c->nranks;
  const size_t es = dsize(ctx->dtype);
  const int64_t lo = shard_lo(c->n, c->rank, R), n_local = shard_lo(c->n, c->rank + 1, R) - lo;
  if (!ctx->rowptr || ctx->row_begin != lo || ctx->n_rows != n_local ||
      (ctx->n_total != c->n && ctx->n_total != c->m * R)) {
    set_error("registered rows are not this rank's shard [N r / R, N (r+1) / R)");
    return FITSNE_EINVAL;
  }
  if (!(alpha >= 1.0)) { set_error("exaggeration alpha must be >= 1"); return FITSNE_EINVAL; }
  // padded column layout (once per registered P)
  if (c->ragged && ctx->col != (const int32_t*)c->colmap.ptr) {
    FITSNE_TRY(ensure(c->colmap, sizeof(int32_t) * (size_t)std::max<int64_t>(ctx->nnz, 1)));
    k_pad_cols<<<8 * ctx->num_sms, 256, 0, st>>>(ctx->col, ctx->nnz, c->n, R, c->m, (int32_t*)c->colmap.ptr);
    FITSNE_CHECK_LAUNCH();
    c->col_src = ctx->col;
    c->nnz_src = ctx->nnz;
    ctx->col = (const int32_t*)c->colmap.ptr;
    ctx->n_total = c->m * R;
    ctx->plogp_valid = false;
    free_tiled(ctx);
  } else if (!c->ragged && ctx->n_total != c->n) {
    set_error("registered affinities do not cover the communicator's points");
    return FITSNE_EINVAL;
  }
  NcclApi* api = nccl();
  const ncclDataType_t ndt = ctx->dtype == FITSNE_F32 ? ncclFloat32 : ncclFloat64;
  // 1. local box, queued first (its blocks get the GPU ahead of the SpMV)
  FITSNE_TRY(ensure(c->bbox, sizeof(double) * 8));
  double* bb = (double*)c->bbox.ptr;
  FITSNE_TRY(bbox_device(ctx, Y_local, n_local, bb, st));
  FITSNE_NCCL(api->all_reduce(bb, bb, (size_t)(2 * S + 1), ncclFloat64, ncclMin, c->comm, st));
  FITSNE_CUDA(cudaMemcpyAsync(c->h_bbox, bb, sizeof(double) * (2 * S + 1), cudaMemcpyDeviceToHost, st));
  FITSNE_CUDA(cudaEventRecord(c->ev_z, st));  // (reused below for Z)
  // 2. all-gather Y (padded layout)
  const void* yfull = Y_local;
  if (R > 1) {
    FITSNE_TRY(ensure(c->yfull, es * S * (size_t)(c->m * R)));
    const void* src = Y_local;
    if (n_local != c->m) {
      FITSNE_TRY(ensure(c->ypad, es * S * (size_t)c->m));
      FITSNE_CUDA(cudaMemcpyAsync(c->ypad.ptr, Y_local, es * S * (size_t)n_local, cudaMemcpyDeviceToDevice, st));
      src = c->ypad.ptr;
    }
    FITSNE_NCCL(api->all_gather(src, c->yfull.ptr, (size_t)(c->m * S), ndt, c->comm, st));
    yfull = c->yfull.ptr;
  }
  // 3. local rows' SpMV on the side stream
  if (!ctx->side) {
    int plo = 0, phi = 0;
    FITSNE_CUDA(cudaDeviceGetStreamPriorityRange(&plo, &phi));
    FITSNE_CUDA(cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, plo));
    FITSNE_CUDA(cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming));
    FITSNE_CUDA(cudaEventCreateWithFlags(&ctx->ev_done, cudaEventDisableTiming));
  }
  FITSNE_TRY(ensure(c->fattr, es * S * (size_t)std::max<int64_t>(n_local, 1)));
  FITSNE_CUDA(cudaEventRecord(c->ev_y, st));
  FITSNE_CUDA(cudaStreamWaitEvent(ctx->side, c->ev_y, 0));
  FITSNE_TRY(attractive(ctx, yfull, nullptr, 1.0, c->fattr.ptr, 0, false, ctx->side));
  FITSNE_CUDA(cudaEventRecord(c->ev_attr, ctx->side));
  // 4. the grid (one readback), private spread, SUM all-reduce, FFT, gather
  FITSNE_CUDA(cudaEventSynchronize(c->ev_z));
  if (c->h_bbox[2 * S] != 0.0) { set_error("points must be finite"); return FITSNE_EPOINTS; }
  double box[4];
  for (int d = 0; d < S; ++d) {
    box[d] = c->h_bbox[d];
    box[S + d] = -c->h_bbox[S + d];
  }
  fitsne_grid g;
  FITSNE_TRY(grid_from_bbox(ctx, box, &g));
  FITSNE_TRY(install_grid(ctx, g, st));
  int64_t G = 1;
  for (int d = 0; d < S; ++d) G *= g.nodes_per_dim;
  const bool wide = ctx->wide;
  const size_t aes = wide ? 8 : es;
  const size_t acc_bytes = aes * (size_t)G * kNodeSlots;
  if (c->acc.cap < acc_bytes) {
    FITSNE_TRY(ensure(c->acc, acc_bytes));
    FITSNE_CUDA(cudaMemsetAsync(c->acc.ptr, 0, c->acc.cap, st));
  }
  FITSNE_TRY(spread_tsne(ctx, Y_local, n_local, c->acc.ptr, st));
  FITSNE_NCCL(api->all_reduce(c->acc.ptr, c->acc.ptr, (size_t)G * kNodeSlots, wide ? ncclFloat64 : ndt, ncclSum,
                              c->comm, st));
  int rc = fft_tsne(ctx, c->acc.ptr, c->n, false, st);  // consumes and clears the accumulator
  if (rc != FITSNE_OK) {
    cudaMemsetAsync(c->acc.ptr, 0, c->acc.cap, st);
    return rc;
  }
  FITSNE_CUDA(cudaMemcpyAsync(c->h_z, ctx->scal.ptr, sizeof(double), cudaMemcpyDeviceToHost, st));
  FITSNE_CUDA(cudaEventRecord(c->ev_z, st));
  FITSNE_TRY(ensure(c->frep, es * S * (size_t)std::max<int64_t>(n_local, 1)));
  FITSNE_TRY(gather_tsne(ctx, Y_local, n_local, c->frep.ptr, nullptr, nullptr, st));
  // 5. combine once the SpMV is done
  FITSNE_CUDA(cudaStreamWaitEvent(st, c->ev_attr, 0));
  FITSNE_TRY(combine_rows(ctx, c->fattr.ptr, c->frep.ptr, n_local, alpha, grad_local, st));
  // Z > 0 (optimizer.py:242-243), checked once the whole step is queued
  FITSNE_CUDA(cudaEventSynchronize(c->ev_z));
  if (z_host) *z_host = *c->h_z;
  if (!(*c->h_z > 0)) { set_error("normalization Z must be positive"); return FITSNE_EZ; }
  return FITSNE_OK;
}

extern "C" int fitsne_gradient_sharded(fitsne_ctx* ctx, const void* Y_local, double alpha, void* grad_local,
                                       double* z_host, void* stream) {
  if (!ctx) { set_error("null context"); return FITSNE_EINVAL; }
  FITSNE_RANGE("fitsne_gradient_sharded");
  if (!ctx->comm) { set_error("no communicator (fitsne_comm_init)"); return FITSNE_EINVAL; }
  FITSNE_CUDA(cudaSetDevice(ctx->device));
  return join_on_error(ctx, gradient_sharded(ctx, Y_local, alpha, grad_local, z_host, (cudaStream_t)stream));
}
