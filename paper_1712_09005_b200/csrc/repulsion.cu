// Repulsive half of the t-SNE gradient on sm_100a: bounding box + grid
// (nbody.py:118-150), box/weights (nbody.py:201-230), charge spreading
// (nbody.py:233-251), circulant-FFT convolution with the Cauchy kernels
// (nbody.py:262-311), gather (nbody.py:344-350) and the t-SNE assembly of
// optimizer.py:193-245.
//
// 2-D convolution layout (all intermediate buffers are L2 resident):
//   accum  : spread charges, kNodeSlots (=4) per node, node-major (x*n + y)
//   F      : [pair][x][k]  complex, x in [0,n), k in [0,L)   (row-FFT output)
//   S      : [i][ky]       complex, i in [0,n), ky in [0,L/2] (kernel row FFT;
//            .x = row transform of K1, .y = of K2, both real-even)
//   pot    : potentials, 4 slots per node
// Two real signals are packed per complex signal ("pairs"): convolving
// a + i b with a real kernel gives K*a + i K*b, so no Hermitian split is
// needed.  t-SNE pairs: A = y_0 + i y_1 (-> K2), B = unit (-> K2 + i K1).
// Z comes from Parseval on B: Z = sum_k K1hat |Bhat|^2 / L^2 - N, equal to
// the reference's sum of K1 potentials (optimizer.py:206, 241).
#include <cmath>
#include <algorithm>
#include <vector>

#include <atomic>

#include "common.cuh"
#include "fft.cuh"
#include "interp.cuh"
#include "internal.h"

namespace fitsne {

static constexpr int kBlock = 256;

static inline int grid_for(int64_t n, int block = kBlock) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > (1LL << 30)) g = (1LL << 30);
  return (int)g;
}

// =============================================================================
// a1: bounding box (nbody.py:131-133) and grid formulas (nbody.py:134-143)
// =============================================================================
// The grid formulas of make_grid (nbody.py:131-143) on the device, operation
// for operation as grid_from_bbox computes them on the host (explicit IEEE
// roundings, no contraction), so both sides derive the same lo, hi, spacing
// and n_intervals from the same box.
__device__ int device_grid(const double* mn, const double* mx, int S, const DevGridReq& rq, fitsne_grid* out) {
  double lo[2] = {0, 0}, hi[2] = {0, 0}, span[2] = {0, 0};
  double widest = -INFINITY;
  for (int d = 0; d < S; ++d) {
    lo[d] = mn[d];
    hi[d] = mx[d];
    if (!isfinite(lo[d]) || !isfinite(hi[d])) return FITSNE_EPOINTS;
    span[d] = __dsub_rn(hi[d], lo[d]);
    widest = fmax(widest, span[d]);
  }
  const double cells = (rq.ipi == 1.0) ? ceil(widest) : ceil(__dmul_rn(widest, rq.ipi));
  if (cells > 1e7) return FITSNE_ETOOBIG;
  const int n_int = max(rq.min_intervals, (int)cells);
  for (int d = 0; d < S; ++d) {
    if (span[d] < 1.0) {
      const double c = __dmul_rn(0.5, __dadd_rn(lo[d], hi[d]));
      lo[d] = __dsub_rn(c, 0.5);
      hi[d] = __dadd_rn(c, 0.5);
    } else {
      const double pad = __dmul_rn(1e-6, span[d]);
      lo[d] = __dsub_rn(lo[d], pad);
      hi[d] = __dadd_rn(hi[d], pad);
    }
  }
  const long long nn = (long long)n_int * rq.p;
  if (nn > (1 << 20)) return FITSNE_ETOOBIG;
  fitsne_grid g{};
  g.dims = S;
  g.n_intervals = n_int;
  g.points_per_interval = rq.p;
  g.nodes_per_dim = (int)nn;
  for (int d = 0; d < S; ++d) {
    g.lo[d] = lo[d];
    g.hi[d] = hi[d];
    g.spacing[d] = __ddiv_rn(__dsub_rn(hi[d], lo[d]), (double)nn);
  }
  g.fft_len = smooth23_at_least(2 * (int)nn - 1);
  *out = g;
  return FITSNE_OK;
}

template <typename T, int S>
__global__ void k_bbox(const T* __restrict__ Y, int64_t n, double* __restrict__ part,
                       int* __restrict__ nonfinite, double* __restrict__ out, int negate_max,
                       GridArgs* __restrict__ dgrid, DevGridReq rq, double* hout = nullptr,
                       unsigned long long seq = 0) {
  // hout: pinned host memory the last block also writes the box to, followed
  // by the sequence number seq at hout[7] -- the host polls that word instead
  // of waiting for a copy and an event (bbox_wait)
  double mn[S], mx[S];
#pragma unroll
  for (int d = 0; d < S; ++d) { mn[d] = INFINITY; mx[d] = -INFINITY; }
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int d = 0; d < S; ++d) {
      double v = (double)Y[i * S + d];
      if (!isfinite(v)) bad = 1;
      mn[d] = fmin(mn[d], v);
      mx[d] = fmax(mx[d], v);
    }
  }
  __shared__ double smn[32][S], smx[32][S];
#pragma unroll
  for (int d = 0; d < S; ++d) {
    for (int o = 16; o > 0; o >>= 1) {
      mn[d] = fmin(mn[d], __shfl_xor_sync(0xffffffffu, mn[d], o));
      mx[d] = fmax(mx[d], __shfl_xor_sync(0xffffffffu, mx[d], o));
    }
  }
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
#pragma unroll
    for (int d = 0; d < S; ++d) { smn[wid][d] = mn[d]; smx[wid][d] = mx[d]; }
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) {
    int nw = (blockDim.x + 31) / 32;
    for (int w = 1; w < nw; ++w)
#pragma unroll
      for (int d = 0; d < S; ++d) { mn[d] = fmin(mn[d], smn[w][d]); mx[d] = fmax(mx[d], smx[w][d]); }
#pragma unroll
    for (int d = 0; d < S; ++d) {
      part[blockIdx.x * 2 * S + d] = mn[d];
      part[blockIdx.x * 2 * S + S + d] = mx[d];
    }
    if (bad) atomicOr(nonfinite, 1);
  }
  if (out == nullptr) return;
  // last block to finish folds the partials (one launch instead of two on
  // the repulsion chain's critical path); nonfinite[1] is the ticket
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(nonfinite + 1, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int k = threadIdx.x; k < rq.zero_words; k += blockDim.x) rq.zero[k] = 0u;
#pragma unroll
  for (int d = 0; d < S; ++d) { mn[d] = INFINITY; mx[d] = -INFINITY; }
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
#pragma unroll
    for (int d = 0; d < S; ++d) {
      mn[d] = fmin(mn[d], __ldcg(part + b * 2 * S + d));
      mx[d] = fmax(mx[d], __ldcg(part + b * 2 * S + S + d));
    }
  }
#pragma unroll
  for (int d = 0; d < S; ++d)
    for (int o = 16; o > 0; o >>= 1) {
      mn[d] = fmin(mn[d], __shfl_xor_sync(0xffffffffu, mn[d], o));
      mx[d] = fmax(mx[d], __shfl_xor_sync(0xffffffffu, mx[d], o));
    }
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int d = 0; d < S; ++d) { smn[wid][d] = mn[d]; smx[wid][d] = mx[d]; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x + 31) / 32; ++w)
#pragma unroll
      for (int d = 0; d < S; ++d) { mn[d] = fmin(mn[d], smn[w][d]); mx[d] = fmax(mx[d], smx[w][d]); }
    const double sg = negate_max ? -1.0 : 1.0;
#pragma unroll
    for (int d = 0; d < S; ++d) { out[d] = mn[d]; out[S + d] = sg * mx[d]; }
    const int bad = __ldcg(nonfinite);
    out[2 * S] = sg * (double)bad;
    nonfinite[1] = 0;  // ticket reset for the next launch
    if (hout) {
#pragma unroll
      for (int d = 0; d < S; ++d) { hout[d] = mn[d]; hout[S + d] = sg * mx[d]; }
      hout[2 * S] = sg * (double)bad;
      __threadfence_system();
      *reinterpret_cast<volatile unsigned long long*>(hout + 7) = seq;
    }
    if (dgrid) {
      // the grid for the stages queued behind this kernel (device-grid schedule)
      fitsne_grid g;
      int rc = bad ? FITSNE_EPOINTS : device_grid(mn, mx, S, rq, &g);
      GridArgs a;
      if (rc == FITSNE_OK) {
        a = grid_args(g);
        double widest = 0;
        for (int d = 0; d < S; ++d) widest = fmax(widest, g.hi[d] - g.lo[d]);
        if (g.n_intervals > rq.cap_nint || g.fft_len > rq.cap_L) a.status = kDevGridCapacity;
        else if (g.n_intervals > rq.max_nint || (rq.wide_span > 0 && widest > rq.wide_span))
          a.status = kDevGridOther;
      } else {
        a = GridArgs{};
        a.status = kDevGridOther;
      }
      DevGrid* blk = reinterpret_cast<DevGrid*>(dgrid);
      if (a.status == kDevGridOk) {
        // the plan of L from the host-built table (binary search by length)
        const FftPlan* tab = reinterpret_cast<const FftPlan*>(rq.plans);
        int lo_i = 0, hi_i = rq.nplans - 1;
        while (lo_i < hi_i) {
          const int mid = (lo_i + hi_i) >> 1;
          if (tab[mid].L < a.L) lo_i = mid + 1; else hi_i = mid;
        }
        if (tab[lo_i].L == a.L) blk->pl = tab[lo_i];
        else a.status = kDevGridOther;
      }
      blk->g = a;
    }
  }
}


// Bounding box in two halves: bbox_launch queues the min/max kernels and the
// 40-byte readback on st (and records ctx->ev_bbox); bbox_wait blocks the host
// on that event only, so work queued on other streams in between (the
// attractive SpMV) is dispatched behind the bbox blocks, not ahead of them.
// k_bbox into out_dev (null: ctx's readback buffer) on st; negate_max for the
// MIN-all-reduce layout of fitsne_bbox_device
static int bbox_kernels(fitsne_ctx* ctx, const void* Y, int64_t n, double* out_dev, int negate_max,
                        cudaStream_t st, double** outd_used, GridArgs* dgrid = nullptr,
                        DevGridReq rq = DevGridReq{}, double* hout = nullptr, unsigned long long seq = 0) {
  const int S = ctx->dims;
  int nblk = (int)std::min<int64_t>(std::max<int64_t>((n + kBlock - 1) / kBlock, 1), 4 * ctx->num_sms);
  FITSNE_TRY(ensure(ctx->bbox_part, sizeof(double) * (size_t)nblk * 2 * S + 64));
  FITSNE_TRY(ensure(ctx->counter, 64 * sizeof(int)));
  double* part = (double*)ctx->bbox_part.ptr;
  double* outd = out_dev ? out_dev : part + (size_t)nblk * 2 * S;
  int* flag = (int*)ctx->counter.ptr;
  // flag[0]: non-finite, flag[1]: last-block ticket (k_bbox folds the partials)
  FITSNE_CUDA(cudaMemsetAsync(flag, 0, 2 * sizeof(int), st));
  if (ctx->dtype == FITSNE_F32) {
    if (S == 1) k_bbox<float, 1><<<nblk, kBlock, 0, st>>>((const float*)Y, n, part, flag, outd, negate_max, dgrid, rq, hout, seq);
    else k_bbox<float, 2><<<nblk, kBlock, 0, st>>>((const float*)Y, n, part, flag, outd, negate_max, dgrid, rq, hout, seq);
  } else {
    if (S == 1) k_bbox<double, 1><<<nblk, kBlock, 0, st>>>((const double*)Y, n, part, flag, outd, negate_max, dgrid, rq, hout, seq);
    else k_bbox<double, 2><<<nblk, kBlock, 0, st>>>((const double*)Y, n, part, flag, outd, negate_max, dgrid, rq, hout, seq);
  }
  FITSNE_CHECK_LAUNCH();
  if (outd_used) *outd_used = outd;
  return FITSNE_OK;
}

int bbox_device(fitsne_ctx* ctx, const void* Y, int64_t n, double* out_dev, cudaStream_t st) {
  return bbox_kernels(ctx, Y, n, out_dev, 1, st, nullptr);
}

int bbox_launch(fitsne_ctx* ctx, const void* Y, int64_t n, cudaStream_t st) {
  const int S = ctx->dims;
  double* outd = nullptr;
  // the kernel's last block writes the box and then a sequence number straight
  // into the pinned h_scal[8 .. 15] (bbox_wait polls it); the event is the
  // fallback and the error path
  // sequence numbers are unique across the process's contexts (a recycled
  // pinned page or a second context can never show this launch's number)
  static std::atomic<unsigned long long> next_seq{1};
  ctx->bbox_seq = next_seq.fetch_add(1, std::memory_order_relaxed);
  FITSNE_TRY(bbox_kernels(ctx, Y, n, nullptr, 0, st, &outd, nullptr, DevGridReq{}, ctx->h_scal + 8, ctx->bbox_seq));
  if (!ctx->ev_bbox) FITSNE_CUDA(cudaEventCreateWithFlags(&ctx->ev_bbox, cudaEventDisableTiming));
  FITSNE_CUDA(cudaEventRecord(ctx->ev_bbox, st));
  return FITSNE_OK;
}

int bbox_wait(fitsne_ctx* ctx, double* bbox_host) {
  FITSNE_RANGE("bbox_wait");
  const int S = ctx->dims;
  {
    // poll the sequence word (a few microseconds after the kernel's last
    // block); give up after ~2 ms of polling and wait for the event instead
    volatile unsigned long long* seq = reinterpret_cast<volatile unsigned long long*>(ctx->h_scal + 15);
    bool seen = false;
    for (int spin = 0; spin < 4000000; ++spin) {
      if (*seq == ctx->bbox_seq) { seen = true; break; }
      if ((spin & 1023) == 1023 && cudaEventQuery(ctx->ev_bbox) != cudaErrorNotReady) break;
    }
    if (!seen) FITSNE_CUDA(cudaEventSynchronize(ctx->ev_bbox));
    std::atomic_thread_fence(std::memory_order_acquire);
    if (*seq != ctx->bbox_seq) { set_error("bounding box kernel did not complete"); return FITSNE_ECUDA; }
  }
  if (ctx->h_scal[8 + 2 * S] != 0.0) {
    set_error("points must be finite");
    return FITSNE_EPOINTS;
  }
  for (int d = 0; d < 2 * S; ++d) bbox_host[d] = ctx->h_scal[8 + d];
  return FITSNE_OK;
}

int compute_bbox(fitsne_ctx* ctx, const void* Y, int64_t n, double* bbox_host, cudaStream_t st) {
  FITSNE_TRY(bbox_launch(ctx, Y, n, st));
  return bbox_wait(ctx, bbox_host);
}

// make_grid in two halves (see bbox_launch)
int make_grid_finish(fitsne_ctx* ctx, cudaStream_t st) {
  double bbox[4];
  FITSNE_TRY(bbox_wait(ctx, bbox));
  fitsne_grid g;
  FITSNE_TRY(grid_from_bbox(ctx, bbox, &g));
  return install_grid(ctx, g, st);
}

// Exact restatement of make_grid's scalar formulas (nbody.py:131-143).  Host
// code compiled with -ffp-contract=off so each operation rounds like numpy.
int grid_from_bbox(fitsne_ctx* ctx, const double* bbox, fitsne_grid* out) {
  const int S = ctx->dims;
  double lo[2] = {0, 0}, hi[2] = {0, 0}, span[2] = {0, 0};
  double widest = -INFINITY;
  for (int d = 0; d < 2 * S; ++d) ctx->raw_bbox[d] = bbox[d];
  for (int d = 0; d < S; ++d) {
    lo[d] = bbox[d];
    hi[d] = bbox[S + d];
    if (!std::isfinite(lo[d]) || !std::isfinite(hi[d])) {
      set_error("points must be finite");
      return FITSNE_EPOINTS;
    }
    span[d] = hi[d] - lo[d];
    widest = std::max(widest, span[d]);
  }
  double cells = (ctx->intervals_per_integer == 1.0) ? std::ceil(widest)
                                                     : std::ceil(widest * ctx->intervals_per_integer);
  if (cells > 1e7) {
    set_error("embedding span too large for the interpolation grid");
    return FITSNE_ETOOBIG;
  }
  int n_int = std::max(ctx->min_intervals, (int)cells);
  for (int d = 0; d < S; ++d) {
    if (span[d] < 1.0) {
      double c = 0.5 * (lo[d] + hi[d]);
      lo[d] = c - 0.5;
      hi[d] = c + 0.5;
    } else {
      double pad = 1e-6 * span[d];
      lo[d] -= pad;
      hi[d] += pad;
    }
  }
  fitsne_grid g{};
  g.dims = S;
  g.n_intervals = n_int;
  g.points_per_interval = ctx->p;
  long long nn = (long long)n_int * ctx->p;
  if (nn > (1 << 20)) {
    set_error("interpolation grid too large");
    return FITSNE_ETOOBIG;
  }
  g.nodes_per_dim = (int)nn;
  for (int d = 0; d < S; ++d) {
    g.lo[d] = lo[d];
    g.hi[d] = hi[d];
    g.spacing[d] = (hi[d] - lo[d]) / (double)nn;
  }
  g.fft_len = smooth23_at_least(2 * (int)nn - 1);
  g.status = 0;
  *out = g;
  return FITSNE_OK;
}

template <typename T>
__global__ void k_twiddles(typename C2<T>::type* tw, int L, const GridArgs* __restrict__ gd = nullptr) {
  if (gd) {
    if (gd->status != kDevGridOk) return;
    L = gd->L;
  }
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < L; m += gridDim.x * blockDim.x) {
    double s, c;
    sincospi(2.0 * (double)m / (double)L, &s, &c);
    typename C2<T>::type w;
    w.x = (T)c;
    w.y = (T)(-s);
    tw[m] = w;
  }
}

// ---------------------------------------------------------------------------
// fp64 grid pipeline for fp32 contexts (FITSNE_OPT_GRID_F64).  The repulsive
// force F_i = y_i (K2*1)_i - (K2*y)_i cancels two terms of size |y| K2*1, so
// fp32 potentials lose accuracy in proportion to the span (rel-L2 3e-4 at
// span 200, 5e-3 at 430, 1.7e-2 at 860 against the fp64 reference).  Above
// kWideSpan the grid stages run on an fp64 twin context (same grid, same
// bit-exact cells): points are widened once per stage, the spread accumulates,
// the FFT stage transforms and the gather interpolates in double, and F_rep
// is rounded to fp32 only at the end.  The attractive SpMV is unaffected.
// ---------------------------------------------------------------------------

__global__ void k_widen(const float* __restrict__ x, int64_t m, double* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (double)x[i];
}

__global__ void k_narrow(const double* __restrict__ x, int64_t m, float* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (float)x[i];
}

static int shadow_ctx(fitsne_ctx* ctx) {
  if (ctx->shadow) return FITSNE_OK;
  fitsne_ctx* sh = nullptr;
  FITSNE_TRY(fitsne_create(&sh, ctx->device, ctx->dims, FITSNE_F64, ctx->p, ctx->min_intervals,
                           ctx->intervals_per_integer));
  sh->sorted_spread = ctx->sorted_spread;
  sh->spread_replicas = ctx->spread_replicas;
  sh->fft_path = ctx->fft_path;
  ctx->shadow = sh;
  return FITSNE_OK;
}

// Y (n, dims) fp32 -> ctx->y64 (double), stream-ordered
const double* widen_points(fitsne_ctx* ctx, const void* Y, int64_t n, cudaStream_t st) {
  const int64_t m = n * ctx->dims;
  if (ensure(ctx->y64, sizeof(double) * (size_t)std::max<int64_t>(m, 1)) != FITSNE_OK) return nullptr;
  if (m > 0) {
    k_widen<<<(int)std::min<int64_t>((m + 255) / 256, 8 * ctx->num_sms), 256, 0, st>>>((const float*)Y, m,
                                                                                     (double*)ctx->y64.ptr);
    if (cudaGetLastError() != cudaSuccess) return nullptr;
  }
  return (const double*)ctx->y64.ptr;
}

int narrow_values(const double* x, int64_t m, float* y, cudaStream_t st) {
  if (m <= 0 || !y) return FITSNE_OK;
  k_narrow<<<(int)std::min<int64_t>((m + 255) / 256, 1184), 256, 0, st>>>(x, m, y);
  FITSNE_CHECK_LAUNCH();
  return FITSNE_OK;
}

// F_rep (n, dims) of the wide pipeline, in double, into ctx->r64
int shadow_frep(fitsne_ctx* ctx, const void* Y, int64_t n, double** frep, cudaStream_t st) {
  const double* y = widen_points(ctx, Y, n, st);
  if (!y) { set_error("fp64 grid: point conversion failed"); return FITSNE_ECUDA; }
  FITSNE_TRY(ensure(ctx->r64, sizeof(double) * (size_t)std::max<int64_t>(n, 1) * (2 * ctx->dims + 2)));
  *frep = (double*)ctx->r64.ptr;
  return gather_tsne(ctx->shadow, y, n, *frep, nullptr, nullptr, st);
}

int install_grid(fitsne_ctx* ctx, const fitsne_grid& g, cudaStream_t st) {
  FITSNE_RANGE("install_grid");
  ctx->spec_ahead = false;  // a spectrum computed ahead belongs to the previous grid
  if (g.dims != ctx->dims) {
    set_error("grid dims do not match the context");
    return FITSNE_EINVAL;
  }
  const int L = g.fft_len;
  // lengths beyond one block's shared memory take the four-step path
  // (bigfft.cu); its launch grid bounds L by 65535
  if (L > 65535) {
    set_error("interpolation grid needs an FFT longer than 65535 (L=" + std::to_string(L) + ")");
    return FITSNE_ETOOBIG;
  }
  ctx->grid = g;
  ctx->grid_valid = true;
  ctx->wide = false;
  if (ctx->dtype == FITSNE_F32 && ctx->grid_f64 != 0) {
    double widest = 0;
    for (int d = 0; d < g.dims; ++d) widest = std::max(widest, g.hi[d] - g.lo[d]);
    if (ctx->grid_f64 == 2 || widest > kWideSpan) {
      FITSNE_TRY(shadow_ctx(ctx));
      for (int d = 0; d < 4; ++d) ctx->shadow->raw_bbox[d] = ctx->raw_bbox[d];
      const int gen0 = ctx->shadow->tw_gen;
      FITSNE_TRY(install_grid(ctx->shadow, g, st));
      ctx->tw_gen += ctx->shadow->tw_gen - gen0;
      ctx->wide = true;
      // the t-SNE stages run on the shadow; this context's own (fp32) FFT
      // still serves the general n-body calls on the same grid
    }
  }
  if (ctx->tw_len != L) {
    size_t es = 2 * dsize(ctx->dtype);
    FITSNE_TRY(ensure(ctx->tw, es * (size_t)L));
    if (ctx->dtype == FITSNE_F32)
      k_twiddles<float><<<grid_for(L), kBlock, 0, st>>>((float2*)ctx->tw.ptr, L);
    else
      k_twiddles<double><<<grid_for(L), kBlock, 0, st>>>((double2*)ctx->tw.ptr, L);
    FITSNE_CHECK_LAUNCH();
    ctx->tw_len = L;
    ++ctx->tw_gen;
  }
  return FITSNE_OK;
}

int make_grid(fitsne_ctx* ctx, const void* Y, int64_t n, cudaStream_t st) {
  double bbox[4];
  FITSNE_TRY(compute_bbox(ctx, Y, n, bbox, st));
  fitsne_grid g;
  FITSNE_TRY(grid_from_bbox(ctx, bbox, &g));
  return install_grid(ctx, g, st);
}

// =============================================================================
// a2/a3: box assignment + Lagrange weights, spreading
// =============================================================================
// t-SNE charges (1, y_0[, y_1]) of each point into 4-slot node records.
// nrep > 1: warps add into one of nrep replicas of the accumulator (replica =
// warp index mod nrep, stride rstride elements) so the points of a crowded
// box do not all serialise on the same L2 addresses; the row-FFT stage sums
// the replicas when it reads the grid.
template <typename T, int S, int P>
__global__ void k_spread_tsne(const T* __restrict__ Y, int64_t n, GridArgs g, T* __restrict__ acc,
                              int nrep, int64_t rstride) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  acc += (int64_t)((threadIdx.x >> 5) & (nrep - 1)) * rstride;
  if constexpr (sizeof(T) == 4 && P == 3 && S == 2) {
    // fp32 mode, p = 3: guarded fp32 box estimate (exact indices), fp32 weights
    const float2 yy = __ldg(reinterpret_cast<const float2*>(Y) + i);
    float wx[3], wy[3];
    const int cx = box_weights3_f32(yy.x, g.lo[0], g.h[0], g.lo_f[0], g.invh_f[0], g.guard[0],
                                    g.n_int, wx);
    const int cy = box_weights3_f32(yy.y, g.lo[1], g.h[1], g.lo_f[1], g.invh_f[1], g.guard[1],
                                    g.n_int, wy);
    const int64_t nn = g.n;
    const float cyx = yy.x - g.cf[0], cyy = yy.y - g.cf[1];  // centred charges
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int64_t rowbase = ((int64_t)cx * 3 + a) * nn + (int64_t)cy * 3;
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const float w = wx[a] * wy[b];
        atomicAdd(reinterpret_cast<float4*>(acc + (rowbase + b) * kNodeSlots),
                  make_float4(w, w * cyx, w * cyy, 0.f));
      }
    }
    return;
  }
  const int p = (P > 0) ? P : g.p;
  PointInterp<T, S> pi;
  double y[S];
  interp_point<T, S>(Y, i, g, pi, y);
  if (S == 1) {
    for (int a = 0; a < p; ++a) {
      int64_t node = (int64_t)pi.cell[0] * p + a;
      double w = pi.w[0][a];
      T* dst = acc + node * kNodeSlots;
      if constexpr (sizeof(T) == 4) {
        atomicAdd(reinterpret_cast<float2*>(dst), make_float2((float)w, (float)(w * (y[0] - g.c[0]))));
      } else {
        atomicAdd((double*)dst, w);
        atomicAdd((double*)dst + 1, w * (y[0] - g.c[0]));
      }
    }
  } else {
    const int64_t nn = g.n;
    for (int a = 0; a < p; ++a) {
      int64_t rowbase = ((int64_t)pi.cell[0] * p + a) * nn + (int64_t)pi.cell[1] * p;
      for (int b = 0; b < p; ++b) {
        double w = pi.w[0][a] * pi.w[1][b];
        T* dst = acc + (rowbase + b) * kNodeSlots;
        if constexpr (sizeof(T) == 4) {
          atomicAdd(reinterpret_cast<float4*>(dst),
                    make_float4((float)w, (float)(w * (y[0] - g.c[0])), (float)(w * (y[1] - g.c[1])), 0.f));
        } else {
          atomicAdd((double*)dst, w);
          atomicAdd((double*)dst + 1, w * (y[0] - g.c[0]));
          atomicAdd((double*)dst + 2, w * (y[1] - g.c[1]));
        }
      }
    }
  }
}

template <typename T, int S>
static void launch_spread_tsne(const T* Y, int64_t n, const GridArgs& g, T* acc, int nrep,
                               int64_t rstride, cudaStream_t st) {
  if (g.p == 3) k_spread_tsne<T, S, 3><<<grid_for(n), kBlock, 0, st>>>(Y, n, g, acc, nrep, rstride);
  else k_spread_tsne<T, S, 0><<<grid_for(n), kBlock, 0, st>>>(Y, n, g, acc, nrep, rstride);
}

static size_t accum_elems(const fitsne_grid& g) {
  size_t G = 1;
  for (int d = 0; d < g.dims; ++d) G *= (size_t)g.nodes_per_dim;
  return G * kNodeSlots;
}

// replicas of the internal accumulator (power of two; 1 for caller buffers)
static int accum_reps(fitsne_ctx* ctx, const void* accum) {
  if (ctx->dims == 1) return 1;
  return (accum == nullptr || accum == ctx->accum.ptr) ? ctx->spread_replicas : 1;
}

// replicas the FFT stage must read (and clear): the spread paths that add
// into replica 0 only leave the others at zero
static int accum_reps_live(fitsne_ctx* ctx, const void* accum) {
  const int r = accum_reps(ctx, accum);
  return r > 1 ? std::min(r, ctx->accum_live_reps) : r;
}

static int ensure_accum(fitsne_ctx* ctx, cudaStream_t st) {
  size_t bytes = accum_elems(ctx->grid) * dsize(ctx->dtype) * (size_t)ctx->spread_replicas;
  if (ctx->accum.cap < bytes) {
    FITSNE_TRY(ensure(ctx->accum, bytes));
    ctx->accum_clean = false;
  }
  if (!ctx->accum_clean) {
    FITSNE_CUDA(cudaMemsetAsync(ctx->accum.ptr, 0, ctx->accum.cap, st));
    ctx->accum_clean = true;
  }
  return FITSNE_OK;
}

int spread_tsne(fitsne_ctx* ctx, const void* Y, int64_t n, void* accum, cudaStream_t st) {
  FITSNE_RANGE("spread");
  ctx->band_sorted = false;  // set again by the band spread below
  if (!ctx->grid_valid) { set_error("no grid"); return FITSNE_EINVAL; }
  if (ctx->wide) {  // fp64 grid: a caller's accumulator is double (fitsne_grid_accum_dtype)
    const double* y = widen_points(ctx, Y, n, st);
    if (!y) { set_error("fp64 grid: point conversion failed"); return FITSNE_ECUDA; }
    return spread_tsne(ctx->shadow, y, n, accum, st);
  }
  GridArgs g = grid_args(ctx->grid);
  const int nrep = accum_reps(ctx, accum);
  const int64_t rstride = (int64_t)accum_elems(ctx->grid);
  if (accum == nullptr) {
    FITSNE_TRY(ensure_accum(ctx, st));
    accum = ctx->accum.ptr;
  }
  // Box-sorted spread when points crowd into few boxes (same-address atomics
  // would serialise): estimate the occupied boxes from the raw bounding box.
  bool use_sorted = ctx->sorted_spread == 2;
  if (ctx->sorted_spread == 1) {
    double occ = 1.0;
    for (int d = 0; d < ctx->dims; ++d) {
      const double w = (ctx->grid.hi[d] - ctx->grid.lo[d]) / ctx->grid.n_intervals;
      const double span = ctx->raw_bbox[ctx->dims + d] - ctx->raw_bbox[d];
      occ *= (span >= 0 && w > 0) ? std::floor(span / w) + 2.0 : 1e30;
    }
    use_sorted = (double)n / occ >= 128.0;
  }
  const bool internal = accum == ctx->accum.ptr;
  // band spread: the fp32 2-D p = 3 default (binning by box row + in-block
  // box sort; no same-address contention, ~1 L2 transaction per node per box
  // run instead of one per point)
  const bool use_band = (ctx->sorted_spread == 3 || (ctx->sorted_spread == 1)) &&
                        band_spread_applies(ctx, n);
  if (use_band) {
    FITSNE_TRY(spread_band(ctx, Y, n, accum, st));
    if (internal) ctx->accum_live_reps = 1;
    ctx->accum_clean = false;
    return FITSNE_OK;
  }
  if (n > 0 && use_sorted && spread_sorted(ctx, Y, n, accum, st) == FITSNE_OK) {
    if (internal) ctx->accum_live_reps = 1;
    ctx->accum_clean = false;
    return FITSNE_OK;
  }
  if (internal) ctx->accum_live_reps = nrep;
  if (n > 0) {
    if (ctx->dtype == FITSNE_F32) {
      if (ctx->dims == 1) launch_spread_tsne<float, 1>((const float*)Y, n, g, (float*)accum, nrep, rstride, st);
      else launch_spread_tsne<float, 2>((const float*)Y, n, g, (float*)accum, nrep, rstride, st);
    } else {
      if (ctx->dims == 1) launch_spread_tsne<double, 1>((const double*)Y, n, g, (double*)accum, nrep, rstride, st);
      else launch_spread_tsne<double, 2>((const double*)Y, n, g, (double*)accum, nrep, rstride, st);
    }
    FITSNE_CHECK_LAUNCH();
  }
  ctx->accum_clean = false;
  return FITSNE_OK;
}

// general charges (N, nq) row-major -> coeffs (nq, G) planar
template <typename T, int S>
__global__ void k_spread_general(const T* __restrict__ Y, int64_t n, GridArgs g,
                                 const T* __restrict__ q, int nq, T* __restrict__ coeffs,
                                 int* __restrict__ outside) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  PointInterp<T, S> pi;
  double y[S];
  bool out = false;
#pragma unroll
  for (int d = 0; d < S; ++d) {
    double v = (double)Y[i * S + d];
    if (v < g.lo[d] || v > g.hi[d]) out = true;
  }
  if (out) { atomicOr(outside, 1); return; }
  interp_point<T, S>(Y, i, g, pi, y);
  const int p = g.p;
  const int64_t nn = g.n;
  const int64_t G = (S == 1) ? nn : nn * nn;
  const int cnt = (S == 1) ? p : p * p;
  for (int k = 0; k < cnt; ++k) {
    int a = (S == 1) ? k : k / p, b = (S == 1) ? 0 : k % p;
    int64_t node = (S == 1) ? ((int64_t)pi.cell[0] * p + a)
                            : (((int64_t)pi.cell[0] * p + a) * nn + (int64_t)pi.cell[1] * p + b);
    double w = (S == 1) ? pi.w[0][a] : pi.w[0][a] * pi.w[1][b];
    for (int c = 0; c < nq; ++c) {
      double v = w * (double)q[i * nq + c];
      atomicAdd(&coeffs[(int64_t)c * G + node], (T)v);
    }
  }
}

template <typename T, int S>
__global__ void k_point_interp(const T* __restrict__ Y, int64_t n, GridArgs g,
                               int64_t* __restrict__ idx, T* __restrict__ wout,
                               int* __restrict__ outside) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool out = false;
#pragma unroll
  for (int d = 0; d < S; ++d) {
    double v = (double)Y[i * S + d];
    if (v < g.lo[d] || v > g.hi[d]) out = true;
  }
  if (out) atomicOr(outside, 1);
  PointInterp<T, S> pi;
  double y[S];
  interp_point<T, S>(Y, i, g, pi, y);
  if constexpr (sizeof(T) == 4) {
    // fp32, p = 3: the node indices come from the guarded fp32 box estimate
    // that the production spread / gather / combine kernels use
    // (box_weights3_f32), so the bit-exactness checks of this entry point
    // cover the production cells; the weights stay the exact fp64 ones
    if (g.p == 3) {
#pragma unroll
      for (int d = 0; d < S; ++d) {
        float wf[3];
        pi.cell[d] = box_weights3_f32((float)Y[i * S + d], g.lo[d], g.h[d], g.lo_f[d], g.invh_f[d],
                                      g.guard[d], g.n_int, wf);
      }
    }
  }
  const int p = g.p;
  const int64_t nn = g.n;
  const int cnt = (S == 1) ? p : p * p;
  for (int k = 0; k < cnt; ++k) {
    int a = (S == 1) ? k : k / p, b = (S == 1) ? 0 : k % p;
    int64_t node = (S == 1) ? ((int64_t)pi.cell[0] * p + a)
                            : (((int64_t)pi.cell[0] * p + a) * nn + (int64_t)pi.cell[1] * p + b);
    double w = (S == 1) ? pi.w[0][a] : pi.w[0][a] * pi.w[1][b];
    idx[i * cnt + k] = node;
    wout[i * cnt + k] = (T)w;
  }
}

static int check_outside(fitsne_ctx* ctx, cudaStream_t st) {
  FITSNE_CUDA(cudaMemcpyAsync(ctx->h_status, ctx->counter.ptr, sizeof(int), cudaMemcpyDeviceToHost, st));
  FITSNE_CUDA(cudaStreamSynchronize(st));
  if (ctx->h_status[0]) {
    set_error("point outside grid bounds");
    return FITSNE_EOUTSIDE;
  }
  return FITSNE_OK;
}

int point_interp(fitsne_ctx* ctx, const void* Y, int64_t n, int64_t* idx, void* w, cudaStream_t st) {
  if (!ctx->grid_valid) { set_error("no grid"); return FITSNE_EINVAL; }
  GridArgs g = grid_args(ctx->grid);
  FITSNE_TRY(ensure(ctx->counter, 64 * sizeof(int)));
  FITSNE_CUDA(cudaMemsetAsync(ctx->counter.ptr, 0, sizeof(int), st));
  if (n > 0) {
    int* flag = (int*)ctx->counter.ptr;
    if (ctx->dtype == FITSNE_F32) {
      if (ctx->dims == 1) k_point_interp<float, 1><<<grid_for(n), kBlock, 0, st>>>((const float*)Y, n, g, idx, (float*)w, flag);
      else k_point_interp<float, 2><<<grid_for(n), kBlock, 0, st>>>((const float*)Y, n, g, idx, (float*)w, flag);
    } else {
      if (ctx->dims == 1) k_point_interp<double, 1><<<grid_for(n), kBlock, 0, st>>>((const double*)Y, n, g, idx, (double*)w, flag);
      else k_point_interp<double, 2><<<grid_for(n), kBlock, 0, st>>>((const double*)Y, n, g, idx, (double*)w, flag);
    }
    FITSNE_CHECK_LAUNCH();
  }
  return check_outside(ctx, st);
}

int spread_general(fitsne_ctx* ctx, const void* Y, int64_t n, const void* q, int nq, void* coeffs,
                   cudaStream_t st) {
  if (!ctx->grid_valid) { set_error("no grid"); return FITSNE_EINVAL; }
  GridArgs g = grid_args(ctx->grid);
  size_t G = accum_elems(ctx->grid) / kNodeSlots;
  FITSNE_CUDA(cudaMemsetAsync(coeffs, 0, G * nq * dsize(ctx->dtype), st));
  FITSNE_TRY(ensure(ctx->counter, 64 * sizeof(int)));
  FITSNE_CUDA(cudaMemsetAsync(ctx->counter.ptr, 0, sizeof(int), st));
  int* flag = (int*)ctx->counter.ptr;
  if (n > 0) {
    if (ctx->dtype == FITSNE_F32) {
      if (ctx->dims == 1) k_spread_general<float, 1><<<grid_for(n), kBlock, 0, st>>>((const float*)Y, n, g, (const float*)q, nq, (float*)coeffs, flag);
      else k_spread_general<float, 2><<<grid_for(n), kBlock, 0, st>>>((const float*)Y, n, g, (const float*)q, nq, (float*)coeffs, flag);
    } else {
      if (ctx->dims == 1) k_spread_general<double, 1><<<grid_for(n), kBlock, 0, st>>>((const double*)Y, n, g, (const double*)q, nq, (double*)coeffs, flag);
      else k_spread_general<double, 2><<<grid_for(n), kBlock, 0, st>>>((const double*)Y, n, g, (const double*)q, nq, (double*)coeffs, flag);
    }
    FITSNE_CHECK_LAUNCH();
  }
  return check_outside(ctx, st);
}

// =============================================================================
// a4/a5: kernel spectrum + circulant convolution (2-D: row / column / row)
// =============================================================================
enum ConvMode { MODE_TSNE = 0, MODE_GENERAL = 1 };

// Device-grid schedule (gd != null): the FFT stages were launched for a
// capacity (n_cap rows, L_cap columns, shared memory for L_cap) before the
// host knew the grid; they read the grid k_bbox computed, blocks beyond its
// n / L return at once, and the Stockham plan of its L is built in shared
// memory.  Returns false when the whole block has nothing to do.
__device__ __forceinline__ bool stage_grid(GridArgs& g, const GridArgs* __restrict__ gd, const FftPlan& pl_arg,
                                           const FftPlan** pl_use) {
  *pl_use = &pl_arg;
  if (!gd) return true;
  g = *gd;
  if (g.status != kDevGridOk) return false;
  *pl_use = dev_plan(gd);
  return true;
}

template <typename T>
__device__ __forceinline__ void kernel_pair(int i, int j, double hx, double hy, T& k1, T& k2) {
  // first[i, j] = K((i hx)^2 + (j hy)^2), nbody.py:272-275
  double dx = (double)i * hx, dy = (double)j * hy;
  double d2 = __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
  double base = 1.0 / (1.0 + d2);
  k1 = (T)base;
  k2 = (T)(base * base);
}

// Row stage.  merged=1: block x transforms data row x (the packed pairs) and
// kernel-spectrum row x in one batched FFT.  merged=0 (large L): blocks [0, n)
// do the data rows, blocks [n, 2n) the spectrum rows.  merged=2 / 3: one
// launch for the data rows, another (spectrum_ahead) for the spectrum rows.  Shared memory: the
// twiddle table (L) then the padded signals (stride plen(L), index pidx).
template <typename T, int MODE>
__global__ void __launch_bounds__(256)
k_rows_forward(T* __restrict__ acc, const T* __restrict__ coeffs, int ncol, int pair0, int npair,
               typename C2<T>::type* __restrict__ F, typename C2<T>::type* __restrict__ Sbuf,
               GridArgs g, const typename C2<T>::type* __restrict__ tw, FftPlan pl_arg, int merged,
               int nrep, int64_t rstride, const GridArgs* __restrict__ gd = nullptr) {
  using V = typename C2<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const FftPlan* plp;
  if (!stage_grid(g, gd, pl_arg, &plp)) return;
  const int L = g.L, n = g.n;
  const int PL = plen(L);
  const int H = L / 2 + 1;
  // unmerged launches put the data rows first: [0, split) data, [split, 2 split) spectrum
  const int split = gd ? (int)gridDim.x / 2 : n;
  // merged: 1 = data + spectrum row in one block, 0 = data blocks then spectrum
  // blocks, 2 = data rows only, 3 = spectrum rows only (spectrum_ahead)
  const bool do_data = merged == 1 || merged == 2 || (merged == 0 && (int)blockIdx.x < split);
  const bool do_spec = merged == 1 || merged == 3 || (merged == 0 && (int)blockIdx.x >= split);
  const int x = (merged != 0 || (int)blockIdx.x < split) ? (int)blockIdx.x : (int)blockIdx.x - split;
  if (x >= n) return;  // capacity beyond the device grid
  const FftPlan& pl = *plp;
  V* s_tw = reinterpret_cast<V*>(smem_raw);
  V* a = s_tw + L;
  const int ns = do_data ? ((MODE == MODE_TSNE) ? 2 : npair) : 0;
  const int nsig = ns + (do_spec ? 1 : 0);
  V* b = a + (size_t)nsig * PL;
  stage_twiddles(s_tw, tw, L);
  for (int y0 = threadIdx.x; y0 < L; y0 += 2 * blockDim.x) {
    if (do_data) {
      if (MODE == MODE_TSNE) {
        T rv[2][3];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int y = y0 + u * blockDim.x;
          rv[u][0] = rv[u][1] = rv[u][2] = 0;
          if (y < n) {
            for (int rp = 0; rp < nrep; ++rp) {  // sum the spread replicas
              T* rec = acc + (size_t)rp * rstride + ((size_t)x * n + y) * kNodeSlots;
              if constexpr (sizeof(T) == 4) {
                const float4 f = *reinterpret_cast<const float4*>(rec);
                rv[u][0] += f.x; rv[u][1] += f.y; rv[u][2] += f.z;
              } else {
                const double2 f0 = *reinterpret_cast<const double2*>(rec);
                rv[u][0] += f0.x; rv[u][1] += f0.y; rv[u][2] += rec[2];
              }
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int y = y0 + u * blockDim.x;
          if (y >= L) continue;
          V A, B;
          B.x = rv[u][0]; B.y = 0;
          A.x = rv[u][1]; A.y = rv[u][2];
          a[pidx(y)] = A;
          a[PL + pidx(y)] = B;
          if (y < n) {
            // consume-and-clear: leaves the accumulator zeroed for the next spread
            for (int rp = 0; rp < nrep; ++rp) {
              T* rec = acc + (size_t)rp * rstride + ((size_t)x * n + y) * kNodeSlots;
              if constexpr (sizeof(T) == 4) *reinterpret_cast<float4*>(rec) = make_float4(0.f, 0.f, 0.f, 0.f);
              else { rec[0] = 0; rec[1] = 0; rec[2] = 0; }
            }
          }
        }
      } else {
        const size_t G = (size_t)n * n;
        for (int u = 0; u < 2; ++u) {
          const int y = y0 + u * blockDim.x;
          if (y >= L) continue;
          for (int q = 0; q < npair; ++q) {
            V v = {0, 0};
            if (y < n) {
              int c0 = 2 * (pair0 + q), c1 = c0 + 1;
              v.x = coeffs[(size_t)c0 * G + (size_t)x * n + y];
              if (c1 < ncol) v.y = coeffs[(size_t)c1 * G + (size_t)x * n + y];
            }
            a[(size_t)q * PL + pidx(y)] = v;
          }
        }
      }
    }
    if (do_spec) {
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int y = y0 + u * blockDim.x;
        if (y >= L) continue;
        // first[x, j] = K((x hx)^2 + (j hy)^2), columns mirrored (nbody.py:272-281)
        V z = {0, 0};
        int jj = (y < n) ? y : ((y > L - n) ? L - y : -1);
        if (jj >= 0) {
          T k1, k2;
          kernel_pair<T>(x, jj, g.h[0], g.h[1], k1, k2);
          z.x = k1;
          z.y = k2;
        }
        a[(size_t)ns * PL + pidx(y)] = z;
      }
    }
  }
  V* r = block_fft<V, T>(a, b, pl, nsig, PL, s_tw, false);
  for (int q = 0; q < ns; ++q)
    for (int k = threadIdx.x; k < L; k += blockDim.x)
      F[((size_t)q * n + x) * L + k] = r[(size_t)q * PL + pidx(k)];
  if (do_spec)
    for (int k = threadIdx.x; k < H; k += blockDim.x)
      Sbuf[(size_t)x * H + k] = r[(size_t)ns * PL + pidx(k)];
}

// Kernel-spectrum column stage: block b transforms spectrum columns
// ky = b*kSpecCols .. (rows mirrored as in the circulant embedding,
// nbody.py:278-281) and stores Khat[ky][kx] = (K1hat, K2hat) / L^2 (real).
constexpr int kSpecCols = 4;

template <typename T>
__global__ void __launch_bounds__(256)
k_spec_cols(const typename C2<T>::type* __restrict__ Sbuf, GridArgs g,
            const typename C2<T>::type* __restrict__ tw, FftPlan pl_arg,
            typename C2<T>::type* __restrict__ Khat, int cpb, const GridArgs* __restrict__ gd = nullptr) {
  using V = typename C2<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const FftPlan* plp;
  if (!stage_grid(g, gd, pl_arg, &plp)) return;
  const int L = g.L, n = g.n, H = L / 2 + 1;
  const int ky0 = blockIdx.x * cpb;  // cpb <= kSpecCols columns per block
  if (ky0 >= H) return;
  const FftPlan& pl = *plp;
  const int PL = plen(L);
  V* s_tw = reinterpret_cast<V*>(smem_raw);
  V* a = s_tw + L;
  V* b = a + (size_t)cpb * PL;
  const int nc = min(cpb, H - ky0);
  stage_twiddles(s_tw, tw, L);
  // each row i contributes kSpecCols consecutive spectrum columns (32 B)
  for (int x = threadIdx.x; x < L; x += blockDim.x) {
    const int ii = (x < n) ? x : ((x > L - n) ? L - x : -1);
    V z[kSpecCols];
#pragma unroll
    for (int c = 0; c < kSpecCols; ++c) {
      z[c].x = 0; z[c].y = 0;
      if (ii >= 0 && c < nc) z[c] = Sbuf[(size_t)ii * H + ky0 + c];
    }
#pragma unroll
    for (int c = 0; c < kSpecCols; ++c)
      if (c < nc) a[(size_t)c * PL + pidx(x)] = z[c];
  }
  V* r = block_fft<V, T>(a, b, pl, nc, PL, s_tw, false);
  const T scale = (T)(1.0 / ((double)L * (double)L));
  for (int c = 0; c < nc; ++c)
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
      V v = r[(size_t)c * PL + pidx(k)];
      v.x *= scale;
      v.y *= scale;
      Khat[(size_t)(ky0 + c) * L + k] = v;
    }
}

// Data column stage: one block per column c in [0, L): forward FFT of the
// pairs, multiply by the kernel spectrum of column min(c, L-c) (+ Parseval
// partial of the unit-charge pair for t-SNE), inverse FFT.
constexpr int kColsMax = 4;  // columns per k_cols block (upper bound)

template <typename T, int MODE>
__global__ void __launch_bounds__(256)
k_cols(typename C2<T>::type* __restrict__ F, const typename C2<T>::type* __restrict__ Khat,
       GridArgs g, const typename C2<T>::type* __restrict__ tw, FftPlan pl_arg, int npair, int kern,
       int with_k1, double* __restrict__ zpart, int cpb, const GridArgs* __restrict__ gd = nullptr) {
  // cpb (<= kColsMax) adjacent columns per block: the strided column reads
  // then use whole 32-byte sectors instead of 8 bytes of each
  using V = typename C2<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const FftPlan* plp;
  if (!stage_grid(g, gd, pl_arg, &plp)) return;
  const int L = g.L, n = g.n;
  const int PL = plen(L);
  const int col0 = blockIdx.x * cpb;
  if (col0 >= L) return;
  const FftPlan& pl = *plp;
  const int nc = min(cpb, L - col0);
  const int nsig = nc * npair;  // signal c * npair + q: column col0 + c, pair q
  V* s_tw = reinterpret_cast<V*>(smem_raw);
  V* a = s_tw + L;
  V* b = a + (size_t)cpb * npair * PL;
  stage_twiddles(s_tw, tw, L);
  for (int q = 0; q < npair; ++q)
    for (int x0 = threadIdx.x; x0 < L; x0 += 2 * blockDim.x) {
      V z[2][kColsMax];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int x = x0 + u * blockDim.x;
#pragma unroll
        for (int c = 0; c < kColsMax; ++c) {
          z[u][c].x = 0;
          z[u][c].y = 0;
          if (x < n && c < nc) z[u][c] = F[((size_t)q * n + x) * L + col0 + c];
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int x = x0 + u * blockDim.x;
        if (x >= L) continue;
#pragma unroll
        for (int c = 0; c < kColsMax; ++c)
          if (c < nc) a[(size_t)(c * npair + q) * PL + pidx(x)] = z[u][c];
      }
    }
  V* fr = block_fft<V, T>(a, b, pl, nsig, PL, s_tw, false);
  V* other = (fr == a) ? b : a;
  double zacc[kColsMax];
#pragma unroll
  for (int c = 0; c < kColsMax; ++c) zacc[c] = 0.0;
#pragma unroll
  for (int c = 0; c < kColsMax; ++c) {
    if (c >= nc) continue;
    const int col = col0 + c;
    const V* Kc = Khat + (size_t)(col <= L - col ? col : L - col) * L;
    for (int k = threadIdx.x; k < L; k += blockDim.x) {
      const V kk = __ldg(Kc + k);
      for (int q = 0; q < npair; ++q) {
        V* p = fr + (size_t)(c * npair + q) * PL + pidx(k);
        const V v = *p;
        V o;
        if (MODE == MODE_TSNE) {
          if (q == 0) {
            o.x = v.x * kk.y;
            o.y = v.y * kk.y;
          } else {
            zacc[c] += (double)kk.x * ((double)v.x * (double)v.x + (double)v.y * (double)v.y);
            if (with_k1) {  // v * (K2 + i K1)
              o.x = v.x * kk.y - v.y * kk.x;
              o.y = v.x * kk.x + v.y * kk.y;
            } else {
              o.x = v.x * kk.y;
              o.y = v.y * kk.y;
            }
          }
        } else {
          const T m = (kern == FITSNE_CAUCHY) ? kk.x : kk.y;
          o.x = v.x * m;
          o.y = v.y * m;
        }
        *p = o;
      }
    }
  }
  V* ir = block_fft<V, T>(fr, other, pl, nsig, PL, s_tw, true);
  for (int q = 0; q < npair; ++q)
    for (int x = threadIdx.x; x < n; x += blockDim.x)
#pragma unroll
      for (int c = 0; c < kColsMax; ++c)
        if (c < nc) F[((size_t)q * n + x) * L + col0 + c] = ir[(size_t)(c * npair + q) * PL + pidx(x)];
  if (MODE == MODE_TSNE) {
    __shared__ double red[kColsMax][32];
#pragma unroll
    for (int c = 0; c < kColsMax; ++c) {
      const double zs = warp_sum(zacc[c]);
      if ((threadIdx.x & 31) == 0) red[c][threadIdx.x >> 5] = zs;
    }
    __syncthreads();
    if (threadIdx.x < nc) {
      double s = 0;
      for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) s += red[threadIdx.x][w];
      zpart[col0 + threadIdx.x] = s;
    }
  }
}

// Row inverse stage: one block per row x.  Block 0 also folds the Parseval
// partials into Z (deterministic order).
template <typename T, int MODE>
__global__ void __launch_bounds__(256)
k_rows_inverse(const typename C2<T>::type* __restrict__ F, GridArgs g,
               const typename C2<T>::type* __restrict__ tw, FftPlan pl_arg, int npair, int ncol,
               int pair0, T* __restrict__ pot, T* __restrict__ out, const double* __restrict__ zpart,
               double* __restrict__ scal, double n_total, const GridArgs* __restrict__ gd = nullptr) {
  using V = typename C2<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const FftPlan* plp;
  if (!stage_grid(g, gd, pl_arg, &plp)) return;
  const int L = g.L, n = g.n;
  const int x = blockIdx.x;
  if (x >= n) return;
  const FftPlan& pl = *plp;
  const int PL = plen(L);
  V* s_tw = reinterpret_cast<V*>(smem_raw);
  V* a = s_tw + L;
  V* b = a + (size_t)npair * PL;
  stage_twiddles(s_tw, tw, L);
  for (int q = 0; q < npair; ++q)
    for (int k0 = threadIdx.x; k0 < L; k0 += 4 * blockDim.x) {
      V z[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + u * blockDim.x;
        if (k < L) z[u] = F[((size_t)q * n + x) * L + k];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int k = k0 + u * blockDim.x;
        if (k < L) a[(size_t)q * PL + pidx(k)] = z[u];
      }
    }
  V* r = block_fft<V, T>(a, b, pl, npair, PL, s_tw, true);
  if (MODE == MODE_TSNE) {
    for (int y = threadIdx.x; y < n; y += blockDim.x) {
      V A = r[pidx(y)], B = r[PL + pidx(y)];
      T* rec = pot + pot_node(x, y, g.p, g.n_int) * kNodeSlots;
      // slots: K2*1, K2*y_0, K2*y_1, K1*1 (the last only with_k1)
      if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4*>(rec) = make_float4(B.x, A.x, A.y, B.y);
      } else {
        reinterpret_cast<double2*>(rec)[0] = make_double2(B.x, A.x);
        reinterpret_cast<double2*>(rec)[1] = make_double2(A.y, B.y);
      }
    }
    if (x == 0) {
      __shared__ double red[32];
      double s = 0;
      for (int k = threadIdx.x; k < L; k += blockDim.x) s += zpart[k];
      s = warp_sum(s);
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0;
        for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) t += red[w];
        scal[0] = t - n_total;  // Z
      }
    }
  } else {
    const size_t G = (size_t)n * n;
    for (int q = 0; q < npair; ++q) {
      int c0 = 2 * (pair0 + q), c1 = c0 + 1;
      for (int y = threadIdx.x; y < n; y += blockDim.x) {
        V v = r[(size_t)q * PL + pidx(y)];
        out[(size_t)c0 * G + (size_t)x * n + y] = v.x;
        if (c1 < ncol) out[(size_t)c1 * G + (size_t)x * n + y] = v.y;
      }
    }
  }
}

// 1-D convolution: a single block holds the whole transform.
template <typename T, int MODE>
__global__ void __launch_bounds__(1024)
k_conv1d(T* __restrict__ acc, const T* __restrict__ coeffs, int ncol, GridArgs g,
         const typename C2<T>::type* __restrict__ tw, FftPlan pl, int kern, int with_k1,
         T* __restrict__ pot, T* __restrict__ out, double* __restrict__ scal, double n_total) {
  using V = typename C2<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int L = g.L, n = g.n;
  const int PL = plen(L);
  V* K = reinterpret_cast<V*>(smem_raw);
  V* a = K + L;
  V* b = a + 2 * (size_t)PL;
  // spectrum: circ[:n] = first, circ[L-n+1:] = mirror (nbody.py:264-271)
  for (int j = threadIdx.x; j < L; j += blockDim.x) {
    V z = {0, 0};
    int jj = (j < n) ? j : ((j > L - n) ? L - j : -1);
    if (jj >= 0) {
      double d = (double)jj * g.h[0];
      double base = 1.0 / (1.0 + __dmul_rn(d, d));
      z.x = (T)base;
      z.y = (T)(base * base);
    }
    a[pidx(j)] = z;
  }
  V* r = block_fft<V, T>(a, b, pl, 1, PL, tw, false);
  const T scale = (T)(1.0 / (double)L);
  for (int k = threadIdx.x; k < L; k += blockDim.x) {
    V v = r[pidx(k)];
    V kk;
    kk.x = v.x * scale;
    kk.y = v.y * scale;
    K[k] = kk;
  }
  __syncthreads();
  const int npair = (MODE == MODE_TSNE) ? 2 : (ncol + 1) / 2;
  double zacc = 0.0;
  for (int q0 = 0; q0 < npair; q0 += 2) {
    const int ns = min(2, npair - q0);
    for (int y = threadIdx.x; y < L; y += blockDim.x) {
      for (int s = 0; s < ns; ++s) {
        V v = {0, 0};
        if (y < n) {
          if (MODE == MODE_TSNE) {
            T* rec = acc + (size_t)y * kNodeSlots;
            if (s == 0) v.x = rec[1]; else v.x = rec[0];
          } else {
            int c0 = 2 * (q0 + s), c1 = c0 + 1;
            v.x = coeffs[(size_t)c0 * n + y];
            if (c1 < ncol) v.y = coeffs[(size_t)c1 * n + y];
          }
        }
        a[(size_t)s * PL + pidx(y)] = v;
      }
    }
    if (MODE == MODE_TSNE) {
      __syncthreads();
      for (int y = threadIdx.x; y < n; y += blockDim.x) {
        T* rec = acc + (size_t)y * kNodeSlots;
        rec[0] = 0; rec[1] = 0;
      }
    }
    V* fr = block_fft<V, T>(a, b, pl, ns, PL, tw, false);
    V* other = (fr == a) ? b : a;
    for (int t = threadIdx.x; t < ns * L; t += blockDim.x) {
      int s = t / L, k = t - s * L;
      V* p = fr + (size_t)s * PL + pidx(k);
      V v = *p;
      V kk = K[k];
      V o;
      if (MODE == MODE_TSNE) {
        if (s == 0) {
          o.x = v.x * kk.y; o.y = v.y * kk.y;
        } else {
          zacc += (double)kk.x * ((double)v.x * (double)v.x + (double)v.y * (double)v.y);
          if (with_k1) {
            o.x = v.x * kk.y - v.y * kk.x;
            o.y = v.x * kk.x + v.y * kk.y;
          } else {
            o.x = v.x * kk.y; o.y = v.y * kk.y;
          }
        }
      } else {
        T m = (kern == FITSNE_CAUCHY) ? kk.x : kk.y;
        o.x = v.x * m; o.y = v.y * m;
      }
      *p = o;
    }
    V* ir = block_fft<V, T>(fr, other, pl, ns, PL, tw, true);
    for (int y = threadIdx.x; y < n; y += blockDim.x) {
      if (MODE == MODE_TSNE) {
        V A = ir[pidx(y)], B = ir[PL + pidx(y)];
        T* rec = pot + (size_t)y * kNodeSlots;
        rec[0] = B.x; rec[1] = A.x; rec[2] = 0; rec[3] = B.y;
      } else {
        for (int s = 0; s < ns; ++s) {
          V v = ir[(size_t)s * PL + pidx(y)];
          int c0 = 2 * (q0 + s), c1 = c0 + 1;
          out[(size_t)c0 * n + y] = v.x;
          if (c1 < ncol) out[(size_t)c1 * n + y] = v.y;
        }
      }
    }
    __syncthreads();
  }
  if (MODE == MODE_TSNE) {
    __shared__ double red[32];
    zacc = warp_sum(zacc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = zacc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0;
      for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) s += red[w];
      scal[0] = s - n_total;
    }
  }
}

template <typename T>
static int set_smem(const void* fn, size_t bytes) {
  // the default 48 KB limit also covers the kernel's static shared memory
  if (bytes > 40 * 1024) {
    FITSNE_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  }
  return FITSNE_OK;
}

// Runs the convolution pipeline.  MODE_TSNE: input accum (4-slot records,
// cleared on the way), output ctx->pot, Z -> scal[0].  MODE_GENERAL: coeffs
// (ncol, G) -> out (ncol, G) with kernel `kern`.
template <typename T, int MODE>
static int run_conv(fitsne_ctx* ctx, T* accum, const T* coeffs, int ncol, int kern, bool with_k1,
                    T* out, int64_t n_total, cudaStream_t st) {
  using V = typename C2<T>::type;
  const fitsne_grid& gr = ctx->grid;
  GridArgs g = grid_args(gr);
  const int L = g.L, n = g.n, H = L / 2 + 1;
  if (big_fft_applies(ctx, L)) {
    if (MODE == MODE_TSNE)
      return conv_big_tsne(ctx, accum, accum_reps_live(ctx, accum), (int64_t)accum_elems(gr), with_k1,
                           n_total, st);
    return conv_big_general(ctx, coeffs, ncol, kern, out, st);
  }
  FftPlan pl;
  make_plan(pl, L);
  const V* tw = (const V*)ctx->tw.ptr;
  double* scal = (double*)ctx->scal.ptr;
  T* pot = (T*)ctx->pot.ptr;
  if (gr.dims == 1) {
    size_t smem = sizeof(V) * ((size_t)L + 4 * (size_t)plen(L));
    FITSNE_TRY(set_smem<T>((const void*)k_conv1d<T, MODE>, smem));
    k_conv1d<T, MODE><<<1, 1024, smem, st>>>(accum, coeffs, ncol, g, tw, pl, kern, with_k1 ? 1 : 0,
                                             pot, out, scal, (double)n_total);
    FITSNE_CHECK_LAUNCH();
    return FITSNE_OK;
  }
  const int maxpair = 2;
  FITSNE_TRY(ensure(ctx->fbuf, sizeof(V) * (size_t)maxpair * n * L));
  // spectrum rows (n x H) followed by the spectrum table Khat (H x L)
  FITSNE_TRY(ensure(ctx->sbuf, sizeof(V) * ((size_t)n * H + (size_t)H * L)));
  FITSNE_TRY(ensure(ctx->zpart, sizeof(double) * (size_t)L));
  V* F = (V*)ctx->fbuf.ptr;
  V* Sb = (V*)ctx->sbuf.ptr;
  V* Kh = Sb + (size_t)n * H;
  double* zp = (double*)ctx->zpart.ptr;
  const int npair_total = (MODE == MODE_TSNE) ? 2 : (ncol + 1) / 2;
  for (int pair0 = 0; pair0 < npair_total; pair0 += maxpair) {
    const int npair = std::min(maxpair, npair_total - pair0);
    // the spectrum rows are recomputed per pair group (one group for t-SNE)
    const int nd = (MODE == MODE_TSNE) ? 2 : npair;
    // the kernel spectrum of this grid may already be on its way (spectrum_ahead)
    const bool ahead = MODE == MODE_TSNE && ctx->spec_ahead && ctx->spec_ahead_L == L && ctx->spec_ahead_n == n;
    ctx->spec_ahead = false;
    const int merged = ahead ? 2 : (sizeof(V) * ((size_t)L + 2 * (size_t)(nd + 1) * plen(L)) <= 113 * 1024 ? 1 : 0);
    size_t smem_r = sizeof(V) * ((size_t)L + 2 * (size_t)(merged == 1 ? nd + 1 : std::max(nd, 1)) * plen(L));
    FITSNE_TRY(set_smem<T>((const void*)k_rows_forward<T, MODE>, smem_r));
    k_rows_forward<T, MODE><<<merged == 0 ? 2 * n : n, 256, smem_r, st>>>(
        accum, coeffs, ncol, pair0, npair, F, Sb, g, tw, pl, merged, accum_reps_live(ctx, accum),
        (int64_t)accum_elems(gr));
    FITSNE_CHECK_LAUNCH();
    if (ahead) {
      FITSNE_CUDA(cudaStreamWaitEvent(st, ctx->ev_spec, 0));  // Khat ready
    } else if (pair0 == 0) {
      // columns per block: as many as fit in shared memory (long transforms
      // take fewer)
      int cpb = kSpecCols;
      auto smem_spec = [&](int c) { return sizeof(V) * ((size_t)L + 2 * (size_t)c * plen(L)); };
      while (cpb > 1 && smem_spec(cpb) > 227 * 1024) cpb /= 2;
      const size_t smem_s = smem_spec(cpb);
      FITSNE_TRY(set_smem<T>((const void*)k_spec_cols<T>, smem_s));
      k_spec_cols<T><<<(H + cpb - 1) / cpb, 256, smem_s, st>>>(Sb, g, tw, pl, Kh, cpb);
      FITSNE_CHECK_LAUNCH();
    }
    // adjacent columns per block (FITSNE_OPT_FFT_COLS; 1 measured fastest at
    // C3 beside the SpMV: 2 and 4 use whole sectors of the strided column
    // reads but fewer blocks fit per SM)
    auto smem_cols = [&](int c) { return sizeof(V) * ((size_t)L + 2 * (size_t)c * npair * plen(L)); };
    int ccols = std::min(kColsMax, ctx->cols_per_block);
    while (ccols > 1 && smem_cols(ccols) > 227 * 1024) ccols /= 2;
    const size_t smem_c = smem_cols(ccols);
    FITSNE_TRY(set_smem<T>((const void*)k_cols<T, MODE>, smem_c));
    k_cols<T, MODE><<<(L + ccols - 1) / ccols, 256, smem_c, st>>>(F, Kh, g, tw, pl, npair, kern,
                                                                  with_k1 ? 1 : 0, zp, ccols);
    FITSNE_CHECK_LAUNCH();
    size_t smem_i = sizeof(V) * ((size_t)L + 2 * (size_t)npair * plen(L));
    FITSNE_TRY(set_smem<T>((const void*)k_rows_inverse<T, MODE>, smem_i));
    k_rows_inverse<T, MODE><<<n, 256, smem_i, st>>>(F, g, tw, pl, npair, ncol, pair0, pot, out, zp,
                                                    scal, (double)n_total);
    FITSNE_CHECK_LAUNCH();
  }
  return FITSNE_OK;
}

// The kernel spectrum depends on the grid only.  In the overlapped schedule it
// is computed on a stream of its own as soon as the grid exists (`from`: the
// stream the grid and its twiddle table were made on), while the spread --
// latency-bound on the few SMs the SpMV leaves -- is still running; the FFT
// stage then transforms the data rows only and joins ev_spec before the
// column stage.  2-D one-block FFT path of this context only (not the fp64
// twin, the four-step path or 1-D).
template <typename T>
static int spectrum_ahead_t(fitsne_ctx* ctx, cudaStream_t from) {
  using V = typename C2<T>::type;
  GridArgs g = grid_args(ctx->grid);
  const int L = g.L, n = g.n, H = L / 2 + 1;
  FftPlan pl;
  make_plan(pl, L);
  FITSNE_TRY(ensure(ctx->fbuf, sizeof(V) * (size_t)2 * n * L));
  FITSNE_TRY(ensure(ctx->sbuf, sizeof(V) * ((size_t)n * H + (size_t)H * L)));
  FITSNE_TRY(ensure(ctx->zpart, sizeof(double) * (size_t)L));
  const V* tw = (const V*)ctx->tw.ptr;
  V* Sb = (V*)ctx->sbuf.ptr;
  V* Kh = Sb + (size_t)n * H;
  if (!ctx->spec) {
    int lo = 0, hi = 0;
    FITSNE_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    FITSNE_CUDA(cudaStreamCreateWithPriority(&ctx->spec, cudaStreamNonBlocking, lo));
    FITSNE_CUDA(cudaEventCreateWithFlags(&ctx->ev_spec_in, cudaEventDisableTiming));
    FITSNE_CUDA(cudaEventCreateWithFlags(&ctx->ev_spec, cudaEventDisableTiming));
  }
  FITSNE_CUDA(cudaEventRecord(ctx->ev_spec_in, from));
  FITSNE_CUDA(cudaStreamWaitEvent(ctx->spec, ctx->ev_spec_in, 0));
  const size_t smem_r = sizeof(V) * ((size_t)L + 2 * (size_t)plen(L));
  FITSNE_TRY(set_smem<T>((const void*)k_rows_forward<T, MODE_TSNE>, smem_r));
  k_rows_forward<T, MODE_TSNE><<<n, 256, smem_r, ctx->spec>>>(nullptr, nullptr, 3, 0, 2, nullptr, Sb, g, tw, pl, 3,
                                                             0, 0);
  FITSNE_CHECK_LAUNCH();
  int cpb = kSpecCols;
  auto smem_spec = [&](int c) { return sizeof(V) * ((size_t)L + 2 * (size_t)c * plen(L)); };
  while (cpb > 1 && smem_spec(cpb) > 227 * 1024) cpb /= 2;
  FITSNE_TRY(set_smem<T>((const void*)k_spec_cols<T>, smem_spec(cpb)));
  k_spec_cols<T><<<(H + cpb - 1) / cpb, 256, smem_spec(cpb), ctx->spec>>>(Sb, g, tw, pl, Kh, cpb);
  FITSNE_CHECK_LAUNCH();
  FITSNE_CUDA(cudaEventRecord(ctx->ev_spec, ctx->spec));
  ctx->spec_ahead = true;
  ctx->spec_ahead_L = L;
  ctx->spec_ahead_n = n;
  return FITSNE_OK;
}

int spectrum_ahead(fitsne_ctx* ctx, cudaStream_t from) {
  ctx->spec_ahead = false;
  if (!ctx->spec_opt || !ctx->grid_valid || ctx->wide || ctx->grid.dims != 2) return FITSNE_OK;
  if (big_fft_applies(ctx, ctx->grid.fft_len)) return FITSNE_OK;
  return ctx->dtype == FITSNE_F32 ? spectrum_ahead_t<float>(ctx, from) : spectrum_ahead_t<double>(ctx, from);
}

int fft_tsne(fitsne_ctx* ctx, void* accum, int64_t n_total, bool with_k1, cudaStream_t st) {
  FITSNE_RANGE("fft_stage");
  if (!ctx->grid_valid) { set_error("no grid"); return FITSNE_EINVAL; }
  if (ctx->wide) {
    FITSNE_TRY(fft_tsne(ctx->shadow, accum, n_total, with_k1, st));
    FITSNE_TRY(ensure(ctx->scal, 64 * sizeof(double)));
    // Z (scal[0]) where this context's consumers read it
    FITSNE_CUDA(cudaMemcpyAsync(ctx->scal.ptr, ctx->shadow->scal.ptr, sizeof(double),
                                cudaMemcpyDeviceToDevice, st));
    return FITSNE_OK;
  }
  if (accum == nullptr) accum = ctx->accum.ptr;
  size_t G = accum_elems(ctx->grid) / kNodeSlots;
  FITSNE_TRY(ensure(ctx->pot, (size_t)pot_records(ctx->grid.dims, ctx->grid.n_intervals, ctx->grid.points_per_interval) *
                                  kNodeSlots * dsize(ctx->dtype)));
  (void)G;
  FITSNE_TRY(ensure(ctx->scal, 64 * sizeof(double)));
  int rc;
  if (ctx->dtype == FITSNE_F32)
    rc = run_conv<float, MODE_TSNE>(ctx, (float*)accum, nullptr, 3, 0, with_k1, nullptr, n_total, st);
  else
    rc = run_conv<double, MODE_TSNE>(ctx, (double*)accum, nullptr, 3, 0, with_k1, nullptr, n_total, st);
  if (rc == FITSNE_OK && accum == ctx->accum.ptr) ctx->accum_clean = true;  // consumed + cleared
  return rc;
}

// FFT stage of the device-grid schedule (fp32, 2-D, t-SNE channels): launch
// shapes and buffers for n_cap nodes per dim and length L_cap, grid read by
// the kernels from gd.  Consumes and clears the accumulator like fft_tsne.
int fft_tsne_dev(fitsne_ctx* ctx, void* accum_v, int64_t n_total, const GridArgs* gd, int n_cap, int L_cap,
                 cudaStream_t st) {
  using T = float;
  using V = float2;
  constexpr int MODE = MODE_TSNE;
  const int H_cap = L_cap / 2 + 1;
  FITSNE_TRY(ensure(ctx->fbuf, sizeof(V) * 2 * (size_t)n_cap * L_cap));
  FITSNE_TRY(ensure(ctx->sbuf, sizeof(V) * ((size_t)n_cap * H_cap + (size_t)H_cap * L_cap)));
  FITSNE_TRY(ensure(ctx->zpart, sizeof(double) * (size_t)L_cap));
  FITSNE_TRY(ensure(ctx->pot, sizeof(T) * (size_t)pot_records(2, n_cap / 3, 3) * kNodeSlots));
  FITSNE_TRY(ensure(ctx->scal, 64 * sizeof(double)));
  FITSNE_TRY(ensure(ctx->tw, sizeof(V) * (size_t)L_cap));
  T* accum = (T*)accum_v;
  V* F = (V*)ctx->fbuf.ptr;
  V* Sb = (V*)ctx->sbuf.ptr;
  V* Kh = Sb + (size_t)n_cap * H_cap;
  double* zp = (double*)ctx->zpart.ptr;
  V* tw = (V*)ctx->tw.ptr;
  const GridArgs g0{};
  const FftPlan pl0{};
  k_twiddles<T><<<grid_for(L_cap), kBlock, 0, st>>>(tw, L_cap, gd);
  FITSNE_CHECK_LAUNCH();
  ctx->tw_len = -1;  // the table now follows the device grid
  const int merged = sizeof(V) * ((size_t)L_cap + 2 * 3 * (size_t)plen(L_cap)) <= 113 * 1024 ? 1 : 0;
  const size_t smem_r = sizeof(V) * ((size_t)L_cap + 2 * (size_t)(merged ? 3 : 2) * plen(L_cap));
  FITSNE_TRY(set_smem<T>((const void*)k_rows_forward<T, MODE>, smem_r));
  k_rows_forward<T, MODE><<<merged ? n_cap : 2 * n_cap, 256, smem_r, st>>>(
      accum, nullptr, 3, 0, 2, F, Sb, g0, tw, pl0, merged, 1, 0, gd);
  FITSNE_CHECK_LAUNCH();
  int cpb = kSpecCols;
  auto smem_spec = [&](int c) { return sizeof(V) * ((size_t)L_cap + 2 * (size_t)c * plen(L_cap)); };
  while (cpb > 1 && smem_spec(cpb) > 227 * 1024) cpb /= 2;
  FITSNE_TRY(set_smem<T>((const void*)k_spec_cols<T>, smem_spec(cpb)));
  k_spec_cols<T><<<(H_cap + cpb - 1) / cpb, 256, smem_spec(cpb), st>>>(Sb, g0, tw, pl0, Kh, cpb, gd);
  FITSNE_CHECK_LAUNCH();
  auto smem_cols = [&](int c) { return sizeof(V) * ((size_t)L_cap + 2 * (size_t)c * 2 * plen(L_cap)); };
  int ccols = std::min(kColsMax, ctx->cols_per_block);
  while (ccols > 1 && smem_cols(ccols) > 227 * 1024) ccols /= 2;
  FITSNE_TRY(set_smem<T>((const void*)k_cols<T, MODE>, smem_cols(ccols)));
  k_cols<T, MODE><<<(L_cap + ccols - 1) / ccols, 256, smem_cols(ccols), st>>>(F, Kh, g0, tw, pl0, 2, 0, 0, zp,
                                                                               ccols, gd);
  FITSNE_CHECK_LAUNCH();
  const size_t smem_i = sizeof(V) * ((size_t)L_cap + 2 * 2 * (size_t)plen(L_cap));
  FITSNE_TRY(set_smem<T>((const void*)k_rows_inverse<T, MODE>, smem_i));
  k_rows_inverse<T, MODE><<<n_cap, 256, smem_i, st>>>(F, g0, tw, pl0, 2, 3, 0, (T*)ctx->pot.ptr, nullptr, zp,
                                                      (double*)ctx->scal.ptr, (double)n_total, gd);
  FITSNE_CHECK_LAUNCH();
  return FITSNE_OK;
}

// the internal accumulator sized for G_cap nodes (one replica suffices for the
// band spread, but the direct scatter of a fallback may use all replicas)
int ensure_accum_nodes(fitsne_ctx* ctx, size_t g_nodes, cudaStream_t st) {
  const size_t bytes = g_nodes * kNodeSlots * dsize(ctx->dtype) * (size_t)ctx->spread_replicas;
  if (ctx->accum.cap < bytes) {
    FITSNE_TRY(ensure(ctx->accum, bytes));
    ctx->accum_clean = false;
  }
  if (!ctx->accum_clean) {
    FITSNE_CUDA(cudaMemsetAsync(ctx->accum.ptr, 0, ctx->accum.cap, st));
    ctx->accum_clean = true;
  }
  return FITSNE_OK;
}

// device-grid schedule: bbox kernels that also compute the grid into gd
// Stockham plans of every 2^a 3^b length up to L_max (ascending), built on the
// host once per context and kept on the device for the device-grid schedule
int device_plan_table(fitsne_ctx* ctx, int L_max, const void** table, int* count) {
  if (ctx->plan_table_max < L_max) {
    std::vector<FftPlan> plans;
    for (long long p2 = 1; p2 <= L_max; p2 *= 2)
      for (long long v = p2; v <= L_max; v *= 3) {
        FftPlan pl;
        make_plan(pl, (int)v);
        plans.push_back(pl);
      }
    std::sort(plans.begin(), plans.end(), [](const FftPlan& a, const FftPlan& b) { return a.L < b.L; });
    FITSNE_TRY(ensure(ctx->plan_table, sizeof(FftPlan) * plans.size()));
    FITSNE_CUDA(cudaMemcpy(ctx->plan_table.ptr, plans.data(), sizeof(FftPlan) * plans.size(),
                           cudaMemcpyHostToDevice));
    ctx->plan_table_max = L_max;
    ctx->plan_table_n = (int)plans.size();
  }
  *table = ctx->plan_table.ptr;
  *count = ctx->plan_table_n;
  return FITSNE_OK;
}

// gd points at a DevGrid block {grid, plan, bbox}; the readback of that
// block goes on copy_st (behind an event), so the stages queued on st after
// the bbox kernel do not wait for it
int bbox_launch_devgrid(fitsne_ctx* ctx, const void* Y, int64_t n, GridArgs* gd, const DevGridReq& rq,
                        GridArgs* gd_host, cudaStream_t st, cudaStream_t copy_st, cudaEvent_t ev_k) {
  double* outd = reinterpret_cast<DevGrid*>(gd)->bbox;
  FITSNE_TRY(bbox_kernels(ctx, Y, n, outd, 0, st, nullptr, gd, rq));
  FITSNE_CUDA(cudaEventRecord(ev_k, st));
  FITSNE_CUDA(cudaStreamWaitEvent(copy_st, ev_k, 0));
  FITSNE_CUDA(cudaMemcpyAsync(gd_host, gd, sizeof(DevGrid), cudaMemcpyDeviceToHost, copy_st));
  if (!ctx->ev_bbox) FITSNE_CUDA(cudaEventCreateWithFlags(&ctx->ev_bbox, cudaEventDisableTiming));
  FITSNE_CUDA(cudaEventRecord(ctx->ev_bbox, copy_st));
  return FITSNE_OK;
}

int matvec_general(fitsne_ctx* ctx, int kernel, const void* coeffs, int ncol, void* out,
                   cudaStream_t st) {
  if (!ctx->grid_valid) { set_error("no grid"); return FITSNE_EINVAL; }
  if (kernel != FITSNE_CAUCHY && kernel != FITSNE_CAUCHY_SQUARED) {
    set_error("unknown kernel");
    return FITSNE_EINVAL;
  }
  FITSNE_TRY(ensure(ctx->pot, 64));
  FITSNE_TRY(ensure(ctx->scal, 64 * sizeof(double)));
  if (ncol <= 0) return FITSNE_OK;
  if (ctx->dtype == FITSNE_F32)
    return run_conv<float, MODE_GENERAL>(ctx, nullptr, (const float*)coeffs, ncol, kernel, false,
                                         (float*)out, 0, st);
  return run_conv<double, MODE_GENERAL>(ctx, nullptr, (const double*)coeffs, ncol, kernel, false,
                                        (double*)out, 0, st);
}

// =============================================================================
// a6/a7/a8: gather + t-SNE assembly
//   k1 = phi_K1(1) - 1, k2[:, c] = phi_K2(y_c) - y_c, k2[:, s] = phi_K2(1) - 1
//   F_rep = (y * k2[:, s] - k2[:, :s]) / Z           (optimizer.py:206-210, 244)
// =============================================================================
template <typename T, int S, int P>
__global__ void k_gather_tsne(const T* __restrict__ Y, int64_t n, GridArgs g,
                              const T* __restrict__ pot, const double* __restrict__ scal,
                              T* __restrict__ forces, T* __restrict__ k1out, T* __restrict__ k2out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int p = (P > 0) ? P : g.p;
  PointInterp<T, S> pi;
  double y[S];
  interp_point<T, S>(Y, i, g, pi, y);
  T phi[4] = {0, 0, 0, 0};
  if (S == 1) {
    for (int a = 0; a < p; ++a) {
      T v[4];
      load_slots<T>(pot + ((int64_t)pi.cell[0] * p + a) * kNodeSlots, v);
      T w = (T)pi.w[0][a];
#pragma unroll
      for (int c = 0; c < 4; ++c) phi[c] += v[c] * w;
    }
  } else {
    for (int a = 0; a < p; ++a) {
      for (int b = 0; b < p; ++b) {
        T v[4];
        load_slots<T>(pot + pot_box_node(pi.cell[0], pi.cell[1], a, b, p, g.n_int) * kNodeSlots, v);
        T w = (T)(pi.w[0][a] * pi.w[1][b]);
#pragma unroll
        for (int c = 0; c < 4; ++c) phi[c] += v[c] * w;
      }
    }
  }
  const T Z = (T)scal[0];
  T h4 = phi[0] - (T)1;
#pragma unroll
  for (int d = 0; d < S; ++d) {
    // phi[1 + d] = K2 * (y_d - c_d) (centred charges)
    const T yc = (T)(y[d] - g.c[d]);
    const T hc = phi[1 + d] - yc;
    forces[i * S + d] = (yc * h4 - hc) / Z;
    // the reference's k2[:, d] = K2 * y_d - y_d
    if (k2out) k2out[i * (S + 1) + d] = (T)((double)phi[1 + d] + g.c[d] * (double)phi[0] - y[d]);
  }
  if (k2out) k2out[i * (S + 1) + S] = h4;
  if (k1out) k1out[i] = phi[3] - (T)1;
}

int gather_tsne(fitsne_ctx* ctx, const void* Y, int64_t n, void* forces, void* k1, void* k2,
                cudaStream_t st) {
  FITSNE_RANGE("gather");
  GridArgs g = grid_args(ctx->grid);
  if (n <= 0) return FITSNE_OK;
  if (ctx->wide) {
    const double* y = widen_points(ctx, Y, n, st);
    if (!y) { set_error("fp64 grid: point conversion failed"); return FITSNE_ECUDA; }
    const int S = ctx->dims;
    FITSNE_TRY(ensure(ctx->r64, sizeof(double) * (size_t)n * (2 * S + 2)));
    double* f = (double*)ctx->r64.ptr;
    double* a1 = f + (size_t)n * S;
    double* a2 = a1 + (size_t)n;
    FITSNE_TRY(gather_tsne(ctx->shadow, y, n, f, k1 ? a1 : nullptr, k2 ? a2 : nullptr, st));
    FITSNE_TRY(narrow_values(f, n * S, (float*)forces, st));
    if (k1) FITSNE_TRY(narrow_values(a1, n, (float*)k1, st));
    if (k2) FITSNE_TRY(narrow_values(a2, n * (S + 1), (float*)k2, st));
    return FITSNE_OK;
  }
  const double* scal = (const double*)ctx->scal.ptr;
#define GATHER_LAUNCH(T, S)                                                                  \
  do {                                                                                       \
    if (g.p == 3)                                                                            \
      k_gather_tsne<T, S, 3><<<grid_for(n), kBlock, 0, st>>>((const T*)Y, n, g,              \
          (const T*)ctx->pot.ptr, scal, (T*)forces, (T*)k1, (T*)k2);                         \
    else                                                                                     \
      k_gather_tsne<T, S, 0><<<grid_for(n), kBlock, 0, st>>>((const T*)Y, n, g,              \
          (const T*)ctx->pot.ptr, scal, (T*)forces, (T*)k1, (T*)k2);                         \
  } while (0)
  if (ctx->dtype == FITSNE_F32) {
    if (ctx->dims == 1) GATHER_LAUNCH(float, 1); else GATHER_LAUNCH(float, 2);
  } else {
    if (ctx->dims == 1) GATHER_LAUNCH(double, 1); else GATHER_LAUNCH(double, 2);
  }
#undef GATHER_LAUNCH
  FITSNE_CHECK_LAUNCH();
  return FITSNE_OK;
}

// values (ncol, G) planar -> out (n, ncol)
template <typename T, int S>
__global__ void k_gather_general(const T* __restrict__ Y, int64_t n, GridArgs g,
                                 const T* __restrict__ vals, int ncol, T* __restrict__ out,
                                 int* __restrict__ outside) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool o = false;
#pragma unroll
  for (int d = 0; d < S; ++d) {
    double v = (double)Y[i * S + d];
    if (v < g.lo[d] || v > g.hi[d]) o = true;
  }
  if (o) { atomicOr(outside, 1); return; }
  PointInterp<T, S> pi;
  double y[S];
  interp_point<T, S>(Y, i, g, pi, y);
  const int p = g.p;
  const int64_t nn = g.n;
  const int64_t G = (S == 1) ? nn : nn * nn;
  const int cnt = (S == 1) ? p : p * p;
  for (int c = 0; c < ncol; ++c) {
    double acc = 0.0;
    for (int k = 0; k < cnt; ++k) {
      int a = (S == 1) ? k : k / p, b = (S == 1) ? 0 : k % p;
      int64_t node = (S == 1) ? ((int64_t)pi.cell[0] * p + a)
                              : (((int64_t)pi.cell[0] * p + a) * nn + (int64_t)pi.cell[1] * p + b);
      double w = (S == 1) ? pi.w[0][a] : pi.w[0][a] * pi.w[1][b];
      acc += (double)vals[(int64_t)c * G + node] * w;
    }
    out[i * ncol + c] = (T)acc;
  }
}

int gather_general(fitsne_ctx* ctx, const void* Y, int64_t n, const void* vals, int ncol, void* out,
                   cudaStream_t st) {
  if (!ctx->grid_valid) { set_error("no grid"); return FITSNE_EINVAL; }
  GridArgs g = grid_args(ctx->grid);
  FITSNE_TRY(ensure(ctx->counter, 64 * sizeof(int)));
  FITSNE_CUDA(cudaMemsetAsync(ctx->counter.ptr, 0, sizeof(int), st));
  int* flag = (int*)ctx->counter.ptr;
  if (n > 0) {
    if (ctx->dtype == FITSNE_F32) {
      if (ctx->dims == 1) k_gather_general<float, 1><<<grid_for(n), kBlock, 0, st>>>((const float*)Y, n, g, (const float*)vals, ncol, (float*)out, flag);
      else k_gather_general<float, 2><<<grid_for(n), kBlock, 0, st>>>((const float*)Y, n, g, (const float*)vals, ncol, (float*)out, flag);
    } else {
      if (ctx->dims == 1) k_gather_general<double, 1><<<grid_for(n), kBlock, 0, st>>>((const double*)Y, n, g, (const double*)vals, ncol, (double*)out, flag);
      else k_gather_general<double, 2><<<grid_for(n), kBlock, 0, st>>>((const double*)Y, n, g, (const double*)vals, ncol, (double*)out, flag);
    }
    FITSNE_CHECK_LAUNCH();
  }
  return check_outside(ctx, st);
}

}  // namespace fitsne
