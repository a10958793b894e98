// Attractive half of the gradient, KL, the momentum/gains update and the
// exact O(N^2) sums, on sm_100a.
//
//   compute_attractive (optimizer.py:150-166): the reference applies every
//   stored upper-triangle pair in both directions with two bincounts; here P
//   is the full symmetric CSR (both triangles) and each row is reduced by one
//   warp: F_i = sum_j p_ij / (1 + |y_i - y_j|^2) (y_i - y_j).
//   _kl_given_z (optimizer.py:265-275): KL = 2 sum_{upper, p>0} p (log p - log q)
//   with q = 1/((1+d^2) Z) equals, over the full matrix,
//   sum p log p + sum p log1p(d^2) + (sum p) log Z; the first sum is fixed and
//   precomputed once, the second is fused into the SpMV row loop.
//   step (optimizer.py:299-323).
//   _exact_repulsion_sums (optimizer.py:169-190).
#include <cmath>
#include <algorithm>

#include "common.cuh"
#include "fft.cuh"
#include "interp.cuh"
#include "internal.h"

namespace fitsne {

static constexpr int kBlock = 256;

static inline int nblocks(int64_t n, int block = kBlock) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > (1LL << 30)) g = (1LL << 30);
  return (int)g;
}

template <typename T>
__device__ __forceinline__ T fast_log1p(T x);
// fp32: SFU log of (1 + x) (2 ulp-level error for 1+x in normal range; for
// x below 2^-24 it returns 0 where log1p returns ~x, a p*x term that is far
// below the KL's fp32 resolution)
template <>
__device__ __forceinline__ float fast_log1p<float>(float x) { return __logf(1.0f + x); }
template <>
__device__ __forceinline__ double fast_log1p<double>(double x) { return log1p(x); }


template <typename T, int S>
__device__ __forceinline__ void load_point(const T* __restrict__ Y, int64_t j, T (&v)[S]) {
  if constexpr (S == 2 && sizeof(T) == 4) {
    float2 a = __ldg(reinterpret_cast<const float2*>(Y) + j);
    v[0] = a.x; v[1] = a.y;
  } else if constexpr (S == 2) {
    double2 a = __ldg(reinterpret_cast<const double2*>(Y) + j);
    v[0] = a.x; v[1] = a.y;
  } else {
    v[0] = __ldg(Y + j);
  }
}

// Neighbour gathers with an L2 evict-last hint: the CSR stream (8-12 B per
// entry, read once) is loaded evict-first, so at large N (C4: Y is 80 MB,
// the stream 7 GB) the embedding stays resident in the 126 MB L2 instead of
// being pushed out by the stream it is gathered against.
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

template <typename T, int S>
__device__ __forceinline__ void load_point_el(const T* __restrict__ Y, int64_t j, T (&v)[S], uint64_t pol) {
  if constexpr (S == 2 && sizeof(T) == 4) {
    float a, b;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;"
                 : "=f"(a), "=f"(b) : "l"(Y + 2 * j), "l"(pol));
    v[0] = a; v[1] = b;
  } else if constexpr (S == 2) {
    double a, b;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(a), "=d"(b) : "l"(Y + 2 * j), "l"(pol));
    v[0] = a; v[1] = b;
  } else if constexpr (sizeof(T) == 4) {
    float a;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(a) : "l"(Y + j), "l"(pol));
    v[0] = a;
  } else {
    double a;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(a) : "l"(Y + j), "l"(pol));
    v[0] = a;
  }
}

// p / (1 + d2): fp32 uses the fast reciprocal-based division (<= 2 ulp, well
// inside the fp32 parity bar); fp64 keeps IEEE division.
template <typename T>
__device__ __forceinline__ T cauchy_weight(T p, T d2) { return p / ((T)1 + d2); }
template <>
__device__ __forceinline__ float cauchy_weight<float>(float p, float d2) {
  return __fdividef(p, 1.0f + d2);
}

// One warp reduces CSR row [beg, end) against y_i: acc += sum_j w_ij (y_i - y_j),
// w_ij = p_ij / (1 + d_ij^2), and (KL) klr += p_ij log1p(d_ij^2).  Each lane
// first issues the (col, val) loads of kU stored entries, then their kU
// neighbour gathers, so 2 kU independent loads are in flight per lane.
constexpr int kRowU = 4;

// (col, val) of the stored entries k0 + 32 u (u < kRowU) of a row ending at end
template <typename T>
__device__ __forceinline__ void row_chunk_load(const int32_t* __restrict__ col, const T* __restrict__ val,
                                               int64_t k0, int64_t end, int32_t (&j)[kRowU],
                                               T (&p)[kRowU]) {
#pragma unroll
  for (int u = 0; u < kRowU; ++u) {
    const int64_t k = k0 + 32 * u;
    const bool ok = k < end;
    j[u] = ok ? __ldcs(col + k) : 0;
    p[u] = ok ? __ldcs(val + k) : (T)0;
  }
}

// gathers y_j of one loaded chunk and accumulates its terms
template <typename T, int S, bool KL>
__device__ __forceinline__ void row_chunk_reduce(const T* __restrict__ Y, int64_t k0, int64_t end,
                                                 const int32_t (&j)[kRowU], const T (&p)[kRowU],
                                                 const T (&yi)[S], T (&acc)[S], T& klr, uint64_t pol) {
  T yj[kRowU][S];
#pragma unroll
  for (int u = 0; u < kRowU; ++u) {
    if (k0 + 32 * u < end) load_point_el<T, S>(Y, j[u], yj[u], pol);
    else {
#pragma unroll
      for (int d = 0; d < S; ++d) yj[u][d] = yi[d];
    }
  }
#pragma unroll
  for (int u = 0; u < kRowU; ++u) {
    T df[S], s2 = 0;
#pragma unroll
    for (int d = 0; d < S; ++d) {
      df[d] = yi[d] - yj[u][d];
      s2 += df[d] * df[d];
    }
    const T w = cauchy_weight<T>(p[u], s2);
#pragma unroll
    for (int d = 0; d < S; ++d) acc[d] += w * df[d];
    if (KL) {
      if (p[u] > (T)0) klr += p[u] * fast_log1p<T>(s2);
    }
  }
}

// One warp reduces CSR row [beg, end) against y_i: acc += sum_j w_ij (y_i - y_j),
// w_ij = p_ij / (1 + d_ij^2), and (KL) klr += p_ij log1p(d_ij^2).  Each lane
// first issues the (col, val) loads of kRowU stored entries, then their
// neighbour gathers, so 2 kRowU independent loads are in flight per lane.
// skip: stored entries of the row already reduced by the caller (row
// pipelining in k_attract reduces the first chunk itself).
template <typename T, int S, bool KL>
__device__ __forceinline__ void row_reduce(const int32_t* __restrict__ col, const T* __restrict__ val,
                                           const T* __restrict__ Y, int64_t beg, int64_t end,
                                           int lane, const T (&yi)[S], T (&acc)[S], T& klr,
                                           uint64_t pol, int skip = 0) {
  for (int64_t k0 = beg + lane + skip; k0 < end; k0 += 32 * kRowU) {
    int32_t j[kRowU];
    T p[kRowU];
    row_chunk_load<T>(col, val, k0, end, j, p);
    row_chunk_reduce<T, S, KL>(Y, k0, end, j, p, yi, acc, klr, pol);
  }
}

#ifndef FITSNE_CSR_PIPE
#define FITSNE_CSR_PIPE 1
#endif

// ---------------------------------------------------------------------------
// warp-per-row CSR SpMV.  MODE 0: F_attr out.  MODE 1: gradient
// 4 (alpha F_attr - F_rep).  KL: per-block partial of sum p log1p(d^2).
// ---------------------------------------------------------------------------
// MODE 2: the repulsive force of row i is gathered in the same warp from the
// potential grid (lanes 0..p^s-1 each interpolate one node), so F_rep never
// round-trips through HBM.
template <typename T, int S, int MODE, bool KL, int P>
#ifndef FITSNE_CSR_MINB
#define FITSNE_CSR_MINB (FITSNE_CSR_PIPE ? 5 : 6)
#endif
__global__ void __launch_bounds__(kBlock, FITSNE_CSR_MINB)
k_attract(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
          const T* __restrict__ val, const T* __restrict__ Y, int64_t n_rows, int64_t row_begin,
          const T* __restrict__ frep, T alpha, T* __restrict__ out, double* __restrict__ klpart,
          GridArgs g, const T* __restrict__ pot, const double* __restrict__ scal) {
  // Each warp owns tiles of 32 consecutive rows.  Per-row scalar work (y_i,
  // row bounds, and for MODE 2 the p^s-node gather of F_rep) is done one row
  // per lane with coalesced loads; the CSR reduction then walks the tile's
  // rows one at a time with the whole warp, and lane m keeps row m's result.
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t ntiles = (n_rows + 31) >> 5;
  // per-warp staging of the tile's row scalars (keeps them out of registers)
  __shared__ int64_t s_rb[kBlock], s_re[kBlock];
  __shared__ T s_y[kBlock * S], s_acc[kBlock * S];
  const int wbase = threadIdx.x & ~31;
  double kl = 0.0;
  T Z = (T)1;
  if (MODE == 2) Z = (T)scal[0];
  const uint64_t pol = l2_evict_last_policy();
  for (int64_t t = warp; t < ntiles; t += nwarps) {
    const int64_t r_mine = t * 32 + lane;
    const bool valid = r_mine < n_rows;
    {
      T ym[S];
#pragma unroll
      for (int d = 0; d < S; ++d) ym[d] = 0;
      int64_t rb = 0, re = 0;
      if (valid) {
        load_point<T, S>(Y, row_begin + r_mine, ym);
        rb = rowptr[r_mine];
        re = rowptr[r_mine + 1];
      }
      s_rb[threadIdx.x] = rb;
      s_re[threadIdx.x] = re;
#pragma unroll
      for (int d = 0; d < S; ++d) s_y[threadIdx.x * S + d] = ym[d];
    }
    __syncwarp();
    const int mcount = (n_rows - t * 32 < 32) ? (int)(n_rows - t * 32) : 32;
#if FITSNE_CSR_PIPE
    // row pipelining: the first (col, val) chunk of row m + 1 is loaded before
    // row m's neighbour gathers, so the HBM stream latency of the next row
    // overlaps the gather latency of this one (short random-graph rows are
    // one chunk each)
    int32_t jn[kRowU];
    T pn[kRowU];
    row_chunk_load<T>(col, val, s_rb[wbase] + lane, s_re[wbase], jn, pn);
#endif
    for (int m = 0; m < mcount; ++m) {
      T yi[S];
#pragma unroll
      for (int d = 0; d < S; ++d) yi[d] = s_y[(wbase + m) * S + d];
      const int64_t beg = s_rb[wbase + m];
      const int64_t end = s_re[wbase + m];
      T acc[S];
#pragma unroll
      for (int d = 0; d < S; ++d) acc[d] = 0;
      T klr = 0;
#if FITSNE_CSR_PIPE
      int32_t jc[kRowU];
      T pc[kRowU];
#pragma unroll
      for (int u = 0; u < kRowU; ++u) { jc[u] = jn[u]; pc[u] = pn[u]; }
      if (m + 1 < mcount)
        row_chunk_load<T>(col, val, s_rb[wbase + m + 1] + lane, s_re[wbase + m + 1], jn, pn);
      row_chunk_reduce<T, S, KL>(Y, beg + lane, end, jc, pc, yi, acc, klr, pol);
      row_reduce<T, S, KL>(col, val, Y, beg, end, lane, yi, acc, klr, pol, 32 * kRowU);
#else
      row_reduce<T, S, KL>(col, val, Y, beg, end, lane, yi, acc, klr, pol);
#endif
#pragma unroll
      for (int d = 0; d < S; ++d) acc[d] = warp_sum(acc[d]);
      if (lane == m) {
#pragma unroll
        for (int d = 0; d < S; ++d) s_acc[threadIdx.x * S + d] = acc[d];
      }
      if (KL) kl += (double)klr;
    }
    __syncwarp();
    if (valid) {
      T ym[S], fr[S];
#pragma unroll
      for (int d = 0; d < S; ++d) { ym[d] = s_y[threadIdx.x * S + d]; fr[d] = 0; }
      if (MODE == 1) {
#pragma unroll
        for (int d = 0; d < S; ++d) fr[d] = frep[r_mine * S + d];
      } else if (MODE == 2) {
        T phi[4];
        point_gather<T, S, P>(ym, g, pot, phi);
#pragma unroll
        for (int d = 0; d < S; ++d) fr[d] = frep_from_phi<T, S>(ym, phi, Z, d, g);
      }
#pragma unroll
      for (int d = 0; d < S; ++d) {
        const T res = s_acc[threadIdx.x * S + d];
        if (MODE == 0) out[r_mine * S + d] = res;
        else out[r_mine * S + d] = (T)4 * (alpha * res - fr[d]);
      }
    }
    __syncwarp();
  }
  if (KL) {
    __shared__ double red[kBlock / 32];
    kl = warp_sum(kl);
    if (lane == 0) red[threadIdx.x >> 5] = kl;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0;
      for (int w = 0; w < kBlock / 32; ++w) s += red[w];
      klpart[blockIdx.x] = s;
    }
  }
}

// deterministic fold of per-block partials into dst[0]
__global__ void k_fold(const double* __restrict__ part, int n, double* __restrict__ dst) {
  __shared__ double red[32];
  double s = 0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) s += part[k];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) t += red[w];
    dst[0] = t;
  }
}

// one 32-row tile per warp (the hardware scheduler balances the tiles)
// Overlap modes use a persistent grid (ctx->spmv_blocks_per_sm blocks per SM,
// warps grid-stride over the 32-row tiles) so all SpMV blocks are resident
// at once and the concurrently launched FFT blocks find free SM slots;
// otherwise one tile per warp.
static int attract_grid(fitsne_ctx* ctx) {
  int64_t tiles = (ctx->n_rows + 31) / 32;
  int64_t blocks = (tiles + kBlock / 32 - 1) / (kBlock / 32);
  if (ctx->overlap != 0 && ctx->spmv_blocks_per_sm > 0) {
    const int64_t cap = (int64_t)ctx->num_sms * ctx->spmv_blocks_per_sm;
    if (blocks > cap) blocks = cap;
  }
  if (blocks < 1) blocks = 1;
  if (blocks > (1LL << 30)) blocks = (1LL << 30);
  return (int)blocks;
}

template <typename T>
static int launch_attract(fitsne_ctx* ctx, const T* Y, const T* frep, T alpha, T* out, int mode,
                          bool kl, double* klpart, int blocks, cudaStream_t st) {
  const T* val = (const T*)ctx->val;
  GridArgs g = grid_args(ctx->grid);
  const T* pot = (const T*)ctx->pot.ptr;
  const double* scal = (const double*)ctx->scal.ptr;
#define ATT(S, M, K, P)                                                                           \
  k_attract<T, S, M, K, P><<<blocks, kBlock, 0, st>>>(ctx->rowptr, ctx->col, val, Y, ctx->n_rows,  \
                                                      ctx->row_begin, frep, alpha, out, klpart, g, \
                                                      pot, scal)
#define ATT_K(S, M, P) do { if (kl) ATT(S, M, true, P); else ATT(S, M, false, P); } while (0)
#define ATT_M(S)                                                    \
  do {                                                              \
    if (mode == 0) ATT_K(S, 0, 3);                                  \
    else if (mode == 1) ATT_K(S, 1, 3);                             \
    else if (g.p == 3) ATT_K(S, 2, 3);                              \
    else ATT_K(S, 2, 0);                                            \
  } while (0)
  if (ctx->dims == 1) ATT_M(1); else ATT_M(2);
#undef ATT_M
#undef ATT_K
#undef ATT
  FITSNE_CHECK_LAUNCH();
  return FITSNE_OK;
}

int attractive(fitsne_ctx* ctx, const void* Yfull, const void* forces, double alpha, void* out,
               int mode, bool kl, cudaStream_t st, bool fold) {
  if (!ctx->rowptr) { set_error("no affinities registered"); return FITSNE_EINVAL; }
  if (mode == 2 && !ctx->grid_valid) { set_error("no grid"); return FITSNE_EINVAL; }
  FITSNE_TRY(ensure(ctx->scal, 64 * sizeof(double)));
  if (mode != 2 && tiled_usable(ctx, Yfull, st)) {
    void* fattr = nullptr;
    double* part = nullptr;
    int np = 0;
    FITSNE_TRY(attract_tiled(ctx, Yfull, kl, st, &fattr, &part, &np));
    FITSNE_TRY(tiled_finish(ctx, forces, alpha, mode, out, st));
    ctx->kl_part = part;
    ctx->kl_nparts = np;
    if (kl && fold) {
      k_fold<<<1, 1024, 0, st>>>(part, np, (double*)ctx->scal.ptr + 1);
      FITSNE_CHECK_LAUNCH();
    }
    return FITSNE_OK;
  }
  const int blocks = attract_grid(ctx);
  FITSNE_TRY(ensure(ctx->part, sizeof(double) * ((size_t)blocks + (size_t)ctx->num_sms * 16 + 64)));
  FITSNE_TRY(ensure(ctx->scal, 64 * sizeof(double)));
  double* part = (double*)ctx->part.ptr;
  if (ctx->dtype == FITSNE_F32)
    FITSNE_TRY(launch_attract<float>(ctx, (const float*)Yfull, (const float*)forces, (float)alpha,
                                     (float*)out, mode, kl, part, blocks, st));
  else
    FITSNE_TRY(launch_attract<double>(ctx, (const double*)Yfull, (const double*)forces, alpha,
                                      (double*)out, mode, kl, part, blocks, st));
  ctx->kl_part = part;
  ctx->kl_nparts = blocks;
  if (kl && fold) {
    k_fold<<<1, 1024, 0, st>>>(part, blocks, (double*)ctx->scal.ptr + 1);
    FITSNE_CHECK_LAUNCH();
  }
  return FITSNE_OK;
}

int kl_sum(fitsne_ctx* ctx, const void* Yfull, cudaStream_t st) {
  // F_attr is computed as a by-product into scratch; only the KL partial is kept
  size_t es = dsize(ctx->dtype);
  FITSNE_TRY(ensure(ctx->gtmp, es * (size_t)std::max<int64_t>(ctx->n_rows, 1) * ctx->dims));
  return attractive(ctx, Yfull, nullptr, 1.0, ctx->gtmp.ptr, 0, true, st);
}

// sum over stored p>0 of p log p and of p (fixed per affinity matrix)
template <typename T>
__global__ void k_plogp(const T* __restrict__ val, int64_t nnz, double* __restrict__ part) {
  double s = 0, m = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz;
       k += (int64_t)gridDim.x * blockDim.x) {
    double p = (double)val[k];
    if (p > 0) { s += p * log(p); m += p; }
  }
  __shared__ double r1[32], r2[32];
  s = warp_sum(s);
  m = warp_sum(m);
  if ((threadIdx.x & 31) == 0) { r1[threadIdx.x >> 5] = s; r2[threadIdx.x >> 5] = m; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0;
    for (int w = 0; w < (int)blockDim.x / 32; ++w) { a += r1[w]; b += r2[w]; }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

__global__ void k_fold2(const double* __restrict__ part, int n, double* __restrict__ dst) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double a = 0, b = 0;
    for (int k = 0; k < n; ++k) { a += part[2 * k]; b += part[2 * k + 1]; }
    dst[0] = a;
    dst[1] = b;
  }
}

int compute_plogp(fitsne_ctx* ctx, cudaStream_t st) {
  FITSNE_TRY(ensure(ctx->part, sizeof(double) * (size_t)ctx->num_sms * 16 + 64));
  FITSNE_TRY(ensure(ctx->scal, 64 * sizeof(double)));
  int blocks = std::min<int64_t>(nblocks(std::max<int64_t>(ctx->nnz, 1)), ctx->num_sms * 4);
  double* part = (double*)ctx->part.ptr;
  double* sc = (double*)ctx->scal.ptr;
  if (ctx->dtype == FITSNE_F32) k_plogp<float><<<blocks, kBlock, 0, st>>>((const float*)ctx->val, ctx->nnz, part);
  else k_plogp<double><<<blocks, kBlock, 0, st>>>((const double*)ctx->val, ctx->nnz, part);
  FITSNE_CHECK_LAUNCH();
  k_fold2<<<1, 32, 0, st>>>(part, blocks, sc + 4);
  FITSNE_CHECK_LAUNCH();
  FITSNE_CUDA(cudaMemcpyAsync(ctx->h_scal + 4, sc + 4, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  FITSNE_CUDA(cudaStreamSynchronize(st));
  ctx->plogp = ctx->h_scal[4];
  ctx->psum = ctx->h_scal[5];
  ctx->plogp_valid = true;
  return FITSNE_OK;
}

// ---------------------------------------------------------------------------
// step (optimizer.py:299-323)
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ int npsign(T v) { return (v > 0) - (v < 0); }

template <typename T>
__global__ void k_step(T* __restrict__ Y, const T* __restrict__ g, T* __restrict__ vel,
                       T* __restrict__ gains, int64_t m, T momentum, T lr) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  T gi = g[i], v = vel[i], gn = gains[i];
  bool agree = npsign(gi) == npsign(v);
  T vn = momentum * v - lr * gn * gi;
  vel[i] = vn;
  Y[i] = Y[i] + vn;
  T ng = agree ? gn * (T)0.8 : gn + (T)0.2;
  gains[i] = ng < (T)0.01 ? (T)0.01 : ng;
}

template <typename T>
__global__ void k_nonfinite(const T* __restrict__ x, int64_t m, int* __restrict__ flag) {
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(x[i])) bad = 1;
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

int nonfinite_count(fitsne_ctx* ctx, const void* x, int64_t count, int* out_host, cudaStream_t st) {
  FITSNE_TRY(ensure(ctx->counter, 64 * sizeof(int)));
  int* flag = (int*)ctx->counter.ptr + 1;
  FITSNE_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
  int blocks = std::min<int64_t>(nblocks(std::max<int64_t>(count, 1)), ctx->num_sms * 8);
  if (ctx->dtype == FITSNE_F32) k_nonfinite<float><<<blocks, kBlock, 0, st>>>((const float*)x, count, flag);
  else k_nonfinite<double><<<blocks, kBlock, 0, st>>>((const double*)x, count, flag);
  FITSNE_CHECK_LAUNCH();
  FITSNE_CUDA(cudaMemcpyAsync(ctx->h_status + 1, flag, sizeof(int), cudaMemcpyDeviceToHost, st));
  FITSNE_CUDA(cudaStreamSynchronize(st));
  *out_host = ctx->h_status[1];
  return FITSNE_OK;
}

int step_update(fitsne_ctx* ctx, void* Y, const void* grad, void* vel, void* gains, int64_t n,
                double momentum, double lr, cudaStream_t st) {
  int64_t m = n * ctx->dims;
  int bad = 0;
  FITSNE_TRY(nonfinite_count(ctx, grad, m, &bad, st));
  if (bad) {
    set_error("non-finite gradient");
    return FITSNE_ENONFINITE;
  }
  if (m == 0) return FITSNE_OK;
  if (ctx->dtype == FITSNE_F32)
    k_step<float><<<nblocks(m), kBlock, 0, st>>>((float*)Y, (const float*)grad, (float*)vel,
                                                 (float*)gains, m, (float)momentum, (float)lr);
  else
    k_step<double><<<nblocks(m), kBlock, 0, st>>>((double*)Y, (const double*)grad, (double*)vel,
                                                  (double*)gains, m, momentum, lr);
  FITSNE_CHECK_LAUNCH();
  return FITSNE_OK;
}

// KL = plogp + sum p log1p(d^2) + psum log Z  -> dst
__global__ void k_kl_final(const double* __restrict__ part, int n, const double* __restrict__ scal,
                           double plogp, double psum, double* __restrict__ dst) {
  __shared__ double red[32];
  double s = 0;
  for (int k = threadIdx.x; k < n; k += blockDim.x) s += part[k];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) t += red[w];
    dst[0] = plogp + t + psum * log(scal[0]);
  }
}

// ---------------------------------------------------------------------------
// Overlapped schedule.  The attractive SpMV does not depend on the grid, so it
// runs on a side stream concurrently with bbox -> spread -> FFT (the SpMV is
// bound by L1/L2 gathers, the FFT stages by shared memory and issue, so they
// share SMs well).  A thread-per-point combine kernel then gathers F_rep from
// the potential grid and finishes the gradient (and, for run_tsne, the
// momentum / gains update, optimizer.py:299-323).
// ---------------------------------------------------------------------------
template <typename T, int S, int P, bool STEP>
__global__ void __launch_bounds__(kBlock)
k_combine(const T* __restrict__ Y, int64_t n, GridArgs g, const T* __restrict__ pot,
          const double* __restrict__ scal, const T* __restrict__ attr, T alpha,
          T* __restrict__ grad, T momentum, T lr, T* __restrict__ Yout, T* __restrict__ vel,
          T* __restrict__ gains, int32_t* __restrict__ status, T* __restrict__ attr_clear,
          const double* __restrict__ frep64, const GridArgs* __restrict__ gd,
          const T* __restrict__ frep_t = nullptr) {
  // frep64: F_rep precomputed by the fp64 grid pipeline (ctx->wide); frep_t:
  // F_rep gathered on the repulsion stream while the SpMV ran (gather_band);
  // else gathered here from the potentials.  gd: the device-computed grid of the
  // device-grid schedule (the block does nothing if it is not valid)
  if (gd) {
    __shared__ GridArgs s_g;
    if (threadIdx.x == 0) s_g = *gd;
    __syncthreads();
    if (s_g.status != kDevGridOk) return;
    g = s_g;
  }
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int bad = 0;
  if (i < n) {
    T yi[S], at[S];
    load_point<T, S>(Y, i, yi);
    load_point<T, S>(attr, i, at);
    if (attr_clear) {  // consume-and-clear the tiled SpMV's accumulator
#pragma unroll
      for (int d = 0; d < S; ++d) attr_clear[i * S + d] = (T)0;
    }
    T phi[4] = {0, 0, 0, 0};
    if (!frep64 && !frep_t) point_gather<T, S, P>(yi, g, pot, phi);
    const T Z = (T)scal[0];
#pragma unroll
    for (int d = 0; d < S; ++d) {
      const int64_t o = i * S + d;
      const T fr = frep_t ? frep_t[o] : (frep64 ? (T)frep64[o] : frep_from_phi<T, S>(yi, phi, Z, d, g));
      const T gd = (T)4 * (alpha * at[d] - fr);
      if (!STEP) {
        grad[o] = gd;
      } else {
        if (!isfinite(gd)) bad |= 1;
        const T v = vel[o], gn = gains[o];
        const bool agree = npsign(gd) == npsign(v);
        const T vn = momentum * v - lr * gn * gd;
        const T ynew = yi[d] + vn;
        if (!isfinite(ynew)) bad |= 2;
        vel[o] = vn;
        Yout[o] = ynew;
        const T ng = agree ? gn * (T)0.8 : gn + (T)0.2;
        gains[o] = ng < (T)0.01 ? (T)0.01 : ng;
      }
    }
  }
  if (STEP) {
    bad = __syncthreads_or(bad);
    if (bad && threadIdx.x == 0 && status) atomicOr(status, bad);
  }
}

// The combine when F_rep was gathered beside the SpMV: a pure stream over the
// points, grad = 4 (alpha F_attr - F_rep), F_attr cleared for the next pass.
// 4 points (float2 each) per thread in flight.
__global__ void __launch_bounds__(256)
k_finish_stream(float2* __restrict__ attr, const float2* __restrict__ frep, int64_t n, float alpha,
                float2* __restrict__ grad, int clear) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    float2 a[4], f[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = attr[i + u * stride];
      f[u] = __ldg(frep + i + u * stride);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      grad[i + u * stride] = make_float2(4.f * (alpha * a[u].x - f[u].x), 4.f * (alpha * a[u].y - f[u].y));
      if (clear) attr[i + u * stride] = make_float2(0.f, 0.f);
    }
  }
  for (; i < n; i += stride) {
    const float2 a = attr[i], f = frep[i];
    grad[i] = make_float2(4.f * (alpha * a.x - f.x), 4.f * (alpha * a.y - f.y));
    if (clear) attr[i] = make_float2(0.f, 0.f);
  }
}

// The repulsion pipeline runs on a HIGH-priority internal stream: the SpMV's
// thousands of blocks would otherwise be dispatched before the bbox / FFT
// blocks queued behind them and the overlap would collapse.
static int side_stream(fitsne_ctx* ctx) {
  if (ctx->side) return FITSNE_OK;
  int lo = 0, hi = 0;
  FITSNE_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  FITSNE_CUDA(cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking,
                                           ctx->overlap == 2 ? hi : lo));
  FITSNE_CUDA(cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming));
  FITSNE_CUDA(cudaEventCreateWithFlags(&ctx->ev_done, cudaEventDisableTiming));
  return FITSNE_OK;
}

template <typename T, bool STEP>
static int launch_combine(fitsne_ctx* ctx, const void* Y, int64_t n, const void* attr, double alpha,
                          void* grad, double momentum, double lr, void* Yout, void* vel,
                          void* gains, int32_t* status, bool clear, cudaStream_t st,
                          const GridArgs* gd = nullptr, size_t frep_off = 0) {
  const GridArgs g = gd ? GridArgs{} : grid_args(ctx->grid);
  const int blocks = nblocks(n);
  double* frep64 = nullptr;
  // F_rep already gathered beside the SpMV (frep_off: byte offset of this point range)
  const T* frep_t = (!gd && ctx->frep_ready && sizeof(T) == 4)
                        ? (const T*)((const unsigned char*)ctx->frep32.ptr + frep_off) : nullptr;
  if (!gd && ctx->wide && !frep_t) FITSNE_TRY(shadow_frep(ctx, Y, n, &frep64, st));
  if constexpr (!STEP && sizeof(T) == 4) {
    if (frep_t && ctx->dims == 2) {
      const int sblocks = (int)std::min<int64_t>((n + 1023) / 1024, 4 * (int64_t)ctx->num_sms);
      k_finish_stream<<<std::max(sblocks, 1), 256, 0, st>>>((float2*)attr, (const float2*)frep_t, n, (float)alpha,
                                                          (float2*)grad, clear ? 1 : 0);
      FITSNE_CHECK_LAUNCH();
      if (clear) tiled_consumed(ctx);
      return FITSNE_OK;
    }
  }
#define CMB(S, P)                                                                              \
  k_combine<T, S, P, STEP><<<blocks, kBlock, 0, st>>>(                                         \
      (const T*)Y, n, g, (const T*)ctx->pot.ptr, (const double*)ctx->scal.ptr, (const T*)attr, \
      (T)alpha, (T*)grad, (T)momentum, (T)lr, (T*)Yout, (T*)vel, (T*)gains, status,            \
      clear ? (T*)attr : (T*)nullptr, frep64, gd, frep_t)
  const int pp = gd ? ctx->p : g.p;  // a device grid has the context's p
  if (ctx->dims == 1) { if (pp == 3) CMB(1, 3); else CMB(1, 0); }
  else { if (pp == 3) CMB(2, 3); else CMB(2, 0); }
#undef CMB
  FITSNE_CHECK_LAUNCH();
  if (clear) tiled_consumed(ctx);
  return FITSNE_OK;
}

int join_on_error(fitsne_ctx* ctx, int rc) {
  if (rc == FITSNE_OK) return rc;
  for (cudaStream_t s : {ctx->side, ctx->hp, ctx->out})
    if (s) cudaStreamSynchronize(s);
  return rc;
}

// Attractive SpMV feeding the combine kernel: the tiled kernel when it applies
// (its accumulator is cleared by the combine), else the CSR kernel into
// ctx->forces.  KL partials are left in ctx->kl_part / kl_nparts.
static int spmv_for_combine(fitsne_ctx* ctx, const void* Y, bool kl, cudaStream_t st, void** attr,
                            bool* clear) {
  if (tiled_usable(ctx, Y, st)) {
    double* part = nullptr;
    int np = 0;
    FITSNE_TRY(attract_tiled(ctx, Y, kl, st, attr, &part, &np));
    ctx->kl_part = part;
    ctx->kl_nparts = np;
    *clear = true;
    ctx->spmv_tiled_live = true;
    return FITSNE_OK;
  }
  ctx->spmv_tiled_live = false;
  FITSNE_TRY(ensure(ctx->forces, dsize(ctx->dtype) * (size_t)ctx->n_total * ctx->dims));
  *attr = ctx->forces.ptr;
  *clear = false;
  return attractive(ctx, Y, nullptr, 1.0, *attr, 0, kl, st, false);
}

// Copy-out stream, per-piece events and the high-priority SpMV-piece stream
// of the host-buffer gradient (created on first use).  The pieces' stream is
// high priority: when piece q drains, the block scheduler hands the freed
// SMs to piece q + 1 before the pending spread / FFT blocks.
static int out_stream(fitsne_ctx* ctx) {
  if (ctx->out) return FITSNE_OK;
  int lo = 0, hi = 0;
  FITSNE_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  FITSNE_CUDA(cudaStreamCreateWithPriority(&ctx->hp, cudaStreamNonBlocking, hi));
  FITSNE_CUDA(cudaStreamCreateWithFlags(&ctx->out, cudaStreamNonBlocking));
  for (cudaEvent_t& e : ctx->ev_piece) FITSNE_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  FITSNE_CUDA(cudaEventCreateWithFlags(&ctx->ev_out, cudaEventDisableTiming));
  return FITSNE_OK;
}

// ---------------------------------------------------------------------------
// Device-grid schedule.  The grid (n_intervals, hence the FFT length) depends
// on the data (nbody.py:134), so the host used to wait for a 40-byte bbox
// readback before it could launch the spread and FFT stages -- ~25 us on the
// repulsion chain, which ends after the SpMV.  Here k_bbox computes the grid
// on the device with the host's formulas and the spread / FFT / combine
// stages, launched at once for a capacity (the previous grid's n_intervals +
// 8), read it from device memory.  The host still reads the box back, but
// after everything is queued, to check the device grid against its own and
// to handle the rare case the capacity was too small (or the grid needs the
// fp64 / non-band pipeline): the device stages then did nothing and the host
// path runs behind them.
// ---------------------------------------------------------------------------
static bool devgrid_applicable(const fitsne_ctx* ctx) {
  return ctx->devgrid && ctx->dg_cap_nint > 0 && ctx->dtype == FITSNE_F32 && ctx->dims == 2 && ctx->p == 3 &&
         (ctx->sorted_spread == 1 || ctx->sorted_spread == 3) && ctx->grid_f64 != 2 && ctx->fft_path != 2 &&
         ctx->n_total < (1LL << 31);
}

// n_intervals capacity for the next call after a grid g (0: the device path
// does not apply to grids like g: wide, too many box rows, long FFT)
static int devgrid_capacity(const fitsne_ctx* ctx, const fitsne_grid& g) {
  if (ctx->dtype != FITSNE_F32 || ctx->dims != 2 || g.points_per_interval != 3) return 0;
  double widest = 0;
  for (int d = 0; d < g.dims; ++d) widest = std::max(widest, g.hi[d] - g.lo[d]);
  if (ctx->grid_f64 == 1 && widest > kWideSpan) return 0;
  const int cap = std::min(1024, g.n_intervals + 8);
  if (smooth23_at_least(2 * 3 * cap - 1) > 5184) return 0;
  return cap;
}

static inline int cap_L(int cap_nint) { return smooth23_at_least(2 * 3 * cap_nint - 1); }

// Queues bbox (side), the SpMV (st, via spmv()), then the repulsion chain on
// the side stream; st waits for the chain.  *gd = the device grid when the
// device-grid schedule was used (the caller passes it to the combine and
// calls devgrid_finish after queueing it), else null (host path, grid known).
template <typename SpmvFn>
static int repulsion_beside_spmv(fitsne_ctx* ctx, const void* Y, int64_t n, cudaStream_t st, SpmvFn spmv,
                                 const GridArgs** gd) {
  *gd = nullptr;
  ctx->frep_ready = false;
  ctx->spmv_tiled_live = false;
  FITSNE_TRY(side_stream(ctx));
  FITSNE_CUDA(cudaEventRecord(ctx->ev_in, st));
  FITSNE_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_in, 0));
  if (devgrid_applicable(ctx)) {
    const int cap = ctx->dg_cap_nint, n_cap = 3 * cap, L_cap = cap_L(cap);
    FITSNE_TRY(ensure(ctx->dgrid, sizeof(DevGrid)));
    if (!ctx->h_dgrid) FITSNE_CUDA(cudaMallocHost(&ctx->h_dgrid, sizeof(DevGrid)));
    FITSNE_TRY(out_stream(ctx));
    GridArgs* dg = (GridArgs*)ctx->dgrid.ptr;
    DevGridReq rq;
    rq.min_intervals = ctx->min_intervals;
    rq.p = ctx->p;
    rq.ipi = ctx->intervals_per_integer;
    rq.cap_nint = cap;
    rq.cap_L = L_cap;
    rq.max_nint = 1024;
    rq.wide_span = ctx->grid_f64 == 1 ? kWideSpan : 0.0;
    rq.zero = band_counters(ctx, n, &rq.zero_words);
    FITSNE_TRY(device_plan_table(ctx, 65536, &rq.plans, &rq.nplans));
    if (!rq.zero) { set_error("device allocation failed"); return FITSNE_ENOMEM; }
    FITSNE_TRY(bbox_launch_devgrid(ctx, Y, n, dg, rq, ctx->h_dgrid, ctx->side, ctx->out, ctx->ev_piece[0]));
    FITSNE_TRY(spmv());
    FITSNE_TRY(ensure_accum_nodes(ctx, (size_t)n_cap * n_cap, ctx->side));
    FITSNE_TRY(spread_band(ctx, Y, n, ctx->accum.ptr, ctx->side, dg));
    FITSNE_TRY(fft_tsne_dev(ctx, ctx->accum.ptr, n, dg, n_cap, L_cap, ctx->side));
    ctx->accum_live_reps = 1;  // consumed and cleared by the FFT stage (or untouched)
    *gd = dg;
  } else {
    // mode 4: the SpMV is dispatched first and the bbox runs on the SMs it leaves
    if (ctx->overlap == 4) FITSNE_TRY(spmv());
    FITSNE_TRY(bbox_launch(ctx, Y, n, ctx->side));
    if (ctx->overlap != 4) FITSNE_TRY(spmv());
    FITSNE_TRY(make_grid_finish(ctx, ctx->side));
    FITSNE_TRY(spectrum_ahead(ctx, ctx->side));  // kernel spectrum beside the spread
    FITSNE_TRY(spread_tsne(ctx, Y, n, nullptr, ctx->side));
    FITSNE_TRY(fft_tsne(ctx, nullptr, n, false, ctx->side));
    if (ctx->side_gather && ctx->band_sorted && ctx->band_n == n && !ctx->wide && ctx->dtype == FITSNE_F32) {
      // F_rep gathered here, in the band spread's box order, while the SpMV
      // still runs: the combine after the SpMV is then a pure stream
      FITSNE_TRY(ensure(ctx->frep32, sizeof(float) * 2 * (size_t)n));
      FITSNE_TRY(gather_band(ctx, n, ctx->frep32.ptr, ctx->side));
      ctx->frep_ready = true;
    }
    if (ctx->spmv_join && ctx->spmv_tiled_live) {
      // the chain is done: its SMs join the SpMV's dynamic schedule
      int np = ctx->kl_nparts;
      FITSNE_TRY(attract_tiled_join(ctx, Y, -1, ctx->side, &np));
      ctx->kl_nparts = np;
    }
    const int cap = devgrid_capacity(ctx, ctx->grid);
    ctx->dg_cap_nint = cap;
  }
  FITSNE_CUDA(cudaEventRecord(ctx->ev_done, ctx->side));
  FITSNE_CUDA(cudaStreamWaitEvent(st, ctx->ev_done, 0));
  return FITSNE_OK;
}

// After the device-grid stages and their consumers are queued: read the box,
// derive the host grid, check the device one; on a capacity miss queue the
// host-grid chain (*fallback = true: the caller re-queues its consumers).
static int devgrid_finish(fitsne_ctx* ctx, const void* Y, int64_t n, cudaStream_t st, bool* fallback) {
  *fallback = false;
  FITSNE_CUDA(cudaEventSynchronize(ctx->ev_bbox));
  const int S = ctx->dims;
  const double* hb = reinterpret_cast<const DevGrid*>(ctx->h_dgrid)->bbox;
  if (hb[2 * S] != 0.0) {
    tiled_mark_dirty(ctx, st);  // the skipped combine did not clear F_attr
    set_error("points must be finite");
    return FITSNE_EPOINTS;
  }
  double bbox[4];
  for (int d = 0; d < 2 * S; ++d) bbox[d] = hb[d];
  fitsne_grid g;
  FITSNE_TRY(grid_from_bbox(ctx, bbox, &g));
  const GridArgs& dgh = *ctx->h_dgrid;
  if (dgh.status == kDevGridOk) {
    bool same = dgh.n_int == g.n_intervals && dgh.L == g.fft_len && dgh.n == g.nodes_per_dim;
    for (int d = 0; d < g.dims; ++d) same = same && dgh.lo[d] == g.lo[d] && dgh.hi[d] == g.hi[d] && dgh.h[d] == g.spacing[d];
    if (!same) {
      set_error("device grid differs from the host grid formulas");
      return FITSNE_ECUDA;
    }
    ctx->grid = g;
    ctx->grid_valid = true;
    ctx->wide = false;
    if (g.n_intervals + 4 > ctx->dg_cap_nint) ctx->dg_cap_nint = devgrid_capacity(ctx, g);
    return FITSNE_OK;
  }
  // the device stages skipped: run the host-grid chain behind them
  *fallback = true;
  ++ctx->dg_fallbacks;
  FITSNE_TRY(install_grid(ctx, g, ctx->side));
  FITSNE_TRY(spread_tsne(ctx, Y, n, nullptr, ctx->side));
  FITSNE_TRY(fft_tsne(ctx, nullptr, n, false, ctx->side));
  FITSNE_CUDA(cudaEventRecord(ctx->ev_done, ctx->side));
  FITSNE_CUDA(cudaStreamWaitEvent(st, ctx->ev_done, 0));
  ctx->dg_cap_nint = devgrid_capacity(ctx, g);
  return FITSNE_OK;
}

static int gradient_overlapped_impl(fitsne_ctx* ctx, const void* Y, double alpha, void* grad,
                                    cudaStream_t st, void* grad_host);

int gradient_overlapped(fitsne_ctx* ctx, const void* Y, double alpha, void* grad, cudaStream_t st,
                        void* grad_host) {
  return join_on_error(ctx, gradient_overlapped_impl(ctx, Y, alpha, grad, st, grad_host));
}

// the gradient's combine (optionally in point ranges with overlapped copy-out)
static int queue_combine(fitsne_ctx* ctx, const void* Y, int64_t n, void* attr, bool clear, double alpha,
                         void* grad, void* grad_host, const GridArgs* gd, cudaStream_t st) {
  if (grad_host) {
    // host result: combine in point ranges, each range's device-to-host copy
    // (copy stream) overlapping the next range's combine
    FITSNE_TRY(out_stream(ctx));
    const size_t row_bytes = dsize(ctx->dtype) * (size_t)ctx->dims;
    constexpr int kParts = 4;
    for (int q = 0; q < kParts; ++q) {
      const int64_t r0 = n * q / kParts, nr = n * (q + 1) / kParts - r0;
      if (nr <= 0) continue;
      const size_t off = row_bytes * (size_t)r0;
      if (ctx->dtype == FITSNE_F32)
        FITSNE_TRY((launch_combine<float, false>(ctx, (const unsigned char*)Y + off, nr,
                                                 (unsigned char*)attr + off, alpha,
                                                 (unsigned char*)grad + off, 0, 0, nullptr, nullptr,
                                                 nullptr, nullptr, clear, st, gd, off)));
      else
        FITSNE_TRY((launch_combine<double, false>(ctx, (const unsigned char*)Y + off, nr,
                                                  (unsigned char*)attr + off, alpha,
                                                  (unsigned char*)grad + off, 0, 0, nullptr, nullptr,
                                                  nullptr, nullptr, clear, st, gd)));
      FITSNE_CUDA(cudaEventRecord(ctx->ev_piece[q], st));
      FITSNE_CUDA(cudaStreamWaitEvent(ctx->out, ctx->ev_piece[q], 0));
      FITSNE_CUDA(cudaMemcpyAsync((unsigned char*)grad_host + off, (unsigned char*)grad + off,
                                  row_bytes * (size_t)nr, cudaMemcpyDeviceToHost, ctx->out));
    }
    FITSNE_CUDA(cudaEventRecord(ctx->ev_out, ctx->out));
    FITSNE_CUDA(cudaStreamWaitEvent(st, ctx->ev_out, 0));
    return FITSNE_OK;
  }
  if (ctx->dtype == FITSNE_F32)
    return launch_combine<float, false>(ctx, Y, n, attr, alpha, grad, 0, 0, nullptr, nullptr, nullptr,
                                        nullptr, clear, st, gd);
  return launch_combine<double, false>(ctx, Y, n, attr, alpha, grad, 0, 0, nullptr, nullptr, nullptr,
                                       nullptr, clear, st, gd);
}

static int gradient_overlapped_impl(fitsne_ctx* ctx, const void* Y, double alpha, void* grad,
                                    cudaStream_t st, void* grad_host) {
  FITSNE_RANGE("gradient_schedule");
  ctx->frep_ready = false;
  const int64_t n = ctx->n_total;
  void* attr = nullptr;
  bool clear = false;
  const GridArgs* gd = nullptr;
  if (ctx->overlap == 0) {
    FITSNE_TRY(make_grid(ctx, Y, n, st));
    FITSNE_TRY(spread_tsne(ctx, Y, n, nullptr, st));
    FITSNE_TRY(fft_tsne(ctx, nullptr, n, false, st));
    FITSNE_TRY(spmv_for_combine(ctx, Y, false, st, &attr, &clear));
  } else if (ctx->overlap == 3) {
    // spread first on the whole GPU, then the SpMV with the FFT stages beside it
    FITSNE_TRY(side_stream(ctx));
    FITSNE_TRY(make_grid(ctx, Y, n, st));
    FITSNE_TRY(spread_tsne(ctx, Y, n, nullptr, st));
    FITSNE_CUDA(cudaEventRecord(ctx->ev_in, st));
    FITSNE_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_in, 0));
    FITSNE_TRY(spmv_for_combine(ctx, Y, false, st, &attr, &clear));
    FITSNE_TRY(fft_tsne(ctx, nullptr, n, false, ctx->side));
    FITSNE_CUDA(cudaEventRecord(ctx->ev_done, ctx->side));
    FITSNE_CUDA(cudaStreamWaitEvent(st, ctx->ev_done, 0));
  } else {
    // bbox kernels first on the side stream (dispatched ahead of the SpMV, so
    // they get the whole GPU for a few microseconds), then the SpMV on st,
    // then spread + FFT on the side stream, which fill the SM slots the SpMV
    // leaves (device-grid schedule: queued at once; host path: after the
    // 40-byte bbox readback)
    FITSNE_TRY(repulsion_beside_spmv(ctx, Y, n, st,
                                     [&]() { return spmv_for_combine(ctx, Y, false, st, &attr, &clear); },
                                     &gd));
  }
  FITSNE_TRY(queue_combine(ctx, Y, n, attr, clear, alpha, grad, grad_host, gd, st));
  if (gd) {
    bool fb = false;
    FITSNE_TRY(devgrid_finish(ctx, Y, n, st, &fb));
    if (fb) FITSNE_TRY(queue_combine(ctx, Y, n, attr, clear, alpha, grad, grad_host, nullptr, st));
  }
  return FITSNE_OK;
}

// Gradient with host buffers (fitsne_gradient_host).  Y is copied in on st;
// the attractive SpMV runs as kTiledPieces launches over consecutive row
// ranges on a high-priority stream while grid + spread + FFT run on the side stream; on the
// copy-out stream the combine of piece k (F_rep gather + 4 (alpha F_attr -
// F_rep)) and its device-to-host copy start as soon as SpMV piece k is done,
// so the gradient leaves the device while the later pieces still run.
static int gradient_host_impl(fitsne_ctx* ctx, const void* Y_host, double alpha, void* grad_host,
                              cudaStream_t st);

int gradient_host(fitsne_ctx* ctx, const void* Y_host, double alpha, void* grad_host, cudaStream_t st) {
  return join_on_error(ctx, gradient_host_impl(ctx, Y_host, alpha, grad_host, st));
}

static int gradient_host_impl(fitsne_ctx* ctx, const void* Y_host, double alpha, void* grad_host,
                              cudaStream_t st) {
  const int64_t n = ctx->n_total;
  ctx->frep_ready = false;
  const size_t row_bytes = dsize(ctx->dtype) * (size_t)ctx->dims;
  const size_t bytes = row_bytes * (size_t)n;
  FITSNE_TRY(ensure(ctx->hy, bytes));
  FITSNE_TRY(ensure(ctx->hg, bytes));
  void* y = ctx->hy.ptr;
  unsigned char* g = (unsigned char*)ctx->hg.ptr;
  FITSNE_CUDA(cudaMemcpyAsync(y, Y_host, bytes, cudaMemcpyHostToDevice, st));
  if (ctx->host_pieces == 2) {  // plain: gradient, then one copy-out
    FITSNE_TRY(gradient_overlapped(ctx, y, alpha, g, st));
    FITSNE_CUDA(cudaMemcpyAsync(grad_host, g, bytes, cudaMemcpyDeviceToHost, st));
    FITSNE_CUDA(cudaStreamSynchronize(st));
    return FITSNE_OK;
  }
  if (ctx->host_pieces == 0 || ctx->overlap == 0 || !tiled_usable(ctx, y, st) ||
      tiled_relabeled(ctx)) {  // row pieces are ranges of the caller's order
    // the combine runs in point ranges whose copy-out overlaps the next range
    FITSNE_TRY(gradient_overlapped(ctx, y, alpha, g, st, grad_host));
    FITSNE_CUDA(cudaStreamSynchronize(st));
    return FITSNE_OK;
  }
  FITSNE_TRY(side_stream(ctx));
  FITSNE_TRY(out_stream(ctx));
  FITSNE_CUDA(cudaEventRecord(ctx->ev_in, st));
  FITSNE_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_in, 0));
  FITSNE_CUDA(cudaStreamWaitEvent(ctx->out, ctx->ev_in, 0));
  FITSNE_CUDA(cudaStreamWaitEvent(ctx->hp, ctx->ev_in, 0));
  void* attr = nullptr;
  FITSNE_TRY(bbox_launch(ctx, y, n, ctx->side));
  for (int q = 0; q < kTiledPieces; ++q) {
    FITSNE_TRY(attract_tiled_piece(ctx, y, q, ctx->hp, &attr));
    FITSNE_CUDA(cudaEventRecord(ctx->ev_piece[q], ctx->hp));
  }
  FITSNE_TRY(make_grid_finish(ctx, ctx->side));
  FITSNE_TRY(spread_tsne(ctx, y, n, nullptr, ctx->side));
  FITSNE_TRY(fft_tsne(ctx, nullptr, n, false, ctx->side));
  FITSNE_CUDA(cudaEventRecord(ctx->ev_done, ctx->side));
  FITSNE_CUDA(cudaStreamWaitEvent(ctx->out, ctx->ev_done, 0));
  int64_t rows[kTiledPieces + 1];
  tiled_piece_rows(ctx, rows);
  for (int q = 0; q < kTiledPieces; ++q) {
    const int64_t r0 = rows[q], nr = rows[q + 1] - rows[q];
    FITSNE_CUDA(cudaStreamWaitEvent(ctx->out, ctx->ev_piece[q], 0));
    if (nr <= 0) continue;
    const size_t off = row_bytes * (size_t)r0;
    FITSNE_TRY((launch_combine<float, false>(ctx, (const unsigned char*)y + off, nr,
                                             (unsigned char*)attr + off, alpha, g + off, 0, 0,
                                             nullptr, nullptr, nullptr, nullptr, true, ctx->out)));
    FITSNE_CUDA(cudaMemcpyAsync((unsigned char*)grad_host + off, g + off, row_bytes * (size_t)nr,
                                cudaMemcpyDeviceToHost, ctx->out));
  }
  FITSNE_CUDA(cudaEventRecord(ctx->ev_out, ctx->out));
  FITSNE_CUDA(cudaStreamWaitEvent(st, ctx->ev_out, 0));
  FITSNE_CUDA(cudaStreamSynchronize(ctx->out));
  return FITSNE_OK;
}

// grad = 4 (alpha F_attr - F_rep) for m values (the sharded path's combine,
// after an F_attr computed concurrently with the repulsion stages)
template <typename T>
__global__ void k_combine_rows(const T* __restrict__ attr, const T* __restrict__ frep, int64_t m,
                               T alpha, T* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m) out[i] = (T)4 * (alpha * attr[i] - frep[i]);
}

int combine_rows(fitsne_ctx* ctx, const void* attr, const void* frep, int64_t n, double alpha,
                 void* out, cudaStream_t st) {
  const int64_t m = n * ctx->dims;
  if (m <= 0) return FITSNE_OK;
  if (ctx->dtype == FITSNE_F32)
    k_combine_rows<float><<<nblocks(m), kBlock, 0, st>>>((const float*)attr, (const float*)frep, m,
                                                        (float)alpha, (float*)out);
  else
    k_combine_rows<double><<<nblocks(m), kBlock, 0, st>>>((const double*)attr, (const double*)frep,
                                                          m, alpha, (double*)out);
  FITSNE_CHECK_LAUNCH();
  return FITSNE_OK;
}

static int iterate_fused_impl(fitsne_ctx* ctx, const void* Yin, void* Yout, void* vel, void* gains,
                              double alpha, double momentum, double lr, double* kl_dev,
                              int32_t* status_dev, cudaStream_t st);

int iterate_fused(fitsne_ctx* ctx, const void* Yin, void* Yout, void* vel, void* gains, double alpha,
                  double momentum, double lr, double* kl_dev, int32_t* status_dev, cudaStream_t st) {
  return join_on_error(ctx, iterate_fused_impl(ctx, Yin, Yout, vel, gains, alpha, momentum, lr, kl_dev,
                                               status_dev, st));
}

static int iterate_fused_impl(fitsne_ctx* ctx, const void* Yin, void* Yout, void* vel, void* gains,
                              double alpha, double momentum, double lr, double* kl_dev,
                              int32_t* status_dev, cudaStream_t st) {
  FITSNE_RANGE("iterate_schedule");
  ctx->frep_ready = false;
  const int64_t n = ctx->n_total;
  if (!ctx->plogp_valid) FITSNE_TRY(compute_plogp(ctx, st));
  void* attr = nullptr;
  bool clear = false;
  const GridArgs* gd = nullptr;
  if (ctx->overlap == 0) {
    FITSNE_TRY(make_grid(ctx, Yin, n, st));
    FITSNE_TRY(spread_tsne(ctx, Yin, n, nullptr, st));
    FITSNE_TRY(fft_tsne(ctx, nullptr, n, false, st));
    FITSNE_TRY(spmv_for_combine(ctx, Yin, kl_dev != nullptr, st, &attr, &clear));
  } else if (ctx->overlap == 3) {
    FITSNE_TRY(side_stream(ctx));
    FITSNE_TRY(make_grid(ctx, Yin, n, st));
    FITSNE_TRY(spread_tsne(ctx, Yin, n, nullptr, st));
    FITSNE_CUDA(cudaEventRecord(ctx->ev_in, st));
    FITSNE_CUDA(cudaStreamWaitEvent(ctx->side, ctx->ev_in, 0));
    FITSNE_TRY(spmv_for_combine(ctx, Yin, kl_dev != nullptr, st, &attr, &clear));
    FITSNE_TRY(fft_tsne(ctx, nullptr, n, false, ctx->side));
    FITSNE_CUDA(cudaEventRecord(ctx->ev_done, ctx->side));
    FITSNE_CUDA(cudaStreamWaitEvent(st, ctx->ev_done, 0));
  } else {
    // bbox on the side stream, SpMV + KL partials on st, spread + FFT on the
    // side stream (device-grid schedule or after the bbox readback)
    FITSNE_TRY(repulsion_beside_spmv(
        ctx, Yin, n, st, [&]() { return spmv_for_combine(ctx, Yin, kl_dev != nullptr, st, &attr, &clear); },
        &gd));
  }
  // the step's combine + update, then the KL of the pre-step embedding
  auto consumers = [&](const GridArgs* g) -> int {
    if (ctx->dtype == FITSNE_F32)
      FITSNE_TRY((launch_combine<float, true>(ctx, Yin, n, attr, alpha, nullptr, momentum, lr, Yout,
                                               vel, gains, status_dev, clear, st, g)));
    else
      FITSNE_TRY((launch_combine<double, true>(ctx, Yin, n, attr, alpha, nullptr, momentum, lr, Yout,
                                                vel, gains, status_dev, clear, st, g)));
    if (kl_dev) {
      k_kl_final<<<1, 1024, 0, st>>>(ctx->kl_part, ctx->kl_nparts, (const double*)ctx->scal.ptr,
                                    ctx->plogp, ctx->psum, kl_dev);
      FITSNE_CHECK_LAUNCH();
    }
    return FITSNE_OK;
  };
  FITSNE_TRY(consumers(gd));
  if (gd) {
    bool fb = false;
    FITSNE_TRY(devgrid_finish(ctx, Yin, n, st, &fb));
    if (fb) FITSNE_TRY(consumers(nullptr));
  }
  return FITSNE_OK;
}

// ---------------------------------------------------------------------------
// exact O(N^2) sums (optimizer.py:169-190): k1_i = sum_{j!=i} q_ij,
// k2_i = sum_{j!=i} q_ij^2 (y_j, 1), q_ij = 1/(1+d^2)
// ---------------------------------------------------------------------------
template <typename T, int S>
__global__ void k_exact(const T* __restrict__ Y, int64_t n, T* __restrict__ k1, T* __restrict__ k2) {
  constexpr int TILE = 256;
  __shared__ T ys[TILE * S];
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  T yi[S];
#pragma unroll
  for (int d = 0; d < S; ++d) yi[d] = (i < n) ? Y[i * S + d] : (T)0;
  double a1 = 0, a2[S + 1];
#pragma unroll
  for (int d = 0; d <= S; ++d) a2[d] = 0;
  for (int64_t t0 = 0; t0 < n; t0 += TILE) {
    __syncthreads();
    for (int k = threadIdx.x; k < TILE * S; k += blockDim.x) {
      int64_t j = t0 + k / S;
      ys[k] = (j < n) ? Y[j * S + (k % S)] : (T)0;
    }
    __syncthreads();
    int lim = (n - t0 < TILE) ? (int)(n - t0) : TILE;
    if (i < n) {
      for (int jj = 0; jj < lim; ++jj) {
        int64_t j = t0 + jj;
        if (j == i) continue;
        T d2 = 0;
#pragma unroll
        for (int d = 0; d < S; ++d) {
          T df = yi[d] - ys[jj * S + d];
          d2 += df * df;
        }
        T a = (T)1 / ((T)1 + d2);
        T b = a * a;
        a1 += (double)a;
#pragma unroll
        for (int d = 0; d < S; ++d) a2[d] += (double)(b * ys[jj * S + d]);
        a2[S] += (double)b;
      }
    }
  }
  if (i < n) {
    k1[i] = (T)a1;
#pragma unroll
    for (int d = 0; d <= S; ++d) k2[i * (S + 1) + d] = (T)a2[d];
  }
}

template <typename T>
__global__ void k_sum(const T* __restrict__ x, int64_t n, double* __restrict__ dst) {
  // single block deterministic sum
  __shared__ double red[32];
  double s = 0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) s += (double)x[k];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) t += red[w];
    dst[0] = t;
  }
}

int exact_sums(fitsne_ctx* ctx, const void* Y, int64_t n, void* k1, void* k2, cudaStream_t st) {
  FITSNE_TRY(ensure(ctx->scal, 64 * sizeof(double)));
  if (ctx->dtype == FITSNE_F32) {
    if (ctx->dims == 1) k_exact<float, 1><<<nblocks(n), 256, 0, st>>>((const float*)Y, n, (float*)k1, (float*)k2);
    else k_exact<float, 2><<<nblocks(n), 256, 0, st>>>((const float*)Y, n, (float*)k1, (float*)k2);
    FITSNE_CHECK_LAUNCH();
    k_sum<float><<<1, 1024, 0, st>>>((const float*)k1, n, (double*)ctx->scal.ptr);
  } else {
    if (ctx->dims == 1) k_exact<double, 1><<<nblocks(n), 256, 0, st>>>((const double*)Y, n, (double*)k1, (double*)k2);
    else k_exact<double, 2><<<nblocks(n), 256, 0, st>>>((const double*)Y, n, (double*)k1, (double*)k2);
    FITSNE_CHECK_LAUNCH();
    k_sum<double><<<1, 1024, 0, st>>>((const double*)k1, n, (double*)ctx->scal.ptr);
  }
  FITSNE_CHECK_LAUNCH();
  return FITSNE_OK;
}

// forces = (y * k2[:, s] - k2[:, :s]) / Z   (optimizer.py:244)
template <typename T, int S>
__global__ void k_forces(const T* __restrict__ Y, int64_t n, const T* __restrict__ k2,
                         const double* __restrict__ scal, T* __restrict__ f) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  T z = (T)scal[0];
#pragma unroll
  for (int d = 0; d < S; ++d) f[i * S + d] = (Y[i * S + d] * k2[i * (S + 1) + S] - k2[i * (S + 1) + d]) / z;
}

int forces_from_sums(fitsne_ctx* ctx, const void* Y, int64_t n, const void* k2, void* forces,
                     cudaStream_t st) {
  const double* sc = (const double*)ctx->scal.ptr;
  if (ctx->dtype == FITSNE_F32) {
    if (ctx->dims == 1) k_forces<float, 1><<<nblocks(n), kBlock, 0, st>>>((const float*)Y, n, (const float*)k2, sc, (float*)forces);
    else k_forces<float, 2><<<nblocks(n), kBlock, 0, st>>>((const float*)Y, n, (const float*)k2, sc, (float*)forces);
  } else {
    if (ctx->dims == 1) k_forces<double, 1><<<nblocks(n), kBlock, 0, st>>>((const double*)Y, n, (const double*)k2, sc, (double*)forces);
    else k_forces<double, 2><<<nblocks(n), kBlock, 0, st>>>((const double*)Y, n, (const double*)k2, sc, (double*)forces);
  }
  FITSNE_CHECK_LAUNCH();
  return FITSNE_OK;
}

// brute_force_nbody (nbody.py:402-419): out[i, c] = sum_j K(d2_ij) q[j, c]
template <typename T, int S>
__global__ void k_exact_nbody(const T* __restrict__ Y, int64_t n, const T* __restrict__ q, int nq,
                              int kern, int include_self, T* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  T yi[S];
#pragma unroll
  for (int d = 0; d < S; ++d) yi[d] = Y[i * S + d];
  for (int c = 0; c < nq; ++c) {
    double acc = 0;
    for (int64_t j = 0; j < n; ++j) {
      double d2 = 0;
#pragma unroll
      for (int d = 0; d < S; ++d) {
        double df = (double)yi[d] - (double)Y[j * S + d];
        d2 += df * df;
      }
      double b = 1.0 / (1.0 + d2);
      if (kern == FITSNE_CAUCHY_SQUARED) b = b * b;
      acc += b * (double)q[j * nq + c];
    }
    if (!include_self) acc -= (double)q[i * nq + c];
    out[i * nq + c] = (T)acc;
  }
}

int exact_nbody(fitsne_ctx* ctx, const void* Y, int64_t n, const void* q, int nq, int kernel,
                int include_self, void* out, cudaStream_t st) {
  if (n <= 0 || nq <= 0) return FITSNE_OK;
  if (ctx->dtype == FITSNE_F32) {
    if (ctx->dims == 1) k_exact_nbody<float, 1><<<nblocks(n), kBlock, 0, st>>>((const float*)Y, n, (const float*)q, nq, kernel, include_self, (float*)out);
    else k_exact_nbody<float, 2><<<nblocks(n), kBlock, 0, st>>>((const float*)Y, n, (const float*)q, nq, kernel, include_self, (float*)out);
  } else {
    if (ctx->dims == 1) k_exact_nbody<double, 1><<<nblocks(n), kBlock, 0, st>>>((const double*)Y, n, (const double*)q, nq, kernel, include_self, (double*)out);
    else k_exact_nbody<double, 2><<<nblocks(n), kBlock, 0, st>>>((const double*)Y, n, (const double*)q, nq, kernel, include_self, (double*)out);
  }
  FITSNE_CHECK_LAUNCH();
  return FITSNE_OK;
}

template <typename T>
__global__ void k_sub(T* __restrict__ out, const T* __restrict__ q, int64_t m) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m) out[i] -= q[i];
}

// out -= q (self-term removal, K(y, y) = 1: nbody.py:374-375)
int sub_inplace(fitsne_ctx* ctx, void* out, const void* q, int64_t count, cudaStream_t st) {
  if (count <= 0) return FITSNE_OK;
  if (ctx->dtype == FITSNE_F32) k_sub<float><<<nblocks(count), kBlock, 0, st>>>((float*)out, (const float*)q, count);
  else k_sub<double><<<nblocks(count), kBlock, 0, st>>>((double*)out, (const double*)q, count);
  FITSNE_CHECK_LAUNCH();
  return FITSNE_OK;
}

int read_scalars(fitsne_ctx* ctx, int count, cudaStream_t st) {
  FITSNE_CUDA(cudaMemcpyAsync(ctx->h_scal, ctx->scal.ptr, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
  FITSNE_CUDA(cudaStreamSynchronize(st));
  return FITSNE_OK;
}

}  // namespace fitsne
