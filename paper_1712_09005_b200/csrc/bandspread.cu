// Band spread: the t-SNE charge spreading (_spread, nbody.py:233-251; the
// unit, y_0 and y_1 charges of _fft_repulsion_sums, optimizer.py:206-210) for
// fp32 2-D embeddings with p = 3, built for running beside the attractive
// SpMV on the few SMs it leaves free.
//
// A direct scatter issues 9 vector reductions per point (one per node), each
// a separate L2 transaction: on ~20 SMs that is LSU-bound (~1 transaction per
// clock per SM) and took ~340 us at N = 1.3M.  Here the points are first
// binned by box row (the x cell) with a counting sort whose histograms live
// in shared memory (<= 864 bins: one global write per bin and block), so a
// block of the reduce pass sees a contiguous piece of one or a few box rows.
// It counting-sorts its piece again by box inside shared memory (key = row
// offset x n_int + y cell, native 32-bit shared atomics), and each thread then
// walks 8 consecutive sorted points, summing the 9 x 3 node contributions of
// a box in registers and flushing one vector reduction per node when the box
// changes.  Crowded boxes -- the case that serialises direct atomics -- cost
// ~1 transaction per node per 8 points.
//
// Cells and weights come from box_weights3_f32 exactly as in k_spread_tsne
// (bit-exact cells); only the summation order differs.
#include <mutex>
#include <set>

#include "common.cuh"
#include "internal.h"
#include "interp.cuh"

namespace fitsne {

#ifndef FITSNE_BAND_BLOCK
#define FITSNE_BAND_BLOCK 256
#endif
#ifndef FITSNE_BAND_KEYS
#define FITSNE_BAND_KEYS 2048
#endif
static constexpr int kBandBlock = FITSNE_BAND_BLOCK;
static constexpr int kBandPts = 4096;                 // points per count / scatter block
static constexpr int kBandChunk = 2048;               // sorted points per reduce block
static constexpr int kBandRun = kBandChunk / kBandBlock;  // sorted points per reduce thread
#ifndef FITSNE_BAND_CROWD
#define FITSNE_BAND_CROWD 4
#endif
static constexpr int kBandCrowd = FITSNE_BAND_CROWD;  // distinct boxes per warp up to which the warp reduces before flushing
static constexpr int kBandKeys = FITSNE_BAND_KEYS;    // (box rows in a chunk) x n_int; 2048 keeps 4 blocks / SM
static constexpr int kBandMaxRows = 1024;             // n_int bound (fp32: n_int <= 864)
static constexpr int kBandSmem = kBandChunk * 16 + kBandKeys * 4 + kBandChunk * 4;

// device-grid schedule: the stage reads the grid k_bbox computed (gd) and
// does nothing when that grid is not for it (status != 0; the host falls back)
__device__ __forceinline__ bool dev_grid(GridArgs& g, const GridArgs* __restrict__ gd) {
  if (!gd) return true;
  __shared__ GridArgs s_g;
  if (threadIdx.x == 0) s_g = *gd;
  __syncthreads();
  g = s_g;
  return g.status == kDevGridOk;
}

__device__ __forceinline__ int band_cell(float y, const GridArgs& g, int d, float* w) {
  return box_weights3_f32(y, g.lo[d], g.h[d], g.lo_f[d], g.invh_f[d], g.guard[d], g.n_int, w);
}

// cell and offset u (the same arithmetic as box_weights3_f32, which derives
// its three weights from u), so the reduce pass can keep u instead of
// recomputing the cell
__device__ __forceinline__ int band_cell_u(float x, const GridArgs& g, int d, float* u_out) {
  const float t = (x - g.lo_f[d]) * g.invh_f[d];
  const float r = t * (1.0f / 3.0f);
  const float q = floorf(r);
  const float fr = r - q;
  int c;
  float u;
  if (fr > g.guard[d] && fr < 1.0f - g.guard[d] && t >= 0.0f) {
    c = (int)q;
    if (c > g.n_int - 1) c = g.n_int - 1;
    u = t - (float)(3 * c) - 0.5f;
  } else {
    double wd[3];
    c = box_weights((double)x, g.lo[d], g.h[d], g.n_int, 3, wd);
    const double td = __ddiv_rn(__dsub_rn((double)x, g.lo[d]), g.h[d]);
    u = (float)__dsub_rn(__dsub_rn(td, (double)(c * 3)), 0.5);
  }
  *u_out = u;
  return c;
}

// box_weights3_f32's weights from u
__device__ __forceinline__ void band_weights(float u, float* w) {
  const float d1 = u - 1.0f, d2 = u - 2.0f;
  w[0] = 0.5f * d1 * d2;
  w[1] = -u * d2;
  w[2] = 0.5f * u * d1;
}

// Two-pass binning by box row without a device-wide scan: pass 1 adds each
// block's row histogram into global row totals; pass 2 recomputes its
// histogram, takes the exclusive scan of the (<= 1024) row totals in shared
// memory, reserves a contiguous range inside each of its rows with one atomic
// per (block, row), and scatters.  (The order of blocks inside a row is
// arbitrary; the reduce pass sorts each piece by box anyway, and the grid
// accumulation is an unordered sum of float reductions already.)
__global__ void __launch_bounds__(kBandBlock)
k_band_rowcount(const float2* __restrict__ Y, int64_t n, GridArgs g, uint32_t* __restrict__ rowtot,
                const GridArgs* __restrict__ gd) {
  if (!dev_grid(g, gd)) return;
  __shared__ uint32_t hist[kBandMaxRows];
  for (int r = threadIdx.x; r < g.n_int; r += kBandBlock) hist[r] = 0;
  __syncthreads();
  const int64_t p0 = blockIdx.x * (int64_t)kBandPts;
  const int64_t p1 = min(n, p0 + kBandPts);
  for (int64_t i = p0 + threadIdx.x; i < p1; i += kBandBlock) {
    float w[3];
    atomicAdd(&hist[band_cell(Y[i].x, g, 0, w)], 1u);
  }
  __syncthreads();
  for (int r = threadIdx.x; r < g.n_int; r += kBandBlock)
    if (hist[r]) atomicAdd(rowtot + r, hist[r]);
}

__global__ void __launch_bounds__(kBandBlock)
k_band_place(const float2* __restrict__ Y, int64_t n, GridArgs g, const uint32_t* __restrict__ rowtot,
             uint32_t* __restrict__ rowcur, float2* __restrict__ sorted, uint32_t* __restrict__ sidx,
             const GridArgs* __restrict__ gd) {
  if (!dev_grid(g, gd)) return;
  __shared__ uint32_t hist[kBandMaxRows];
  __shared__ uint32_t start[kBandMaxRows];
  __shared__ uint32_t part[kBandBlock];
  const int ni = g.n_int, tid = threadIdx.x;
  for (int r = tid; r < ni; r += kBandBlock) hist[r] = 0;
  __syncthreads();
  const int64_t p0 = blockIdx.x * (int64_t)kBandPts;
  const int64_t p1 = min(n, p0 + kBandPts);
  for (int64_t i = p0 + tid; i < p1; i += kBandBlock) {
    float w[3];
    atomicAdd(&hist[band_cell(Y[i].x, g, 0, w)], 1u);
  }
  // exclusive scan of the row totals: kBandMaxRows / kBandBlock per thread
  constexpr int E = kBandMaxRows / kBandBlock;
  uint32_t loc[E], run = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int r = tid * E + e;
    loc[e] = run;
    run += r < ni ? rowtot[r] : 0u;
  }
  part[tid] = run;
  __syncthreads();
  if (tid < 32) {
    uint32_t v[kBandBlock / 32], t = 0;
#pragma unroll
    for (int j = 0; j < kBandBlock / 32; ++j) {
      v[j] = part[tid * (kBandBlock / 32) + j];
      t += v[j];
    }
    uint32_t x = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if ((tid & 31) >= o) x += y;
    }
    uint32_t ex = x - t;
#pragma unroll
    for (int j = 0; j < kBandBlock / 32; ++j) {
      const uint32_t vj = v[j];
      part[tid * (kBandBlock / 32) + j] = ex;
      ex += vj;
    }
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) start[tid * E + e] = loc[e] + part[tid];
  __syncthreads();
  // this block's range inside each row it touches
  for (int r = tid; r < ni; r += kBandBlock)
    if (hist[r]) hist[r] = start[r] + atomicAdd(rowcur + r, hist[r]);
  __syncthreads();
  for (int64_t i = p0 + tid; i < p1; i += kBandBlock) {
    const float2 y = Y[i];
    float w[3];
    const uint32_t at = atomicAdd(&hist[band_cell(y.x, g, 0, w)], 1u);
    FITSNE_DCHECK(at < n);
    sorted[at] = y;
    sidx[at] = (uint32_t)i;
  }
}

// 9 vector reductions of one box's (or one point's) 27 node sums
__device__ __forceinline__ void band_flush(float* __restrict__ acc, int nn, int cx, int cy,
                                           const float (&s)[3][3][3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const int64_t rowbase = ((int64_t)cx * 3 + a) * nn + (int64_t)cy * 3;
#pragma unroll
    for (int b = 0; b < 3; ++b)
      atomicAdd(reinterpret_cast<float4*>(acc + (rowbase + b) * kNodeSlots),
                make_float4(s[a][b][0], s[a][b][1], s[a][b][2], 0.f));
  }
}

// reduce pass over the box-row-sorted points: in-block counting sort by box,
// then per-thread runs of kBandRun sorted points with one flush per box
__global__ void __launch_bounds__(kBandBlock)
k_band_reduce(const float2* __restrict__ ys, const uint32_t* __restrict__ sidx, int64_t n, GridArgs g,
              float* __restrict__ acc, float2* __restrict__ bs_pts, uint32_t* __restrict__ bs_idx,
              const GridArgs* __restrict__ gd) {
  // bs_pts / bs_idx: the chunk's points and original indices in box order,
  // kept for the box-ordered gather of F_rep (k_band_gather)
  if (!dev_grid(g, gd)) return;
  // dynamic shared memory (kBandSmem bytes): hist, points, (u_x, u_y), order, keys
  extern __shared__ __align__(16) unsigned char band_smem[];
  float2* pts = reinterpret_cast<float2*>(band_smem);
  float2* uvs = pts + kBandChunk;
  uint32_t* hist = reinterpret_cast<uint32_t*>(uvs + kBandChunk);
  uint16_t* order = reinterpret_cast<uint16_t*>(hist + kBandKeys);
  uint16_t* keyof = order + kBandChunk;
  __shared__ uint32_t part[kBandBlock];
  __shared__ int s_cx0, s_direct;
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t c0 = blockIdx.x * (int64_t)kBandChunk;
  const int cnt = (int)min((int64_t)kBandChunk, n - c0);
  const int nn = g.n, ni = g.n_int;
  if (tid == 0) {
    float w[3];
    const int a = band_cell(ys[c0].x, g, 0, w);
    const int b = band_cell(ys[c0 + cnt - 1].x, g, 0, w);
    s_cx0 = a;
    s_direct = (b - a + 1) * ni > kBandKeys;  // piece spans too many rows: direct scatter
  }
  for (int k = tid; k < kBandKeys; k += kBandBlock) hist[k] = 0;
  __syncthreads();
  const int cx0 = s_cx0;
  if (s_direct) {
    for (int k = tid; k < cnt; k += kBandBlock) {
      const float2 y = ys[c0 + k];
      float wx[3], wy[3], s[3][3][3];
      const int cx = band_cell(y.x, g, 0, wx), cy = band_cell(y.y, g, 1, wy);
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const float w = wx[a] * wy[b];
          s[a][b][0] = w;
          s[a][b][1] = w * (y.x - g.cf[0]);
          s[a][b][2] = w * (y.y - g.cf[1]);
        }
      band_flush(acc, nn, cx, cy, s);
      bs_pts[c0 + k] = y;
      bs_idx[c0 + k] = sidx[c0 + k];
    }
    return;
  }
  // keys + histogram (shared atomics)
  for (int k = tid; k < cnt; k += kBandBlock) {
    const float2 y = ys[c0 + k];
    float2 uv;
    const int cx = band_cell_u(y.x, g, 0, &uv.x), cy = band_cell_u(y.y, g, 1, &uv.y);
    const int key = (cx - cx0) * ni + cy;
    FITSNE_DCHECK(key >= 0 && key < kBandKeys && cx < ni && cy < ni);
    pts[k] = y;
    uvs[k] = uv;
    keyof[k] = (uint16_t)key;
    atomicAdd(&hist[key], 1u);
  }
  __syncthreads();
  // exclusive scan of hist: kBandKeys / kBandBlock = 16 entries per thread
  constexpr int E = kBandKeys / kBandBlock;
  uint32_t loc[E], run = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    loc[e] = run;
    run += hist[tid * E + e];
  }
  part[tid] = run;
  __syncthreads();
  if (tid < 32) {
    uint32_t v[kBandBlock / 32], t = 0;
#pragma unroll
    for (int j = 0; j < kBandBlock / 32; ++j) {
      v[j] = part[tid * (kBandBlock / 32) + j];
      t += v[j];
    }
    uint32_t x = t;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    uint32_t ex = x - t;
#pragma unroll
    for (int j = 0; j < kBandBlock / 32; ++j) {
      const uint32_t vj = v[j];
      part[tid * (kBandBlock / 32) + j] = ex;
      ex += vj;
    }
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) hist[tid * E + e] = loc[e] + part[tid];
  __syncthreads();
  // scatter local indices into box order
  for (int k = tid; k < cnt; k += kBandBlock) {
    order[atomicAdd(&hist[keyof[k]], 1u)] = (uint16_t)k;
  }
  __syncthreads();
  for (int q = tid; q < cnt; q += kBandBlock) {
    const int k = order[q];
    bs_pts[c0 + q] = pts[k];
    bs_idx[c0 + q] = sidx[c0 + k];
  }
  // runs of kBandRun sorted points per thread: register sums per box
  const int s0 = tid * kBandRun, s1 = min(cnt, s0 + kBandRun);
  float s[3][3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) s[a][b][0] = s[a][b][1] = s[a][b][2] = 0.f;
  int cur = -1, ccx = 0, ccy = 0;
  for (int q = s0; q < s1; ++q) {
    const int k = order[q];
    FITSNE_DCHECK(k < cnt);
    const int key = keyof[k];
    const float2 y = pts[k];
    const float2 uv = uvs[k];
    float wx[3], wy[3];
    band_weights(uv.x, wx);
    band_weights(uv.y, wy);
    if (key != cur) {
      if (cur >= 0) band_flush(acc, nn, ccx, ccy, s);
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) s[a][b][0] = s[a][b][1] = s[a][b][2] = 0.f;
      cur = key;
      ccx = cx0 + key / ni;
      ccy = key - (ccx - cx0) * ni;
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const float w = wx[a] * wy[b];
        s[a][b][0] += w;
        s[a][b][1] += w * (y.x - g.cf[0]);
        s[a][b][2] += w * (y.y - g.cf[1]);
      }
  }
  // Crowded boxes (a collapsed embedding early in a run: hundreds of points
  // per box): the lanes' runs are consecutive in box order, so a warp whose
  // 32 runs end in at most kBandCrowd distinct boxes adds the partials of a
  // box up with a segmented shuffle reduction and flushes once per box
  // instead of once per lane -- the per-lane flushes then serialise in the
  // L2 atomic units on a few thousand addresses (C3, span 1e-4: 570 us alone
  // on the GPU, and the SpMV beside it slows down by 1.8x).
  const unsigned all = 0xffffffffu;
  const int prev = __shfl_up_sync(all, cur, 1);
  const bool head = cur >= 0 && (lane == 0 || prev != cur);
  const unsigned heads = __ballot_sync(all, head);
  if (__popc(heads) <= kBandCrowd) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ko = __shfl_down_sync(all, cur, o);
      const bool take = lane + o < 32 && ko == cur;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const float v = __shfl_down_sync(all, s[a][b][c], o);
            if (take) s[a][b][c] += v;
          }
    }
    if (head) band_flush(acc, nn, ccx, ccy, s);
  } else if (cur >= 0) {
    band_flush(acc, nn, ccx, ccy, s);
  }
}

// F_rep of every point from the potentials (gather_potentials, nbody.py:344-350;
// optimizer.py:203-210, 244), in the box order the reduce pass left: a thread
// walks kBandRun consecutive points, which mostly share a box, and re-reads the
// box's 160-byte record block only when the box changes; neighbouring threads
// read neighbouring boxes.  Same arithmetic per point as k_combine's
// point_gather + frep_from_phi (bit-identical F_rep), written at the point's
// original index.
__global__ void __launch_bounds__(kBandBlock)
k_band_gather(const float2* __restrict__ bs_pts, const uint32_t* __restrict__ bs_idx, int64_t n, GridArgs g,
              const float* __restrict__ pot, const double* __restrict__ scal, float2* __restrict__ frep) {
  const int64_t q0 = (blockIdx.x * (int64_t)kBandBlock + threadIdx.x) * kBandRun;
  if (q0 >= n) return;
  const float Z = (float)scal[0];
  float r[40];
  int b0 = -1, b1 = -1;
  const int cnt = (int)min((int64_t)kBandRun, n - q0);
  for (int k = 0; k < cnt; ++k) {
    const float2 y = bs_pts[q0 + k];
    float w0[3], w1[3];
    const int c0 = band_cell(y.x, g, 0, w0), c1 = band_cell(y.y, g, 1, w1);
    if (c0 != b0 || c1 != b1) {
      b0 = c0;
      b1 = c1;
      const float* bp = pot + pot_box_node(c0, c1, 0, 0, 3, g.n_int) * kNodeSlots;
#pragma unroll
      for (int j = 0; j < 5; ++j)
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r[8 * j]), "=f"(r[8 * j + 1]), "=f"(r[8 * j + 2]), "=f"(r[8 * j + 3]),
                       "=f"(r[8 * j + 4]), "=f"(r[8 * j + 5]), "=f"(r[8 * j + 6]), "=f"(r[8 * j + 7])
                     : "l"(bp + 8 * j));
    }
    float phi[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const float wt = w0[a] * w1[b];
#pragma unroll
        for (int c = 0; c < 4; ++c) phi[c] += r[(a * 3 + b) * 4 + c] * wt;
      }
    const float yi[2] = {y.x, y.y};
    frep[bs_idx[q0 + k]] = make_float2(frep_from_phi<float, 2>(yi, phi, Z, 0, g),
                                       frep_from_phi<float, 2>(yi, phi, Z, 1, g));
  }
}

// scratch layout: row totals + row cursors, then (256-byte aligned) the
// row-sorted points and indices, then their box-ordered copies
struct BandBufs {
  uint32_t *rowtot, *rowcur, *sidx, *bs_idx;
  float2 *sorted, *bs_pts;
};
static inline size_t band_align(size_t x) { return (x + 255) & ~(size_t)255; }
static size_t band_bytes(int64_t n) {
  return band_align(2 * sizeof(uint32_t) * kBandMaxRows) + 2 * band_align(sizeof(float2) * (size_t)n) +
         2 * band_align(sizeof(uint32_t) * (size_t)n);
}
static BandBufs band_bufs(unsigned char* base, int64_t n) {
  BandBufs b;
  b.rowtot = (uint32_t*)base;
  b.rowcur = b.rowtot + kBandMaxRows;
  unsigned char* p = base + band_align(2 * sizeof(uint32_t) * kBandMaxRows);
  b.sorted = (float2*)p;
  p += band_align(sizeof(float2) * (size_t)n);
  b.sidx = (uint32_t*)p;
  p += band_align(sizeof(uint32_t) * (size_t)n);
  b.bs_pts = (float2*)p;
  p += band_align(sizeof(float2) * (size_t)n);
  b.bs_idx = (uint32_t*)p;
  return b;
}

// F_rep (n x 2 floats, original point order) from ctx->pot and Z (ctx->scal[0])
// for the points of the last spread_band call (same grid)
int gather_band(fitsne_ctx* ctx, int64_t n, void* frep, cudaStream_t st) {
  if (!ctx->band_sorted || ctx->band_n != n || !ctx->sortbuf.ptr) {
    set_error("band gather without a band spread of the same points");
    return FITSNE_EINVAL;
  }
  const BandBufs b = band_bufs((unsigned char*)ctx->sortbuf.ptr, n);
  const GridArgs g = grid_args(ctx->grid);
  const int nblk = (int)((n + (int64_t)kBandBlock * kBandRun - 1) / ((int64_t)kBandBlock * kBandRun));
  k_band_gather<<<nblk, kBandBlock, 0, st>>>(b.bs_pts, b.bs_idx, n, g, (const float*)ctx->pot.ptr,
                                             (const double*)ctx->scal.ptr, (float2*)frep);
  FITSNE_CHECK_LAUNCH();
  return FITSNE_OK;
}

// the row counters the band spread needs zeroed (the device-grid schedule
// has k_bbox clear them instead of a memset on the chain)
uint32_t* band_counters(fitsne_ctx* ctx, int64_t n, int* words) {
  if (ensure(ctx->sortbuf, band_bytes(n)) != FITSNE_OK) return nullptr;
  *words = 2 * kBandMaxRows;
  return (uint32_t*)ctx->sortbuf.ptr;
}

bool band_spread_applies(const fitsne_ctx* ctx, int64_t n) {
  return ctx->dtype == FITSNE_F32 && ctx->dims == 2 && ctx->grid.points_per_interval == 3 &&
         ctx->grid.n_intervals <= kBandMaxRows && n > 0 && n < (1LL << 31);
}

int spread_band(fitsne_ctx* ctx, const void* Y, int64_t n, void* accum, cudaStream_t st,
                const GridArgs* gd) {
  // gd: the device-computed grid (the host's ctx->grid is not known yet)
  const GridArgs g = gd ? GridArgs{} : grid_args(ctx->grid);
  const int nblk = (int)((n + kBandPts - 1) / kBandPts);
  FITSNE_TRY(ensure(ctx->sortbuf, band_bytes(n)));
  const BandBufs bb = band_bufs((unsigned char*)ctx->sortbuf.ptr, n);
  uint32_t* rowtot = bb.rowtot;
  uint32_t* rowcur = bb.rowcur;
  float2* sorted = bb.sorted;
  if (!gd) FITSNE_CUDA(cudaMemsetAsync(rowtot, 0, 2 * sizeof(uint32_t) * kBandMaxRows, st));
  k_band_rowcount<<<nblk, kBandBlock, 0, st>>>((const float2*)Y, n, g, rowtot, gd);
  FITSNE_CHECK_LAUNCH();
  k_band_place<<<nblk, kBandBlock, 0, st>>>((const float2*)Y, n, g, rowtot, rowcur, sorted, bb.sidx, gd);
  FITSNE_CHECK_LAUNCH();
  const int nred = (int)((n + kBandChunk - 1) / kBandChunk);
  {
    static std::mutex mu;
    static std::set<int> configured;
    std::lock_guard<std::mutex> lock(mu);
    if (!configured.count(ctx->device)) {
      FITSNE_CUDA(cudaFuncSetAttribute(k_band_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kBandSmem));
      configured.insert(ctx->device);
    }
  }
  k_band_reduce<<<nred, kBandBlock, kBandSmem, st>>>(sorted, bb.sidx, n, g, (float*)accum, bb.bs_pts,
                                                     bb.bs_idx, gd);
  FITSNE_CHECK_LAUNCH();
  // the box-ordered copy is usable by gather_band only with a host-known grid
  ctx->band_sorted = gd == nullptr;
  ctx->band_n = n;
  return FITSNE_OK;
}

}  // namespace fitsne
