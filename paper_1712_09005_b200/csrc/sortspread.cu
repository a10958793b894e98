// Box-sorted charge spreading (replaces one global atomic per point and node
// with one per box segment).
//
// The reference spreads with np.bincount over (N, p^s) node indices
// (nbody.py:233-237).  On the GPU a direct scatter makes ~27 atomics per point
// and collapses when points concentrate in a few boxes (the first t-SNE
// iterations put all points into 4 boxes: same-address atomics serialise).
// Here the points are first sorted by box with a stable LSD radix sort
// (8-bit digits, block-local stable ranks, no global atomics), then each warp
// walks a contiguous range of the sorted order, reduces the 9 x 3 node
// contributions of each box segment with a segmented warp scan, and flushes
// one vector atomic per node per (warp, box) piece.  A box that spans many
// warps gets at most one flush per warp, so contention is bounded by
// N / kWarpRange instead of N.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "interp.cuh"
#include "internal.h"

namespace fitsne {

static constexpr int kSortBlock = 256;
static constexpr int kItemsPerThread = 8;
static constexpr int kTile = kSortBlock * kItemsPerThread;  // items per sort block
static constexpr int kRadixBins = 256;
static constexpr int kWarpRange = 1024;                      // sorted items per reduce warp

// box id of a point (exact), shared by the key pass
template <typename T, int S>
__device__ __forceinline__ uint32_t point_box(const T* __restrict__ Y, int64_t i, const GridArgs& g) {
  int cell[S];
  if constexpr (sizeof(T) == 4) {
    if (g.p == 3) {
#pragma unroll
      for (int d = 0; d < S; ++d) {
        float w[3];
        cell[d] = box_weights3_f32(Y[i * S + d], g.lo[d], g.h[d], g.lo_f[d], g.invh_f[d],
                                   g.guard[d], g.n_int, w);
      }
    } else {
#pragma unroll
      for (int d = 0; d < S; ++d) {
        double w[kMaxP];
        cell[d] = box_weights((double)Y[i * S + d], g.lo[d], g.h[d], g.n_int, g.p, w);
      }
    }
  } else {
#pragma unroll
    for (int d = 0; d < S; ++d) {
      double w[kMaxP];
      cell[d] = box_weights((double)Y[i * S + d], g.lo[d], g.h[d], g.n_int, g.p, w);
    }
  }
  return (S == 1) ? (uint32_t)cell[0] : (uint32_t)cell[0] * (uint32_t)g.n_int + (uint32_t)cell[S - 1];
}

// histogram of one 8-bit digit over a block's tile, written digit-major
__device__ __forceinline__ void tile_hist_flush(uint32_t* s_hist, uint32_t* __restrict__ hist,
                                                int nblk) {
  __syncthreads();
  for (int d = threadIdx.x; d < kRadixBins; d += blockDim.x) hist[(size_t)d * nblk + blockIdx.x] = s_hist[d];
}

__device__ __forceinline__ void warp_hist_add(uint32_t* s_hist, uint32_t digit, bool valid) {
  const unsigned act = __ballot_sync(0xffffffffu, valid);
  if (!valid) return;
  const unsigned peers = __match_any_sync(act, digit);
  const int leader = __ffs(peers) - 1;
  if ((int)(threadIdx.x & 31) == leader) atomicAdd(&s_hist[digit], (uint32_t)__popc(peers));
}

// keys = box ids, vals = point indices, plus the histogram of digit 0
template <typename T, int S>
__global__ void __launch_bounds__(kSortBlock)
k_box_keys(const T* __restrict__ Y, int64_t n, GridArgs g, uint32_t* __restrict__ keys,
           uint32_t* __restrict__ vals, uint32_t* __restrict__ hist) {
  __shared__ uint32_t s_hist[kRadixBins];
  for (int d = threadIdx.x; d < kRadixBins; d += blockDim.x) s_hist[d] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTile;
#pragma unroll 1
  for (int r = 0; r < kItemsPerThread; ++r) {
    const int64_t i = base + (int64_t)r * kSortBlock + threadIdx.x;
    const bool valid = i < n;
    uint32_t key = 0;
    if (valid) {
      key = point_box<T, S>(Y, i, g);
      keys[i] = key;
      vals[i] = (uint32_t)i;
    }
    warp_hist_add(s_hist, key & 0xffu, valid);
  }
  tile_hist_flush(s_hist, hist, gridDim.x);
}

__global__ void __launch_bounds__(kSortBlock)
k_digit_hist(const uint32_t* __restrict__ keys, int64_t n, int shift, uint32_t* __restrict__ hist) {
  __shared__ uint32_t s_hist[kRadixBins];
  for (int d = threadIdx.x; d < kRadixBins; d += blockDim.x) s_hist[d] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kTile;
#pragma unroll 1
  for (int r = 0; r < kItemsPerThread; ++r) {
    const int64_t i = base + (int64_t)r * kSortBlock + threadIdx.x;
    const bool valid = i < n;
    const uint32_t key = valid ? __ldg(keys + i) : 0u;
    warp_hist_add(s_hist, (key >> shift) & 0xffu, valid);
  }
  tile_hist_flush(s_hist, hist, gridDim.x);
}

// Exclusive scan of each digit's row of the (digit-major) histogram matrix:
// one block per digit, coalesced chunks of blockDim items; the row total goes
// to totals[d].  The prefix over digits is added by the scatter kernel.
__global__ void __launch_bounds__(256)
k_scan_rows(uint32_t* __restrict__ hist, int nblk, uint32_t* __restrict__ totals) {
  __shared__ uint32_t s_warp[8];
  __shared__ uint32_t s_carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t* row = hist + (size_t)blockIdx.x * nblk;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int c0 = 0; c0 < nblk; c0 += blockDim.x) {
    const int k = c0 + threadIdx.x;
    const uint32_t x = (k < nblk) ? row[k] : 0u;
    uint32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[wid] = incl;
    __syncthreads();
    uint32_t wpre = 0, chunk = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (w < wid) wpre += s_warp[w];
      chunk += s_warp[w];
    }
    const uint32_t carry = s_carry;
    if (k < nblk) row[k] = carry + wpre + incl - x;
    __syncthreads();
    if (threadIdx.x == 0) s_carry = carry + chunk;
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = s_carry;
}

// stable scatter by one digit: block-local ranks in original order
__global__ void __launch_bounds__(kSortBlock)
k_digit_scatter(const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
                int64_t n, int shift, const uint32_t* __restrict__ offsets,
                const uint32_t* __restrict__ totals,
                uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out) {
  constexpr int kWarps = kSortBlock / 32;
  __shared__ uint32_t s_run[kRadixBins];             // items of each digit already placed
  __shared__ uint32_t s_wcnt[kWarps][kRadixBins];    // this round: per-warp digit counts
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // digit bases: exclusive prefix of the digit totals (kSortBlock == kRadixBins)
  {
    const uint32_t x = totals[threadIdx.x];
    uint32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_wcnt[0][wid] = incl;
    __syncthreads();
    uint32_t wpre = 0;
    for (int w = 0; w < wid; ++w) wpre += s_wcnt[0][w];
    s_run[threadIdx.x] = wpre + incl - x + offsets[(size_t)threadIdx.x * gridDim.x + blockIdx.x];
    __syncthreads();
  }
  const int64_t base = (int64_t)blockIdx.x * kTile;
#pragma unroll 1
  for (int r = 0; r < kItemsPerThread; ++r) {
    for (int t = threadIdx.x; t < kWarps * kRadixBins; t += blockDim.x) (&s_wcnt[0][0])[t] = 0;
    __syncthreads();
    const int64_t i = base + (int64_t)r * kSortBlock + threadIdx.x;
    const bool valid = i < n;
    const uint32_t key = valid ? keys_in[i] : 0u;
    const uint32_t val = valid ? vals_in[i] : 0u;
    const uint32_t digit = (key >> shift) & 0xffu;
    const unsigned act = __ballot_sync(0xffffffffu, valid);
    unsigned peers = 0;
    uint32_t rank = 0;
    if (valid) {
      peers = __match_any_sync(act, digit);
      rank = __popc(peers & ((1u << lane) - 1u));
      if (lane == __ffs(peers) - 1) s_wcnt[wid][digit] = __popc(peers);
    }
    __syncthreads();
    // exclusive prefix over warps (in warp order) for this item's digit
    if (valid) {
      uint32_t pre = 0;
      for (int w = 0; w < wid; ++w) pre += s_wcnt[w][digit];
      const uint32_t pos = s_run[digit] + pre + rank;
      keys_out[pos] = key;
      vals_out[pos] = val;
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadixBins; d += blockDim.x) {
      uint32_t tot = 0;
      for (int w = 0; w < kWarps; ++w) tot += s_wcnt[w][d];
      s_run[d] += tot;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// segmented spread over the box-sorted points
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ void flush_node(T* __restrict__ acc, int64_t node, T a, T b, T c) {
  T* dst = acc + node * kNodeSlots;
  if constexpr (sizeof(T) == 4) {
    atomicAdd(reinterpret_cast<float4*>(dst), make_float4(a, b, c, 0.f));
  } else {
    atomicAdd(dst, a);
    atomicAdd(dst + 1, b);
    if (c != (T)0) atomicAdd(dst + 2, c);
  }
}

// S = 2, p = 3: 9 nodes x 3 channels = 27 values per point.  S = 1, p = 3:
// 3 nodes x 2 channels.  (other p use the direct-scatter kernel)
template <typename T, int S>
__global__ void __launch_bounds__(256)
k_spread_sorted(const T* __restrict__ Y, const uint32_t* __restrict__ keys,
                const uint32_t* __restrict__ vals, int64_t n, GridArgs g, T* __restrict__ acc) {
  constexpr int NV = (S == 2) ? 27 : 6;   // nodes x channels
  constexpr int NN = (S == 2) ? 9 : 3;    // nodes per box
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t beg = warp * kWarpRange;
  if (beg >= n) return;
  const int64_t end = (beg + kWarpRange < n) ? beg + kWarpRange : n;
  T carry[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) carry[v] = 0;
  uint32_t carry_key = 0xffffffffu;
  for (int64_t k0 = beg; k0 < end; k0 += 32) {
    const int64_t k = k0 + lane;
    const bool valid = k < end;
    uint32_t key = valid ? __ldg(keys + k) : 0xfffffffeu;
    T v[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = 0;
    if (valid) {
      const uint32_t i = __ldg(vals + k);
      T y[S];
#pragma unroll
      for (int d = 0; d < S; ++d) y[d] = Y[(int64_t)i * S + d];
      using W = typename std::conditional<sizeof(T) == 4, float, double>::type;
      W wx[3], wy[3] = {1, 0, 0};
      if constexpr (sizeof(T) == 4) {
        box_weights3_f32((float)y[0], g.lo[0], g.h[0], g.lo_f[0], g.invh_f[0], g.guard[0], g.n_int, wx);
        if (S == 2)
          box_weights3_f32((float)y[S - 1], g.lo[S - 1], g.h[S - 1], g.lo_f[S - 1], g.invh_f[S - 1],
                           g.guard[S - 1], g.n_int, wy);
      } else {
        box_weights((double)y[0], g.lo[0], g.h[0], g.n_int, 3, wx);
        if (S == 2) box_weights((double)y[S - 1], g.lo[S - 1], g.h[S - 1], g.n_int, 3, wy);
      }
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < ((S == 2) ? 3 : 1); ++b) {
          const W w = wx[a] * wy[b];
          const int m = (S == 2) ? a * 3 + b : a;
          v[m * (NV / NN) + 0] = (T)w;
          v[m * (NV / NN) + 1] = (T)(w * ((W)y[0] - gcentre<W>(g, 0)));
          if (S == 2) v[m * (NV / NN) + 2] = (T)(w * ((W)y[S - 1] - gcentre<W>(g, S - 1)));
        }
    }
    // carry from the previous step joins lane 0's segment if the key continues
    const uint32_t key0 = __shfl_sync(0xffffffffu, key, 0);
    const bool carry_live = (carry_key != 0xffffffffu);
    const bool carry_joins = carry_live && carry_key == key0;
    if (lane == 0 && carry_joins) {
#pragma unroll
      for (int q = 0; q < NV; ++q) v[q] += carry[q];
    }
    // flush a carry that does not continue (lane 0 owns the carry)
    if (carry_live && !carry_joins && lane == 0) {
      const uint32_t cx = (S == 2) ? carry_key / (uint32_t)g.n_int : carry_key;
      const uint32_t cy = (S == 2) ? carry_key - cx * (uint32_t)g.n_int : 0;
#pragma unroll
      for (int m = 0; m < NN; ++m) {
        const int a = (S == 2) ? m / 3 : m, b = (S == 2) ? m % 3 : 0;
        const int64_t node = (S == 2) ? (((int64_t)cx * 3 + a) * g.n + (int64_t)cy * 3 + b)
                                      : ((int64_t)cx * 3 + a);
        flush_node<T>(acc, node, carry[m * (NV / NN)], carry[m * (NV / NN) + 1],
                      (S == 2) ? carry[m * (NV / NN) + 2] : (T)0);
      }
    }
    // inclusive segmented scan (keys are sorted, so equal neighbours are contiguous)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t nk = __shfl_up_sync(0xffffffffu, key, o);
      const bool add = lane >= o && nk == key;
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const T nv = __shfl_up_sync(0xffffffffu, v[q], o);
        if (add) v[q] += nv;
      }
    }
    const uint32_t next_key = __shfl_down_sync(0xffffffffu, key, 1);
    const bool tail = valid && (lane == 31 || next_key != key);
    // the segment ending at lane 31 continues into the next step: carry it
    const uint32_t k31 = __shfl_sync(0xffffffffu, key, 31);
    const bool last_step = (k0 + 32 >= end);
#pragma unroll
    for (int q = 0; q < NV; ++q) carry[q] = __shfl_sync(0xffffffffu, v[q], 31);
    carry_key = (last_step || !__shfl_sync(0xffffffffu, (int)valid, 31)) ? 0xffffffffu : k31;
    const bool flush = tail && (lane != 31 || last_step);
    if (flush) {
      const uint32_t cx = (S == 2) ? key / (uint32_t)g.n_int : key;
      const uint32_t cy = (S == 2) ? key - cx * (uint32_t)g.n_int : 0;
#pragma unroll
      for (int m = 0; m < NN; ++m) {
        const int a = (S == 2) ? m / 3 : m, b = (S == 2) ? m % 3 : 0;
        const int64_t node = (S == 2) ? (((int64_t)cx * 3 + a) * g.n + (int64_t)cy * 3 + b)
                                      : ((int64_t)cx * 3 + a);
        flush_node<T>(acc, node, v[m * (NV / NN)], v[m * (NV / NN) + 1],
                      (S == 2) ? v[m * (NV / NN) + 2] : (T)0);
      }
    }
  }
}

// =============================================================================
// v2 (grids with <= kSmemBoxes boxes): counting sort by box with a full
// per-block shared-memory histogram, then one warp per (box, part).
//   k_box_count   : keys + block histogram -> global counts (<= 1 atomic per
//                   (block, box): contention bounded by the block count)
//   k_box_scan    : exclusive scan of the counts (box offsets) and of the
//                   per-box part counts ceil(cnt / kPart) (work items)
//   k_box_scatter : block histogram again, one global reservation per
//                   (block, box), then shared-memory slots; writes the
//                   points' coordinates in box order
//   k_box_reduce  : warp per (box, part): coalesced reads of the sorted
//                   coordinates, register accumulation of the 9 x 3 node
//                   values, one warp reduction, plain stores when the box has
//                   one part (no atomics, no contention), atomics otherwise
// =============================================================================
static constexpr int kSmemBoxes = 48 * 1024;   // 192 KB of int counters
static constexpr int kCountBlock = 1024;
static constexpr int kPart = 256;              // points per reduce work item
static constexpr int kGroup = 32;              // lanes per reduce work item (a warp)

template <typename T, int S>
__global__ void __launch_bounds__(kCountBlock)
k_box_count(const T* __restrict__ Y, int64_t n, GridArgs g, int nbox, int64_t chunk,
            uint32_t* __restrict__ keys, uint32_t* __restrict__ counts) {
  extern __shared__ uint32_t s_cnt[];
  for (int b = threadIdx.x; b < nbox; b += blockDim.x) s_cnt[b] = 0;
  __syncthreads();
  const int64_t beg = blockIdx.x * chunk;
  const int64_t end = (beg + chunk < n) ? beg + chunk : n;
  for (int64_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
    const uint32_t key = point_box<T, S>(Y, i, g);
    keys[i] = key;
    atomicAdd(&s_cnt[key], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nbox; b += blockDim.x) {
    const uint32_t c = s_cnt[b];
    if (c) atomicAdd(&counts[b], c);
  }
}

// one block: offsets = exclusive scan of counts; items = exclusive scan of
// ceil(count / kPart); cursor = offsets (for the scatter's reservations)
__global__ void __launch_bounds__(1024)
k_box_scan(const uint32_t* __restrict__ counts, int nbox, uint32_t* __restrict__ offsets,
           uint32_t* __restrict__ cursor, uint32_t* __restrict__ items,
           uint32_t* __restrict__ item_box) {
  __shared__ uint32_t s_w[2][32];
  __shared__ uint32_t s_carry[2];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x == 0) { s_carry[0] = 0; s_carry[1] = 0; }
  __syncthreads();
  for (int c0 = 0; c0 <= nbox; c0 += blockDim.x) {
    const int b = c0 + threadIdx.x;
    const uint32_t x = (b < nbox) ? counts[b] : 0u;
    const uint32_t y = (b < nbox) ? (x + kPart - 1) / kPart : 0u;
    uint32_t ix = x, iy = y;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t ux = __shfl_up_sync(0xffffffffu, ix, o);
      const uint32_t uy = __shfl_up_sync(0xffffffffu, iy, o);
      if (lane >= o) { ix += ux; iy += uy; }
    }
    if (lane == 31) { s_w[0][wid] = ix; s_w[1][wid] = iy; }
    __syncthreads();
    uint32_t px = 0, py = 0, tx = 0, ty = 0;
    for (int w = 0; w < nw; ++w) {
      if (w < wid) { px += s_w[0][w]; py += s_w[1][w]; }
      tx += s_w[0][w];
      ty += s_w[1][w];
    }
    const uint32_t cx = s_carry[0], cy = s_carry[1];
    if (b <= nbox) {
      const uint32_t ox = cx + px + ix - x, oy = cy + py + iy - y;
      offsets[b] = ox;
      items[b] = oy;
      if (b < nbox) {
        cursor[b] = ox;
        for (uint32_t k = 0; k < y; ++k) item_box[oy + k] = (uint32_t)b;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) { s_carry[0] = cx + tx; s_carry[1] = cy + ty; }
    __syncthreads();
  }
}

template <typename T, int S>
__global__ void __launch_bounds__(kCountBlock)
k_box_scatter(const T* __restrict__ Y, int64_t n, int nbox, int64_t chunk,
              const uint32_t* __restrict__ keys, uint32_t* __restrict__ cursor,
              T* __restrict__ ysorted) {
  extern __shared__ uint32_t s_cnt[];
  for (int b = threadIdx.x; b < nbox; b += blockDim.x) s_cnt[b] = 0;
  __syncthreads();
  const int64_t beg = blockIdx.x * chunk;
  const int64_t end = (beg + chunk < n) ? beg + chunk : n;
  for (int64_t i = beg + threadIdx.x; i < end; i += blockDim.x) atomicAdd(&s_cnt[__ldg(keys + i)], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < nbox; b += blockDim.x) {
    const uint32_t c = s_cnt[b];
    s_cnt[b] = c ? atomicAdd(&cursor[b], c) : 0u;   // this block's base in box b
  }
  __syncthreads();
  for (int64_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
    const uint32_t slot = atomicAdd(&s_cnt[__ldg(keys + i)], 1u);
#pragma unroll
    for (int d = 0; d < S; ++d) ysorted[(size_t)slot * S + d] = Y[i * S + d];
  }
}

template <typename T, int S>
__global__ void __launch_bounds__(256)
k_box_reduce(const T* __restrict__ ysorted, const uint32_t* __restrict__ offsets,
             const uint32_t* __restrict__ items, const uint32_t* __restrict__ item_box, int nbox,
             GridArgs g, T* __restrict__ acc) {
  // one group of kGroup lanes per work item (box, part); kGroup-lane shuffles
  constexpr int NN = (S == 2) ? 9 : 3;
  constexpr int NC = S + 1;
  const int gl = threadIdx.x & (kGroup - 1);
  const int64_t item = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / kGroup;
  const uint32_t total = __ldg(items + nbox);
  const bool live = item < (int64_t)total;
  int box = 0;
  uint32_t p0 = 0, p1 = 0;
  bool whole = true;
  if (live) {
    box = (int)__ldg(item_box + item);
    const uint32_t part = (uint32_t)item - __ldg(items + box);
    const uint32_t b0 = __ldg(offsets + box), b1 = __ldg(offsets + box + 1);
    p0 = b0 + part * kPart;
    p1 = (p0 + kPart < b1) ? p0 + kPart : b1;
    whole = (b1 - b0) <= (uint32_t)kPart;
  }
  using W = typename std::conditional<sizeof(T) == 4, float, double>::type;
  W v[NN][NC];
#pragma unroll
  for (int m = 0; m < NN; ++m)
#pragma unroll
    for (int c = 0; c < NC; ++c) v[m][c] = 0;
  for (uint32_t k = p0 + gl; k < p1; k += kGroup) {
    T y[S];
#pragma unroll
    for (int d = 0; d < S; ++d) y[d] = ysorted[(size_t)k * S + d];
    W wx[3], wy[3] = {1, 0, 0};
    if constexpr (sizeof(T) == 4) {
      box_weights3_f32((float)y[0], g.lo[0], g.h[0], g.lo_f[0], g.invh_f[0], g.guard[0], g.n_int, wx);
      if (S == 2)
        box_weights3_f32((float)y[S - 1], g.lo[S - 1], g.h[S - 1], g.lo_f[S - 1], g.invh_f[S - 1],
                         g.guard[S - 1], g.n_int, wy);
    } else {
      box_weights((double)y[0], g.lo[0], g.h[0], g.n_int, 3, wx);
      if (S == 2) box_weights((double)y[S - 1], g.lo[S - 1], g.h[S - 1], g.n_int, 3, wy);
    }
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int bb = 0; bb < ((S == 2) ? 3 : 1); ++bb) {
        const int m = (S == 2) ? a * 3 + bb : a;
        const W w = wx[a] * wy[bb];
        v[m][0] += w;
        v[m][1] += w * ((W)y[0] - gcentre<W>(g, 0));
        if (S == 2) v[m][2] += w * ((W)y[S - 1] - gcentre<W>(g, S - 1));
      }
  }
#pragma unroll
  for (int m = 0; m < NN; ++m)
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int o = kGroup / 2; o > 0; o >>= 1) v[m][c] += __shfl_xor_sync(0xffffffffu, v[m][c], o, kGroup);
  if (!live) return;
  const uint32_t cx = (S == 2) ? (uint32_t)box / (uint32_t)g.n_int : (uint32_t)box;
  const uint32_t cy = (S == 2) ? (uint32_t)box - cx * (uint32_t)g.n_int : 0u;
#pragma unroll
  for (int m = 0; m < NN; ++m) {
    if ((m % kGroup) != gl) continue;   // group lane gl writes nodes gl, gl + kGroup
    const int a = (S == 2) ? m / 3 : m, bb = (S == 2) ? m % 3 : 0;
    const int64_t node = (S == 2) ? (((int64_t)cx * 3 + a) * g.n + (int64_t)cy * 3 + bb)
                                  : ((int64_t)cx * 3 + a);
    T* dst = acc + node * kNodeSlots;
    if (whole) {
      dst[0] = (T)v[m][0];
      dst[1] = (T)v[m][1];
      if (S == 2) dst[2] = (T)v[m][2];
    } else {
      flush_node<T>(acc, node, (T)v[m][0], (T)v[m][1], (S == 2) ? (T)v[m][2] : (T)0);
    }
  }
}

static int spread_counting(fitsne_ctx* ctx, const void* Y, int64_t n, void* accum, int nbox,
                           cudaStream_t st) {
  const GridArgs g = grid_args(ctx->grid);
  const int S = ctx->dims;
  const size_t es = dsize(ctx->dtype);
  // blocks: ~2 per SM, contiguous chunks
  int nblk = 2 * ctx->num_sms;
  int64_t chunk = (n + nblk - 1) / nblk;
  if (chunk < 4096) { chunk = 4096; nblk = (int)((n + chunk - 1) / chunk); }
  const int64_t max_items = (int64_t)nbox + (n + kPart - 1) / kPart;
  const size_t ints = 4 * (size_t)nbox + (size_t)max_items + 16;
  const size_t bytes = sizeof(uint32_t) * ((size_t)n + ints) + es * S * (size_t)n + 256;
  FITSNE_TRY(ensure(ctx->sortbuf, bytes));
  uint32_t* keys = (uint32_t*)ctx->sortbuf.ptr;
  uint32_t* counts = keys + n;
  uint32_t* offsets = counts + nbox + 1;
  uint32_t* cursor = offsets + nbox + 1;
  uint32_t* items = cursor + nbox + 1;
  uint32_t* item_box = items + nbox + 2;
  void* ysorted = (void*)(((uintptr_t)(item_box + max_items + 2) + 15) & ~(uintptr_t)15);
  FITSNE_CUDA(cudaMemsetAsync(counts, 0, sizeof(uint32_t) * nbox, st));
  const size_t smem = sizeof(uint32_t) * (size_t)nbox;
#define LAUNCH2(T, SS)                                                                          \
  do {                                                                                         \
    FITSNE_CUDA(cudaFuncSetAttribute((const void*)k_box_count<T, SS>,                          \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));  \
    FITSNE_CUDA(cudaFuncSetAttribute((const void*)k_box_scatter<T, SS>,                        \
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));  \
    k_box_count<T, SS><<<nblk, kCountBlock, smem, st>>>((const T*)Y, n, g, nbox, chunk, keys,  \
                                                        counts);                               \
    FITSNE_CHECK_LAUNCH();                                                                     \
    k_box_scan<<<1, 1024, 0, st>>>(counts, nbox, offsets, cursor, items, item_box);            \
    FITSNE_CHECK_LAUNCH();                                                                     \
    k_box_scatter<T, SS><<<nblk, kCountBlock, smem, st>>>((const T*)Y, n, nbox, chunk, keys,   \
                                                          cursor, (T*)ysorted);                \
    FITSNE_CHECK_LAUNCH();                                                                     \
    k_box_reduce<T, SS><<<(int)((max_items * kGroup + 255) / 256), 256, 0, st>>>(              \
        (const T*)ysorted, offsets, items, item_box, nbox, g, (T*)accum);                      \
    FITSNE_CHECK_LAUNCH();                                                                     \
  } while (0)
  if (ctx->dtype == FITSNE_F32) { if (S == 1) LAUNCH2(float, 1); else LAUNCH2(float, 2); }
  else { if (S == 1) LAUNCH2(double, 1); else LAUNCH2(double, 2); }
#undef LAUNCH2
  return FITSNE_OK;
}

// Sorted spread entry: returns FITSNE_EINVAL when this path does not apply
// (p != 3), in which case the caller uses the direct scatter.
int spread_sorted(fitsne_ctx* ctx, const void* Y, int64_t n, void* accum, cudaStream_t st) {
  const GridArgs g = grid_args(ctx->grid);
  if (g.p != 3 || n <= 0 || n > 0x7fffffffLL) return FITSNE_EINVAL;
  const int S = ctx->dims;
  const uint64_t nbox = (S == 2) ? (uint64_t)g.n_int * g.n_int : (uint64_t)g.n_int;
  if (nbox <= (uint64_t)kSmemBoxes) return spread_counting(ctx, Y, n, accum, (int)nbox, st);
  int bits = 1;
  while (bits < 32 && ((uint64_t)1 << bits) < nbox) ++bits;
  const int passes = (bits + 7) / 8;
  const int nblk = (int)((n + kTile - 1) / kTile);
  const size_t hist_n = (size_t)kRadixBins * nblk;
  // scratch: keys/vals x 2 buffers + histogram
  const size_t bytes = sizeof(uint32_t) * (4 * (size_t)n + hist_n + kRadixBins) + 256;
  FITSNE_TRY(ensure(ctx->sortbuf, bytes));
  uint32_t* k0 = (uint32_t*)ctx->sortbuf.ptr;
  uint32_t* v0 = k0 + n;
  uint32_t* k1 = v0 + n;
  uint32_t* v1 = k1 + n;
  uint32_t* hist = v1 + n;
  uint32_t* totals = hist + hist_n;
  if (ctx->dtype == FITSNE_F32) {
    if (S == 1) k_box_keys<float, 1><<<nblk, kSortBlock, 0, st>>>((const float*)Y, n, g, k0, v0, hist);
    else k_box_keys<float, 2><<<nblk, kSortBlock, 0, st>>>((const float*)Y, n, g, k0, v0, hist);
  } else {
    if (S == 1) k_box_keys<double, 1><<<nblk, kSortBlock, 0, st>>>((const double*)Y, n, g, k0, v0, hist);
    else k_box_keys<double, 2><<<nblk, kSortBlock, 0, st>>>((const double*)Y, n, g, k0, v0, hist);
  }
  FITSNE_CHECK_LAUNCH();
  for (int p = 0; p < passes; ++p) {
    if (p > 0) {
      k_digit_hist<<<nblk, kSortBlock, 0, st>>>(k0, n, 8 * p, hist);
      FITSNE_CHECK_LAUNCH();
    }
    k_scan_rows<<<kRadixBins, 256, 0, st>>>(hist, nblk, totals);
    FITSNE_CHECK_LAUNCH();
    k_digit_scatter<<<nblk, kSortBlock, 0, st>>>(k0, v0, n, 8 * p, hist, totals, k1, v1);
    FITSNE_CHECK_LAUNCH();
    std::swap(k0, k1);
    std::swap(v0, v1);
  }
  const int64_t warps = (n + kWarpRange - 1) / kWarpRange;
  const int blocks = (int)((warps * 32 + 255) / 256);
  if (ctx->dtype == FITSNE_F32) {
    if (S == 1) k_spread_sorted<float, 1><<<blocks, 256, 0, st>>>((const float*)Y, k0, v0, n, g, (float*)accum);
    else k_spread_sorted<float, 2><<<blocks, 256, 0, st>>>((const float*)Y, k0, v0, n, g, (float*)accum);
  } else {
    if (S == 1) k_spread_sorted<double, 1><<<blocks, 256, 0, st>>>((const double*)Y, k0, v0, n, g, (double*)accum);
    else k_spread_sorted<double, 2><<<blocks, 256, 0, st>>>((const double*)Y, k0, v0, n, g, (double*)accum);
  }
  FITSNE_CHECK_LAUNCH();
  return FITSNE_OK;
}

}  // namespace fitsne
