// Tiled attractive SpMV (compute_attractive, optimizer.py:150-166) for fp32
// 2-D embeddings.
//
// The row-per-warp CSR kernel (attract.cu) is bound by its neighbour gathers:
// every stored entry reads y_j from a different 32-byte L2 sector (a kNN
// graph has no index locality to exploit), so it moves ~4x more bytes through
// L2->L1 than the CSR stream itself.  Here P is re-laid out once, on first
// use, as tiles of (row block of R rows) x (column chunk of C points):
//
//   * a persistent CTA walks its share of the tiles in row-block-major order;
//     the Y rows of the current block and their force accumulators live in
//     shared memory, and the tile's column chunk of Y (C points, 64 KB) is
//     bulk-copied into shared memory (cp.async.bulk + mbarrier, double
//     buffered: the next tile's chunk lands while this one is processed);
//   * inside a tile the rows present are sorted by their entry count and
//     packed 32 per slab (sliced ELL): lane l of a warp owns row rows[l] of
//     the slab and walks its entries at slots (off + k) * 32 + l, so the
//     16-bit chunk-local column and the fp32 value streams are read fully
//     coalesced (6 bytes per slot instead of the CSR's 8), y_j comes from
//     shared memory, and each row is flushed once per tile with no atomics;
//   * row-block partial forces are added to the output with vector
//     reductions (a row block may be split between two CTAs).
//
// Only the summation order differs from the CSR kernel.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace fitsne {

// What the producer warp needs per tile: which Y chunk to stage and where the
// tile's header blob is.  The blob (16-byte aligned, copied into shared memory
// with the chunk) holds
//   int32 meta[4] = {row block, slab count, first group, group count}
//   int32 wlo[32]            first group of consumer warp w's run (cost-balanced cuts)
//   int32 wstart[32]         slab holding the first group of consumer warp w
//                            (whole-slab split: warp w owns slabs [wstart[w], wstart[w + 1]))
//   int32 wdesc[32][4]       consumer warp w's run in one 16-byte word: {first group, end group,
//                            first slab | (first slab is shared with another warp) << 31,
//                            end group of the first slab}
//   uint32 goff[nslab + 1]   group offsets of the slabs (padded to 4 entries)
//   uint16 rows[nslab][32]   tile-local row of each lane (0xFFFF: empty lane)
// where a "group" is 32 consecutive slots, one per lane.
struct TileLoad {
  int32_t chunk;
  int32_t hdr_bytes;
  int64_t hdr_off;
  int32_t g0, ng;  // the tile's slot groups
  int32_t pad[2];
};

__host__ __device__ inline int hdr_goff_words(int nslab) { return (nslab + 1 + 3) & ~3; }
constexpr int kHdrWstart = 16;                 // int32 wstart[32] after meta
constexpr int kHdrWlo = kHdrWstart + 128;      // int32 wlo[32]: first group of consumer warp w's run
constexpr int kHdrWdesc = kHdrWlo + 128;       // int4 wdesc[32]: {lo, hi, first slab | shared << 31, its end}
constexpr int kHdrGoff = kHdrWdesc + 512;      // uint32 goff[] after wdesc
__host__ __device__ inline int hdr_bytes_for(int nslab) {
  return kHdrGoff + 4 * hdr_goff_words(nslab) + 64 * nslab;
}

#ifndef FITSNE_TILED_THREADS
#define FITSNE_TILED_THREADS 1024
#endif
static constexpr int kTiledThreads = FITSNE_TILED_THREADS;  // consumer warps + 1 producer warp
static constexpr int kTiledConsumers = kTiledThreads / 32 - 1;
#ifndef FITSNE_TILED_U
#define FITSNE_TILED_U 4
#endif
#ifndef FITSNE_TILED_HOIST
#define FITSNE_TILED_HOIST 0
#endif
#ifndef FITSNE_TILED_L2PF
#define FITSNE_TILED_L2PF 1
#endif
#ifndef FITSNE_TILED_DEPTH
#define FITSNE_TILED_DEPTH 2
#endif
#ifndef FITSNE_TILED_FASTPATH
#define FITSNE_TILED_FASTPATH 0
#endif
// slabs cut by a warp-range boundary: 1 = add into the shared row-block
// accumulator with a compare-and-swap loop, 0 = vector reduction to global
#ifndef FITSNE_TILED_SCUT
#define FITSNE_TILED_SCUT 1
#endif
// whole-slab work split: every slab of a tile belongs to one consumer warp
// (slabs are dealt to the warps longest-first at build time and stored in
// that order), so no slab is cut by a warp-range boundary, each slab's header
// words / row points / accumulators are touched once, and every flush is a
// plain shared-memory read-modify-write.  The rows of a tile are also ordered
// so that the 16 (2-D) / 32 (1-D) rows of a half-warp / warp fall in distinct
// shared-memory banks.  0 = equal group ranges per warp (cut slabs).
#ifndef FITSNE_TILED_WSLAB
#define FITSNE_TILED_WSLAB 0
#endif
// dynamic schedule: the tail of every CTA's static share is cut into small
// work units drawn from a global counter (0 = static shares only)
#ifndef FITSNE_TILED_DYN
#define FITSNE_TILED_DYN 1
#endif
// share of a CTA's static run kept as its first (large) unit, in percent
#ifndef FITSNE_TILED_DYN_HEAD
#define FITSNE_TILED_DYN_HEAD 70
#endif
// small units per mean CTA share (a unit costs about share / this)
#ifndef FITSNE_TILED_DYN_UNIT
#define FITSNE_TILED_DYN_UNIT 24
#endif
// probe: per-CTA busy time written to the KL partials, printed by fitsne_tiled_stats
#ifndef FITSNE_TILED_TIMING
#define FITSNE_TILED_TIMING 0
#endif
static constexpr bool kWslab = FITSNE_TILED_WSLAB != 0;
// rows of a tile ordered so that the lanes of a slab hit distinct shared-memory
// banks with their row point / accumulator (second sort pass of the build)
#ifndef FITSNE_TILED_BANKROWS
#define FITSNE_TILED_BANKROWS 1
#endif
static constexpr bool kBankRows = FITSNE_TILED_BANKROWS != 0;
// a slab's rows placed in the lanes where their bank is free (k_slab_lanes)
#ifndef FITSNE_TILED_LANEDEAL
#define FITSNE_TILED_LANEDEAL 1
#endif
static constexpr bool kLaneDeal = FITSNE_TILED_LANEDEAL != 0;
// Consumer-warp runs inside a tile: cut points balance groups + BETA per slab
// start (a slab boundary costs about that many groups), and a cut within SNAP
// groups of a slab boundary moves onto it (the slab is then not shared by two
// warps).  Tenths of a group; 0 / 0 = equal group counts.
#ifndef FITSNE_TILED_CUT_BETA
#define FITSNE_TILED_CUT_BETA 10
#endif
#ifndef FITSNE_TILED_CUT_SNAP
#define FITSNE_TILED_CUT_SNAP 15
#endif
#ifndef FITSNE_TILED_WSLAB_BCOST
#define FITSNE_TILED_WSLAB_BCOST 1
#endif
static constexpr int kWslabBoundaryCost = FITSNE_TILED_WSLAB_BCOST;  // slab boundary, in groups
static constexpr int kKeyTileShift = 32;  // sort key: tile << 32 | (0xFFFF - count) << 16 | rank << 5 | bank
static constexpr int kTiledU = FITSNE_TILED_U;    // groups per lane per pipeline step
static constexpr int kTiledPad = 4 * kTiledU * 32;  // tail padding of the slot arrays

// Slot layout.  FITSNE_TILED_VEC = 1 (default): batches of four groups, lane-
// major inside a batch -- slot (g, lane) at (g / 4) * 128 + lane * 4 + g % 4 --
// so a lane reads a batch's four columns with one 8-byte and its four values
// with one 16-byte load (two coalesced global loads per four groups instead of
// eight).  FITSNE_TILED_VEC = 0: group-major, lane-minor (one 64-byte and one
// 128-byte warp load per group).
#ifndef FITSNE_TILED_VEC
#define FITSNE_TILED_VEC 1
#endif
#if FITSNE_TILED_VEC
static_assert(FITSNE_TILED_U == 4, "the vector slot layout is built for batches of four groups");
__host__ __device__ inline int64_t slot_index(int64_t g, int lane) {
  return ((g >> 2) << 7) + ((int64_t)lane << 2) + (g & 3);
}
#else
__host__ __device__ inline int64_t slot_index(int64_t g, int lane) { return g * 32 + lane; }
#endif
#ifndef FITSNE_TILED_STAGES
#define FITSNE_TILED_STAGES 2
#endif
static constexpr int kTiledStages = FITSNE_TILED_STAGES;  // chunk + header ring depth

// First group of consumer warp w's run in a tile of ng groups: equal shares
// (group granularity: all consumers meet at every tile, so the longest run
// sets the pace).  32-bit unsigned arithmetic (a tile holds < 2^32 / 32
// groups; a 64-bit division was ~90 instructions per warp and tile).
__host__ __device__ inline int tiled_run_lo(int ng, int w) {
  return (int)(((uint32_t)ng * (uint32_t)w) / (uint32_t)kTiledConsumers);
}

struct TiledP {
  DevBuf tiles, sched, psched, slab_off, rows, hdr, cols, vals, fattr, part;
  DevBuf units, counter;  // dynamic schedule: work units (int2 tile ranges) and the ticket counter
  int nunits = 0;
  unsigned ticket_base = 0;  // first ticket of the next launch
  // the pass in flight (attract_tiled), for the joining launch (attract_tiled_join)
  unsigned cur_base = 0;
  bool cur_kl = false, cur_dynamic = false;
  int join_grid = 0;         // CTAs of the last joining launch (0: none)
  int cur_grid = 0;          // CTAs of the pass's main launch (main_grid(): the build's grid or a few more)
  cudaEvent_t ev_perm = nullptr;  // relabelled Y copy ready
  // locality relabelling (reorder.cu): tiles are built over P[order][:, order];
  // order[new] = old.  The kernel reads Y through yp = Y[order] and adds each
  // row's force at its original index.
  DevBuf order, yp;
  bool relabeled = false;
  int relabel_mode = -1;
  int bank_mode = -1;
  int64_t nseg_natural = 0;  // (row, chunk) segments of the caller's order
  int64_t piece_rows[kTiledPieces + 1] = {};  // row ranges of the piece schedules
  int64_t ntiles = 0, nslabs = 0, nslots = 0, nseg = 0;
  int hdr_max = 0;  // largest header blob (bytes)
  int R = 0, C = 0, grid = 0;
  // the CSR this copy was built from
  const int64_t* rowptr = nullptr;
  const int32_t* col = nullptr;
  const void* val = nullptr;
  int64_t n_rows = 0, row_begin = 0, n_total = 0, nnz = 0;
  bool failed = false;  // build impossible for this CSR (size limits / memory)
  // fattr holds forces of a pass whose consumer (combine / finish kernel, which
  // clears it) was never queued -- an error between the SpMV and its consumer.
  // The next pass clears it first (after the stream that ran the stale pass).
  bool dirty = false;
  cudaStream_t dirty_stream = nullptr;
};

// points per column chunk: the option's value for 2-D, twice that for 1-D
// (same bytes per staged chunk); column indices are 16-bit
static int tile_cols_eff(const fitsne_ctx* ctx) {
  return std::min(ctx->dims == 1 ? 2 * ctx->tile_cols : ctx->tile_cols, 65536);
}

static void release_buf(DevBuf& b) {
  if (b.ptr) cudaFree(b.ptr);
  b.ptr = nullptr;
  b.cap = 0;
}

// exact-size allocation (the tiled arrays are large; no growth headroom)
static int alloc_exact(DevBuf& b, size_t bytes) {
  release_buf(b);
  if (bytes == 0) bytes = 16;
  if (cudaMalloc(&b.ptr, bytes) != cudaSuccess) {
    cudaGetLastError();
    b.ptr = nullptr;
    set_error("device allocation failed while tiling P");
    return FITSNE_ENOMEM;
  }
  b.cap = bytes;
  return FITSNE_OK;
}

void free_tiled(fitsne_ctx* ctx) {
  if (!ctx->tiled) return;
  TiledP* t = ctx->tiled;
  if (t->ev_perm) cudaEventDestroy(t->ev_perm);
  DevBuf* bufs[] = {&t->tiles, &t->sched, &t->psched, &t->slab_off, &t->rows, &t->hdr, &t->cols,
                    &t->vals, &t->fattr, &t->part, &t->order, &t->yp, &t->units, &t->counter};
  for (DevBuf* b : bufs) release_buf(*b);
  delete t;
  ctx->tiled = nullptr;
}

// ---------------------------------------------------------------------------
// build: CSR -> segments (row, chunk) -> sort by (tile, count desc) -> slabs
// ---------------------------------------------------------------------------
__global__ void k_rows_unsorted(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                int64_t n_rows, int32_t* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (r >= n_rows) return;
  const int64_t b = rowptr[r], e = rowptr[r + 1];
  bool bad = false;
  for (int64_t k = b + 1 + lane; k < e; k += 32) bad |= col[k] < col[k - 1];
  if (__any_sync(0xffffffffu, bad) && lane == 0) *flag = 1;
}

// segments of one row = maximal runs of entries in the same column chunk
// (columns are sorted inside a row, so a chunk's entries are contiguous)
__global__ void k_seg_count(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                            int64_t n_rows, int C, int32_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (r >= n_rows) return;
  const int64_t b = rowptr[r], e = rowptr[r + 1];
  int total = 0;
  for (int64_t k0 = b; k0 < e; k0 += 32) {
    const int64_t k = k0 + lane;
    bool f = false;
    if (k < e) f = (k == b) || (col[k] / C != col[k - 1] / C);
    total += __popc(__ballot_sync(0xffffffffu, f));
  }
  if (lane == 0) cnt[r] = total;
}

__global__ void k_seg_emit(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                           int64_t n_rows, int C, int nch, int R, const int64_t* __restrict__ segstart,
                           int64_t* __restrict__ seg_begin, int32_t* __restrict__ seg_row,
                           uint64_t* __restrict__ key) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (r >= n_rows) return;
  const int64_t b = rowptr[r], e = rowptr[r + 1];
  int64_t base = segstart[r];
  const int64_t tile_row = (r / R) * (int64_t)nch;
  for (int64_t k0 = b; k0 < e; k0 += 32) {
    const int64_t k = k0 + lane;
    bool f = false;
    int ch = 0;
    if (k < e) {
      ch = col[k] / C;
      f = (k == b) || (ch != col[k - 1] / C);
    }
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (f) {
      const int64_t s = base + __popc(m & ((1u << lane) - 1u));
      seg_begin[s] = k;
      seg_row[s] = (int32_t)r;
      key[s] = (uint64_t)(tile_row + ch) << kKeyTileShift;  // count filled in by k_seg_finish
    }
    base += __popc(m);
  }
}

__global__ void k_seg_finish(const int64_t* __restrict__ rowptr, const int64_t* __restrict__ segstart,
                             const int64_t* __restrict__ seg_begin, const int32_t* __restrict__ seg_row,
                             int64_t nseg, int R, int bank_mask, uint64_t* __restrict__ key,
                             uint32_t* __restrict__ idx, int32_t* __restrict__ seg_cnt) {
  const int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const int32_t r = seg_row[s];
  const int64_t end = (s + 1 < segstart[r + 1]) ? seg_begin[s + 1] : rowptr[r + 1];
  const int32_t c = (int32_t)(end - seg_begin[s]);
  seg_cnt[s] = c;
  // larger counts first inside a tile (sliced-ELL sorting window = the tile);
  // then the shared-memory bank of the row's point / accumulator
  key[s] |= ((uint64_t)(0xFFFF - c) << 16) | (uint64_t)((r % R) & bank_mask);
  idx[s] = (uint32_t)s;
}

// Second sort key.  After the first sort the segments of one (tile, count,
// bank) class are contiguous; rank = position inside the class.  Sorting by
// (tile, count, rank, bank) deals a class's banks round-robin, so consecutive
// rows -- the lanes of a slab -- fall in distinct banks.
__global__ void k_run_heads(const uint64_t* __restrict__ key, int64_t nseg, int64_t* __restrict__ head) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nseg) return;
  head[q] = (q == 0 || key[q] != key[q - 1]) ? q : 0;
}
__global__ void k_rank_key(uint64_t* __restrict__ key, const int64_t* __restrict__ head, int64_t nseg) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nseg) return;
  const int64_t rank = q - head[q];
  key[q] |= (uint64_t)(rank < 2047 ? rank : 2047) << 5;
}
struct MaxI64 {
  __host__ __device__ int64_t operator()(int64_t a, int64_t b) const { return a > b ? a : b; }
};

__global__ void k_tile_bounds(const uint64_t* __restrict__ key, int64_t nseg,
                              int32_t* __restrict__ tfirst, int32_t* __restrict__ tcount) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nseg) return;
  const uint64_t t = key[q] >> kKeyTileShift;
  if (q == 0 || (key[q - 1] >> kKeyTileShift) != t) {
    int64_t e = q + 1;
    // count: find the end of this tile's run (runs are short relative to nseg;
    // binary search over the sorted keys)
    int64_t lo = q, hi = nseg;  // first index with tile > t
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((key[mid] >> kKeyTileShift) > t) hi = mid; else lo = mid + 1;
    }
    e = lo;
    tfirst[t] = (int32_t)q;
    tcount[t] = (int32_t)(e - q);
  }
}

__global__ void k_tile_nslab(const int32_t* __restrict__ tcount, int64_t nt, int32_t* __restrict__ nslab) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t < nt) nslab[t] = (tcount[t] + 31) / 32;
}

__global__ void k_slab_kmax(const int32_t* __restrict__ tfirst, const int32_t* __restrict__ nslab,
                            const int32_t* __restrict__ slab_begin, const uint32_t* __restrict__ sidx,
                            const int32_t* __restrict__ seg_cnt, int64_t nt, uint32_t* __restrict__ kmax) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= nt) return;
  const int ns = nslab[t];
  for (int j = 0; j < ns; ++j) kmax[slab_begin[t] + j] = (uint32_t)seg_cnt[sidx[tfirst[t] + 32 * j]];
}

// Lane of each row inside its slab.  The sort deals a (tile, count) class's
// rows round-robin over the shared-memory banks of their point / accumulator,
// but a slab -- 32 consecutive rows of that order -- still mixes the tails of
// two rank groups, and a 64-bit access conflicts inside a half-warp on row mod
// 16.  The slab's rows may sit in any lane: put each row in a half-warp (2-D;
// the whole warp in 1-D) where its bank is still free, the rest wherever room
// is left.  One thread per slab; lane_of[q] for the sorted segment q.
__global__ void k_slab_lanes(const uint64_t* __restrict__ key, const int32_t* __restrict__ tfirst,
                             const int32_t* __restrict__ tcount, const int32_t* __restrict__ nslab,
                             int64_t ntd, int nbanks, unsigned char* __restrict__ lane_of) {
  const int64_t t = blockIdx.x;
  if (t >= ntd) return;
  const int ns = nslab[t];
  for (int j = threadIdx.x; j < ns; j += blockDim.x) {
    const int64_t q0 = (int64_t)tfirst[t] + 32 * j;
    const int n = min(32, tcount[t] - 32 * j);
    const int ngrp = 32 / nbanks;          // 2 half-warps of 16 banks, or 1 group of 32
    unsigned used[2] = {0u, 0u};
    unsigned taken = 0u;                   // lanes in use
    unsigned deferred = 0u;
    for (int i = 0; i < n; ++i) {
      const int b = (int)(key[q0 + i] & (uint64_t)(nbanks - 1));
      int g = -1;
      for (int h = 0; h < ngrp; ++h)
        if (g < 0 && !((used[h] >> b) & 1u)) g = h;
      if (g < 0) { deferred |= 1u << i; continue; }
      used[g] |= 1u << b;
      // the bank's own lane of the group: lanes of one group then hold distinct banks by construction
      const int lane = g * nbanks + b;
      taken |= 1u << lane;
      lane_of[q0 + i] = (unsigned char)lane;
    }
    for (int i = 0; i < n; ++i) {
      if (!((deferred >> i) & 1u)) continue;
      const int lane = __ffs(~taken) - 1;
      taken |= 1u << lane;
      lane_of[q0 + i] = (unsigned char)lane;
    }
  }
}

__global__ void k_tile_fill(const uint64_t* __restrict__ key, const uint32_t* __restrict__ sidx,
                            int64_t nseg, const int32_t* __restrict__ tfirst,
                            const int32_t* __restrict__ slab_begin, const int32_t* __restrict__ slab_pos,
                            const uint32_t* __restrict__ slab_off,
                            const int64_t* __restrict__ seg_begin, const int32_t* __restrict__ seg_row,
                            const int32_t* __restrict__ seg_cnt, const int32_t* __restrict__ col,
                            const float* __restrict__ val, int nch, int R, int C,
                            const unsigned char* __restrict__ lane_of,
                            uint16_t* __restrict__ rows, uint16_t* __restrict__ cols,
                            float* __restrict__ vals) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nseg) return;
  const int64_t t = (int64_t)(key[q] >> kKeyTileShift);
  const int64_t rel = q - tfirst[t];
  // slab_pos: the slab's place in the tile's stored order (whole-slab split)
  const int64_t slab = slab_begin[t] + (slab_pos ? slab_pos[slab_begin[t] + rel / 32] : rel / 32);
  const int lane = lane_of ? (int)lane_of[q] : (int)(rel & 31);
  const uint32_t s = sidx[q];
  const int32_t r = seg_row[s];
  const int rb = (int)(t / nch), ch = (int)(t % nch);
  rows[slab * 32 + lane] = (uint16_t)(r - (int64_t)rb * R);
  const int64_t b = seg_begin[s];
  const int c = seg_cnt[s];
  const int64_t o = (int64_t)slab_off[slab];
  for (int k = 0; k < c; ++k) {
    const int64_t slot = slot_index(o + k, lane);
    cols[slot] = (uint16_t)(col[b + k] - ch * C);
    vals[slot] = val[b + k];
  }
}

// Bank-aware slot order.  Inside a slab, lane l may visit its row's entries in
// any order; the y_j gather of step k is a 64-bit shared-memory load whose
// half-warps conflict when two lanes hit the same bank pair (column mod 16).
// Greedily pick, step by step and lane by lane, the remaining entry whose bank
// pair is least used in the lane's half-warp.  Slabs longer than kBankCap keep
// their order.  One warp per slab.
static constexpr int kBankCap = 32;
static constexpr int kBankWarps = 4;
__global__ void __launch_bounds__(kBankWarps * 32)
k_slab_bankorder(const uint32_t* __restrict__ slab_off, int64_t nslabs, uint16_t* __restrict__ cols,
                 float* __restrict__ vals) {
  __shared__ uint16_t lc[kBankWarps][32][kBankCap];
  __shared__ float lv[kBankWarps][32][kBankCap];
  __shared__ int cnt[kBankWarps][2][16];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int64_t sl = blockIdx.x * (int64_t)kBankWarps + wl;
  if (sl >= nslabs) return;
  const int64_t o = slab_off[sl];
  const int kmax = (int)(slab_off[sl + 1] - o);
  if (kmax > kBankCap || kmax < 2) return;
  // this lane's non-zero entries
  int n = 0;
  for (int k = 0; k < kmax; ++k) {
    const size_t slot = (size_t)slot_index(o + k, lane);
    const float v = vals[slot];
    if (v != 0.f) {
      lc[wl][lane][n] = cols[slot];
      lv[wl][lane][n] = v;
      ++n;
    }
  }
  unsigned used = 0;
  const int half = lane >> 4, hl = lane & 15;
  for (int k = 0; k < kmax; ++k) {
    if (lane < 32) {
      if (hl == 0) {
        for (int b = 0; b < 16; ++b) cnt[wl][half][b] = 0;
      }
    }
    __syncwarp();
    // lanes past their entries read column 0 (bank pair 0)
    const unsigned pad = __ballot_sync(0xffffffffu, k >= n);
    if (hl == 0) {
      const unsigned mine = half ? (pad >> 16) : (pad & 0xffffu);
      if (mine) cnt[wl][half][0] += 1;
    }
    __syncwarp();
    uint16_t pc = 0;
    float pv = 0.f;
    for (int i = 0; i < 16; ++i) {
      if (hl == i && k < n) {
        int best = -1, bc = 1 << 30;
        for (int e = 0; e < n; ++e) {
          if (used & (1u << e)) continue;
          const int c = cnt[wl][half][lc[wl][lane][e] & 15];
          if (c < bc) { bc = c; best = e; }
        }
        used |= 1u << best;
        pc = lc[wl][lane][best];
        pv = lv[wl][lane][best];
        cnt[wl][half][pc & 15] += 1;
      }
      __syncwarp();
    }
    const size_t slot = (size_t)slot_index(o + k, lane);
    cols[slot] = k < n ? pc : (uint16_t)0;
    vals[slot] = k < n ? pv : 0.f;
  }
}

// Bank-aware order for slabs longer than kBankCap (up to kBankCapLong slots
// per lane): one warp per slab.  Each lane buckets its entries by bank pair
// (column mod 16); at every step the lanes of a half-warp pick, in turn, an
// entry from the bucket whose bank pair is least used so far at that step.
static constexpr int kBankCapLong = 256;
__global__ void __launch_bounds__(32)
k_slab_bankorder_long(const uint32_t* __restrict__ slab_off, int64_t nslabs, uint16_t* __restrict__ cols,
                      float* __restrict__ vals) {
  extern __shared__ __align__(16) unsigned char bo_smem[];
  float* lv = reinterpret_cast<float*>(bo_smem);                       // [32][cap]
  uint16_t* lc = reinterpret_cast<uint16_t*>(lv + 32 * kBankCapLong);  // [32][cap]
  uint16_t* bstart = lc + 32 * kBankCapLong;                           // [32][17]
  uint16_t* btaken = bstart + 32 * 17;                                 // [32][16]
  __shared__ int use[2][16];
  const int lane = threadIdx.x;
  const int64_t sl = blockIdx.x;
  if (sl >= nslabs) return;
  const int64_t o = slab_off[sl];
  const int kmax = (int)(slab_off[sl + 1] - o);
  if (kmax <= kBankCap || kmax > kBankCapLong) return;
  uint16_t* st = bstart + lane * 17;
  uint16_t* tk = btaken + lane * 16;
  for (int b = 0; b < 17; ++b) st[b] = 0;
  for (int b = 0; b < 16; ++b) tk[b] = 0;
  int n = 0;
  for (int k = 0; k < kmax; ++k) {
    const size_t slot = (size_t)slot_index(o + k, lane);
    if (vals[slot] != 0.f) {
      ++st[(cols[slot] & 15) + 1];
      ++n;
    }
  }
  for (int b = 0; b < 16; ++b) st[b + 1] += st[b];
  for (int k = 0; k < kmax; ++k) {
    const size_t slot = (size_t)slot_index(o + k, lane);
    const float v = vals[slot];
    if (v != 0.f) {
      const int b = cols[slot] & 15;
      const int at = st[b] + tk[b]++;
      lc[lane * kBankCapLong + at] = cols[slot];
      lv[lane * kBankCapLong + at] = v;
    }
  }
  for (int b = 0; b < 16; ++b) tk[b] = 0;
  __syncwarp();
  const int half = lane >> 4, hl = lane & 15;
  for (int k = 0; k < kmax; ++k) {
    if (hl == 0)
      for (int b = 0; b < 16; ++b) use[half][b] = 0;
    __syncwarp();
    const unsigned pad = __ballot_sync(0xffffffffu, k >= n);
    if (hl == 0 && (half ? (pad >> 16) : (pad & 0xffffu))) use[half][0] += 1;  // pads broadcast col 0
    __syncwarp();
    uint16_t pc = 0;
    float pv = 0.f;
    for (int i = 0; i < 16; ++i) {
      if (hl == i && k < n) {
        int best = -1, bu = 1 << 30;
        for (int b = 0; b < 16; ++b) {
          if (tk[b] < st[b + 1] - st[b] && use[half][b] < bu) {
            bu = use[half][b];
            best = b;
          }
        }
        const int at = st[best] + tk[best]++;
        pc = lc[lane * kBankCapLong + at];
        pv = lv[lane * kBankCapLong + at];
        use[half][best] += 1;
      }
      __syncwarp();
    }
    const size_t slot = (size_t)slot_index(o + k, lane);
    cols[slot] = k < n ? pc : (uint16_t)0;
    vals[slot] = k < n ? pv : 0.f;
  }
}

static size_t bankorder_long_smem() {
  return (size_t)32 * kBankCapLong * (sizeof(float) + sizeof(uint16_t)) + (size_t)32 * 33 * sizeof(uint16_t);
}

// one warp per tile: assemble its header blob
__global__ void k_tile_headers(const int32_t* __restrict__ t_dense, const int32_t* __restrict__ t_sb,
                               const int32_t* __restrict__ t_ns, const int64_t* __restrict__ t_hoff,
                               int64_t ntiles, int nch, const uint32_t* __restrict__ slab_off,
                               const uint16_t* __restrict__ rows, const int32_t* __restrict__ t_wfirst,
                               unsigned char* __restrict__ hdr) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (t >= ntiles) return;
  const int sb = t_sb[t], ns = t_ns[t];
  unsigned char* h = hdr + t_hoff[t];
  int32_t* meta = reinterpret_cast<int32_t*>(h);
  int32_t* wstart = reinterpret_cast<int32_t*>(h + kHdrWstart);
  uint32_t* goff = reinterpret_cast<uint32_t*>(h + kHdrGoff);
  uint16_t* hr = reinterpret_cast<uint16_t*>(h + kHdrGoff + 4 * hdr_goff_words(ns));
  const uint32_t g0 = slab_off[sb];
  const uint32_t ng = slab_off[sb + ns] - g0;
  if (lane == 0) {
    meta[0] = t_dense[t] / nch;
    meta[1] = ns;
    meta[2] = (int32_t)g0;
    meta[3] = (int32_t)ng;
  }
  int32_t* wlo = reinterpret_cast<int32_t*>(h + kHdrWlo);
  if (t_wfirst) {
    // whole-slab split: warp `lane` owns the stored slabs [wstart[lane], wstart[lane + 1])
    wstart[lane] = t_wfirst[t * 32 + lane];
    wlo[lane] = (int32_t)(slab_off[sb + wstart[lane]] - g0);
  } else {
    // consumer warp `lane` starts where the cumulative cost (groups + beta per
    // slab start) reaches lane / kTiledConsumers of the tile's
    const float beta = FITSNE_TILED_CUT_BETA * 0.1f, snap = FITSNE_TILED_CUT_SNAP * 0.1f;
    auto cum = [&](int j) { return (float)(slab_off[sb + j] - g0) + beta * (float)j; };  // cost before slab j
    uint32_t lo;
    int a = 0;
    if (lane >= kTiledConsumers) {
      lo = ng;
      a = ns - 1;
    } else {
      const float target = cum(ns) * (float)lane / (float)kTiledConsumers;
      int z = ns;
      while (z - a > 1) {  // last slab whose start cost is <= target
        const int m = (a + z) >> 1;
        if (cum(m) <= target) a = m; else z = m;
      }
      const uint32_t s0 = slab_off[sb + a] - g0, s1 = slab_off[sb + a + 1] - g0;
      float into = target - cum(a) - beta;  // groups of slab a before the cut
      if (into < snap) into = 0.f;                          // onto the slab's start
      if ((float)(s1 - s0) - into < snap) into = (float)(s1 - s0);  // onto its end
      lo = s0 + (uint32_t)(into + 0.5f);
      if (lo > s1) lo = s1;
      if (lo == s1 && a + 1 < ns) a = a + 1;  // the run starts with the next slab
      if (lane == 0) { lo = 0; a = 0; }
    }
    wlo[lane] = (int32_t)lo;
    wstart[lane] = a;
  }
  for (int j = lane; j < hdr_goff_words(ns); j += 32) goff[j] = j <= ns ? slab_off[sb + j] - g0 : 0u;
  for (int64_t k = lane; k < (int64_t)ns * 32; k += 32) hr[k] = rows[(int64_t)sb * 32 + k];
  {
    // the run of consumer warp `lane` in one 16-byte word
    const int lo = wlo[lane], a = wstart[lane];
    int hi = __shfl_down_sync(0xffffffffu, lo, 1);
    if (lane >= kTiledConsumers - 1) hi = (int)ng;
    if (lane >= kTiledConsumers) hi = lo;
    const int a_lo = (int)(slab_off[sb + a] - g0), a_end = (int)(slab_off[sb + a + 1] - g0);
    const bool shared = a_lo < lo || a_end > hi;
    int4 d;
    d.x = lo;
    d.y = hi;
    d.z = a | (shared ? (int)0x80000000u : 0);
    d.w = a_end;
    reinterpret_cast<int4*>(h + kHdrWdesc)[lane] = d;
  }
}

// The stored column of a slot becomes its byte offset inside the staged chunk
// (column x sizeof(point): < 65536 for 8192 2-D or 16384 1-D points), so the
// consumers add it to the chunk's base without a shift.  Last build pass.
__global__ void k_cols_to_offsets(uint16_t* __restrict__ cols, int64_t nslots, int shift) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < nslots) cols[i] = (uint16_t)((uint32_t)cols[i] << shift);
}

// Persistent grid: with the overlapped schedule ~3/16 of the SMs stay free
// for the bbox / spread / FFT / gather chain running concurrently on the side
// stream (the tiled kernel fills an SM: 1024 threads x 64 registers, ~218 KB
// of shared memory); serial schedules use every SM.  The chain is ~1/3 of the
// step's SM-time at C3: with 120 of 148 SMs on the SpMV both end together
// (104: 1876, 112: 1879, 120: 1907, 128: 1868, 136: 1838 evaluations/s).
static int tiled_grid(const fitsne_ctx* ctx) {
  if (ctx->tiled_ctas > 0) return ctx->tiled_ctas;
  if (ctx->overlap != 0) return std::max(1, ctx->num_sms - (3 * ctx->num_sms + 8) / 16);
  return ctx->num_sms;
}

// Build temporaries come from the stream-ordered pool (no device-wide sync
// on free, memory reused by the next build).
struct TmpBufs {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit TmpBufs(cudaStream_t s) : st(s) {}
  ~TmpBufs() { for (void* p : ptrs) cudaFreeAsync(p, st); }
  template <typename T>
  int alloc(T** out, size_t count) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, std::max<size_t>(count, 1) * sizeof(T), st) != cudaSuccess) {
      cudaGetLastError();
      set_error("device allocation failed while tiling P");
      return FITSNE_ENOMEM;
    }
    ptrs.push_back(p);
    *out = (T*)p;
    return FITSNE_OK;
  }
};

static inline int nb(int64_t n, int block) { return (int)std::max<int64_t>(1, (n + block - 1) / block); }

// Exclusive scan of n items in -> out (CUB), temp storage from `tmp`.
template <typename In, typename Out>
static int excl_scan(TmpBufs& tmp, In* in, Out* out, int64_t n, cudaStream_t st) {
  size_t bytes = 0;
  FITSNE_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, st));
  void* t = nullptr;
  unsigned char* tb = nullptr;
  FITSNE_TRY(tmp.alloc(&tb, bytes));
  t = tb;
  FITSNE_CUDA(cub::DeviceScan::ExclusiveSum(t, bytes, in, out, n, st));
  return FITSNE_OK;
}

// P[order][:, order] as CSR: new row r is old row order[r] with its columns
// relabelled by pos_of (rows come out unsorted; the build sorts them)
__global__ void k_perm_degree(const int64_t* __restrict__ rowptr, const int* __restrict__ order, int64_t n,
                              int64_t* __restrict__ deg) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r < n) deg[r] = rowptr[order[r] + 1] - rowptr[order[r]];
  if (r == n) deg[n] = 0;
}

__global__ void k_perm_rows(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                            const float* __restrict__ val, const int* __restrict__ order,
                            const int* __restrict__ pos_of, int64_t n, const int64_t* __restrict__ nrowptr,
                            int32_t* __restrict__ ncol, float* __restrict__ nval) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (r >= n) return;
  const int64_t b = rowptr[order[r]], e = rowptr[order[r] + 1], o = nrowptr[r];
  for (int64_t k = b + lane; k < e; k += 32) {
    ncol[o + (k - b)] = pos_of[col[k]];
    nval[o + (k - b)] = val[k];
  }
}

static int build_tiled_csr(fitsne_ctx* ctx, TiledP* T, const int64_t* rowptr, const int32_t* col_in,
                           const float* val_in, cudaStream_t st);

// total (row, chunk) segments of a row-sorted CSR (one host read)
static int count_segments(const int64_t* rowptr, const int32_t* col, int64_t n_rows, int C, TmpBufs& tmp,
                          int64_t* out, cudaStream_t st) {
  int32_t* cnt;
  int64_t* start;
  FITSNE_TRY(tmp.alloc(&cnt, n_rows + 1));
  FITSNE_TRY(tmp.alloc(&start, n_rows + 1));
  FITSNE_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * (n_rows + 1), st));
  k_seg_count<<<nb(n_rows * 32, 256), 256, 0, st>>>(rowptr, col, n_rows, C, cnt);
  FITSNE_CHECK_LAUNCH();
  FITSNE_TRY(excl_scan(tmp, cnt, start, n_rows + 1, st));
  FITSNE_CUDA(cudaMemcpyAsync(out, start + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FITSNE_CUDA(cudaStreamSynchronize(st));
  return FITSNE_OK;
}

// (row, chunk) segments of the registered CSR in the caller's order (rows may
// list their columns unsorted: counted on a sorted copy then)
static int natural_segments(fitsne_ctx* ctx, TmpBufs& tmp, int64_t* out, cudaStream_t st) {
  const int64_t n = ctx->n_total, nnz = ctx->nnz;
  const int32_t* c0 = ctx->col;
  int32_t* flag;
  FITSNE_TRY(tmp.alloc(&flag, 1));
  FITSNE_CUDA(cudaMemsetAsync(flag, 0, sizeof(int32_t), st));
  k_rows_unsorted<<<nb(n * 32, 256), 256, 0, st>>>(ctx->rowptr, c0, n, flag);
  int32_t hf = 0;
  FITSNE_CUDA(cudaMemcpyAsync(&hf, flag, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  FITSNE_CUDA(cudaStreamSynchronize(st));
  if (hf) {
    int32_t* oc;
    float* ov;
    FITSNE_TRY(tmp.alloc(&oc, nnz));
    FITSNE_TRY(tmp.alloc(&ov, nnz));
    size_t bytes = 0;
    FITSNE_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, bytes, ctx->col, oc, (const float*)ctx->val, ov,
                                                    nnz, n, ctx->rowptr, ctx->rowptr + 1, st));
    unsigned char* tb;
    FITSNE_TRY(tmp.alloc(&tb, bytes));
    FITSNE_CUDA(cub::DeviceSegmentedSort::SortPairs(tb, bytes, ctx->col, oc, (const float*)ctx->val, ov,
                                                    nnz, n, ctx->rowptr, ctx->rowptr + 1, st));
    c0 = oc;
  }
  return count_segments(ctx->rowptr, c0, n, tile_cols_eff(ctx), tmp, out, st);
}

// Auto relabelling skips the search for an ordering on a large matrix (many
// column chunks) whose caller order already gives this many entries per (row,
// chunk) segment: the Cuthill-McKee orderings of the large kNN graphs
// measured reach ~7, so an input at 4 or more cannot have its segments halved
// (the bar for using the ordering), and the search costs ~0.9 s at C3, 10x
// the layout build itself.  Small matrices (few chunks: an ordering can bring
// a row's neighbours into one or two of them) always search; it is cheap there.
static constexpr double kRelabelSkipDensity = 4.0;
static constexpr int64_t kRelabelSkipChunks = 64;

static int build_tiled(fitsne_ctx* ctx, TiledP* T, cudaStream_t st) {
  FITSNE_RANGE("tiled_build");
  // relabel (FITSNE_OPT_RELABEL) only a whole matrix: the sharded layout's
  // rows are one rank's range of the global columns
  const bool whole = ctx->row_begin == 0 && ctx->n_rows == ctx->n_total;
  if (ctx->relabel == 0 || !whole || ctx->n_total > 0x7fffffffLL)
    return build_tiled_csr(ctx, T, ctx->rowptr, ctx->col, (const float*)ctx->val, st);
  const int64_t n = ctx->n_total, nnz = ctx->nnz;
  int64_t seg_natural = -1;
  if (ctx->relabel == 1) {
    TmpBufs tmp0(st);
    FITSNE_TRY(natural_segments(ctx, tmp0, &seg_natural, st));
    T->nseg_natural = seg_natural;
    const int64_t nch = (ctx->n_total + tile_cols_eff(ctx) - 1) / tile_cols_eff(ctx);
    if (nch >= kRelabelSkipChunks && (double)nnz >= kRelabelSkipDensity * (double)seg_natural)
      return build_tiled_csr(ctx, T, ctx->rowptr, ctx->col, (const float*)ctx->val, st);
  }
  TmpBufs tmp(st);
  FITSNE_TRY(alloc_exact(T->order, sizeof(int) * (size_t)n));
  int* order = (int*)T->order.ptr;
  int* pos_of;
  FITSNE_TRY(tmp.alloc(&pos_of, n));
  FITSNE_TRY(cuthill_mckee(ctx->rowptr, ctx->col, (int)n, order, pos_of, ctx->num_sms, st));
  int64_t *nrowptr, *deg;
  int32_t* ncol;
  float* nval;
  FITSNE_TRY(tmp.alloc(&deg, n + 1));
  FITSNE_TRY(tmp.alloc(&nrowptr, n + 1));
  FITSNE_TRY(tmp.alloc(&ncol, nnz));
  FITSNE_TRY(tmp.alloc(&nval, nnz));
  k_perm_degree<<<nb(n + 1, 256), 256, 0, st>>>(ctx->rowptr, order, n, deg);
  FITSNE_CHECK_LAUNCH();
  FITSNE_TRY(excl_scan(tmp, deg, nrowptr, n + 1, st));
  k_perm_rows<<<nb(n * 32, 256), 256, 0, st>>>(ctx->rowptr, ctx->col, (const float*)ctx->val, order, pos_of,
                                               n, nrowptr, ncol, nval);
  FITSNE_CHECK_LAUNCH();
  // sort each relabelled row's columns (the segment count needs them sorted)
  int32_t* scol;
  float* sval;
  FITSNE_TRY(tmp.alloc(&scol, nnz));
  FITSNE_TRY(tmp.alloc(&sval, nnz));
  {
    size_t bytes = 0;
    FITSNE_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, bytes, ncol, scol, nval, sval, nnz, n, nrowptr,
                                                    nrowptr + 1, st));
    unsigned char* tb;
    FITSNE_TRY(tmp.alloc(&tb, bytes));
    FITSNE_CUDA(cub::DeviceSegmentedSort::SortPairs(tb, bytes, ncol, scol, nval, sval, nnz, n, nrowptr,
                                                    nrowptr + 1, st));
  }
  bool use = ctx->relabel == 2;
  if (!use) {
    // auto: keep the caller's order unless relabelling at least halves the
    // (row, chunk) segments.  Measured at C3: a cluster-ordered input (41M ->
    // 28M segments) runs 7% slower relabelled, a randomly ordered one (117M
    // segments, no tiled layout at all) gets the tiled SpMV back.
    int64_t seg_new = 0, seg_old = 0;
    FITSNE_TRY(count_segments(nrowptr, scol, n, tile_cols_eff(ctx), tmp, &seg_new, st));
    seg_old = seg_natural;  // counted above (auto mode)
    T->nseg_natural = seg_old;
    use = (double)seg_new <= 0.5 * (double)seg_old;
  }
  if (!use) {
    release_buf(T->order);
    return build_tiled_csr(ctx, T, ctx->rowptr, ctx->col, (const float*)ctx->val, st);
  }
  FITSNE_TRY(alloc_exact(T->yp, sizeof(float) * 2 * (size_t)n));
  T->relabeled = true;
  return build_tiled_csr(ctx, T, nrowptr, scol, sval, st);
}

static int build_tiled_csr(fitsne_ctx* ctx, TiledP* T, const int64_t* rowptr, const int32_t* col_in,
                           const float* val_in, cudaStream_t st) {
  const int64_t n_rows = ctx->n_rows, n_total = ctx->n_total, nnz = ctx->nnz;
  const int R = ctx->tile_rows, C = tile_cols_eff(ctx);
  const int64_t nrb = (n_rows + R - 1) / R, nch = (n_total + C - 1) / C;
  const int64_t ntd = nrb * nch;  // dense tile count
  if ((int64_t)C * (ctx->dims == 1 ? 4 : 8) > 65536) {
    set_error("tile_cols too large: a staged chunk holds at most 64 KB of points");
    return FITSNE_EINVAL;
  }
  if (ntd >= (1LL << 31) || nnz >= (1LL << 31) || nrb >= (1LL << 31)) {
    set_error("P too large for the tiled layout");
    return FITSNE_ETOOBIG;
  }
  TmpBufs tmp(st);
  // rows must list their columns in ascending order (one segment per row and
  // chunk); sort a copy if the registered CSR does not
  const int32_t* col = col_in;
  const float* val = val_in;
  {
    int32_t* flag;
    FITSNE_TRY(tmp.alloc(&flag, 1));
    FITSNE_CUDA(cudaMemsetAsync(flag, 0, sizeof(int32_t), st));
    k_rows_unsorted<<<nb(n_rows * 32, 256), 256, 0, st>>>(rowptr, col, n_rows, flag);
    FITSNE_CHECK_LAUNCH();
    int32_t h_flag = 0;
    FITSNE_CUDA(cudaMemcpyAsync(&h_flag, flag, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    FITSNE_CUDA(cudaStreamSynchronize(st));
    if (h_flag) {
      int32_t* scol;
      float* sval;
      FITSNE_TRY(tmp.alloc(&scol, nnz));
      FITSNE_TRY(tmp.alloc(&sval, nnz));
      size_t bytes = 0;
      FITSNE_CUDA(cub::DeviceSegmentedSort::SortPairs(nullptr, bytes, col, scol, val, sval, nnz, n_rows,
                                                      rowptr, rowptr + 1, st));
      unsigned char* tb;
      FITSNE_TRY(tmp.alloc(&tb, bytes));
      FITSNE_CUDA(cub::DeviceSegmentedSort::SortPairs(tb, bytes, col, scol, val, sval, nnz, n_rows,
                                                      rowptr, rowptr + 1, st));
      col = scol;
      val = sval;
    }
  }
  int32_t* segcnt;
  int64_t* segstart;
  FITSNE_TRY(tmp.alloc(&segcnt, n_rows + 1));
  FITSNE_TRY(tmp.alloc(&segstart, n_rows + 1));
  FITSNE_CUDA(cudaMemsetAsync(segcnt, 0, sizeof(int32_t) * (n_rows + 1), st));
  k_seg_count<<<nb(n_rows * 32, 256), 256, 0, st>>>(rowptr, col, n_rows, C, segcnt);
  FITSNE_CHECK_LAUNCH();
  FITSNE_TRY(excl_scan(tmp, segcnt, segstart, n_rows + 1, st));
  int64_t nseg = 0;
  FITSNE_CUDA(cudaMemcpyAsync(&nseg, segstart + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FITSNE_CUDA(cudaStreamSynchronize(st));
  if (nseg <= 0) { set_error("empty P"); return FITSNE_EINVAL; }
  // A graph without index locality (e.g. random kNN partners) leaves ~1
  // entry per (row, chunk) segment: every tile would stage a whole Y chunk
  // for a few hundred entries.  The row-per-warp CSR kernel is the right one
  // there; keep the tiled layout for >= 2 entries per segment on average
  // (C3's clustered kNN graph: 5.4).
  if (ctx->tiled_spmv == 1 && nnz < 2 * nseg) {
    set_error("P has no column locality for the tiled layout");
    return FITSNE_EINVAL;
  }

  int64_t* seg_begin;
  int32_t *seg_row, *seg_cnt;
  uint64_t *key, *key2;
  uint32_t *idx, *idx2;
  FITSNE_TRY(tmp.alloc(&seg_begin, nseg));
  FITSNE_TRY(tmp.alloc(&seg_row, nseg));
  FITSNE_TRY(tmp.alloc(&seg_cnt, nseg));
  FITSNE_TRY(tmp.alloc(&key, nseg));
  FITSNE_TRY(tmp.alloc(&key2, nseg));
  FITSNE_TRY(tmp.alloc(&idx, nseg));
  FITSNE_TRY(tmp.alloc(&idx2, nseg));
  k_seg_emit<<<nb(n_rows * 32, 256), 256, 0, st>>>(rowptr, col, n_rows, C, (int)nch, R,
                                                   segstart, seg_begin, seg_row, key);
  FITSNE_CHECK_LAUNCH();
  // bank of a row's point / accumulator in shared memory: 8-byte float2 (2-D)
  // conflicts inside a half-warp on row mod 16, 4-byte float (1-D) on row mod 32
  const int bank_mask = kBankRows ? (ctx->dims == 1 ? 31 : 15) : 0;
  k_seg_finish<<<nb(nseg, 256), 256, 0, st>>>(rowptr, segstart, seg_begin, seg_row, nseg, R, bank_mask, key,
                                              idx, seg_cnt);
  FITSNE_CHECK_LAUNCH();
  int end_bit = kKeyTileShift;
  while ((1LL << (end_bit - kKeyTileShift)) < ntd) ++end_bit;
  auto sort_pairs = [&](uint64_t* kin, uint64_t* kout, uint32_t* vin, uint32_t* vout) -> int {
    size_t bytes = 0;
    FITSNE_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, nseg, 0, end_bit, st));
    unsigned char* tb;
    FITSNE_TRY(tmp.alloc(&tb, bytes));
    FITSNE_CUDA(cub::DeviceRadixSort::SortPairs(tb, bytes, kin, kout, vin, vout, nseg, 0, end_bit, st));
    return FITSNE_OK;
  };
  FITSNE_TRY(sort_pairs(key, key2, idx, idx2));
  if (kBankRows) {
    // second pass: (tile, count, rank inside the (tile, count, bank) class, bank)
    int64_t *head, *hpos;
    FITSNE_TRY(tmp.alloc(&head, nseg));
    FITSNE_TRY(tmp.alloc(&hpos, nseg));
    k_run_heads<<<nb(nseg, 256), 256, 0, st>>>(key2, nseg, head);
    FITSNE_CHECK_LAUNCH();
    {
      size_t bytes = 0;
      FITSNE_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, head, hpos, MaxI64(), nseg, st));
      unsigned char* tb;
      FITSNE_TRY(tmp.alloc(&tb, bytes));
      FITSNE_CUDA(cub::DeviceScan::InclusiveScan(tb, bytes, head, hpos, MaxI64(), nseg, st));
    }
    k_rank_key<<<nb(nseg, 256), 256, 0, st>>>(key2, hpos, nseg);
    FITSNE_CHECK_LAUNCH();
    FITSNE_TRY(sort_pairs(key2, key, idx2, idx));
    std::swap(key, key2);   // key2 / idx2: the final order, as below
    std::swap(idx, idx2);
  }
  int32_t *tfirst, *tcount, *nslab, *slab_begin;
  FITSNE_TRY(tmp.alloc(&tfirst, ntd));
  FITSNE_TRY(tmp.alloc(&tcount, ntd));
  FITSNE_TRY(tmp.alloc(&nslab, ntd + 1));
  FITSNE_TRY(tmp.alloc(&slab_begin, ntd + 1));
  FITSNE_CUDA(cudaMemsetAsync(tfirst, 0, sizeof(int32_t) * ntd, st));
  FITSNE_CUDA(cudaMemsetAsync(tcount, 0, sizeof(int32_t) * ntd, st));
  FITSNE_CUDA(cudaMemsetAsync(nslab, 0, sizeof(int32_t) * (ntd + 1), st));
  k_tile_bounds<<<nb(nseg, 256), 256, 0, st>>>(key2, nseg, tfirst, tcount);
  FITSNE_CHECK_LAUNCH();
  k_tile_nslab<<<nb(ntd, 256), 256, 0, st>>>(tcount, ntd, nslab);
  FITSNE_CHECK_LAUNCH();
  FITSNE_TRY(excl_scan(tmp, nslab, slab_begin, ntd + 1, st));
  int32_t nslabs = 0;
  FITSNE_CUDA(cudaMemcpyAsync(&nslabs, slab_begin + ntd, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  FITSNE_CUDA(cudaStreamSynchronize(st));

  uint32_t* kmax;
  FITSNE_TRY(tmp.alloc(&kmax, (size_t)nslabs + 1));
  FITSNE_CUDA(cudaMemsetAsync(kmax, 0, sizeof(uint32_t) * ((size_t)nslabs + 1), st));
  k_slab_kmax<<<nb(ntd, 256), 256, 0, st>>>(tfirst, nslab, slab_begin, idx2, seg_cnt, ntd, kmax);
  FITSNE_CHECK_LAUNCH();
  std::vector<int32_t> h_nslab(ntd), h_sb(ntd);
  FITSNE_CUDA(cudaMemcpyAsync(h_nslab.data(), nslab, sizeof(int32_t) * ntd, cudaMemcpyDeviceToHost, st));
  FITSNE_CUDA(cudaMemcpyAsync(h_sb.data(), slab_begin, sizeof(int32_t) * ntd, cudaMemcpyDeviceToHost, st));
  // Whole-slab split (host): deal each tile's slabs, longest first, to the
  // consumer warp with the least work so far (a slab costs its groups plus a
  // fixed boundary term); store the slabs warp by warp.  slab_pos[j] = stored
  // position of the tile's j-th slab of the sorted order, wfirst[w] = first
  // stored slab of warp w.
  int32_t* slab_pos = nullptr;
  std::vector<int32_t> h_wfirst;  // per dense tile with slabs: 32 entries, filled below
  std::vector<int64_t> wf_of(kWslab ? ntd : 0, -1);
  if (kWslab) {
    std::vector<uint32_t> h_kmax((size_t)nslabs + 1), h_kperm((size_t)nslabs + 1, 0u);
    std::vector<int32_t> h_pos((size_t)nslabs);
    FITSNE_CUDA(cudaMemcpyAsync(h_kmax.data(), kmax, sizeof(uint32_t) * ((size_t)nslabs + 1),
                                cudaMemcpyDeviceToHost, st));
    FITSNE_CUDA(cudaStreamSynchronize(st));
    std::vector<int> owner;
    for (int64_t t = 0; t < ntd; ++t) {
      const int ns = h_nslab[t];
      if (ns == 0) continue;
      const int64_t sb = h_sb[t];
      owner.assign(ns, 0);
      int64_t load[32] = {};
      int cnt[32] = {};
      for (int j = 0; j < ns; ++j) {  // sorted order: longest slabs first
        int best = 0;
        for (int w = 1; w < kTiledConsumers; ++w)
          if (load[w] < load[best]) best = w;
        owner[j] = best;
        load[best] += (int64_t)h_kmax[sb + j] + kWslabBoundaryCost;
        ++cnt[best];
      }
      wf_of[t] = (int64_t)h_wfirst.size();
      int first[33];
      first[0] = 0;
      for (int w = 0; w < 32; ++w) first[w + 1] = first[w] + (w < kTiledConsumers ? cnt[w] : 0);
      for (int w = 0; w < 32; ++w) h_wfirst.push_back(first[w]);
      int at[32];
      for (int w = 0; w < 32; ++w) at[w] = first[w];
      for (int j = 0; j < ns; ++j) {
        const int p = at[owner[j]]++;
        h_pos[sb + j] = p;
        h_kperm[sb + p] = h_kmax[sb + j];
      }
    }
    FITSNE_TRY(tmp.alloc(&slab_pos, (size_t)nslabs));
    FITSNE_CUDA(cudaMemcpyAsync(slab_pos, h_pos.data(), sizeof(int32_t) * (size_t)nslabs, cudaMemcpyHostToDevice, st));
    FITSNE_CUDA(cudaMemcpyAsync(kmax, h_kperm.data(), sizeof(uint32_t) * ((size_t)nslabs + 1),
                                cudaMemcpyHostToDevice, st));
    FITSNE_CUDA(cudaStreamSynchronize(st));  // the host vectors go out of scope
  }
  FITSNE_TRY(alloc_exact(T->slab_off, sizeof(uint32_t) * ((size_t)nslabs + 1)));
  uint32_t* slab_off = (uint32_t*)T->slab_off.ptr;
  FITSNE_TRY(excl_scan(tmp, kmax, slab_off, (int64_t)nslabs + 1, st));
  uint32_t total_k = 0;
  FITSNE_CUDA(cudaMemcpyAsync(&total_k, slab_off + nslabs, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  FITSNE_CUDA(cudaStreamSynchronize(st));
  const int64_t nslots = (int64_t)total_k * 32;

  FITSNE_TRY(alloc_exact(T->rows, sizeof(uint16_t) * (size_t)nslabs * 32));
  // kTiledPad extra slots: the kernel reads whole groups of slots past a
  // slab's end (values masked), so the last slab must not run off the array
  FITSNE_TRY(alloc_exact(T->cols, sizeof(uint16_t) * (size_t)(nslots + kTiledPad)));
  FITSNE_TRY(alloc_exact(T->vals, sizeof(float) * (size_t)(nslots + kTiledPad)));
  FITSNE_CUDA(cudaMemsetAsync(T->rows.ptr, 0xFF, sizeof(uint16_t) * (size_t)nslabs * 32, st));
  FITSNE_CUDA(cudaMemsetAsync(T->cols.ptr, 0, sizeof(uint16_t) * (size_t)(nslots + kTiledPad), st));
  FITSNE_CUDA(cudaMemsetAsync(T->vals.ptr, 0, sizeof(float) * (size_t)(nslots + kTiledPad), st));
  unsigned char* lane_of = nullptr;
  if (kBankRows && kLaneDeal) {
    FITSNE_TRY(tmp.alloc(&lane_of, (size_t)nseg));
    k_slab_lanes<<<(unsigned)ntd, 128, 0, st>>>(key2, tfirst, tcount, nslab, ntd, bank_mask + 1, lane_of);
    FITSNE_CHECK_LAUNCH();
  }
  k_tile_fill<<<nb(nseg, 256), 256, 0, st>>>(key2, idx2, nseg, tfirst, slab_begin, slab_pos, slab_off, seg_begin,
                                             seg_row, seg_cnt, col, val,
                                             (int)nch, R, C, lane_of, (uint16_t*)T->rows.ptr,
                                             (uint16_t*)T->cols.ptr, (float*)T->vals.ptr);
  FITSNE_CHECK_LAUNCH();
  if (ctx->tiled_bank_order) {
    k_slab_bankorder<<<nb(nslabs, kBankWarps), kBankWarps * 32, 0, st>>>(
        slab_off, nslabs, (uint16_t*)T->cols.ptr, (float*)T->vals.ptr);
    FITSNE_CHECK_LAUNCH();
    if (ctx->tiled_bank_order == 1) {
      const size_t sm = bankorder_long_smem();
      FITSNE_CUDA(cudaFuncSetAttribute(k_slab_bankorder_long, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sm));
      k_slab_bankorder_long<<<(unsigned)std::max<int64_t>(nslabs, 1), 32, sm, st>>>(
          slab_off, nslabs, (uint16_t*)T->cols.ptr, (float*)T->vals.ptr);
      FITSNE_CHECK_LAUNCH();
    }
  }
  // columns -> byte offsets inside the staged chunk (after the bank ordering,
  // which reads columns)
  k_cols_to_offsets<<<nb(nslots + kTiledPad, 256), 256, 0, st>>>((uint16_t*)T->cols.ptr, nslots + kTiledPad,
                                                               ctx->dims == 1 ? 2 : 3);
  FITSNE_CHECK_LAUNCH();

  // host: compact tile list, header blobs, static schedule balanced on cost
  std::vector<uint32_t> h_off((size_t)nslabs + 1);
  FITSNE_CUDA(cudaMemcpyAsync(h_off.data(), slab_off, sizeof(uint32_t) * ((size_t)nslabs + 1),
                              cudaMemcpyDeviceToHost, st));
  FITSNE_CUDA(cudaStreamSynchronize(st));
  if ((uint64_t)h_off[nslabs] + 2 * kTiledU >= (1ULL << 31)) {
    set_error("P too large for the tiled layout");
    return FITSNE_ETOOBIG;
  }
  std::vector<TileLoad> tiles;
  std::vector<int32_t> t_dense, t_sb, t_ns;
  std::vector<int64_t> t_hoff;
  std::vector<double> cost;
  int64_t hoff = 0;
  int hmax = 16;
  for (int64_t t = 0; t < ntd; ++t) {
    if (h_nslab[t] == 0) continue;
    const int ns = h_nslab[t];
    TileLoad d;
    d.chunk = (int32_t)(t % nch);
    d.hdr_bytes = hdr_bytes_for(ns);
    d.hdr_off = hoff;
    d.g0 = (int32_t)h_off[h_sb[t]];
    d.ng = (int32_t)(h_off[h_sb[t] + ns] - h_off[h_sb[t]]);
    d.pad[0] = d.pad[1] = 0;
    hoff += d.hdr_bytes;
    hmax = std::max(hmax, d.hdr_bytes);
    const double groups = (double)(h_off[h_sb[t] + ns] - h_off[h_sb[t]]);
    // streamed groups + per-slab flush + chunk / header staging
    cost.push_back(32.0 * groups + 48.0 * ns + 0.5 * C);
    tiles.push_back(d);
    t_dense.push_back((int32_t)t);
    t_sb.push_back(h_sb[t]);
    t_ns.push_back(ns);
    t_hoff.push_back(d.hdr_off);
  }
  const int64_t nt = (int64_t)tiles.size();
  FITSNE_TRY(alloc_exact(T->hdr, (size_t)std::max<int64_t>(hoff, 16)));
  {
    int32_t *d_dense, *d_sb, *d_ns, *d_wfirst = nullptr;
    int64_t* d_hoff;
    if (kWslab) {
      std::vector<int32_t> wf((size_t)nt * 32);
      for (int64_t i = 0; i < nt; ++i)
        std::memcpy(wf.data() + (size_t)i * 32, h_wfirst.data() + wf_of[t_dense[i]], 32 * sizeof(int32_t));
      FITSNE_TRY(tmp.alloc(&d_wfirst, (size_t)nt * 32));
      FITSNE_CUDA(cudaMemcpyAsync(d_wfirst, wf.data(), sizeof(int32_t) * (size_t)nt * 32, cudaMemcpyHostToDevice, st));
      FITSNE_CUDA(cudaStreamSynchronize(st));
    }
    FITSNE_TRY(tmp.alloc(&d_dense, nt));
    FITSNE_TRY(tmp.alloc(&d_sb, nt));
    FITSNE_TRY(tmp.alloc(&d_ns, nt));
    FITSNE_TRY(tmp.alloc(&d_hoff, nt));
    FITSNE_CUDA(cudaMemcpyAsync(d_dense, t_dense.data(), sizeof(int32_t) * nt, cudaMemcpyHostToDevice, st));
    FITSNE_CUDA(cudaMemcpyAsync(d_sb, t_sb.data(), sizeof(int32_t) * nt, cudaMemcpyHostToDevice, st));
    FITSNE_CUDA(cudaMemcpyAsync(d_ns, t_ns.data(), sizeof(int32_t) * nt, cudaMemcpyHostToDevice, st));
    FITSNE_CUDA(cudaMemcpyAsync(d_hoff, t_hoff.data(), sizeof(int64_t) * nt, cudaMemcpyHostToDevice, st));
    k_tile_headers<<<nb(nt * 32, 256), 256, 0, st>>>(d_dense, d_sb, d_ns, d_hoff, nt, (int)nch, slab_off,
                                                    (const uint16_t*)T->rows.ptr, d_wfirst,
                                                    (unsigned char*)T->hdr.ptr);
    FITSNE_CHECK_LAUNCH();
    FITSNE_CUDA(cudaStreamSynchronize(st));
  }
  const int grid = tiled_grid(ctx);
  // static schedule of tiles [ta, tb) over the persistent grid: contiguous
  // runs of the row-block-major order balanced on cost
  auto balance = [&](int64_t ta, int64_t tb, int32_t* sched) {
    double total = 0;
    for (int64_t t = ta; t < tb; ++t) total += cost[t];
    double acc = 0;
    int k = 1;
    sched[0] = (int32_t)ta;
    for (int64_t t = ta; t < tb && k < grid; ++t) {
      acc += cost[t];
      while (k < grid && acc >= total * k / grid) sched[k++] = (int32_t)(t + 1);
    }
    for (; k <= grid; ++k) sched[k] = (int32_t)tb;
  };
  std::vector<int32_t> sched(grid + 1), psched((size_t)kTiledPieces * (grid + 1));
  balance(0, nt, sched.data());
  // dynamic schedule: unit b < grid = the head of CTA b's static share
  // (FITSNE_TILED_DYN_HEAD percent of its cost), then every share's tail in
  // units of FITSNE_TILED_DYN_UNIT tiles, in tile order
  std::vector<int2> units;
  if (FITSNE_TILED_DYN) {
    std::vector<int32_t> cut(grid);
    for (int b = 0; b < grid; ++b) {
      double total = 0, acc = 0;
      for (int64_t t = sched[b]; t < sched[b + 1]; ++t) total += cost[t];
      int64_t t = sched[b];
      for (; t < sched[b + 1]; ++t) {
        if (acc + cost[t] > total * (FITSNE_TILED_DYN_HEAD / 100.0)) break;
        acc += cost[t];
      }
      cut[b] = (int32_t)t;
      units.push_back(make_int2(sched[b], cut[b]));
    }
    // tails: units of about 1 / FITSNE_TILED_DYN_UNIT of a CTA's mean share
    // (by cost; a tile is never split, so the heavy diagonal tiles make large
    // units), drawn largest first so the small ones level the finish
    double total = 0;
    for (int64_t t = 0; t < nt; ++t) total += cost[t];
    const double target = total / grid / FITSNE_TILED_DYN_UNIT;
    std::vector<std::pair<double, int2>> tail;
    for (int b = 0; b < grid; ++b) {
      int32_t t = cut[b];
      while (t < sched[b + 1]) {
        double acc = 0;
        int32_t e = t;
        do { acc += cost[e]; ++e; } while (e < sched[b + 1] && acc + 0.5 * cost[e] <= target);
        tail.push_back({acc, make_int2(t, e)});
        t = e;
      }
    }
    std::stable_sort(tail.begin(), tail.end(),
                     [](const std::pair<double, int2>& a, const std::pair<double, int2>& b) { return a.first > b.first; });
    for (const auto& u : tail) units.push_back(u.second);
  }
  // piece schedules: row blocks split in kTiledPieces near-equal-cost ranges
  {
    const int64_t nrb = (n_rows + R - 1) / R;
    std::vector<double> rb_cost(nrb, 0.0);
    for (int64_t t = 0; t < nt; ++t) rb_cost[t_dense[t] / nch] += cost[t];
    double total = 0;
    for (double c : rb_cost) total += c;
    std::vector<int64_t> rb_cut(kTiledPieces + 1, nrb);
    rb_cut[0] = 0;
    double acc = 0;
    int k = 1;
    for (int64_t b = 0; b < nrb && k < kTiledPieces; ++b) {
      acc += rb_cost[b];
      while (k < kTiledPieces && acc >= total * k / kTiledPieces) rb_cut[k++] = b + 1;
    }
    int64_t t = 0;
    for (int q = 0; q < kTiledPieces; ++q) {
      const int64_t ta = t;
      while (t < nt && t_dense[t] / nch < rb_cut[q + 1]) ++t;
      balance(ta, t, psched.data() + (size_t)q * (grid + 1));
      T->piece_rows[q] = std::min<int64_t>(rb_cut[q] * R, n_rows);
    }
    T->piece_rows[kTiledPieces] = n_rows;
  }
  FITSNE_TRY(alloc_exact(T->tiles, sizeof(TileLoad) * (size_t)std::max<int64_t>(nt, 1)));
  FITSNE_TRY(alloc_exact(T->sched, sizeof(int32_t) * (grid + 1)));
  FITSNE_TRY(alloc_exact(T->psched, sizeof(int32_t) * psched.size()));
  FITSNE_CUDA(cudaMemcpyAsync(T->psched.ptr, psched.data(), sizeof(int32_t) * psched.size(),
                              cudaMemcpyHostToDevice, st));
  FITSNE_CUDA(cudaMemcpyAsync(T->tiles.ptr, tiles.data(), sizeof(TileLoad) * nt, cudaMemcpyHostToDevice, st));
  FITSNE_CUDA(cudaMemcpyAsync(T->sched.ptr, sched.data(), sizeof(int32_t) * (grid + 1),
                              cudaMemcpyHostToDevice, st));
  FITSNE_TRY(alloc_exact(T->fattr, sizeof(float) * 2 * (size_t)std::max<int64_t>(n_rows, 1)));
  FITSNE_CUDA(cudaMemsetAsync(T->fattr.ptr, 0, sizeof(float) * 2 * (size_t)n_rows, st));
  FITSNE_TRY(alloc_exact(T->part, sizeof(double) * (grid + ctx->num_sms + 1)));  // + a joining launch
  T->nunits = (int)units.size();
  T->ticket_base = 0;
  if (!units.empty()) {
    FITSNE_TRY(alloc_exact(T->units, sizeof(int2) * units.size()));
    FITSNE_TRY(alloc_exact(T->counter, sizeof(unsigned)));
    FITSNE_CUDA(cudaMemcpyAsync(T->units.ptr, units.data(), sizeof(int2) * units.size(), cudaMemcpyHostToDevice, st));
    FITSNE_CUDA(cudaMemsetAsync(T->counter.ptr, 0, sizeof(unsigned), st));
  }
  FITSNE_CUDA(cudaStreamSynchronize(st));  // host vectors and temporaries go out of scope
  release_buf(T->rows);      // folded into the header blobs
  release_buf(T->slab_off);
  T->ntiles = nt;
  T->nseg = nseg;
  T->nslabs = nslabs;
  T->nslots = nslots;
  T->hdr_max = hmax;
  T->R = R;
  T->C = C;
  T->grid = grid;
  return FITSNE_OK;
}

// es: bytes per point (8 for 2-D float2, 4 for 1-D float)
static size_t stage_bytes(int C, int hdr_max, size_t es) {
  return (size_t)C * es + (size_t)((hdr_max + 15) & ~15);
}
static size_t tiled_smem(int R, int C, int hdr_max, size_t es) {
  return ((es * 3 * (size_t)R + 15) & ~(size_t)15) + kTiledStages * stage_bytes(C, hdr_max, es);
}

// Use the tiled kernel for this call?  Builds the tiled copy on first use.
bool tiled_usable(fitsne_ctx* ctx, const void* Y, cudaStream_t st) {
  if (ctx->tiled_spmv == 0 || ctx->dtype != FITSNE_F32 || !ctx->rowptr) return false;
  if (((uintptr_t)Y & 15) != 0) return false;
  if (ctx->tiled_spmv == 1 && ctx->nnz < (1LL << 22)) return false;
  if (tiled_smem(ctx->tile_rows, tile_cols_eff(ctx), hdr_bytes_for((ctx->tile_rows + 31) / 32),
                 ctx->dims == 1 ? sizeof(float) : sizeof(float2)) >
      227 * 1024 - 1024)
    return false;  // tile shape does not fit in shared memory
  TiledP* T = ctx->tiled;
  const bool same = T && T->rowptr == ctx->rowptr && T->col == ctx->col && T->val == ctx->val &&
                    T->n_rows == ctx->n_rows && T->row_begin == ctx->row_begin &&
                    T->n_total == ctx->n_total && T->nnz == ctx->nnz && T->R == ctx->tile_rows &&
                    T->C == tile_cols_eff(ctx) && T->relabel_mode == ctx->relabel &&
                    T->bank_mode == ctx->tiled_bank_order &&
                    T->grid == (tiled_grid(ctx));
  if (same) return !T->failed;
  if (T && T->failed && T->rowptr == ctx->rowptr && T->col == ctx->col && T->val == ctx->val &&
      T->nnz == ctx->nnz)
    return false;
  free_tiled(ctx);
  T = new TiledP();
  ctx->tiled = T;
  T->rowptr = ctx->rowptr;
  T->col = ctx->col;
  T->val = ctx->val;
  T->n_rows = ctx->n_rows;
  T->row_begin = ctx->row_begin;
  T->n_total = ctx->n_total;
  T->nnz = ctx->nnz;
  T->R = ctx->tile_rows;
  T->C = tile_cols_eff(ctx);
  T->relabel_mode = ctx->relabel;
  T->bank_mode = ctx->tiled_bank_order;
  T->grid = tiled_grid(ctx);
  if (ctx->n_rows < 1 || ctx->nnz < 1 || build_tiled(ctx, T, st) != FITSNE_OK) {
    // keep the CSR kernel for this P; release what the attempt allocated
    cudaStreamSynchronize(st);
    cudaGetLastError();
    DevBuf* bufs[] = {&T->tiles, &T->sched, &T->psched, &T->slab_off, &T->rows, &T->hdr, &T->cols,
                      &T->vals, &T->fattr, &T->part, &T->order, &T->yp, &T->units, &T->counter};
    for (DevBuf* b : bufs) release_buf(*b);
    T->failed = true;
    return false;
  }
  return true;
}

// ---------------------------------------------------------------------------
// kernel
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra LAB_WAIT;\n"
      "}\n" ::"r"(smem_addr(b)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(b))
      : "memory");
}

// L2 eviction policy for the Y chunks, which every row block re-reads while
// the slot stream passes through L2 once
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* b,
                                              uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
      "[%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(b)), "l"(pol)
      : "memory");
}

// L2 prefetch of a global range (bulk, no destination, no completion)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Point type of the tiles: float2 (2-D) or float (1-D embeddings; a chunk of
// C points is then 4C bytes, so 1-D uses twice the points per chunk).
template <int S> struct TPt;
template <> struct TPt<2> {
  using T = float2;
  static __device__ __forceinline__ T zero() { return make_float2(0.f, 0.f); }
  static __device__ __forceinline__ T make(float a, float b) { return make_float2(a, b); }
  static __device__ __forceinline__ T add(T a, T b) { return make_float2(a.x + b.x, a.y + b.y); }
  static __device__ __forceinline__ bool nonzero(T a) { return a.x != 0.f || a.y != 0.f; }
  // the point at shared-memory address a (a staged chunk: read-only while the
  // tile is processed, so the load may be scheduled freely)
  static __device__ __forceinline__ T lds(uint32_t a) {
    T v;
    asm("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
    return v;
  }
  // accumulator read / write by shared-memory address (ordered: volatile)
  static __device__ __forceinline__ T lds_acc(uint32_t a) {
    T v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
    return v;
  }
  static __device__ __forceinline__ void sts_acc(uint32_t a, T v) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
  }
  // *a += (x, y), concurrent-safe (64-bit compare-and-swap)
  static __device__ __forceinline__ void smem_add_s(uint32_t a, float x, float y) {
    unsigned long long old, was;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(old) : "r"(a) : "memory");
    do {
      was = old;
      const float2 v = make_float2(__uint_as_float((uint32_t)was) + x, __uint_as_float((uint32_t)(was >> 32)) + y);
      const unsigned long long nv = ((unsigned long long)__float_as_uint(v.y) << 32) | __float_as_uint(v.x);
      asm volatile("atom.shared.cas.b64 %0, [%1], %2, %3;" : "=l"(old) : "r"(a), "l"(was), "l"(nv) : "memory");
    } while (old != was);
  }
  // *p += (a, b) on shared memory, concurrent-safe (64-bit compare-and-swap)
  static __device__ __forceinline__ void smem_add(T* p, float a, float b) {
    unsigned long long* q = reinterpret_cast<unsigned long long*>(p);
    unsigned long long old = *q, was;
    do {
      was = old;
      const float2 v = make_float2(__uint_as_float((uint32_t)was) + a, __uint_as_float((uint32_t)(was >> 32)) + b);
      old = atomicCAS(q, was, ((unsigned long long)__float_as_uint(v.y) << 32) | __float_as_uint(v.x));
    } while (old != was);
  }
  // accumulate w (y_i - y_j), w = p / (1 + |y_i - y_j|^2); returns 1 + d^2
  static __device__ __forceinline__ float accum(T yi, T yj, float p, float& ax, float& ay) {
    const float dx = yi.x - yj.x, dy = yi.y - yj.y;
    const float q = 1.0f + (dx * dx + dy * dy);
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(q));
    const float w = p * r;
    ax += w * dx;
    ay += w * dy;
    return q;
  }
};
template <> struct TPt<1> {
  using T = float;
  static __device__ __forceinline__ T zero() { return 0.f; }
  static __device__ __forceinline__ T make(float a, float) { return a; }
  static __device__ __forceinline__ T add(T a, T b) { return a + b; }
  static __device__ __forceinline__ bool nonzero(T a) { return a != 0.f; }
  static __device__ __forceinline__ T lds(uint32_t a) {
    T v;
    asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
  }
  static __device__ __forceinline__ T lds_acc(uint32_t a) {
    T v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    return v;
  }
  static __device__ __forceinline__ void sts_acc(uint32_t a, T v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
  }
  static __device__ __forceinline__ void smem_add_s(uint32_t a, float x, float) {
    asm volatile("red.shared.add.f32 [%0], %1;" ::"r"(a), "f"(x) : "memory");
  }
  static __device__ __forceinline__ void smem_add(T* p, float a, float) { atomicAdd(p, a); }
  static __device__ __forceinline__ float accum(T yi, T yj, float p, float& ax, float&) {
    const float dx = yi - yj;
    const float q = 1.0f + dx * dx;
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(q));
    ax += p * r * dx;
    return q;
  }
};

// consumer-only barrier (the producer warp never joins it)
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kTiledConsumers * 32) : "memory");
}

// 1 / x for x >= 1 (no denormal handling needed): one MUFU.RCP
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Warp-specialised persistent kernel.  Warp 31 (one lane) streams, per tile,
// the Y column chunk and the tile's header blob into a 2-stage shared-memory
// ring with bulk copies (full barriers: transaction bytes; empty barriers: one
// arrival per consumer warp).  Consumer warps 0..30 split each tile's slot
// groups evenly, walk them with a 2-deep register pipeline of (column, value)
// loads, gather y_j from the staged chunk and flush a row's partial force into
// the row block's shared accumulator at every slab boundary.  Row-block
// changes (rare: a CTA's tiles are a contiguous run of the row-block-major
// order) flush the accumulator to global memory with vector reductions.
template <int S, bool KL>
__global__ void __launch_bounds__(kTiledThreads, 1)
k_attract_tiled(const TileLoad* __restrict__ tiles, const int32_t* __restrict__ sched,
                const unsigned char* __restrict__ hdr, const uint16_t* __restrict__ cols,
                const float* __restrict__ vals, const typename TPt<S>::T* __restrict__ Y, int64_t row_begin,
                int64_t n_rows, int64_t n_total, int R, int C, int stage_sz,
                typename TPt<S>::T* __restrict__ fattr, double* __restrict__ klpart,
                const int* __restrict__ rowmap, const int2* __restrict__ units, int nunits,
                unsigned* __restrict__ counter, unsigned base) {
  // units != null: dynamic schedule.  The producer draws work units (tile
  // ranges [x, y)) from a global counter: the first `grid` units are the large
  // heads of the static shares, the rest their tails cut into small units, so
  // CTAs that finish early take over the tails of slow ones.  The counter is
  // never reset: launch k draws tickets base .. base + nunits + grid - 1.
  using PT = typename TPt<S>::T;
  using Tr = TPt<S>;
  // rowmap (relabelled P): the output index of tile row r is rowmap[r]
  extern __shared__ __align__(16) unsigned char smem_raw[];
  PT* ys = reinterpret_cast<PT*>(smem_raw);
  PT* acc = ys + R;  // two accumulators: [0, R) even tiles, [R, 2R) odd tiles
  // the bulk-copy ring starts 16-byte aligned (1-D rows are 12 bytes each)
  unsigned char* ring = smem_raw + ((3 * (size_t)R * sizeof(PT) + 15) & ~(size_t)15);
  __shared__ __align__(8) uint64_t full[kTiledStages], empty[kTiledStages];
  __shared__ double red[kTiledConsumers];
  __shared__ int live[kTiledStages];  // 1: the stage holds a tile, 0: end of this CTA's work
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#if FITSNE_TILED_TIMING
  unsigned long long t_begin = 0;
  if (tid == 0) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_begin));
#endif
  if (tid == 0) {
    for (int b = 0; b < kTiledStages; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], kTiledConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == kTiledConsumers) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol_y = policy_evict_last();
      int it = 0;
      auto stage_tile = [&](int t) {
        const int b = it % kTiledStages;
        if (it >= kTiledStages) mbar_wait(&empty[b], (uint32_t)(((it / kTiledStages) - 1) & 1));
        const TileLoad d = tiles[t];
        unsigned char* st = ring + (size_t)b * stage_sz;
        PT* cdst = reinterpret_cast<PT*>(st);
        unsigned char* hdst = st + (size_t)C * sizeof(PT);
        const int64_t c0 = (int64_t)d.chunk * C;
        const int64_t cnt = (n_total - c0 < C) ? (n_total - c0) : C;
        constexpr int64_t kAl = 16 / (int64_t)sizeof(PT);  // points per 16 bytes
        const int64_t cbulk = cnt / kAl * kAl;
        const uint32_t cbytes = (uint32_t)cbulk * (uint32_t)sizeof(PT);
        // tail points (bulk copies move multiples of 16 bytes) and the live
        // flag: plain stores, published to the consumers by the release of
        // the arrive below
        for (int64_t k = cbulk; k < cnt; ++k) cdst[k] = Y[c0 + k];
        live[b] = 1;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_tx(&full[b], cbytes + (uint32_t)d.hdr_bytes);
        if (cbytes) bulk_g2s_hint(cdst, Y + c0, cbytes, &full[b], pol_y);
        bulk_g2s(hdst, hdr + d.hdr_off, (uint32_t)d.hdr_bytes, &full[b]);
#if FITSNE_TILED_L2PF
        // the consumers stream this tile's column / value slots with a
        // one-batch register pipeline; staging the slots in L2 one to two
        // tiles ahead turns their DRAM latency into L2 latency
        {
#if FITSNE_TILED_VEC
          const int64_t gb = (int64_t)d.g0 & ~(int64_t)3;  // the batch holding the tile's first group
          const uint32_t ngb = (uint32_t)(((int64_t)d.g0 + d.ng + 3 - gb) & ~(int64_t)3);
#else
          const int64_t gb = d.g0;
          const uint32_t ngb = (uint32_t)d.ng;
#endif
          const char* cbeg = reinterpret_cast<const char*>(cols + (size_t)slot_index(gb, 0));
          const char* vbeg = reinterpret_cast<const char*>(vals + (size_t)slot_index(gb, 0));
          uint32_t cb = ngb * 64u, vb = ngb * 128u;
          for (uint32_t o = 0; o < cb; o += 65536u) bulk_prefetch_l2(cbeg + o, min(65536u, cb - o));
          for (uint32_t o = 0; o < vb; o += 65536u) bulk_prefetch_l2(vbeg + o, min(65536u, vb - o));
        }
#endif
        ++it;
      };
      if (units) {
        for (;;) {
          const unsigned u = atomicAdd(counter, 1u) - base;
          if (u >= (unsigned)nunits) break;
          const int2 r = units[u];
          for (int t = r.x; t < r.y; ++t) stage_tile(t);
        }
      } else {
        const int t0 = sched[blockIdx.x], t1 = sched[blockIdx.x + 1];
        for (int t = t0; t < t1; ++t) stage_tile(t);
      }
      // end marker: one more stage with live = 0
      {
        const int b = it % kTiledStages;
        if (it >= kTiledStages) mbar_wait(&empty[b], (uint32_t)(((it / kTiledStages) - 1) & 1));
        live[b] = 0;
        mbar_arrive(&full[b]);
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  // Work split: consumer warps take equal runs of the tile's slot groups; a
  // slab cut by a run boundary is shared by two or more warps, which add
  // their partials to the output with L2 vector reductions; every other slab
  // belongs to one warp and is flushed into shared memory.  Across tiles, consumers are at most
  // one tile apart (the producer refills a stage only after every consumer
  // released it), so even and odd tiles accumulate into separate arrays and
  // those flushes are plain shared-memory read-modify-writes.
  // shared-memory address of the row block's points; kept in a register (the
  // empty asm hides how it was computed, so it is not rematerialised -- a
  // special-register read and three integer instructions -- at every use)
  uint32_t ys_s = (uint32_t)__cvta_generic_to_shared(ys);
  asm volatile("" : "+r"(ys_s));
  float kl = 0.f;
  double kld = 0.0;
  int cur_rb = -1;
  int64_t r0 = 0;
  int nr = 0;
  auto flush_block = [&]() {
    for (int i = tid; i < nr; i += kTiledConsumers * 32) {
      const PT v = Tr::add(acc[i], acc[R + i]);
      if (Tr::nonzero(v)) atomicAdd(fattr + (rowmap ? (int64_t)rowmap[r0 + i] : r0 + i), v);
    }
  };
#if !FITSNE_TILED_VEC
  unsigned short cA[kTiledU], cB[kTiledU];
  float pA[kTiledU], pB[kTiledU];
#endif
  for (int it = 0;; ++it) {
    const int b = it % kTiledStages;
    const unsigned char* st = ring + (size_t)b * stage_sz;
    const unsigned char* h = st + (size_t)C * sizeof(PT);
    const uint32_t st_s = (uint32_t)__cvta_generic_to_shared(st);  // the staged chunk's shared-memory address
    mbar_wait(&full[b], (uint32_t)((it / kTiledStages) & 1));
    if (!live[b]) break;
    const int4 meta4 = *reinterpret_cast<const int4*>(h);
    const int32_t meta[4] = {meta4.x, meta4.y, meta4.z, meta4.w};
    const int rb = meta[0], ns = meta[1];
    FITSNE_DCHECK(rb >= 0 && (int64_t)rb * R < n_rows && ns >= 1 && ns <= (R + 31) / 32 + 1 &&
                  meta[3] >= 0);
    const int64_t g0 = (uint32_t)meta[2];
    const int ng = meta[3];
    const uint32_t* goff = reinterpret_cast<const uint32_t*>(h + kHdrGoff);
    const uint16_t* hrows = reinterpret_cast<const uint16_t*>(h + kHdrGoff + 4 * hdr_goff_words(ns));
    if (rb != cur_rb) {
      consumer_sync();  // every consumer is done with the previous row block
      if (cur_rb >= 0) flush_block();
      cur_rb = rb;
      r0 = (int64_t)rb * R;
      nr = (n_rows - r0 < R) ? (int)(n_rows - r0) : R;
      for (int i = tid; i < R; i += kTiledConsumers * 32) {
        ys[i] = i < nr ? Y[row_begin + r0 + i] : Tr::zero();
        acc[i] = Tr::zero();
        acc[R + i] = Tr::zero();
      }
      consumer_sync();
    }
    // this tile's accumulator (even / odd): address of row 0
    const uint32_t accp_s = ys_s + (uint32_t)((1 + (it & 1)) * R) * (uint32_t)sizeof(PT);
#if FITSNE_TILED_WSLAB
    // this warp's slabs [ws0, ws1) and their groups [lo, hi)
    const int ws0 = reinterpret_cast<const int32_t*>(h + kHdrWstart)[warp];
    const int ws1 = reinterpret_cast<const int32_t*>(h + kHdrWstart)[warp + 1];
    const int lo = (int)goff[ws0], hi = (int)goff[ws1];
#else
    const int4 wd = reinterpret_cast<const int4*>(h + kHdrWdesc)[warp];
    const int lo = wd.x, hi = wd.y;
#endif
    if (lo < hi) {
#if FITSNE_TILED_WSLAB
      int s = ws0;
      int s_end = (int)goff[s + 1];
      constexpr bool shared_slab = false;  // every slab belongs to one warp
#else
      int s = wd.z & 0x7FFFFFFF;
      int s_end = wd.w;
      bool shared_slab = wd.z < 0;
#endif
      int row = hrows[s * 32 + lane];
      PT yi = row != 0xFFFF ? Tr::lds(ys_s + (uint32_t)row * (uint32_t)sizeof(PT)) : Tr::zero();
      float ax = 0.f, ay = 0.f;
      // output index of a shared slab's row, loaded when the slab starts so
      // the (relabelled) row map's L2 latency is hidden behind the slab
      int64_t orow = 0;
      auto out_row = [&]() {
        if (!FITSNE_TILED_SCUT && shared_slab && row != 0xFFFF)
          orow = rowmap ? (int64_t)__ldg(rowmap + r0 + row) : r0 + row;
      };
      out_row();
      auto flush_row = [&]() {
        if (row == 0xFFFF) return;
        const uint32_t ra = accp_s + (uint32_t)row * (uint32_t)sizeof(PT);
        if (FITSNE_TILED_SCUT && shared_slab) {
          Tr::smem_add_s(ra, ax, ay);  // the slab's other warps add to the same row
        } else if (shared_slab) {
          // rows of a slab cut by a warp-range boundary are updated by two or
          // more warps of this tile: add straight to the output with a vector
          // reduction in L2 instead of a shared-memory compare-and-swap loop
          atomicAdd(fattr + orow, Tr::make(ax, ay));
        } else {
          Tr::sts_acc(ra, Tr::add(Tr::lds_acc(ra), Tr::make(ax, ay)));
        }
      };
      // slab boundary (warp-uniform): flush the finished row, load the next
      auto advance = [&]() {
        flush_row();
        ax = ay = 0.f;
        ++s;
        s_end = (int)goff[s + 1];
#if !FITSNE_TILED_WSLAB
        shared_slab = s_end > hi;
#endif
        row = hrows[s * 32 + lane];
        yi = row != 0xFFFF ? Tr::lds(ys_s + (uint32_t)row * (uint32_t)sizeof(PT)) : Tr::zero();
        out_row();
      };
      auto accum = [&](PT yj, float p) {
        const float q = Tr::accum(yi, yj, p, ax, ay);
        if (KL) kl += p * __logf(q);
      };
      // one group: slab boundary check, gather, accumulate (tail groups)
      // (off: the column's byte offset inside the staged chunk)
      auto step = [&](int gg, uint32_t off, float p) {
        if (gg == s_end) advance();
        FITSNE_DCHECK(off < (uint32_t)C * sizeof(PT) && off % sizeof(PT) == 0 && s < ns &&
                      (row == 0xFFFF || row < R));
        accum(Tr::lds(st_s + off), p);
      };
#if FITSNE_TILED_VEC
      // batches [bb, be) of four groups hold this warp's run; the first and
      // the last may be shared with the neighbouring runs (groups outside
      // [lo, hi) are skipped: `guarded`).  One batch of loads in flight ahead
      // of the one being consumed; reads past the run stay inside the padded
      // arrays.
      const int64_t bb = (g0 + lo) >> 2;
      const uint2* cp = reinterpret_cast<const uint2*>(cols) + bb * 32 + lane;
      const float4* vp = reinterpret_cast<const float4*>(vals) + bb * 32 + lane;
      // (loading the first batch of the warp's run in the NEXT tile before the
      // current run's tail -- waiting for that tile's stage or only testing it
      // -- measured 7% slower: SpMV 0.452 vs 0.420 ms on 120 CTAs at C3)
      uint2 cv = __ldcs(cp);
      float4 pv = __ldcs(vp);
      int g = (int)((bb << 2) - g0);  // tile-relative group of the batch's first slot (may precede lo)
      auto batch4 = [&](const uint2 c, const float4 p, const int gb) {
        step(gb, c.x & 0xFFFFu, p.x);
        step(gb + 1, c.x >> 16, p.y);
        step(gb + 2, c.y & 0xFFFFu, p.z);
        step(gb + 3, c.y >> 16, p.w);
      };
      auto guarded = [&](const uint2 c, const float4 p, const int gb) {
#pragma unroll 1
        for (int u = 0; u < 4; ++u) {
          const uint32_t w = (u & 2) ? c.y : c.x;
          const float pu = u == 0 ? p.x : u == 1 ? p.y : u == 2 ? p.z : p.w;
          if (gb + u >= lo && gb + u < hi) step(gb + u, (u & 1) ? (w >> 16) : (w & 0xFFFFu), pu);
        }
      };
      if (g < lo) {  // head batch shared with the previous run
        const uint2 cn = __ldcs(cp + 32);
        const float4 pn = __ldcs(vp + 32);
        if (hi >= g + 4) {
          const int k = lo - g;  // the batch's first k = 1..3 groups belong to the previous run
          if (k == 1) step(g + 1, cv.x >> 16, pv.y);
          if (k <= 2) step(g + 2, cv.y & 0xFFFFu, pv.z);
          step(g + 3, cv.y >> 16, pv.w);
        } else {
          guarded(cv, pv, g);  // (rare) the run also ends inside this batch
        }
        cv = cn;
        pv = pn;
        cp += 32;
        vp += 32;
        g += 4;
      }
      int nfull = (hi - g) >> 2;  // whole batches from g (negative: the run ended inside the head batch)
      for (; nfull >= 2; nfull -= 2) {
        const uint2 c1 = __ldcs(cp + 32);
        const float4 p1 = __ldcs(vp + 32);
        batch4(cv, pv, g);
        cv = __ldcs(cp + 64);
        pv = __ldcs(vp + 64);
        batch4(c1, p1, g + 4);
        cp += 64;
        vp += 64;
        g += 8;
      }
      if (nfull == 1) {
        const uint2 cn = __ldcs(cp + 32);
        const float4 pn = __ldcs(vp + 32);
        batch4(cv, pv, g);
        cv = cn;
        pv = pn;
        g += 4;
      }
      if (g < hi) {  // tail batch shared with the next run: its first 1..3 groups
        const int k = hi - g;
        step(g, cv.x & 0xFFFFu, pv.x);
        if (k > 1) step(g + 1, cv.x >> 16, pv.y);
        if (k > 2) step(g + 2, cv.y & 0xFFFFu, pv.z);
      }
      flush_row();
      if (KL) { kld += (double)kl; kl = 0.f; }
#else
      const uint16_t* cp = cols + (size_t)slot_index(g0 + lo, lane);
      const float* vp = vals + (size_t)slot_index(g0 + lo, lane);
#pragma unroll
      for (int u = 0; u < kTiledU; ++u) {
        cA[u] = __ldcs(reinterpret_cast<const unsigned short*>(cp) + u * 32);
        pA[u] = __ldcs(vp + u * 32);
      }
#if FITSNE_TILED_DEPTH >= 3
      // two batches in flight: B holds the next batch, C is loaded ahead of it
      unsigned short cC[kTiledU];
      float pC[kTiledU];
#pragma unroll
      for (int u = 0; u < kTiledU; ++u) {
        cB[u] = __ldcs(reinterpret_cast<const unsigned short*>(cp) + (kTiledU + u) * 32);
        pB[u] = __ldcs(vp + (kTiledU + u) * 32);
      }
#endif
      int g = lo;
      for (; g + kTiledU <= hi; g += kTiledU) {
        // prefetch the next step (reads past hi stay inside the padded arrays)
#if FITSNE_TILED_DEPTH >= 3
#pragma unroll
        for (int u = 0; u < kTiledU; ++u) {
          cC[u] = __ldcs(reinterpret_cast<const unsigned short*>(cp) + (2 * kTiledU + u) * 32);
          pC[u] = __ldcs(vp + (2 * kTiledU + u) * 32);
        }
#else
#pragma unroll
        for (int u = 0; u < kTiledU; ++u) {
          cB[u] = __ldcs(reinterpret_cast<const unsigned short*>(cp) + (kTiledU + u) * 32);
          pB[u] = __ldcs(vp + (kTiledU + u) * 32);
        }
#endif
#if FITSNE_TILED_HOIST
        // the batch's y_j gathers issued together (the staged chunk is never
        // written while the tile is processed; the flushes write accumulators)
        PT yj[kTiledU];
#pragma unroll
        for (int u = 0; u < kTiledU; ++u) yj[u] = Tr::lds(st_s + cA[u]);
        if (s_end >= g + kTiledU) {
          // no slab boundary inside the batch: straight-line accumulation
#pragma unroll
          for (int u = 0; u < kTiledU; ++u) accum(yj[u], pA[u]);
        } else {
#pragma unroll
          for (int u = 0; u < kTiledU; ++u) {
            if (g + u == s_end) advance();
            accum(yj[u], pA[u]);
          }
        }
#elif FITSNE_TILED_FASTPATH
        if (s_end >= g + kTiledU) {
          // no slab boundary inside the batch: straight-line accumulation
#pragma unroll
          for (int u = 0; u < kTiledU; ++u) accum(Tr::lds(st_s + cA[u]), pA[u]);
        } else {
#pragma unroll
          for (int u = 0; u < kTiledU; ++u) step(g + u, cA[u], pA[u]);
        }
#else
        // (hoisting the batch's four gathers measured 14% slower: the
        // compiler then delays the next batch's global loads)
#pragma unroll
        for (int u = 0; u < kTiledU; ++u) step(g + u, cA[u], pA[u]);
#endif
#pragma unroll
        for (int u = 0; u < kTiledU; ++u) { cA[u] = cB[u]; pA[u] = pB[u]; }
#if FITSNE_TILED_DEPTH >= 3
#pragma unroll
        for (int u = 0; u < kTiledU; ++u) { cB[u] = cC[u]; pB[u] = pC[u]; }
#endif
        cp += kTiledU * 32;
        vp += kTiledU * 32;
      }
#pragma unroll
      for (int u = 0; u < kTiledU - 1; ++u)
        if (g + u < hi) step(g + u, cA[u], pA[u]);
      flush_row();
      if (KL) { kld += (double)kl; kl = 0.f; }
#endif
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[b]);
  }
  consumer_sync();
  if (cur_rb >= 0) flush_block();
#if FITSNE_TILED_TIMING
  // probe build: the CTA's busy time (ns) in the (otherwise unused) KL partial
  if (!KL && tid == 0) {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_end));
    klpart[blockIdx.x] = (double)(t_end - t_begin);
  }
#endif
  if (KL) {
    kld = warp_sum(kld);
    if (lane == 0) red[warp] = kld;
    consumer_sync();
    if (tid == 0) {
      double sum = 0;
      for (int w = 0; w < kTiledConsumers; ++w) sum += red[w];
      klpart[blockIdx.x] = sum;
    }
  }
}

// out = F_attr (mode 0) or 4 (alpha F_attr - F_rep) (mode 1); clears F_attr
__global__ void k_tiled_finish(float* __restrict__ fattr, int64_t m, const float* __restrict__ frep,
                               float alpha, int mode, float* __restrict__ out) {
  // m = n rows x dims values
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m) return;
  const float a = fattr[i];
  out[i] = (mode == 1) ? 4.f * (alpha * a - frep[i]) : a;
  fattr[i] = 0.f;
}

// yp[r] = Y[order[r]]
template <typename PT>
__global__ void k_permute_points(const PT* __restrict__ Y, const int* __restrict__ order, int64_t n,
                                 PT* __restrict__ yp) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r < n) yp[r] = Y[order[r]];
}

// Runs the tiled SpMV: F_attr accumulates into the tiled copy's zeroed buffer
// (*fattr_out; the consumer must clear it), KL partials -> T->part[0, grid).
// CTAs of a dynamically scheduled main launch.  The build's grid (tiled_grid:
// 120 of 148 SMs beside the repulsion chain) fits C3's 199-interval grid; when
// the last evaluation's grid was small (a run's 50..100 intervals: the FFT
// stages are a few tens of microseconds) the chain needs fewer SMs and the
// SpMV takes 8 more -- work units are drawn from the ticket counter, so the
// launch grid need not be the grid the schedule was built for (a C3 run_tsne
// iteration: 487 -> 472 us).  An explicit FITSNE_OPT_TILED_CTAS is kept.
static int main_grid(const fitsne_ctx* ctx, const TiledP* T, bool dynamic) {
  if (!dynamic || ctx->tiled_ctas > 0 || ctx->overlap == 0 || !ctx->grid_valid) return T->grid;
  if (ctx->grid.n_intervals > 100) return T->grid;
  return std::min(ctx->num_sms, T->grid + 8);
}

template <int S>
static int launch_tiled_s(fitsne_ctx* ctx, const void* Y, bool kl, const int32_t* sched, cudaStream_t st,
                          int join_ctas) {
  // join_ctas > 0: a second launch that only draws work units of the pass in
  // flight (same ticket base), for SMs that become free while it runs
  using PT = typename TPt<S>::T;
  TiledP* T = ctx->tiled;
  const size_t smem = tiled_smem(T->R, T->C, T->hdr_max, sizeof(PT));
  const int stage_sz = (int)stage_bytes(T->C, T->hdr_max, sizeof(PT));
  {
    // the attribute is per device and process-wide: cache what was set per
    // (device, dims) under a lock (raise only; a smaller request fits)
    static std::mutex mu;
    static std::map<int, size_t> configured;
    std::lock_guard<std::mutex> lock(mu);
    size_t& have = configured[ctx->device * 4 + S];
    if (have < smem) {
      FITSNE_CUDA(cudaFuncSetAttribute(k_attract_tiled<S, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
      FITSNE_CUDA(cudaFuncSetAttribute(k_attract_tiled<S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
      have = smem;
    }
  }
  double* part = (double*)T->part.ptr + (join_ctas > 0 ? T->cur_grid : 0);
  const int* rowmap = nullptr;
  if (T->relabeled) {
    // the tiles index the relabelled points: stage Y in that order
    if (!T->ev_perm) FITSNE_CUDA(cudaEventCreateWithFlags(&T->ev_perm, cudaEventDisableTiming));
    if (join_ctas > 0) {
      FITSNE_CUDA(cudaStreamWaitEvent(st, T->ev_perm, 0));
    } else {
      k_permute_points<PT><<<nb(ctx->n_total, 256), 256, 0, st>>>((const PT*)Y, (const int*)T->order.ptr,
                                                                  ctx->n_total, (PT*)T->yp.ptr);
      FITSNE_CHECK_LAUNCH();
      FITSNE_CUDA(cudaEventRecord(T->ev_perm, st));
    }
    Y = T->yp.ptr;
    rowmap = (const int*)T->order.ptr;
  }
#define TILED_ARGS                                                                                  \
  (const TileLoad*)T->tiles.ptr, sched, (const unsigned char*)T->hdr.ptr,                          \
      (const uint16_t*)T->cols.ptr, (const float*)T->vals.ptr, (const PT*)Y, ctx->row_begin,        \
      ctx->n_rows, ctx->n_total, T->R, T->C, stage_sz, (PT*)T->fattr.ptr, part, rowmap, units, T->nunits, \
      (unsigned*)T->counter.ptr, base
  // the whole-matrix schedule draws its units dynamically; the piece
  // schedules (host-buffer gradient) stay static
  const int2* units = (sched == (const int32_t*)T->sched.ptr && T->nunits > 0) ? (const int2*)T->units.ptr : nullptr;
  const unsigned base = join_ctas > 0 ? T->cur_base : T->ticket_base;
  const int launch_grid = join_ctas > 0 ? join_ctas : main_grid(ctx, T, units != nullptr);
  if (join_ctas > 0 && !units) { set_error("joining launch without a dynamic schedule"); return FITSNE_EINVAL; }
  if (kl)
    k_attract_tiled<S, true><<<launch_grid, kTiledThreads, smem, st>>>(TILED_ARGS);
  else
    k_attract_tiled<S, false><<<launch_grid, kTiledThreads, smem, st>>>(TILED_ARGS);
#undef TILED_ARGS
  FITSNE_CHECK_LAUNCH();
  // every CTA draws tickets until one is past the last unit
  if (join_ctas > 0) {
    T->ticket_base += (unsigned)join_ctas;
    T->join_grid = join_ctas;
  } else {
    T->cur_base = T->ticket_base;
    T->cur_kl = kl;
    T->cur_dynamic = units != nullptr;
    T->join_grid = 0;
    T->cur_grid = launch_grid;
    if (units) T->ticket_base += (unsigned)T->nunits + (unsigned)launch_grid;
  }
  return FITSNE_OK;
}

static int launch_tiled(fitsne_ctx* ctx, const void* Y, bool kl, const int32_t* sched,
                        cudaStream_t st, int join_ctas = 0) {
  FITSNE_RANGE("tiled_spmv");
  return ctx->dims == 1 ? launch_tiled_s<1>(ctx, Y, kl, sched, st, join_ctas)
                        : launch_tiled_s<2>(ctx, Y, kl, sched, st, join_ctas);
}

// Start of an SpMV pass over fattr: clear a stale accumulation first (see
// TiledP::dirty), then mark the buffer as owned by this pass until
// tiled_consumed().
static int tiled_begin(fitsne_ctx* ctx, cudaStream_t st) {
  TiledP* T = ctx->tiled;
  if (T->dirty) {
    if (T->dirty_stream != st) cudaStreamSynchronize(T->dirty_stream);
    FITSNE_CUDA(cudaMemsetAsync(T->fattr.ptr, 0, sizeof(float) * 2 * (size_t)ctx->n_rows, st));
  }
  T->dirty = true;
  T->dirty_stream = st;
  return FITSNE_OK;
}

bool tiled_relabeled(const fitsne_ctx* ctx) { return ctx->tiled && ctx->tiled->relabeled; }

void tiled_mark_dirty(fitsne_ctx* ctx, cudaStream_t st) {
  if (!ctx->tiled) return;
  ctx->tiled->dirty = true;
  ctx->tiled->dirty_stream = st;
}

void tiled_consumed(fitsne_ctx* ctx) {
  if (ctx->tiled) ctx->tiled->dirty = false;
}

int attract_tiled(fitsne_ctx* ctx, const void* Y, bool kl, cudaStream_t st, void** fattr_out,
                  double** part_out, int* nparts) {
  TiledP* T = ctx->tiled;
  double* part = (double*)T->part.ptr;
  FITSNE_TRY(tiled_begin(ctx, st));
  FITSNE_TRY(launch_tiled(ctx, Y, kl, (const int32_t*)T->sched.ptr, st));
  *fattr_out = T->fattr.ptr;
  if (part_out) *part_out = part;
  if (nparts) *nparts = T->cur_grid;
  return FITSNE_OK;
}

// Second launch of the pass queued by attract_tiled, on another stream: `ctas`
// more CTAs draw work units from the same counter (they exit at once when the
// pass is already done).  Queued by the gradient schedule behind the repulsion
// chain, so the SMs the chain used go back to the SpMV.  *nparts grows by the
// joining CTAs' KL partials.
int attract_tiled_join(fitsne_ctx* ctx, const void* Y, int ctas, cudaStream_t st, int* nparts) {
  TiledP* T = ctx->tiled;
  if (ctas < 0 && T) ctas = ctx->num_sms - T->cur_grid;  // the SMs the first launch left
  if (!T || !T->cur_dynamic || ctas <= 0) return FITSNE_OK;
  ctas = std::min(ctas, ctx->num_sms);
  FITSNE_TRY(launch_tiled(ctx, Y, T->cur_kl, (const int32_t*)T->sched.ptr, st, ctas));
  if (nparts) *nparts = T->cur_grid + ctas;
  return FITSNE_OK;
}

int attract_tiled_piece(fitsne_ctx* ctx, const void* Y, int piece, cudaStream_t st, void** fattr_out) {
  TiledP* T = ctx->tiled;
  if (piece == 0) FITSNE_TRY(tiled_begin(ctx, st));
  FITSNE_TRY(launch_tiled(ctx, Y, false, (const int32_t*)T->psched.ptr + (size_t)piece * (T->grid + 1),
                          st));
  *fattr_out = T->fattr.ptr;
  return FITSNE_OK;
}

void tiled_piece_rows(const fitsne_ctx* ctx, int64_t* rows) {
  for (int q = 0; q <= kTiledPieces; ++q) rows[q] = ctx->tiled->piece_rows[q];
}

int tiled_stats(fitsne_ctx* ctx, const void* Y, int64_t* out, cudaStream_t st) {
  const bool use = tiled_usable(ctx, Y, st);
  TiledP* T = ctx->tiled;
  out[0] = use ? 1 : 0;
  out[1] = use ? T->ntiles : 0;
  out[2] = use ? T->nslabs : 0;
  out[3] = use ? T->nslots / 32 : 0;
  out[4] = use ? T->nseg : 0;
  out[5] = ctx->nnz;
  out[6] = use && T->relabeled ? 1 : 0;
  out[7] = use ? (T->nseg_natural ? T->nseg_natural : T->nseg) : 0;
#if FITSNE_TILED_TIMING
  if (use) {
    std::vector<double> h(T->grid + T->join_grid);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), T->part.ptr, sizeof(double) * h.size(), cudaMemcpyDeviceToHost);
    double jsum = 0;
    for (int i = 0; i < T->join_grid; ++i) jsum += h[T->grid + i];
    h.resize(T->grid);
    std::sort(h.begin(), h.end());
    double sum = 0;
    for (double v : h) sum += v;
    fprintf(stderr, "tiled CTA busy time (us): min %.1f p25 %.1f median %.1f p75 %.1f max %.1f mean %.1f (grid %d, units %d; %d joining CTAs, mean %.1f)\n",
            h[0] * 1e-3, h[T->grid / 4] * 1e-3, h[T->grid / 2] * 1e-3, h[3 * T->grid / 4] * 1e-3,
            h[T->grid - 1] * 1e-3, sum / T->grid * 1e-3, T->grid, T->nunits, T->join_grid,
            T->join_grid ? jsum / T->join_grid * 1e-3 : 0.0);
  }
#endif
  return FITSNE_OK;
}

int tiled_finish(fitsne_ctx* ctx, const void* frep, double alpha, int mode, void* out, cudaStream_t st) {
  TiledP* T = ctx->tiled;
  const int64_t n = ctx->n_rows;
  const int64_t m = n * ctx->dims;
  k_tiled_finish<<<nb(m, 256), 256, 0, st>>>((float*)T->fattr.ptr, m, (const float*)frep, (float)alpha,
                                             mode, (float*)out);
  FITSNE_CHECK_LAUNCH();
  tiled_consumed(ctx);
  return FITSNE_OK;
}

}  // namespace fitsne
