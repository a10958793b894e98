// Locality relabelling of the points, computed from P alone on the device.
//
// The tiled attractive SpMV (tiled.cu) needs index locality: the rows of a
// row block should find their neighbours in few column chunks.  A kNN graph
// has it only if the points arrive grouped (e.g. by cluster); real data come
// in any order.  This computes a Cuthill-McKee ordering of the symmetric
// pattern of P: breadth-first search, level by level, where the nodes found
// in a level are numbered in the order of the parent that found them first
// (ties by node id), restarting at the next unvisited node when a component
// is exhausted.  Components (clusters) become contiguous label ranges and
// neighbours get nearby labels.  Cost: every stored entry is examined once
// (the visited array, 4 B per point, is L2 resident) plus one radix sort per
// level; one host read of the level size per level.
//
// The relabelling is internal to the tiled copy of P (tiled.cu): the SpMV
// reads a permuted copy of Y and scatters each row's force to its original
// index, so callers see the original order (the reference's compute_attractive,
// optimizer.py:150-166, is order-independent up to summation order).
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace fitsne {

static constexpr int kUnvisited = -1;

// the seed of the first component: a node of minimum degree (a cheap
// pseudo-peripheral choice, as in RCM)
__global__ void k_min_degree(const int64_t* __restrict__ rowptr, int n, unsigned long long* __restrict__ best) {
  unsigned long long b = ~0ull;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const unsigned long long deg = (unsigned long long)(rowptr[i + 1] - rowptr[i]);
    b = min(b, (deg << 32) | (unsigned)i);
  }
  for (int o = 16; o > 0; o >>= 1) b = min(b, __shfl_xor_sync(0xffffffffu, b, o));
  if ((threadIdx.x & 31) == 0) atomicMin(best, b);
}

__global__ void k_visit_seed(int* __restrict__ pos_of, int* __restrict__ order, int seed, int pos) {
  pos_of[seed] = pos;
  order[pos] = seed;
}

// Expand the frontier order[f0, f1): a warp per frontier node walks its
// neighbours; an unvisited neighbour is claimed by the smallest position
// among the frontier nodes that reach it (atomicMin on claim); the first
// claimer appends it to the candidate list.
__global__ void k_expand(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                         const int* __restrict__ order, int f0, int f1, const int* __restrict__ pos_of,
                         int* __restrict__ claim, int* __restrict__ cand, int* __restrict__ ncand) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int f = f0 + w; f < f1; f += nw) {
    const int u = order[f];
    const int64_t b = rowptr[u], e = rowptr[u + 1];
    for (int64_t k = b + lane; k < e; k += 32) {
      const int c = col[k];
      if (__ldcg(pos_of + c) != kUnvisited) continue;
      const int old = atomicMin(claim + c, f);
      if (old == INT_MAX) cand[atomicAdd(ncand, 1)] = c;
    }
  }
}

// candidate keys: (claiming position, node id)
__global__ void k_cand_keys(const int* __restrict__ cand, int m, const int* __restrict__ claim,
                            unsigned long long* __restrict__ key) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int c = cand[i];
  key[i] = ((unsigned long long)(unsigned)claim[c] << 32) | (unsigned)c;
}

// number the sorted candidates pos, pos + 1, ... and reset their claims
__global__ void k_number(const unsigned long long* __restrict__ key, int m, int pos, int* __restrict__ pos_of,
                         int* __restrict__ order, int* __restrict__ claim) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  const int c = (int)(unsigned)(key[i] & 0xffffffffull);
  pos_of[c] = pos + i;
  order[pos + i] = c;
  claim[c] = INT_MAX;
}

// next unvisited node at or after `from` (restart of the search)
__global__ void k_first_unvisited(const int* __restrict__ pos_of, int from, int n, int* __restrict__ out) {
  for (int i = from + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (pos_of[i] == kUnvisited) {
      atomicMin(out, i);
      return;
    }
}

static inline int nblk(int64_t n, int b) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + b - 1) / b, 1 << 20));
}

__global__ void k_fill_int(int* __restrict__ a, int n, int v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = v;
}

// order[new] = old, pos_of[old] = new (device, n ints each)
int cuthill_mckee(const int64_t* rowptr, const int32_t* col, int n, int* order, int* pos_of, int num_sms,
                  cudaStream_t st) {
  FITSNE_RANGE("relabel");
  if (n <= 0) return FITSNE_OK;
  int *claim = nullptr, *cand = nullptr, *cnt = nullptr;
  unsigned long long *key = nullptr, *key2 = nullptr, *best = nullptr;
  void* tmp = nullptr;
  int* h = nullptr;
  size_t tmp_bytes = 0;
  FITSNE_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, key, key2, n, 0, 64, st));
  cudaError_t e = cudaMallocAsync(&claim, sizeof(int) * (size_t)n, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&cand, sizeof(int) * (size_t)n, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&cnt, sizeof(int) * 4, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&key, sizeof(unsigned long long) * (size_t)n, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&key2, sizeof(unsigned long long) * (size_t)n, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&best, sizeof(unsigned long long), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&tmp, std::max<size_t>(tmp_bytes, 16), st);
  if (e == cudaSuccess) e = cudaMallocHost(&h, sizeof(int) * 4);
  int rc = FITSNE_OK;
  const int fb = 8 * num_sms;
  if (e == cudaSuccess) {
    k_fill_int<<<fb, 256, 0, st>>>(pos_of, n, kUnvisited);
    k_fill_int<<<fb, 256, 0, st>>>(claim, n, INT_MAX);
    cudaMemsetAsync(best, 0xff, sizeof(unsigned long long), st);
    k_min_degree<<<fb, 256, 0, st>>>(rowptr, n, best);
    unsigned long long hb = 0;
    cudaMemcpyAsync(&hb, best, sizeof(hb), cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    int seed = (int)(unsigned)(hb & 0xffffffffull);
    int pos = 0;       // labels handed out
    int scan_from = 0; // restarts look for unvisited nodes from here on
    while (e == cudaSuccess && pos < n) {
      k_visit_seed<<<1, 1, 0, st>>>(pos_of, order, seed, pos);
      int f0 = pos, f1 = pos + 1;
      pos += 1;
      // breadth-first levels of this component
      while (e == cudaSuccess && f1 > f0) {
        cudaMemsetAsync(cnt, 0, sizeof(int), st);
        const int64_t warps = (int64_t)(f1 - f0);
        k_expand<<<nblk(warps * 32, 256), 256, 0, st>>>(rowptr, col, order, f0, f1, pos_of, claim, cand, cnt);
        cudaMemcpyAsync(h, cnt, sizeof(int), cudaMemcpyDeviceToHost, st);
        e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) break;
        const int m = h[0];
        if (m == 0) break;
        k_cand_keys<<<nblk(m, 256), 256, 0, st>>>(cand, m, claim, key);
        e = cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, key, key2, m, 0, 64, st);
        if (e != cudaSuccess) break;
        k_number<<<nblk(m, 256), 256, 0, st>>>(key2, m, pos, pos_of, order, claim);
        f0 = pos;
        f1 = pos + m;
        pos += m;
      }
      if (e != cudaSuccess || pos >= n) break;
      // restart at the first unvisited node (labels are handed out in
      // increasing node order for the seeds, so the scan only moves forward)
      h[1] = n;
      cudaMemcpyAsync(cnt + 1, h + 1, sizeof(int), cudaMemcpyHostToDevice, st);
      k_first_unvisited<<<nblk(n - scan_from, 256), 256, 0, st>>>(pos_of, scan_from, n, cnt + 1);
      cudaMemcpyAsync(h + 2, cnt + 1, sizeof(int), cudaMemcpyDeviceToHost, st);
      e = cudaStreamSynchronize(st);
      seed = h[2];
      if (seed >= n) break;  // cannot happen while pos < n
      scan_from = seed + 1;
    }
    if (e == cudaSuccess) e = cudaGetLastError();
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error(std::string("relabelling failed: ") + cudaGetErrorString(e));
    rc = FITSNE_ECUDA;
  }
  if (h) cudaFreeHost(h);
  for (void* p : {(void*)claim, (void*)cand, (void*)cnt, (void*)key, (void*)key2, (void*)best, tmp})
    if (p) cudaFreeAsync(p, st);
  return rc;
}

}  // namespace fitsne
