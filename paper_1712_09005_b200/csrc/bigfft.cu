// Four-step FFT convolution for grids whose FFT length does not fit one
// block's shared memory (the circulant convolution of nbody.py:262-311 at
// any span: the reference sizes every grid with next_fast_len, nbody.py:134,
// 267, 276, and has no length cap).
//
// A length-L transform along an axis is split L = L1 * L2 (both 2^a 3^b,
// L1 the largest such divisor <= sqrt(L)).  With index j = j1 L2 + j2:
//   pass 1: for each j2, FFT_L1 over j1, then multiply by W_L^(j2 k1);
//   pass 2: for each k1, FFT_L2 over j2.
// Frequency k1 + L1 k2 ends at position k1 L2 + k2 (a fixed permutation), so
// no transposition is needed: the kernel spectrum goes through the same
// passes, the pointwise product is order-free (Parseval's Z too), and the
// inverse passes take the permuted order back to natural order.  Every pass is
// one launch of k_fft_pass: a block loads `cb` sub-transforms (consecutive in
// memory along their batch index, so loads and stores are coalesced) into
// shared memory, runs the Stockham block FFT of fft.cuh, applies the twiddle
// and writes back in place.  Buffers: planes [plane][x][y] of L x L complex
// (2-D) or L complex (1-D), in the context dtype, in HBM.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "fft.cuh"
#include "internal.h"

namespace fitsne {

static constexpr int kBigThreads = 256;

struct PassArgs {
  int m;          // sub-transform length
  int64_t es;     // element stride
  int nb_in;      // inner batch count (a block takes cb consecutive ones)
  int64_t bs_in;  // inner batch stride
  int64_t bs_o2;  // stride of blockIdx.y (outer batch inside a plane)
  int64_t ps;     // plane stride (blockIdx.z)
  int tw_src;     // 0: no twiddle; 1: W_L^(inner index * k); 2: W_L^(blockIdx.y * k)
  int inv;
};

// L = L1 * L2 with L1 the largest 2^a 3^b divisor of L that is <= sqrt(L)
static void split_len(int L, int& L1, int& L2) {
  int best = 1;
  for (long long p2 = 1; p2 <= L; p2 *= 2)
    for (long long v = p2; v <= L; v *= 3)
      if (L % v == 0 && v * v <= L && v > best) best = (int)v;
  L1 = best;
  L2 = L / best;
}

template <typename V, typename T>
__global__ void __launch_bounds__(kBigThreads)
k_fft_pass(V* __restrict__ data, PassArgs a, FftPlan pl, const V* __restrict__ tw_m,
           const V* __restrict__ tw_L, int cb) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int m = a.m, PL = plen(m);
  V* s_tw = reinterpret_cast<V*>(smem_raw);
  V* b0buf = s_tw + m;
  V* b1buf = b0buf + (size_t)cb * PL;
  const int t0 = blockIdx.x * cb;
  const int nt = min(cb, a.nb_in - t0);
  V* base = data + (int64_t)blockIdx.z * a.ps + (int64_t)blockIdx.y * a.bs_o2 + (int64_t)t0 * a.bs_in;
  stage_twiddles(s_tw, tw_m, m);
  const int total = nt * m;
  // element e of sub-transform t: consecutive threads take consecutive
  // addresses (e fastest when the elements are contiguous, else t)
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    int t, e;
    if (a.es == 1) { t = idx / m; e = idx - t * m; }
    else { e = idx / nt; t = idx - e * nt; }
    FITSNE_DCHECK(t < nt && e < m);
    b0buf[(size_t)t * PL + pidx(e)] = base[(int64_t)t * a.bs_in + (int64_t)e * a.es];
  }
  V* r = block_fft<V, T>(b0buf, b1buf, pl, nt, PL, s_tw, a.inv != 0);
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    int t, e;
    if (a.es == 1) { t = idx / m; e = idx - t * m; }
    else { e = idx / nt; t = idx - e * nt; }
    V v = r[(size_t)t * PL + pidx(e)];
    if (a.tw_src) {
      const int64_t ti = (a.tw_src == 1) ? (int64_t)(t0 + t) : (int64_t)blockIdx.y;
      V w = tw_L[ti * e];  // ti * e < L: the two factors index complementary splits
      if (a.inv) w.y = -w.y;
      v = cmul(v, w);
    }
    base[(int64_t)t * a.bs_in + (int64_t)e * a.es] = v;
  }
}

// circulant embedding of (K1 + i K2) (nbody.py:264-281): first[i, j] =
// K((i hx)^2 + (j hy)^2) mirrored into the four quadrants; zero elsewhere
template <typename V, typename T>
__global__ void k_big_kernel(V* __restrict__ K, GridArgs g, int dims) {
  const int L = g.L, n = g.n;
  const int64_t total = (dims == 1) ? (int64_t)L : (int64_t)L * L;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int x = (dims == 1) ? 0 : (int)(q / L);
    const int y = (dims == 1) ? (int)q : (int)(q - (int64_t)x * L);
    const int i = (dims == 1) ? 0 : (x < n ? x : (x > L - n ? L - x : -1));
    const int j = y < n ? y : (y > L - n ? L - y : -1);
    V z;
    z.x = 0;
    z.y = 0;
    if (i >= 0 && j >= 0) {
      double dx = (double)i * g.h[0], dy = (double)j * g.h[dims - 1];
      double d2 = (dims == 1) ? __dmul_rn(dy, dy) : __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
      double base = 1.0 / (1.0 + d2);
      z.x = (T)base;
      z.y = (T)(base * base);
    }
    K[q] = z;
  }
}

// t-SNE charges -> planes W0 = y_0 + i y_1 (centred), W1 = unit; sums and
// clears the accumulator replicas (consume-and-clear, as the fast path)
template <typename V, typename T>
__global__ void k_big_load_tsne(T* __restrict__ acc, int nrep, int64_t rstride, V* __restrict__ W,
                                int64_t ps, int n, int L, int dims) {
  const int64_t G = (dims == 1) ? (int64_t)n : (int64_t)n * n;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < G;
       q += (int64_t)gridDim.x * blockDim.x) {
    T v[3] = {0, 0, 0};
    for (int rp = 0; rp < nrep; ++rp) {
      T* rec = acc + (size_t)rp * rstride + q * kNodeSlots;
      v[0] += rec[0];
      v[1] += rec[1];
      v[2] += rec[2];
      rec[0] = 0;
      rec[1] = 0;
      rec[2] = 0;
    }
    const int64_t pos = (dims == 1) ? q : (q / n) * L + (q % n);
    V a, b;
    a.x = v[1];
    a.y = v[2];
    b.x = v[0];
    b.y = 0;
    W[pos] = a;
    W[ps + pos] = b;
  }
}

// general coefficients (ncol, G) -> pair planes W_q = c_{2q} + i c_{2q+1}
template <typename V, typename T>
__global__ void k_big_load_general(const T* __restrict__ coeffs, int ncol, V* __restrict__ W, int64_t ps,
                                   int n, int L, int dims) {
  const int64_t G = (dims == 1) ? (int64_t)n : (int64_t)n * n;
  const int npair = (ncol + 1) / 2;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < G;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = (dims == 1) ? q : (q / n) * L + (q % n);
    for (int pr = 0; pr < npair; ++pr) {
      V v;
      v.x = coeffs[(int64_t)(2 * pr) * G + q];
      v.y = (2 * pr + 1 < ncol) ? coeffs[(int64_t)(2 * pr + 1) * G + q] : (T)0;
      W[pr * ps + pos] = v;
    }
  }
}

// pointwise product with the (permuted-order) spectrum; t-SNE also forms the
// Parseval partials of Z = sum K1hat |B|^2 / L^dims - N (optimizer.py:206, 241)
template <typename V, typename T, int MODE>
__global__ void k_big_mul(V* __restrict__ W, int64_t ps, int npl, const V* __restrict__ K, int64_t total,
                          double scale, int kern, int with_k1, double* __restrict__ zpart) {
  double zacc = 0.0;
  const T s = (T)scale;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const V kk = K[q];
    const T k1 = kk.x * s, k2 = kk.y * s;
    if (MODE == 0) {  // t-SNE: W0 * K2, W1 * (K2 + i K1)
      V a = W[q], b = W[ps + q];
      zacc += (double)k1 * ((double)b.x * (double)b.x + (double)b.y * (double)b.y);
      a.x *= k2;
      a.y *= k2;
      V o;
      if (with_k1) {
        o.x = b.x * k2 - b.y * k1;
        o.y = b.x * k1 + b.y * k2;
      } else {
        o.x = b.x * k2;
        o.y = b.y * k2;
      }
      W[q] = a;
      W[ps + q] = o;
    } else {
      const T mk = (kern == FITSNE_CAUCHY) ? k1 : k2;
      for (int pr = 0; pr < npl; ++pr) {
        V v = W[pr * ps + q];
        v.x *= mk;
        v.y *= mk;
        W[pr * ps + q] = v;
      }
    }
  }
  if (MODE == 0) {
    __shared__ double red[kBigThreads / 32];
    zacc = warp_sum(zacc);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = zacc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0;
      for (int w = 0; w < kBigThreads / 32; ++w) t += red[w];
      zpart[blockIdx.x] = t;
    }
  }
}

__global__ void k_big_zfold(const double* __restrict__ zpart, int nb, double n_total, double* __restrict__ scal) {
  __shared__ double red[32];
  double s = 0;
  for (int k = threadIdx.x; k < nb; k += blockDim.x) s += zpart[k];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) t += red[w];
    scal[0] = t - n_total;
  }
}

// planes -> potentials (t-SNE: K2*1, K2*y_0, K2*y_1, K1*1 per node) or
// general outputs (ncol, G); crops the circulant to the n^dims grid
template <typename V, typename T, int MODE>
__global__ void k_big_store(const V* __restrict__ W, int64_t ps, int ncol, int n, int L, int dims, int p,
                            T* __restrict__ pot, T* __restrict__ out) {
  const int64_t G = (dims == 1) ? (int64_t)n : (int64_t)n * n;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < G;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t pos = (dims == 1) ? q : (q / n) * L + (q % n);
    if (MODE == 0) {
      const V a = W[pos], b = W[ps + pos];
      T* rec = pot + ((dims == 1) ? q : pot_node(q / n, q % n, p, n / p)) * kNodeSlots;
      rec[0] = b.x;
      rec[1] = a.x;
      rec[2] = (dims == 1) ? (T)0 : a.y;
      rec[3] = b.y;
    } else {
      const int npair = (ncol + 1) / 2;
      for (int pr = 0; pr < npair; ++pr) {
        const V v = W[pr * ps + pos];
        out[(int64_t)(2 * pr) * G + q] = v.x;
        if (2 * pr + 1 < ncol) out[(int64_t)(2 * pr + 1) * G + q] = v.y;
      }
    }
  }
}

template <typename T>
__global__ void k_big_twiddles(typename C2<T>::type* tw, int L) {
  for (int m = blockIdx.x * blockDim.x + threadIdx.x; m < L; m += gridDim.x * blockDim.x) {
    double s, c;
    sincospi(2.0 * (double)m / (double)L, &s, &c);
    typename C2<T>::type w;
    w.x = (T)c;
    w.y = (T)(-s);
    tw[m] = w;
  }
}

// transforms per block: enough adjacent sub-transforms for 128-byte loads,
// bounded by ~96 KB of shared memory (two blocks per SM)
template <typename V>
static int pass_cb(int m, bool contiguous_elems) {
  int cb = contiguous_elems ? 4 : (int)std::max<size_t>(1, 128 / sizeof(V));
  while (cb > 1 && sizeof(V) * ((size_t)m + 2 * (size_t)cb * plen(m)) > 96 * 1024) cb /= 2;
  return cb;
}

template <typename V, typename T>
static int run_pass(V* data, const PassArgs& a, int nb_o2, int planes, const V* tw_m, const V* tw_L,
                    cudaStream_t st) {
  FftPlan pl;
  make_plan(pl, a.m);
  const int cb = pass_cb<V>(a.m, a.es == 1);
  const size_t smem = sizeof(V) * ((size_t)a.m + 2 * (size_t)cb * plen(a.m));
  if (smem > 48 * 1024)
    FITSNE_CUDA(cudaFuncSetAttribute(k_fft_pass<V, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((a.nb_in + cb - 1) / cb, nb_o2, planes);
  k_fft_pass<V, T><<<grid, kBigThreads, smem, st>>>(data, a, pl, tw_m, tw_L, cb);
  FITSNE_CHECK_LAUNCH();
  return FITSNE_OK;
}

static PassArgs pa(int m, int64_t es, int nb_in, int64_t bs_in, int64_t bs_o2, int64_t ps, int tw_src,
                   int inv) {
  PassArgs a;
  a.m = m;
  a.es = es;
  a.nb_in = nb_in;
  a.bs_in = bs_in;
  a.bs_o2 = bs_o2;
  a.ps = ps;
  a.tw_src = tw_src;
  a.inv = inv;
  return a;
}

// forward (natural -> permuted) or inverse (permuted -> natural) transform
// along the contiguous axis of `nrows` rows (stride L) of `planes` planes
template <typename V, typename T>
static int rows_passes(V* d, int planes, int64_t ps, int nrows, int L, int L1, int L2, const V* tw1,
                       const V* tw2, const V* twL, bool inv, cudaStream_t st) {
  if (!inv) {
    FITSNE_TRY((run_pass<V, T>(d, pa(L1, L2, L2, 1, L, ps, 1, 0), nrows, planes, tw1, twL, st)));
    FITSNE_TRY((run_pass<V, T>(d, pa(L2, 1, L1, L2, L, ps, 0, 0), nrows, planes, tw2, twL, st)));
  } else {
    FITSNE_TRY((run_pass<V, T>(d, pa(L2, 1, L1, L2, L, ps, 1, 1), nrows, planes, tw2, twL, st)));
    FITSNE_TRY((run_pass<V, T>(d, pa(L1, L2, L2, 1, L, ps, 0, 1), nrows, planes, tw1, twL, st)));
  }
  return FITSNE_OK;
}

// the same along the strided axis (x, stride L) of all L columns
template <typename V, typename T>
static int cols_passes(V* d, int planes, int64_t ps, int L, int L1, int L2, const V* tw1, const V* tw2,
                       const V* twL, bool inv, cudaStream_t st) {
  const int64_t Ll = L;
  if (!inv) {
    FITSNE_TRY((run_pass<V, T>(d, pa(L1, (int64_t)L2 * Ll, L, 1, Ll, ps, 2, 0), L2, planes, tw1, twL, st)));
    FITSNE_TRY((run_pass<V, T>(d, pa(L2, Ll, L, 1, (int64_t)L2 * Ll, ps, 0, 0), L1, planes, tw2, twL, st)));
  } else {
    FITSNE_TRY((run_pass<V, T>(d, pa(L2, Ll, L, 1, (int64_t)L2 * Ll, ps, 2, 1), L1, planes, tw2, twL, st)));
    FITSNE_TRY((run_pass<V, T>(d, pa(L1, (int64_t)L2 * Ll, L, 1, Ll, ps, 0, 1), L2, planes, tw1, twL, st)));
  }
  return FITSNE_OK;
}

bool big_fft_applies(const fitsne_ctx* ctx, int L) {
  if (ctx->fft_path == 2) return true;
  if (ctx->fft_path == 1) return false;
  return L > (ctx->dtype == FITSNE_F32 ? 5184 : 2592);
}

template <typename T, int MODE>
static int conv_big_t(fitsne_ctx* ctx, T* accum, int nrep, int64_t rstride, const T* coeffs, int ncol,
                      int kern, bool with_k1, T* out, int64_t n_total, cudaStream_t st) {
  FITSNE_RANGE("four_step_fft");
  using V = typename C2<T>::type;
  const GridArgs g = grid_args(ctx->grid);
  const int L = g.L, n = g.n, dims = ctx->grid.dims;
  if (L > 65535) {
    set_error("interpolation grid needs an FFT longer than 65535");
    return FITSNE_ETOOBIG;
  }
  int L1, L2;
  split_len(L, L1, L2);
  const int64_t plane = (dims == 1) ? (int64_t)L : (int64_t)L * L;
  const int nw = (MODE == 0) ? 2 : (ncol + 1) / 2;  // data planes, then the kernel plane
  const size_t bytes = sizeof(V) * (size_t)plane * (size_t)(nw + 1);
  FITSNE_TRY(ensure(ctx->big, bytes));
  // twiddle tables: W_L (ctx->tw, installed with the grid), W_L1, W_L2
  FITSNE_TRY(ensure(ctx->bigtw, sizeof(V) * (size_t)(L1 + L2)));
  V* tw1 = (V*)ctx->bigtw.ptr;
  V* tw2 = tw1 + L1;
  if (ctx->big_tw_l1 != L1 || ctx->big_tw_l2 != L2) {
    k_big_twiddles<T><<<(L1 + 255) / 256, 256, 0, st>>>(tw1, L1);
    k_big_twiddles<T><<<(L2 + 255) / 256, 256, 0, st>>>(tw2, L2);
    FITSNE_CHECK_LAUNCH();
    ctx->big_tw_l1 = L1;
    ctx->big_tw_l2 = L2;
  }
  const V* twL = (const V*)ctx->tw.ptr;
  V* W = (V*)ctx->big.ptr;
  V* K = W + (size_t)nw * plane;
  const int nb = 4 * ctx->num_sms;
  FITSNE_TRY(ensure(ctx->zpart, sizeof(double) * (size_t)std::max(L, nb)));
  // data planes: zero padding, then the charges / coefficients
  FITSNE_CUDA(cudaMemsetAsync(W, 0, sizeof(V) * (size_t)plane * nw, st));
  if (MODE == 0)
    k_big_load_tsne<V, T><<<nb, 256, 0, st>>>(accum, nrep, rstride, W, plane, n, L, dims);
  else
    k_big_load_general<V, T><<<nb, 256, 0, st>>>(coeffs, ncol, W, plane, n, L, dims);
  FITSNE_CHECK_LAUNCH();
  k_big_kernel<V, T><<<nb, 256, 0, st>>>(K, g, dims);
  FITSNE_CHECK_LAUNCH();
  // forward transforms (only the first n rows of the data planes are non-zero)
  if (dims == 1) {
    FITSNE_TRY((rows_passes<V, T>(W, nw + 1, plane, 1, L, L1, L2, tw1, tw2, twL, false, st)));
  } else {
    FITSNE_TRY((rows_passes<V, T>(W, nw, plane, n, L, L1, L2, tw1, tw2, twL, false, st)));
    FITSNE_TRY((rows_passes<V, T>(K, 1, plane, L, L, L1, L2, tw1, tw2, twL, false, st)));
    FITSNE_TRY((cols_passes<V, T>(W, nw + 1, plane, L, L1, L2, tw1, tw2, twL, false, st)));
  }
  const double scale = 1.0 / (double)plane;
  double* zp = (double*)ctx->zpart.ptr;
  k_big_mul<V, T, MODE><<<nb, kBigThreads, 0, st>>>(W, plane, nw, K, plane, scale, kern, with_k1 ? 1 : 0, zp);
  FITSNE_CHECK_LAUNCH();
  if (MODE == 0) {
    k_big_zfold<<<1, 1024, 0, st>>>(zp, nb, (double)n_total, (double*)ctx->scal.ptr);
    FITSNE_CHECK_LAUNCH();
  }
  // inverse transforms: all columns, then only the n output rows
  if (dims == 1) {
    FITSNE_TRY((rows_passes<V, T>(W, nw, plane, 1, L, L1, L2, tw1, tw2, twL, true, st)));
  } else {
    FITSNE_TRY((cols_passes<V, T>(W, nw, plane, L, L1, L2, tw1, tw2, twL, true, st)));
    FITSNE_TRY((rows_passes<V, T>(W, nw, plane, n, L, L1, L2, tw1, tw2, twL, true, st)));
  }
  k_big_store<V, T, MODE><<<nb, 256, 0, st>>>(W, plane, ncol, n, L, dims, g.p, (T*)ctx->pot.ptr, out);
  FITSNE_CHECK_LAUNCH();
  return FITSNE_OK;
}

int conv_big_tsne(fitsne_ctx* ctx, void* accum, int nrep, int64_t rstride, bool with_k1, int64_t n_total,
                  cudaStream_t st) {
  if (ctx->dtype == FITSNE_F32)
    return conv_big_t<float, 0>(ctx, (float*)accum, nrep, rstride, nullptr, 3, 0, with_k1, nullptr, n_total, st);
  return conv_big_t<double, 0>(ctx, (double*)accum, nrep, rstride, nullptr, 3, 0, with_k1, nullptr, n_total, st);
}

int conv_big_general(fitsne_ctx* ctx, const void* coeffs, int ncol, int kern, void* out, cudaStream_t st) {
  if (ctx->dtype == FITSNE_F32)
    return conv_big_t<float, 1>(ctx, nullptr, 1, 0, (const float*)coeffs, ncol, kern, false, (float*)out, 0, st);
  return conv_big_t<double, 1>(ctx, nullptr, 1, 0, (const double*)coeffs, ncol, kern, false, (double*)out, 0,
                               st);
}

}  // namespace fitsne
