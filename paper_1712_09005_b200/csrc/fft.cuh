// Block-cooperative mixed-radix (2, 3, 4) Stockham FFT in shared memory.
//
// This replaces scipy.fft's pocketfft calls of the reference
// (nbody.py:271, 282, 291-297).  Lengths are L = 2^a 3^b, chosen as the
// smallest such L >= 2n-1 (the reference takes next_fast_len(2n-1) over
// 5-smooth numbers; any L >= 2n-1 gives the same circulant product).
//
// Formulation (autosort, out of place, one pass per radix stage):
//   Ns = product of the radices already applied; for j in [0, L/R):
//     k = j mod Ns, v_r = in[j + r L/R] * w_L^{r k L/(Ns R)}, v = DFT_R(v),
//     out[(j/Ns) Ns R + k + r Ns] = v_r.
// The twiddles come from a table tw[m] = exp(-2 pi i m / L) in global memory
// (L1/L2 resident); the inverse transform uses conjugated twiddles and is
// unnormalised (callers fold 1/L^2 into the kernel spectrum).
#pragma once

#include "common.cuh"

namespace fitsne {

struct FftPlan {
  int nstage;
  int L;
  int radix[24];
  int ns[24];      // Ns before the stage
  int stride[24];  // L / (Ns * R): twiddle index multiplier
  unsigned mlr[24];  // ceil(2^32 / (L/R)): exact x / (L/R) = umulhi(x, mlr) for x < 2^32/(L/R)
  unsigned mns[24];  // ceil(2^32 / Ns)
};

// m = ceil(2^32 / d) for d >= 2; d == 1 is encoded as m = 0 (2^32 does not fit)
__host__ __device__ inline unsigned magic_div(unsigned d) {
  if (d <= 1) return 0u;
  return (unsigned)((((unsigned long long)1 << 32) + d - 1) / d);
}

// exact x / d for x * d < 2^32 (here x < 16 L <= 2^17 and d <= 2^13)
__device__ __forceinline__ unsigned fast_div(unsigned x, unsigned m) {
  return m ? __umulhi(x, m) : x;
}

__host__ __device__ inline bool is_smooth23(int L) {
  if (L < 1) return false;
  while (L % 2 == 0) L /= 2;
  while (L % 3 == 0) L /= 3;
  return L == 1;
}

// smallest 2^a 3^b >= m
__host__ __device__ inline int smooth23_at_least(int m) {
  if (m <= 1) return 1;
  long long best = -1;
  for (long long p2 = 1; p2 < 4LL * m; p2 *= 2) {
    long long v = p2;
    while (v < m) v *= 3;
    if (best < 0 || v < best) best = v;
  }
  return (int)best;
}

__host__ __device__ inline void make_plan(FftPlan& pl, int L) {
  int a = 0, b = 0, m = L;
  while (m % 2 == 0) { m /= 2; ++a; }
  while (m % 3 == 0) { m /= 3; ++b; }
  int s = 0, ns = 1;
  for (int i = 0; i < a / 2; ++i) { pl.radix[s] = 4; pl.ns[s] = ns; ns *= 4; ++s; }
  if (a % 2) { pl.radix[s] = 2; pl.ns[s] = ns; ns *= 2; ++s; }
  for (int i = 0; i < b; ++i) { pl.radix[s] = 3; pl.ns[s] = ns; ns *= 3; ++s; }
  pl.nstage = s;
  pl.L = L;
  for (int i = 0; i < s; ++i) {
    pl.stride[i] = L / (pl.ns[i] * pl.radix[i]);
    pl.mlr[i] = magic_div((unsigned)(L / pl.radix[i]));
    pl.mns[i] = magic_div((unsigned)pl.ns[i]);
  }
}

template <typename V>
__device__ __forceinline__ V twiddle(const V* __restrict__ tw, int idx, bool inv) {
  V w = __ldg(&tw[idx]);
  if (inv) w.y = -w.y;
  return w;
}

// radix butterflies: forward uses e^{-2 pi i / R}, inverse e^{+2 pi i / R}
template <typename V, typename T>
__device__ __forceinline__ void dft2(V& a, V& b) {
  V t = a;
  a.x = t.x + b.x; a.y = t.y + b.y;
  b.x = t.x - b.x; b.y = t.y - b.y;
}

template <typename V, typename T>
__device__ __forceinline__ void dft4(V& a0, V& a1, V& a2, V& a3, bool inv) {
  V s02 = cadd(a0, a2), d02 = csub(a0, a2);
  V s13 = cadd(a1, a3), d13 = csub(a1, a3);
  // -i * d13 (forward) or +i * d13 (inverse)
  V r;
  if (!inv) { r.x = d13.y; r.y = -d13.x; } else { r.x = -d13.y; r.y = d13.x; }
  a0 = cadd(s02, s13);
  a2 = csub(s02, s13);
  a1 = cadd(d02, r);
  a3 = csub(d02, r);
}

template <typename V, typename T>
__device__ __forceinline__ void dft3(V& a0, V& a1, V& a2, bool inv) {
  const T c = (T)-0.5;
  const T s = inv ? (T)0.86602540378443864676 : (T)-0.86602540378443864676;
  V t1 = cadd(a1, a2);
  V t2 = csub(a1, a2);
  V m;  // a0 - t1/2
  m.x = a0.x + c * t1.x;
  m.y = a0.y + c * t1.y;
  // i*s*t2
  V r;
  r.x = -s * t2.y;
  r.y = s * t2.x;
  a0 = cadd(a0, t1);
  a1 = cadd(m, r);
  a2 = csub(m, r);
}

// One Stockham stage over `nsig` signals laid out at in[s*sig + i].
template <typename V, typename T>
__device__ __forceinline__ void fft_stage(const V* __restrict__ in, V* __restrict__ out, int L,
                                          int R, int Ns, int tstride, unsigned mlr, unsigned mns,
                                          int nsig, int sig, const V* __restrict__ tw, bool inv) {
  const int LR = L / R;
  const int total = nsig * LR;
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    int s = (int)fast_div((unsigned)t, mlr);
    int j = t - s * LR;
    int k = j - (int)fast_div((unsigned)j, mns) * Ns;
    const V* src = in + (size_t)s * sig;
    V* dst = out + (size_t)s * sig;
    int base = (j - k) * R + k;  // (j/Ns)*Ns*R + k
    if (R == 4) {
      V a0 = src[j], a1 = src[j + LR], a2 = src[j + 2 * LR], a3 = src[j + 3 * LR];
      if (Ns > 1) {
        int e = k * tstride;
        a1 = cmul(a1, twiddle(tw, e, inv));
        a2 = cmul(a2, twiddle(tw, 2 * e, inv));
        a3 = cmul(a3, twiddle(tw, 3 * e, inv));
      }
      dft4<V, T>(a0, a1, a2, a3, inv);
      dst[base] = a0;
      dst[base + Ns] = a1;
      dst[base + 2 * Ns] = a2;
      dst[base + 3 * Ns] = a3;
    } else if (R == 2) {
      V a0 = src[j], a1 = src[j + LR];
      if (Ns > 1) a1 = cmul(a1, twiddle(tw, k * tstride, inv));
      dft2<V, T>(a0, a1);
      dst[base] = a0;
      dst[base + Ns] = a1;
    } else {  // R == 3
      V a0 = src[j], a1 = src[j + LR], a2 = src[j + 2 * LR];
      if (Ns > 1) {
        int e = k * tstride;
        a1 = cmul(a1, twiddle(tw, e, inv));
        a2 = cmul(a2, twiddle(tw, 2 * e, inv));
      }
      dft3<V, T>(a0, a1, a2, inv);
      dst[base] = a0;
      dst[base + Ns] = a1;
      dst[base + 2 * Ns] = a2;
    }
  }
}

// Full transform of `nsig` signals (stride `sig` elements) held in `a`; `b` is
// scratch of the same size.  Returns the buffer holding the result.  Must be
// called by every thread of the block; begins and ends with a barrier.
template <typename V, typename T>
__device__ V* block_fft(V* a, V* b, const FftPlan& pl, int nsig, int sig,
                        const V* __restrict__ tw, bool inv) {
  __syncthreads();
  for (int st = 0; st < pl.nstage; ++st) {
    fft_stage<V, T>(a, b, pl.L, pl.radix[st], pl.ns[st], pl.stride[st], pl.mlr[st], pl.mns[st],
                    nsig, sig, tw, inv);
    __syncthreads();
    V* t = a; a = b; b = t;
  }
  return a;
}

}  // namespace fitsne
