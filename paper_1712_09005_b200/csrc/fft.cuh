// Block-cooperative mixed-radix Stockham FFT in shared memory with
// register-resident radix-{2,3,4,6,8,9,12,16} butterflies.
//
// This replaces scipy.fft's pocketfft calls of the reference
// (nbody.py:271, 282, 291-297).  Lengths are L = 2^a 3^b, chosen as the
// smallest such L >= 2n-1 (the reference takes next_fast_len(2n-1) over
// 5-smooth numbers; any L >= 2n-1 gives the same circulant product).
//
// Formulation (autosort, out of place, one smem pass per radix stage):
//   Ns = product of the radices already applied; for j in [0, L/R):
//     k = j mod Ns, v_r = in[j + r L/R] * w_L^{r k L/(Ns R)}, v = DFT_R(v),
//     out[(j/Ns) Ns R + k + r Ns] = v_r.
// Radices up to 16 are evaluated in registers (R = A*B split, compile-time
// twiddles), so L = 1296 takes three passes (16, 9, 9) instead of six.
// Shared-memory signals are stored with one pad word per 32 elements
// (pidx) so the strided stores of the first stages are bank-conflict free.
// The global twiddle table holds tw[m] = exp(-2 pi i m / L); the inverse
// transform uses conjugates and is unnormalised.
#pragma once

#include "common.cuh"
#include "twiddles.cuh"

namespace fitsne {

// padded shared-memory layout of one signal
__host__ __device__ __forceinline__ int pidx(int i) { return i + (i >> 5); }
__host__ __device__ __forceinline__ int plen(int L) { return L + (L >> 5) + 1; }

struct FftPlan {
  int nstage;
  int L;
  int radix[16];
  int ns[16];        // Ns before the stage
  int stride[16];    // L / (Ns * R): twiddle index multiplier
  unsigned mlr[16];  // magic for x / (L/R)
  unsigned mns[16];  // magic for x / Ns
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

// radices: 16 while 2^4 | L, 9 while 3^2 | L, then the remainder 2^a 3^b
// (a <= 3, b <= 1) as one radix in {2,3,4,6,8,12} (24 -> 8, 3)
__host__ __device__ inline void make_plan(FftPlan& pl, int L) {
  int a = 0, b = 0, m = L;
  while (m % 2 == 0) { m /= 2; ++a; }
  while (m % 3 == 0) { m /= 3; ++b; }
  int rs[16], nr = 0;
  while (a >= 4) { rs[nr++] = 16; a -= 4; }
  while (b >= 2) { rs[nr++] = 9; b -= 2; }
  int rem = (1 << a) * (b ? 3 : 1);
  if (rem == 24) { rs[nr++] = 8; rs[nr++] = 3; }
  else if (rem > 1) rs[nr++] = rem;
  int ns = 1;
  for (int i = 0; i < nr; ++i) {
    pl.radix[i] = rs[i];
    pl.ns[i] = ns;
    pl.stride[i] = L / (ns * rs[i]);
    pl.mlr[i] = magic_div((unsigned)(L / rs[i]));
    pl.mns[i] = magic_div((unsigned)ns);
    ns *= rs[i];
  }
  pl.nstage = nr;
  pl.L = L;
}

// Device-grid block (device-grid schedule, attract.cu): the grid k_bbox
// computes on the device, the Stockham plan of its FFT length (built once
// there instead of in every FFT block) and the box it came from.
struct DevGrid {
  GridArgs g;
  FftPlan pl;
  double bbox[8];
};
__device__ __forceinline__ const FftPlan* dev_plan(const GridArgs* gd) {
  return &reinterpret_cast<const DevGrid*>(gd)->pl;
}

// `tw` is normally the block's shared-memory copy of the table (stage_twiddles)
template <typename V>
__device__ __forceinline__ V twiddle(const V* __restrict__ tw, int idx, bool inv) {
  V w = tw[idx];
  if (inv) w.y = -w.y;
  return w;
}

// Copy the global twiddle table into shared memory (4 loads in flight per
// thread).  The caller's later block_fft begins with a barrier.
template <typename V>
__device__ __forceinline__ void stage_twiddles(V* __restrict__ s_tw, const V* __restrict__ tw, int L) {
  for (int m0 = threadIdx.x; m0 < L; m0 += 4 * blockDim.x) {
    V w[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int m = m0 + u * blockDim.x;
      if (m < L) w[u] = __ldg(tw + m);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int m = m0 + u * blockDim.x;
      if (m < L) s_tw[m] = w[u];
    }
  }
}

// ---------------------------------------------------------------------------
// register DFTs
// ---------------------------------------------------------------------------
template <int R> struct Split;
template <> struct Split<6> { static constexpr int A = 2, B = 3; };
template <> struct Split<8> { static constexpr int A = 2, B = 4; };
template <> struct Split<9> { static constexpr int A = 3, B = 3; };
template <> struct Split<12> { static constexpr int A = 3, B = 4; };
template <> struct Split<16> { static constexpr int A = 4, B = 4; };

template <typename V, typename T, int R, bool INV>
__device__ __forceinline__ void dft_reg(V (&x)[R]) {
  if constexpr (R == 2) {
    V t = x[0];
    x[0].x = t.x + x[1].x; x[0].y = t.y + x[1].y;
    x[1].x = t.x - x[1].x; x[1].y = t.y - x[1].y;
  } else if constexpr (R == 3) {
    const T c = (T)-0.5;
    const T s = INV ? (T)0.86602540378443864676 : (T)-0.86602540378443864676;
    V t1 = cadd(x[1], x[2]);
    V t2 = csub(x[1], x[2]);
    V m;
    m.x = x[0].x + c * t1.x;
    m.y = x[0].y + c * t1.y;
    V r;
    r.x = -s * t2.y;
    r.y = s * t2.x;
    x[0] = cadd(x[0], t1);
    x[1] = cadd(m, r);
    x[2] = csub(m, r);
  } else if constexpr (R == 4) {
    V s02 = cadd(x[0], x[2]), d02 = csub(x[0], x[2]);
    V s13 = cadd(x[1], x[3]), d13 = csub(x[1], x[3]);
    V r;
    if (!INV) { r.x = d13.y; r.y = -d13.x; } else { r.x = -d13.y; r.y = d13.x; }
    x[0] = cadd(s02, s13);
    x[2] = csub(s02, s13);
    x[1] = cadd(d02, r);
    x[3] = csub(d02, r);
  } else {
    // R = A B: input n = B n1 + n2, output k = k1 + A k2
    constexpr int A = Split<R>::A, B = Split<R>::B;
#pragma unroll
    for (int n2 = 0; n2 < B; ++n2) {
      V t[A];
#pragma unroll
      for (int n1 = 0; n1 < A; ++n1) t[n1] = x[B * n1 + n2];
      dft_reg<V, T, A, INV>(t);
#pragma unroll
      for (int k1 = 0; k1 < A; ++k1) {
        V u = t[k1];
        const int e = (n2 * k1) % R;
        if (e != 0) {
          V w;
          w.x = (T)twc(R, e);
          w.y = INV ? (T)-tws(R, e) : (T)tws(R, e);
          u = cmul(u, w);
        }
        x[B * k1 + n2] = u;
      }
    }
    V o[R];
#pragma unroll
    for (int k1 = 0; k1 < A; ++k1) {
      V t[B];
#pragma unroll
      for (int n2 = 0; n2 < B; ++n2) t[n2] = x[B * k1 + n2];
      dft_reg<V, T, B, INV>(t);
#pragma unroll
      for (int k2 = 0; k2 < B; ++k2) o[k1 + A * k2] = t[k2];
    }
#pragma unroll
    for (int r = 0; r < R; ++r) x[r] = o[r];
  }
}

// One Stockham stage of radix R over `nsig` padded signals (stride `sig`).
template <typename V, typename T, int R, bool INV>
__device__ __forceinline__ void fft_stage_r(const V* __restrict__ in, V* __restrict__ out, int L,
                                            int Ns, int tstride, unsigned mlr, unsigned mns,
                                            int nsig, int sig, const V* __restrict__ tw) {
  const int LR = L / R;
  const int total = nsig * LR;
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const int s = (int)fast_div((unsigned)t, mlr);
    const int j = t - s * LR;
    const int k = j - (int)fast_div((unsigned)j, mns) * Ns;
    const V* src = in + (size_t)s * sig;
    V* dst = out + (size_t)s * sig;
    V v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[pidx(j + r * LR)];
    if (Ns > 1) {
      const int e = k * tstride;
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], twiddle(tw, r * e, INV));
    }
    dft_reg<V, T, R, INV>(v);
    const int base = (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) dst[pidx(base + r * Ns)] = v[r];
  }
}

template <typename V, typename T, bool INV>
__device__ __forceinline__ void fft_stage_dispatch(const V* in, V* out, const FftPlan& pl, int st,
                                                   int nsig, int sig, const V* tw) {
  const int L = pl.L, Ns = pl.ns[st], ts = pl.stride[st];
  const unsigned ml = pl.mlr[st], mn = pl.mns[st];
  switch (pl.radix[st]) {
    case 16: fft_stage_r<V, T, 16, INV>(in, out, L, Ns, ts, ml, mn, nsig, sig, tw); break;
    case 12: fft_stage_r<V, T, 12, INV>(in, out, L, Ns, ts, ml, mn, nsig, sig, tw); break;
    case 9: fft_stage_r<V, T, 9, INV>(in, out, L, Ns, ts, ml, mn, nsig, sig, tw); break;
    case 8: fft_stage_r<V, T, 8, INV>(in, out, L, Ns, ts, ml, mn, nsig, sig, tw); break;
    case 6: fft_stage_r<V, T, 6, INV>(in, out, L, Ns, ts, ml, mn, nsig, sig, tw); break;
    case 4: fft_stage_r<V, T, 4, INV>(in, out, L, Ns, ts, ml, mn, nsig, sig, tw); break;
    case 3: fft_stage_r<V, T, 3, INV>(in, out, L, Ns, ts, ml, mn, nsig, sig, tw); break;
    default: fft_stage_r<V, T, 2, INV>(in, out, L, Ns, ts, ml, mn, nsig, sig, tw); break;
  }
}

// Full transform of `nsig` padded signals (stride `sig` elements) held in `a`;
// `b` is scratch of the same size.  Returns the buffer holding the result.
// Must be called by every thread of the block; begins and ends with a barrier.
template <typename V, typename T>
__device__ V* block_fft(V* a, V* b, const FftPlan& pl, int nsig, int sig,
                        const V* __restrict__ tw, bool inv) {
  __syncthreads();
  for (int st = 0; st < pl.nstage; ++st) {
    if (inv) fft_stage_dispatch<V, T, true>(a, b, pl, st, nsig, sig, tw);
    else fft_stage_dispatch<V, T, false>(a, b, pl, st, nsig, sig, tw);
    __syncthreads();
    V* t = a; a = b; b = t;
  }
  return a;
}

}  // namespace fitsne
