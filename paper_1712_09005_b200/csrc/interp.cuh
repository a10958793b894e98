// Per-point interpolation helpers shared by the spread, gather and fused
// SpMV kernels (nbody.py:201-230, 344-350; optimizer.py:203-210, 244).
#pragma once

#include <type_traits>

#include "common.cuh"

namespace fitsne {

template <typename T, int S>
struct PointInterp {
  int cell[S];
  double w[S][kMaxP];
};

template <typename T, int S>
__device__ __forceinline__ void interp_point(const T* __restrict__ Y, int64_t i, const GridArgs& g,
                                             PointInterp<T, S>& pi, double* y) {
#pragma unroll
  for (int d = 0; d < S; ++d) {
    y[d] = (double)Y[i * S + d];
    pi.cell[d] = box_weights(y[d], g.lo[d], g.h[d], g.n_int, g.p, pi.w[d]);
  }
}

// one 4-slot potential record (float4 / 2 x double2)
template <typename T>
__device__ __forceinline__ void load_slots(const T* p, T (&v)[4]) {
  if constexpr (sizeof(T) == 4) {
    float4 f = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
  } else {
    double2 a = __ldg(reinterpret_cast<const double2*>(p));
    double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
}

// Warp-cooperative gather for point i: lane m < p^S interpolates node m of
// the point's box; returns this lane's partial potentials phi[0..3] (to be
// summed over the warp).  All lanes must call it (no divergence required).
// P = 3: compile-time fast path (registers only); P = 0: any p in [2, 8].
template <typename T, int S, int P>
__device__ __forceinline__ void warp_gather_partial(const T (&yi)[S], const GridArgs& g,
                                                    const T* __restrict__ pot, int lane,
                                                    T (&phi)[4]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) phi[c] = 0;
  if constexpr (P == 3) {
    // p = 3 fast path: everything in registers (no runtime-indexed arrays)
    const int cnt = (S == 1) ? 3 : 9;
    if (lane >= cnt) return;
    const int a = (S == 1) ? lane : lane / 3, b = (S == 1) ? 0 : lane - (lane / 3) * 3;
    using W = typename std::conditional<sizeof(T) == 4, float, double>::type;
    W w0[3], w1[3];
    int c0, c1 = 0;
    if constexpr (sizeof(T) == 4) {
      c0 = box_weights3_f32((float)yi[0], g.lo[0], g.h[0], g.lo_f[0], g.invh_f[0], g.guard[0],
                            g.n_int, w0);
      if (S == 2)
        c1 = box_weights3_f32((float)yi[S - 1], g.lo[S - 1], g.h[S - 1], g.lo_f[S - 1],
                              g.invh_f[S - 1], g.guard[S - 1], g.n_int, w1);
    } else {
      c0 = box_weights((double)yi[0], g.lo[0], g.h[0], g.n_int, 3, w0);
      if (S == 2) c1 = box_weights((double)yi[S - 1], g.lo[S - 1], g.h[S - 1], g.n_int, 3, w1);
    }
    const W wa = (a == 0) ? w0[0] : ((a == 1) ? w0[1] : w0[2]);
    W wt = wa;
    int64_t node = (int64_t)c0 * 3 + a;
    if (S == 2) {
      wt = wa * ((b == 0) ? w1[0] : ((b == 1) ? w1[1] : w1[2]));
      node = pot_box_node(c0, c1, a, b, 3, g.n_int);
    }
    T v[4];
    load_slots<T>(pot + node * kNodeSlots, v);
    const T tw = (T)wt;
#pragma unroll
    for (int c = 0; c < 4; ++c) phi[c] = v[c] * tw;
    return;
  } else {
  const int p = g.p;
  const int cnt = (S == 1) ? p : p * p;
  if (lane >= cnt && cnt <= 32) return;
  double w[S][kMaxP];
  int cell[S];
#pragma unroll
  for (int d = 0; d < S; ++d) cell[d] = box_weights((double)yi[d], g.lo[d], g.h[d], g.n_int, p, w[d]);
  for (int m = lane; m < cnt; m += 32) {
    int64_t node;
    double wt;
    if (S == 1) {
      node = (int64_t)cell[0] * p + m;
      wt = w[0][m];
    } else {
      const int a = m / p, b = m - (m / p) * p;
      node = pot_box_node(cell[0], cell[1], a, b, p, g.n_int);
      wt = w[0][a] * w[S - 1][b];
    }
    T v[4];
    load_slots<T>(pot + node * kNodeSlots, v);
    const T tw = (T)wt;
#pragma unroll
    for (int c = 0; c < 4; ++c) phi[c] += v[c] * tw;
  }
  }
}

// Thread-per-point gather of the 4 potentials of point y (all p^S nodes).
template <typename T, int S, int P>
__device__ __forceinline__ void point_gather(const T (&yi)[S], const GridArgs& g,
                                             const T* __restrict__ pot, T (&phi)[4]) {
#pragma unroll
  for (int c = 0; c < 4; ++c) phi[c] = 0;
  if constexpr (P == 3 && sizeof(T) == 4) {
    float w0[3], w1[3] = {1.f, 0.f, 0.f};
    const int c0 = box_weights3_f32((float)yi[0], g.lo[0], g.h[0], g.lo_f[0], g.invh_f[0],
                                    g.guard[0], g.n_int, w0);
    int c1 = 0;
    if (S == 2)
      c1 = box_weights3_f32((float)yi[S - 1], g.lo[S - 1], g.h[S - 1], g.lo_f[S - 1],
                            g.invh_f[S - 1], g.guard[S - 1], g.n_int, w1);
    FITSNE_DCHECK(c0 >= 0 && c0 < g.n_int && c1 >= 0 && c1 < g.n_int);
    if constexpr (S == 2) {
      // box-major potentials: the 9 records of box (c0, c1) are one 32-byte
      // aligned 160-byte block, read with five 256-bit loads
      const float* bp = reinterpret_cast<const float*>(pot) + pot_box_node(c0, c1, 0, 0, 3, g.n_int) * kNodeSlots;
      float r[40];
#pragma unroll
      for (int k = 0; k < 5; ++k)
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r[8 * k]), "=f"(r[8 * k + 1]), "=f"(r[8 * k + 2]), "=f"(r[8 * k + 3]),
                       "=f"(r[8 * k + 4]), "=f"(r[8 * k + 5]), "=f"(r[8 * k + 6]), "=f"(r[8 * k + 7])
                     : "l"(bp + 8 * k));
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const float wt = w0[a] * w1[b];
#pragma unroll
          for (int c = 0; c < 4; ++c) phi[c] += r[(a * 3 + b) * 4 + c] * wt;
        }
      return;
    }
    // 1-D: the three records of the box are contiguous
    const int64_t box0 = (int64_t)c0 * 3;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int64_t rowbase = box0 + a * ((S == 1) ? 1 : 3);
#pragma unroll
      for (int b = 0; b < ((S == 1) ? 1 : 3); ++b) {
        T v[4];
        load_slots<T>(pot + (rowbase + b) * kNodeSlots, v);
        const float wt = w0[a] * w1[b];
#pragma unroll
        for (int c = 0; c < 4; ++c) phi[c] += v[c] * wt;
      }
    }
  } else {
    const int p = (P > 0) ? P : g.p;
    double w[S][kMaxP];
    int cell[S];
#pragma unroll
    for (int d = 0; d < S; ++d) cell[d] = box_weights((double)yi[d], g.lo[d], g.h[d], g.n_int, p, w[d]);
    const int cnt = (S == 1) ? p : p * p;
    for (int m = 0; m < cnt; ++m) {
      const int a = (S == 1) ? m : m / p, b = (S == 1) ? 0 : m - (m / p) * p;
      const int64_t node = (S == 1) ? ((int64_t)cell[0] * p + a)
                                    : pot_box_node(cell[0], cell[1], a, b, p, g.n_int);
      const double wt = (S == 1) ? w[0][a] : w[0][a] * w[S - 1][b];
      T v[4];
      load_slots<T>(pot + node * kNodeSlots, v);
#pragma unroll
      for (int c = 0; c < 4; ++c) phi[c] += v[c] * (T)wt;
    }
  }
}

// F_rep_i = (y_i (phi_0 - 1) - (phi_{1+d} - y_d)) / Z  (optimizer.py:206-210, 244),
// with the y charges spread centred (phi_{1+d} = K2 * (y_d - c_d)): the same
// value, y_i K2*1 - K2*y, without the fp32 cancellation of two |y|-sized terms
template <typename T, int S>
__device__ __forceinline__ T frep_from_phi(const T (&yi)[S], const T (&phi)[4], T Z, int d,
                                           const GridArgs& g) {
  const T h4 = phi[0] - (T)1;
  const T yc = yi[d] - gcentre<T>(g, d);
  return (yc * h4 - (phi[1 + d] - yc)) / Z;
}

}  // namespace fitsne
