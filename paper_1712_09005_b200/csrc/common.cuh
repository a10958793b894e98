// Shared definitions of the sm_100a FIt-SNE library: context, grid arguments,
// status handling, complex arithmetic and the bit-exact box/weight helpers.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <stdint.h>
#include <cstddef>
#include <string>

#include "../../include/fitsne_b200.h"

namespace fitsne {

// ----------------------------------------------------------------------------
// error handling
// ----------------------------------------------------------------------------
void set_error(const std::string& msg);

struct Status {
  int code;
  Status(int c = FITSNE_OK) : code(c) {}
  bool ok() const { return code == FITSNE_OK; }
};

#define FITSNE_CUDA(expr)                                                          \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess) {                                                       \
      ::fitsne::set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) +   \
                          " at " __FILE__ ":" + std::to_string(__LINE__));         \
      return FITSNE_ECUDA;                                                         \
    }                                                                              \
  } while (0)

#define FITSNE_CHECK_LAUNCH() FITSNE_CUDA(cudaGetLastError())

// Device-side bounds checks of the debug build variant (python -m
// paper_1712_09005_b200.build --variant=debug -DFITSNE_DEBUG_BOUNDS=1; the
// test suite runs against it with FITSNE_LIB=libfitsne_b200_debug.so).  They
// stand in for compute-sanitizer memcheck, which is closed on the GPU pool.
#ifndef FITSNE_DEBUG_BOUNDS
#define FITSNE_DEBUG_BOUNDS 0
#endif
#if FITSNE_DEBUG_BOUNDS
#define FITSNE_DCHECK(c)                                                                  \
  do {                                                                                    \
    if (!(c)) {                                                                           \
      printf("FITSNE_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
             #c, (int)blockIdx.x, (int)threadIdx.x);                                      \
      __trap();                                                                           \
    }                                                                                     \
  } while (0)
#else
#define FITSNE_DCHECK(c) \
  do {                   \
  } while (0)
#endif

// NVTX range for the lifetime of a scope (C-ABI entry points and pipeline
// stages show up by name in Nsight timelines; a push/pop pair when no tool
// is attached)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
#define FITSNE_RANGE(name) ::fitsne::NvtxRange _fitsne_nvtx_range(name)

#define FITSNE_TRY(expr)              \
  do {                                \
    int _s = (expr);                  \
    if (_s != FITSNE_OK) return _s;   \
  } while (0)

// ----------------------------------------------------------------------------
// grid arguments passed by value to kernels (the device twin of InterpGrid)
// ----------------------------------------------------------------------------
struct GridArgs {
  double lo[2];
  double hi[2];
  double h[2];
  float lo_f[2];    // fp32 copies for the guarded fp32 box estimate
  float invh_f[2];
  float guard[2];   // margin in units of t/p (>= 0.5 disables the fast path)
  // centre of the grid: the t-SNE y charges are spread as (y - c) so fp32
  // potentials do not carry |y| ~ span (the repulsion is translation
  // invariant; F = (y_i - c) K2*1 - K2*(y - c) = y_i K2*1 - K2*y)
  double c[2];
  float cf[2];
  int dims;
  int n_int;
  int p;
  int n;   // nodes per dim
  int L;   // FFT length
  // device-computed grids (kDevGrid*): 0 = valid for the launched stages,
  // else why the stages skipped it and the host must run the fallback
  int status;
};

// What the device-grid schedule asks k_bbox for: the make_grid options and
// the capacity the dependent stages were launched with
struct DevGridReq {
  int min_intervals = 20;
  int p = 3;
  double ipi = 1.0;
  int cap_nint = 0;      // n_intervals the launch shapes cover
  int cap_L = 0;         // FFT length they cover
  int max_nint = 1024;   // band spread limit
  double wide_span = 0;  // > 0: wider spans need the fp64 grid (host path)
  uint32_t* zero = nullptr;  // words the dependent stages need zeroed (band spread row counters)
  int zero_words = 0;
  const void* plans = nullptr;  // FftPlan table for the 2^a 3^b lengths (ascending), host-built
  int nplans = 0;
};

// fp32 contexts run their grid stages in fp64 beyond this span (repulsion.cu)
constexpr double kWideSpan = 256.0;

// status values of a device-computed grid
constexpr int kDevGridOk = 0;
constexpr int kDevGridCapacity = 100;  // larger than the capacity the stages were launched for
constexpr int kDevGridOther = 101;     // needs another pipeline (fp64 grid, other spread, error)

__host__ __device__ inline GridArgs grid_args(const fitsne_grid& g) {
  GridArgs a;
  for (int d = 0; d < 2; ++d) {
    a.lo[d] = g.lo[d];
    a.hi[d] = g.hi[d];
    a.h[d] = g.spacing[d];
    a.lo_f[d] = (float)g.lo[d];
    a.invh_f[d] = g.spacing[d] > 0 ? (float)(1.0 / g.spacing[d]) : 0.f;
    // |t32 - t| <= (|lo| 2^-24 + |x - lo| 2^-24) / h + t 2^-22 (rounding of
    // lo, of x - lo, of 1/h and of the product); bound it with x - lo <= span
    double span = g.hi[d] - g.lo[d];
    double lo_abs = g.lo[d] < 0 ? -g.lo[d] : g.lo[d];
    double et = g.spacing[d] > 0
                    ? (lo_abs + span) * 5.96e-8 / g.spacing[d] + (double)g.nodes_per_dim * 2.4e-7
                    : 1.0;
    double gd = 4.0 * et / (g.points_per_interval > 0 ? g.points_per_interval : 3) + 1e-3;
    a.guard[d] = gd > 0.5 ? 0.5f : (float)gd;
    a.c[d] = 0.5 * (g.lo[d] + g.hi[d]);
    a.cf[d] = (float)a.c[d];
  }
  a.dims = g.dims;
  a.n_int = g.n_intervals;
  a.p = g.points_per_interval;
  a.n = g.nodes_per_dim;
  a.L = g.fft_len;
  a.status = kDevGridOk;
  return a;
}

// nodes in a box per point: p^dims
constexpr int kMaxP = 8;

// The t-SNE potentials (ctx->pot) are stored box-major in 2-D: the p x p
// nodes of box (bx, by) are one contiguous run of p^2 records, so a point's
// p^2-node gather reads 9 x 16 B = 144 contiguous bytes (p = 3) instead of
// three 48-byte pieces n records apart.  (Boxes own their nodes: node x
// belongs to box x / p.)  1-D: the node order is already box-major.
// records per box: p^2 rounded up to even, so each box starts 32-byte
// aligned in fp32 (p = 3: 10 records = 160 B, read with five 256-bit loads)
__host__ __device__ __forceinline__ int pot_box_records(int p) { return (p * p + 1) & ~1; }
__host__ __device__ __forceinline__ int64_t pot_box_node(int64_t bx, int64_t by, int a, int b, int p,
                                                         int n_int) {
  return (bx * n_int + by) * pot_box_records(p) + a * p + b;
}
// records of the potential buffer for a grid (2-D box-major, 1-D node order)
__host__ __device__ __forceinline__ int64_t pot_records(int dims, int n_int, int p) {
  return dims == 1 ? (int64_t)n_int * p : (int64_t)n_int * n_int * pot_box_records(p);
}
__host__ __device__ __forceinline__ int64_t pot_node(int64_t x, int64_t y, int p, int n_int) {
  const int64_t bx = x / p, by = y / p;
  return pot_box_node(bx, by, (int)(x - bx * p), (int)(y - by * p), p, n_int);
}

// Channel layout of the t-SNE spread / potentials: one 4-slot record per node.
//   spread:     [0] unit charge, [1] y_0, [2] y_1, [3] unused
//   potentials: [0] K2*1, [1] K2*y_0, [2] K2*y_1, [3] K1*1
constexpr int kNodeSlots = 4;

// ----------------------------------------------------------------------------
// the context
// ----------------------------------------------------------------------------
struct DevBuf {
  void* ptr = nullptr;
  size_t cap = 0;
};

struct TiledP;  // tiled copy of P (tiled.cu)
struct GridArgs;
struct Comm;    // NCCL communicator state (comm.cu)

}  // namespace fitsne

struct fitsne_ctx {
  int device = 0;
  int dims = 2;
  int dtype = FITSNE_F32;
  int p = 3;
  int min_intervals = 20;
  double intervals_per_integer = 1.0;

  fitsne_grid grid{};
  bool grid_valid = false;

  // scratch (grow-only)
  fitsne::DevBuf accum;     // spread accumulator, kNodeSlots per node, ctx dtype
  bool accum_clean = false; // accum holds zeros over its whole capacity
  fitsne::DevBuf fbuf;      // FFT work: 2 pairs x n x L complex
  fitsne::DevBuf sbuf;      // kernel spectrum rows: n x (L/2+1) complex
  fitsne::DevBuf pot;       // potentials: kNodeSlots per node
  fitsne::DevBuf tw;        // twiddles exp(-2 pi i m / L)
  int tw_len = 0;
  int tw_gen = 0;           // twiddle regenerations (this context and its shadow)
  fitsne::DevBuf zpart;     // Parseval partials (double), L/2+1
  fitsne::DevBuf bbox_part; // per-block bbox partials (double)
  fitsne::DevBuf scal;      // device scalars (double): [0] Z, [1] KL sum, [2..] misc
  fitsne::DevBuf counter;   // int32 counters / status words
  fitsne::DevBuf forces;    // (N, s) repulsive forces scratch
  fitsne::DevBuf gtmp;      // (N, s) gradient scratch
  fitsne::DevBuf part;      // per-block partial sums (double)
  fitsne::DevBuf gen;       // generic scratch
  fitsne::DevBuf sortbuf;   // box sort keys / values / histograms
  bool band_sorted = false; // sortbuf holds the last band spread's box-ordered points (for gather_band)
  int64_t band_n = 0;       //   ... of this many points
  fitsne::DevBuf frep32;    // (N, 2) fp32 F_rep gathered on the repulsion stream
  int spmv_join = 1;        // a second tiled-SpMV launch behind the repulsion chain joins the dynamic schedule
  bool spmv_tiled_live = false;  // the evaluation being queued runs the tiled SpMV
  bool frep_ready = false;  // frep32 holds F_rep of the evaluation being queued
  int side_gather = 1;      // gather F_rep on the repulsion stream (band spread), stream-combine after the SpMV
  fitsne::DevBuf big;       // four-step FFT planes (bigfft.cu)
  fitsne::DevBuf bigtw;     // its sub-length twiddle tables
  int big_tw_l1 = 0, big_tw_l2 = 0;
  int fft_path = 0;         // 0 auto (four-step above the shared-memory lengths), 1 fast only, 2 four-step
  // fp64 grid pipeline of an fp32 context (spread accumulation, FFT stage,
  // potentials and F_rep in double; points and the SpMV stay fp32): used when
  // the embedding is wide (grid_f64: 0 never, 1 auto, 2 always)
  int grid_f64 = 1;
  bool wide = false;             // the current grid runs on the fp64 shadow
  fitsne_ctx* shadow = nullptr;  // fp64 twin context holding that pipeline
  fitsne::DevBuf y64;            // points converted for the shadow
  // device-grid schedule (attract.cu): the grid k_bbox computes on the
  // device, its pinned host copy, and the n_intervals capacity the stages
  // are launched for (0: not yet known -- the next call takes the host path)
  int devgrid = 0;
  fitsne::DevBuf dgrid;
  fitsne::GridArgs* h_dgrid = nullptr;
  int dg_cap_nint = 0;
  int dg_fallbacks = 0;          // calls that fell back to the host grid (diagnostics)
  fitsne::DevBuf plan_table;     // FftPlan of every 2^a 3^b length <= plan_table_max
  int plan_table_max = 0, plan_table_n = 0;
  fitsne::DevBuf r64;            // shadow gather outputs (F_rep, k1, k2)
  int sorted_spread = 1;      // 0 direct scatter, 1 auto (band spread for fp32 2-D p = 3, else box-sorted when crowded), 2 box-sorted, 3 band
  int spread_replicas = 4;    // replicas of the internal spread accumulator (power of two)
  int accum_live_reps = 4;    // replicas the last spread into the internal accumulator wrote
  int overlap = 1;                 // 0 serial, 1 SpMV || repulsion, 2 same + priority repulsion
  int spmv_blocks_per_sm = 0;      // >0: persistent SpMV grid in the overlap modes
  int tiled_spmv = 1;              // 0 CSR kernel, 1 auto, 2 tiled when applicable
  int tile_rows = 3072, tile_cols = 8192, tiled_ctas = 0;
  int tiled_bank_order = 1;        // bank-aware slot order inside slabs (tiled build)
  int relabel = 1;                 // tiled build over a Cuthill-McKee relabelling of P: 0 off, 1 auto, 2 on
  int cols_per_block = 1;          // adjacent FFT columns per k_cols block (1, 2 or 4)
  int host_pieces = 0;             // fitsne_gradient_host: SpMV row pieces + overlapped copy-out
  fitsne::TiledP* tiled = nullptr; // built lazily from the registered CSR
  fitsne::Comm* comm = nullptr;    // fitsne_comm_init
  double* kl_part = nullptr;       // where the last SpMV left its KL partials
  int kl_nparts = 0;
  cudaStream_t side = nullptr;     // repulsion stream (overlaps the attractive SpMV)
  cudaEvent_t ev_in = nullptr, ev_done = nullptr;
  // kernel spectrum computed ahead of the charges (spectrum_ahead): its own
  // stream, fork / join events, and the grid it was computed for
  cudaStream_t spec = nullptr;
  cudaEvent_t ev_spec_in = nullptr, ev_spec = nullptr;
  bool spec_ahead = false;
  int spec_ahead_L = 0, spec_ahead_n = 0;
  int spec_opt = 0;  // FITSNE_OPT_SPEC_AHEAD (measured: no gain, off)
  cudaEvent_t ev_bbox = nullptr;   // bbox readback landed (bbox_launch / bbox_wait)
  // host-buffer gradient (fitsne_gradient_host): copy-out stream, one event
  // per SpMV row piece, device copies of Y and the gradient
  cudaStream_t out = nullptr, hp = nullptr;
  cudaEvent_t ev_piece[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_out = nullptr;
  fitsne::DevBuf hy, hg;
  double raw_bbox[4] = {0, 0, 0, 0};  // unpadded min/max of the last grid's points

  fitsne_grid* h_grid = nullptr;  // pinned mirror
  double* h_scal = nullptr;       // pinned scalars
  unsigned long long bbox_seq = 0;  // sequence number of the last bbox_launch (polled in h_scal[15])
  int32_t* h_status = nullptr;    // pinned status

  // affinities (borrowed device pointers)
  const int64_t* rowptr = nullptr;
  const int32_t* col = nullptr;
  const void* val = nullptr;
  int64_t n_rows = 0, row_begin = 0, n_total = 0, nnz = 0;
  bool plogp_valid = false;
  double plogp = 0.0;   // sum over stored (full, both triangles) p>0 of p log p
  double psum = 0.0;    // sum over stored p>0 entries

  int num_sms = 148;
};

namespace fitsne {

int ensure(DevBuf& b, size_t bytes);
inline size_t dsize(int dtype) { return dtype == FITSNE_F64 ? 8 : 4; }

// ----------------------------------------------------------------------------
// complex helpers
// ----------------------------------------------------------------------------
template <typename T> struct C2;
template <> struct C2<float> { using type = float2; };
template <> struct C2<double> { using type = double2; };

template <typename V>
__device__ __forceinline__ V cmul(V a, V b) {
  V r;
  r.x = a.x * b.x - a.y * b.y;
  r.y = a.x * b.y + a.y * b.x;
  return r;
}
template <typename V>
__device__ __forceinline__ V cadd(V a, V b) { V r; r.x = a.x + b.x; r.y = a.y + b.y; return r; }
template <typename V>
__device__ __forceinline__ V csub(V a, V b) { V r; r.x = a.x - b.x; r.y = a.y - b.y; return r; }
template <typename V>
__device__ __forceinline__ V cconj(V a) { a.y = -a.y; return a; }

// ----------------------------------------------------------------------------
// Bit-exact box assignment + Lagrange weights (nbody.py:201-230).
//
// Follows numpy's arithmetic: t = (x - lo)/h (IEEE double), cell =
// clip(floor_divide(t, p), 0, n_int-1) with numpy's npy_divmod semantics,
// u = (t - cell*p) - 0.5, w_j = prod_{i != j}(u - i) / prod_{i != j}(j - i)
// multiplied left to right (nbody.py:183-190).  All in double with explicit
// _rn intrinsics so that no FMA contraction can change a rounding.
// ----------------------------------------------------------------------------
__device__ __forceinline__ double npy_floor_divide(double a, double b) {
  // numpy/_core/src/npymath/npy_math_internal.h.src : npy_divmod
  double mod = fmod(a, b);
  double div = __ddiv_rn(__dsub_rn(a, mod), b);
  if (mod != 0.0) {
    if ((b < 0) != (mod < 0)) {
      div = __dsub_rn(div, 1.0);
    }
  }
  double floordiv;
  if (div != 0.0) {
    floordiv = floor(div);
    if (__dsub_rn(div, floordiv) > 0.5) floordiv = __dadd_rn(floordiv, 1.0);
  } else {
    floordiv = copysign(0.0, __ddiv_rn(a, b));
  }
  return floordiv;
}

// returns the cell (box) index along one dimension and fills w[0..p-1]
// floor_divide(t, p) for t >= 0 and integer p in [2, 8]: numpy's divmod
// computes mod = fmod(t, p) exactly, then (t - mod) = k p and k p / p = k
// exactly, i.e. the floor of the EXACT quotient.  The correctly rounded IEEE
// quotient RN(t/p) has the same floor: it could only differ if t < k p while
// RN(t/p) = k.  But t <= k p - d, with d the double spacing below k p, and
// d >= 2^floor(log2 p) u_k (u_k the spacing below k), so k - t/p >=
// (2^floor(log2 p) / p) u_k > u_k / 2 for p in {3, 5, 6, 7} (powers of two
// divide exactly): RN(t/p) <= k - u_k.  Hence floor(t / p) == numpy's t // p
// without the costly fmod.  Negative t (out-of-bounds points) keeps numpy's
// algorithm verbatim.
__device__ __forceinline__ double floor_div_small(double t, int p) {
  if (t >= 0.0) return floor(__ddiv_rn(t, (double)p));
  return npy_floor_divide(t, (double)p);
}

__device__ __forceinline__ int box_weights(double x, double lo, double h, int n_int, int p,
                                           double* w) {
  double t = __ddiv_rn(__dsub_rn(x, lo), h);
  double q = floor_div_small(t, p);
  long long c = (long long)q;
  if (c < 0) c = 0;
  if (c > n_int - 1) c = n_int - 1;
  double u = __dsub_rn(__dsub_rn(t, (double)(c * p)), 0.5);
  if (p == 3) {
    // denominators 2, -1, 2 (nbody.py:176-180); x/2 == x*0.5 and x/-1 == -x exactly
    double d0 = u, d1 = __dsub_rn(u, 1.0), d2 = __dsub_rn(u, 2.0);
    w[0] = __dmul_rn(__dmul_rn(d1, d2), 0.5);
    w[1] = -__dmul_rn(d0, d2);
    w[2] = __dmul_rn(__dmul_rn(d0, d1), 0.5);
  } else {
    for (int j = 0; j < p; ++j) {
      double num = 1.0, den = 1.0;
      bool first = true;
      for (int i = 0; i < p; ++i) {
        if (i == j) continue;
        double di = __dsub_rn(u, (double)i);
        num = first ? di : __dmul_rn(num, di);
        den = __dmul_rn(den, (double)(j - i));
        first = false;
      }
      w[j] = __ddiv_rn(num, den);
    }
  }
  return (int)c;
}

// fp32 fast path for p = 3 (fp32 mode): the box index must stay bit-exact,
// the weights only need fp32 accuracy.  t is estimated in fp32; `guard` (set
// by grid_args from a rounding-error bound, >= 1e-3) is a safe margin in
// units of t/3: when t/3 lies within it of an integer the exact fp64 path
// decides the cell.  Returns the cell and the three fp32 Lagrange weights.
__device__ __forceinline__ int box_weights3_f32(float x, double lo, double h, float lo_f,
                                                float invh_f, float guard, int n_int, float* w) {
  const float t = (x - lo_f) * invh_f;
  const float r = t * (1.0f / 3.0f);
  const float q = floorf(r);
  const float fr = r - q;
  int c;
  float u;
  if (fr > guard && fr < 1.0f - guard && t >= 0.0f) {
    c = (int)q;
    if (c > n_int - 1) c = n_int - 1;
    u = t - (float)(3 * c) - 0.5f;
  } else {
    double wd[3];
    c = box_weights((double)x, lo, h, n_int, 3, wd);
    double td = __ddiv_rn(__dsub_rn((double)x, lo), h);
    u = (float)__dsub_rn(__dsub_rn(td, (double)(c * 3)), 0.5);
  }
  const float d1 = u - 1.0f, d2 = u - 2.0f;
  w[0] = 0.5f * d1 * d2;
  w[1] = -u * d2;
  w[2] = 0.5f * u * d1;
  return c;
}

// grid centre in the working precision (float: cf, double: c)
template <typename W>
__device__ __forceinline__ W gcentre(const GridArgs& g, int d) {
  if constexpr (sizeof(W) == 4) return g.cf[d];
  else return g.c[d];
}

// block-wide reductions ------------------------------------------------------
template <typename V>
__device__ __forceinline__ V warp_sum(V v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace fitsne
