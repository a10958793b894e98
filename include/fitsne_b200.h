/*
 * fitsne_b200.h -- C-ABI of the B200 (sm_100a) FIt-SNE gradient library.
 *
 * The reference (`fftsne`, /root/reference/pkg/src/fftsne) is a pure-Python
 * package with no FFI of its own: its boundary for this path is the Python API
 * of fftsne.nbody and fftsne.optimizer.  Every entry point below replaces the
 * reference function named beside it; the Python mirror
 * (paper_1712_09005_b200/{nbody,optimizer}.py) binds them through ctypes with
 * the reference's names, argument meaning and exceptions, and INTEGRATION.md
 * shows the ctypes stub a maintainer of the reference would add.
 *
 * Conventions
 *   - All array arguments are DEVICE pointers (cudaMalloc / torch CUDA tensors)
 *     unless the name ends in `_host`.  The caller owns every buffer; the
 *     library owns only the context (scratch grids, FFT work areas, twiddles).
 *   - Embeddings Y are row-major (N, dims) in the context dtype
 *     (FITSNE_F32 -> float, FITSNE_F64 -> double).  The point index is the
 *     row; dims in {1, 2}.
 *   - Every call is stream-ordered on `stream` (a cudaStream_t; 0 = legacy
 *     default).  The only host synchronisation is the grid-size readback in
 *     fitsne_make_grid (the FFT length depends on the data, nbody.py:134).
 *   - Return value: FITSNE_OK or an error code; fitsne_last_error() gives a
 *     thread-local message.  The Python layer maps FITSNE_EINVAL/FITSNE_EOUTSIDE/
 *     FITSNE_EZ/FITSNE_EPOINTS to ValueError and FITSNE_ENONFINITE to FloatingPointError,
 *     exactly as the reference raises (optimizer.py:242-243, 310-313;
 *     nbody.py:127-128, 210-211).
 */
#ifndef FITSNE_B200_H
#define FITSNE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FITSNE_ABI_VERSION 1

enum fitsne_status {
  FITSNE_OK = 0,
  FITSNE_EINVAL = 1,      /* bad argument / shape / config -> ValueError */
  FITSNE_ENONFINITE = 2,  /* non-finite input or gradient -> FloatingPointError */
  FITSNE_EZ = 3,          /* normalisation Z <= 0 -> ValueError (optimizer.py:242) */
  FITSNE_ECUDA = 4,       /* CUDA runtime error */
  FITSNE_ENOMEM = 5,      /* device allocation failed */
  FITSNE_EOUTSIDE = 6,    /* point outside grid bounds -> ValueError (nbody.py:210) */
  FITSNE_ETOOBIG = 7,     /* grid larger than the FFT kernels support */
  FITSNE_EPOINTS = 8,     /* non-finite point met while building the grid -> ValueError
                             ("points must be finite", nbody.py:127-128); the fused
                             iteration reports it for a diverged embedding */
  FITSNE_ENCCL = 9        /* NCCL missing or failed (fitsne_comm_init / sharded gradient) */
};

enum fitsne_dtype { FITSNE_F32 = 0, FITSNE_F64 = 1 };
enum fitsne_kernel { FITSNE_CAUCHY = 0, FITSNE_CAUCHY_SQUARED = 1 };  /* nbody.py:38-42 */

/* Interpolation grid, the device-side twin of nbody.InterpGrid (nbody.py:62-104). */
typedef struct fitsne_grid {
  double lo[2];
  double hi[2];
  double spacing[2];   /* (hi - lo) / nodes_per_dim, nbody.py:97-99 */
  int32_t dims;
  int32_t n_intervals;
  int32_t points_per_interval;
  int32_t nodes_per_dim;   /* n = n_intervals * points_per_interval */
  int32_t fft_len;         /* L >= 2n-1, 2^a 3^b (reference: next_fast_len, nbody.py:267) */
  int32_t status;          /* 0, or FITSNE_ENONFINITE if a coordinate was not finite */
} fitsne_grid;

typedef struct fitsne_ctx fitsne_ctx;

const char* fitsne_last_error(void);
int fitsne_abi_version(void);

/* Context: one per (device, dtype, dims, interpolation options).
 * intervals_per_integer: FIt-SNE's option; the reference hard-codes 1.0
 * (nbody.py:134) and only 1.0 has an oracle. */
int fitsne_create(fitsne_ctx** out, int device, int dims, int dtype,
                  int points_per_interval, int min_intervals,
                  double intervals_per_integer);
int fitsne_destroy(fitsne_ctx* ctx);
int fitsne_set_interp(fitsne_ctx* ctx, int points_per_interval, int min_intervals,
                      double intervals_per_integer);

/* Implementation switches (no reference counterpart; for A/B tests).
 *   FITSNE_OPT_SORTED_SPREAD: 0 = one atomic per point and node; 1 (default)
 *   = band spread for fp32 2-D p = 3 (points binned by box row, then sorted
 *   by box per block, one reduction per node per box run), otherwise the
 *   box-sorted segmented spread (p = 3) when the points crowd into few boxes
 *   (>= 128 points per occupied box); 2 = always box-sorted; 3 = band spread
 *   whenever it applies. */
enum fitsne_option {
  FITSNE_OPT_SORTED_SPREAD = 1,
  FITSNE_OPT_OVERLAP = 2,
  FITSNE_OPT_SPMV_BLOCKS_PER_SM = 3,
  FITSNE_OPT_SPREAD_REPLICAS = 4,
  FITSNE_OPT_TILED_SPMV = 5,
  FITSNE_OPT_TILE_ROWS = 6,
  FITSNE_OPT_TILE_COLS = 7,
  FITSNE_OPT_TILED_CTAS = 8,
  FITSNE_OPT_TILED_BANK_ORDER = 9,
  FITSNE_OPT_HOST_PIECES = 10,
  FITSNE_OPT_FFT_COLS = 11,
  FITSNE_OPT_FFT_PATH = 12,
  FITSNE_OPT_GRID_F64 = 13,
  FITSNE_OPT_RELABEL = 14,
  FITSNE_OPT_DEVICE_GRID = 15,
  FITSNE_OPT_SIDE_GATHER = 16,
  FITSNE_OPT_SPMV_JOIN = 17,
  FITSNE_OPT_SPEC_AHEAD = 18
};
/*   FITSNE_OPT_TILED_SPMV: 0 = row-per-warp CSR SpMV; 1 (default) = for fp32
 *   2-D embeddings with >= 2^22 stored entries, a copy of P in row-block x
 *   column-chunk tiles (sliced-ELL inside each tile) whose column chunk of Y
 *   is staged in shared memory by bulk copies; 2 = tiled whenever applicable.
 *   The tiled copy is built on first use after fitsne_set_affinities.
 *   FITSNE_OPT_TILE_ROWS / FITSNE_OPT_TILE_COLS: tile shape (rows per row
 *   block, default 3072; points per column chunk, default 8192); both even and
 *   <= 16384.  Shapes whose shared-memory footprint (24 rows + 16 cols + 4.3
 *   rows bytes) exceeds 226 KiB use the CSR kernel.  FITSNE_OPT_TILED_CTAS:
 *   persistent grid of the tiled kernel (default 0 = 11/12 of the SMs when the
 *   repulsion runs concurrently on the side stream, else one CTA per SM).
 *   FITSNE_OPT_HOST_PIECES: fitsne_gradient_host schedule; 0 (default) = copy
 *   in, gradient with the final combine in point ranges whose copy-out
 *   overlaps the next range; 1 = tiled SpMV in row pieces on a high-priority
 *   stream with each piece's combine + copy-out overlapping later pieces;
 *   2 = copy in, gradient, one copy out.
 *   FITSNE_OPT_TILED_BANK_ORDER: slot order inside the tiles' slabs chosen
 *   to spread each step's y_j gathers over shared-memory bank pairs; 0 = off,
 *   1 (default) = every slab up to 256 slots per lane, 2 = slabs up to 32 only.
 *   FITSNE_OPT_FFT_COLS: adjacent columns per block of the column FFT stage
 *   (1 = default, 2, 4; fewer when shared memory does not fit).
 *   FITSNE_OPT_FFT_PATH: 0 (default) = one-block-per-transform kernels while
 *   the transform fits shared memory (L <= 5184 fp32 / 2592 fp64), the
 *   four-step path (L = L1 L2, two shared-memory passes per axis through HBM)
 *   beyond; 1 = shared-memory kernels only; 2 = four-step always.
 *   FITSNE_OPT_GRID_F64 (fp32 contexts): 0 = fp32 grid pipeline; 1 (default)
 *   = spread accumulation, FFT stage, potentials and F_rep in fp64 when the
 *   embedding's widest span exceeds 256 (fp32's repulsive force loses
 *   accuracy with the span: F = y K2*1 - K2*y cancels |y|-sized terms); 2 =
 *   always.  Points, the attractive SpMV and the gradient stay fp32.
 *   FITSNE_OPT_RELABEL: the tiled copy of P over a Cuthill-McKee relabelling
 *   of the points computed from P's pattern on the device (components and
 *   neighbourhoods get contiguous labels; results stay in the caller's
 *   order).  0 = caller's order; 1 (default) = relabel when that at least
 *   halves the (row, column chunk) segments of the tiles; 2 = always.
 *   FITSNE_OPT_SIDE_GATHER: 1 (default) = with the band spread (fp32 2-D p = 3)
 *   F_rep is gathered on the repulsion stream, in the spread's box order,
 *   while the attractive SpMV still runs, and the combine after the SpMV only
 *   streams 4 (alpha F_attr - F_rep); 0 = the combine gathers F_rep itself.
 *   FITSNE_OPT_SPMV_JOIN: 1 (default) = when the repulsion chain beside the
 *   tiled SpMV is done, a second SpMV launch on its stream joins the dynamic
 *   work-unit schedule with the SMs the chain used; 0 = one launch only.
 *   FITSNE_OPT_SPEC_AHEAD: 1 = in the overlapped schedule the kernel spectrum
 *   (it depends on the grid only: nbody.py:264-283) is computed on a stream of
 *   its own while the charges are still being spread, instead of in the FFT
 *   stage behind the spread; 0 (default) = inside the FFT stage.  Measured at
 *   C3: the spectrum kernels and the spread share the same ~28 SMs, the chain
 *   ends 5 us earlier and the step is 0.6% slower, so it is off.
 *   FITSNE_OPT_DEVICE_GRID: 1 = fitsne_gradient / _host / _iterate compute
 *   the grid on the device and queue the spread and FFT stages without
 *   waiting for the bbox readback (the host checks the grid after queueing
 *   and re-runs the chain in the rare case the stages' launch capacity was
 *   exceeded); 0 (default) = wait for the readback first.  At C3 the chain
 *   then starts ~20 us earlier but its stages run no faster on the SMs the
 *   SpMV leaves, so the step measured 1.5% slower; kept as an option. */
int fitsne_set_option(fitsne_ctx* ctx, int option, int value);
/* Layout of the tiled copy of P (diagnostics; builds it if needed, using Y
 * only for its alignment): out[0..7] = {in use (0/1), tiles, slabs, slot
 * groups, (row, chunk) segments, stored entries, relabelled (0/1), segments
 * in the caller's order}. */
int fitsne_tiled_stats(fitsne_ctx* ctx, const void* Y, int64_t* out, void* stream);

/* --- a1: make_grid (nbody.py:118-150).  Device bbox reduction + fp64 grid
 * formulas; the grid is copied to *grid_host (one host sync) and kept as the
 * context's current grid. */
int fitsne_make_grid(fitsne_ctx* ctx, const void* Y, int64_t n, fitsne_grid* grid_host,
                     void* stream);
/* Local bounding box only (multi-GPU: the caller all-reduces MIN/MAX, then
 * calls fitsne_grid_from_bbox on every rank).  bbox_host = {min_0..min_{s-1},
 * max_0..max_{s-1}}. */
int fitsne_bbox(fitsne_ctx* ctx, const void* Y, int64_t n, double* bbox_host, void* stream);
/* The same into DEVICE memory, stream-ordered, no host sync (multi-GPU: the
 * ranks all-reduce it on the device and read it back once):
 * bbox_dev[0 .. 2s] = {min_0..min_{s-1}, -max_0..-max_{s-1}, -nonfinite}, so a
 * single MIN all-reduce combines every field. */
int fitsne_bbox_device(fitsne_ctx* ctx, const void* Y, int64_t n, double* bbox_dev, void* stream);
int fitsne_grid_from_bbox(fitsne_ctx* ctx, const double* bbox_host, fitsne_grid* grid_host);
/* Install an explicit grid (nbody.InterpGrid built by the caller). */
int fitsne_set_grid(fitsne_ctx* ctx, const fitsne_grid* grid_host);

/* --- a2: _point_interp (nbody.py:201-230): node_index (n, p^s) int64 and
 * weights (n, p^s) in ctx dtype.  Bit-exact node indices. */
int fitsne_point_interp(fitsne_ctx* ctx, const void* Y, int64_t n, int64_t* node_index,
                        void* weights, void* stream);

/* --- a3: spread_charges (nbody.py:233-251).  charges (n, ncharge) row-major
 * ctx dtype; coeffs out (ncharge, G) ctx dtype. */
int fitsne_spread(fitsne_ctx* ctx, const void* Y, int64_t n, const void* charges,
                  int ncharge, void* coeffs, void* stream);

/* --- a4/a5: kernel_matvec_fft (nbody.py:262-311): v = Toeplitz(K) w on the
 * current grid for `ncol` coefficient vectors (ncol, G). */
int fitsne_kernel_matvec(fitsne_ctx* ctx, int kernel, const void* coeffs, int ncol,
                         void* out, void* stream);

/* --- a6: gather_potentials (nbody.py:344-350): values (ncol, G) -> out (n, ncol). */
int fitsne_gather(fitsne_ctx* ctx, const void* Y, int64_t n, const void* values, int ncol,
                  void* out, void* stream);

/* --- a16: evaluate_nbody (nbody.py:353-399): builds the grid from the points,
 * charges (n, ncharge) -> out (n, ncharge). */
int fitsne_evaluate_nbody(fitsne_ctx* ctx, const void* Y, int64_t n, const void* charges,
                          int ncharge, int kernel, int include_self, void* out, void* stream);

/* --- a7/a8: compute_repulsive(method="fft") (optimizer.py:193-245).
 * forces (n, s); z_host gets Z; k1 (n,) and k2 (n, s+1) optional (NULL). */
int fitsne_repulsive(fitsne_ctx* ctx, const void* Y, int64_t n, void* forces, double* z_host,
                     void* k1, void* k2, void* stream);
/* --- a14: compute_repulsive(method="exact") (optimizer.py:169-190, 236). */
int fitsne_repulsive_exact(fitsne_ctx* ctx, const void* Y, int64_t n, void* forces,
                           double* z_host, void* k1, void* k2, void* stream);

/* --- a15 -> CSR: the symmetric affinities (both triangles) of
 * affinities.SparseAffinities (affinities.py:78-104).  Registers device
 * arrays (kept alive by the caller): rows [row_begin, row_begin+n_rows) of the
 * full matrix; col indices are global point indices. */
int fitsne_set_affinities(fitsne_ctx* ctx, const int64_t* rowptr, const int32_t* col,
                          const void* val, int64_t n_rows, int64_t row_begin, int64_t n_total,
                          int64_t nnz);

/* --- a9: compute_attractive (optimizer.py:150-166) over the registered rows.
 * Y_full (n_total, s); out (n_rows, s). */
int fitsne_attractive(fitsne_ctx* ctx, const void* Y_full, void* out, void* stream);

/* --- a10: gradient (optimizer.py:248-262), method="fft": 4(alpha F_attr - F_rep).
 * Single-GPU (registered rows must be all rows).  grad (n, s); z_host optional. */
int fitsne_gradient(fitsne_ctx* ctx, const void* Y, double alpha, void* grad, double* z_host,
                    void* stream);

/* --- a10 with HOST buffers: the reference's gradient() call shape (numpy in,
 * numpy out; optimizer.py:248-262).  Y_host (n, s) and grad_host (n, s) in the
 * context dtype, pinned for full PCIe speed.  Copies Y in on `stream`, runs the
 * gradient with the attractive SpMV split into row pieces and copies each
 * piece of the gradient out while the later pieces still run.  Returns when
 * grad_host is written. */
int fitsne_gradient_host(fitsne_ctx* ctx, const void* Y_host, double alpha, void* grad_host,
                         void* stream);

/* --- a12: _kl_given_z (optimizer.py:265-275) over the registered rows. */
int fitsne_kl(fitsne_ctx* ctx, const void* Y_full, double z, double* kl_host, void* stream);

/* --- a11: step (optimizer.py:299-323): in-place Y, velocity, gains update.
 * FITSNE_ENONFINITE if grad has a non-finite entry (Y, state untouched). */
int fitsne_step(fitsne_ctx* ctx, void* Y, const void* grad, void* velocity, void* gains,
                int64_t n, double momentum, double learning_rate, void* stream);

/* --- a13 inner loop (optimizer.py:383-413): one fused t-SNE iteration on the
 * device: grid, spread, FFT, Z, gather, SpMV, KL, update.  kl_dev (double*)
 * receives KL of the pre-step Y at kl_dev[0] (device pointer, may be NULL);
 * status_dev (int32*, device) gets FITSNE_ENONFINITE if the gradient or the new Y
 * is non-finite (sticky, may be NULL).  One host sync (grid size). */
int fitsne_iterate(fitsne_ctx* ctx, const void* Y, void* Y_out, void* velocity, void* gains,
                   double alpha, double momentum, double learning_rate, double* kl_dev,
                   int32_t* status_dev, void* stream);

/* --- a16 helper: brute_force_nbody (nbody.py:402-419) on the device. */
int fitsne_exact_nbody(fitsne_ctx* ctx, const void* Y, int64_t n, const void* charges,
                       int ncharge, int kernel, int include_self, void* out, void* stream);

/* Stage entry points for the sharded (multi-GPU) gradient: the host performs
 * the NCCL collectives between them (parallel.py).  The grid accumulator holds
 * 4 slots per node in the context dtype, fitsne_grid_accum_len() elements, and
 * must be zero before the first spread (it is cleared again by fitsne_fft_tsne). */
int64_t fitsne_grid_accum_len(fitsne_ctx* ctx);
/* dtype (FITSNE_F32 / FITSNE_F64) of that accumulator for the current grid:
 * FITSNE_F64 when an fp32 context runs the grid in fp64 (FITSNE_OPT_GRID_F64). */
int fitsne_grid_accum_dtype(fitsne_ctx* ctx);
int fitsne_spread_tsne(fitsne_ctx* ctx, const void* Y_local, int64_t n_local, void* accum,
                       void* stream);
int fitsne_fft_tsne(fitsne_ctx* ctx, void* accum, int64_t n_total, int with_k1,
                    double* z_host, void* stream);
int fitsne_gather_tsne(fitsne_ctx* ctx, const void* Y_local, int64_t n_local, void* forces,
                       void* k1, void* k2, void* stream);
int fitsne_gradient_rows(fitsne_ctx* ctx, const void* Y_full, const void* forces_local,
                         double alpha, void* grad_local, void* stream);
/* The combine of the sharded path (optimizer.py:262): grad = 4 (alpha F_attr
 * - F_rep) over n rows of the context's dims, when F_attr (fitsne_attractive,
 * run concurrently with the repulsion stages) and F_rep (fitsne_gather_tsne)
 * were computed separately. */
int fitsne_combine_rows(fitsne_ctx* ctx, const void* attr, const void* frep, int64_t n, double alpha,
                        void* grad, void* stream);
/* Stream-ordered copy of the last FFT stage's Z (device scalar) to z_dst
 * (host pinned or device memory), so a caller can check Z > 0
 * (optimizer.py:242-243) without a synchronisation inside the step. */
int fitsne_read_z(fitsne_ctx* ctx, double* z_dst, void* stream);

/* --- Multi-GPU over NCCL inside the library: one context
 * and one process per GPU.  Rank 0 makes the id (128 bytes) and sends it to
 * the others by any means; every rank then calls fitsne_comm_init, registers
 * the CSR rows of its shard [N r / R, N (r+1) / R) with fitsne_set_affinities
 * (global column indices, n_total = N) and calls fitsne_gradient_sharded each
 * evaluation: device bbox + MIN all-reduce (one 40-byte readback), all-gather
 * of Y, the shard's attractive SpMV on a side stream, private spread + SUM
 * all-reduce of the grid, replicated FFT stage, gather, combine.  NCCL is
 * loaded at run time (libnccl.so.2; the copy already in the process first). */
int fitsne_nccl_unique_id(void* unique_id_out);
int fitsne_comm_init(fitsne_ctx* ctx, const void* unique_id, int rank, int nranks, int64_t n_total);
int fitsne_comm_destroy(fitsne_ctx* ctx);
int fitsne_gradient_sharded(fitsne_ctx* ctx, const void* Y_local, double alpha, void* grad_local,
                            double* z_host, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FITSNE_B200_H */
