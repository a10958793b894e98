// Host-side orchestration functions shared by the C-ABI translation unit.
#pragma once

#include "common.cuh"

namespace fitsne {

// grid ------------------------------------------------------------------------
int grid_from_bbox(fitsne_ctx* ctx, const double* bbox, fitsne_grid* out);
int compute_bbox(fitsne_ctx* ctx, const void* Y, int64_t n, double* bbox_host,
                 cudaStream_t st);
int install_grid(fitsne_ctx* ctx, const fitsne_grid& g, cudaStream_t st);
// fp64 grid pipeline of an fp32 context (ctx->wide): F_rep (n, dims) in
// double from the shadow context's potentials
int shadow_frep(fitsne_ctx* ctx, const void* Y, int64_t n, double** frep, cudaStream_t st);
int make_grid(fitsne_ctx* ctx, const void* Y, int64_t n, cudaStream_t st);
// make_grid split around other launches: bbox kernels + readback queued on st
// (bbox_launch), then the host waits for the readback only and installs the
// grid for work queued on st (make_grid_finish)
int bbox_launch(fitsne_ctx* ctx, const void* Y, int64_t n, cudaStream_t st);
int bbox_wait(fitsne_ctx* ctx, double* bbox_host);
int bbox_device(fitsne_ctx* ctx, const void* Y, int64_t n, double* out_dev, cudaStream_t st);
int make_grid_finish(fitsne_ctx* ctx, cudaStream_t st);

// device-grid schedule (the grid computed by k_bbox on the device; no host
// round trip before the spread / FFT stages) -----------------------------------
int bbox_launch_devgrid(fitsne_ctx* ctx, const void* Y, int64_t n, GridArgs* gd, const DevGridReq& rq,
                        GridArgs* gd_host, cudaStream_t st, cudaStream_t copy_st, cudaEvent_t ev_k);
int fft_tsne_dev(fitsne_ctx* ctx, void* accum, int64_t n_total, const GridArgs* gd, int n_cap, int L_cap,
                 cudaStream_t st);
int ensure_accum_nodes(fitsne_ctx* ctx, size_t g_nodes, cudaStream_t st);
int device_plan_table(fitsne_ctx* ctx, int L_max, const void** table, int* count);

// repulsion pipeline ------------------------------------------------------------
// spread of the t-SNE charges (1, y_0[, y_1]) into ctx->accum (or `accum`)
int spread_tsne(fitsne_ctx* ctx, const void* Y, int64_t n, void* accum, cudaStream_t st);
// box-sorted spread (p = 3); FITSNE_EINVAL when not applicable
int spread_sorted(fitsne_ctx* ctx, const void* Y, int64_t n, void* accum, cudaStream_t st);
// FFT stage: accum -> ctx->pot, Z -> ctx->scal[0] (needs n_total for Z)
int fft_tsne(fitsne_ctx* ctx, void* accum, int64_t n_total, bool with_k1, cudaStream_t st);
// start the kernel spectrum of the current grid on the context's spectrum
// stream (after `from`); the next fft_tsne on this grid joins it
int spectrum_ahead(fitsne_ctx* ctx, cudaStream_t from);
// gather: pot -> forces (n, s) [+ k1 (n,), k2 (n, s+1)]
int gather_tsne(fitsne_ctx* ctx, const void* Y, int64_t n, void* forces, void* k1, void* k2,
                cudaStream_t st);

// general n-body pieces (nbody.py public API) ------------------------------------
int point_interp(fitsne_ctx* ctx, const void* Y, int64_t n, int64_t* idx, void* w,
                 cudaStream_t st);
int spread_general(fitsne_ctx* ctx, const void* Y, int64_t n, const void* q, int nq,
                   void* coeffs, cudaStream_t st);
int matvec_general(fitsne_ctx* ctx, int kernel, const void* coeffs, int ncol, void* out,
                   cudaStream_t st);
int gather_general(fitsne_ctx* ctx, const void* Y, int64_t n, const void* vals, int ncol,
                   void* out, cudaStream_t st);

// exact O(N^2) sums: k1 (n,), k2 (n, s+1) both ctx dtype; Z -> scal[0]
int exact_sums(fitsne_ctx* ctx, const void* Y, int64_t n, void* k1, void* k2, cudaStream_t st);
int forces_from_sums(fitsne_ctx* ctx, const void* Y, int64_t n, const void* k2, void* forces,
                     cudaStream_t st);
int exact_nbody(fitsne_ctx* ctx, const void* Y, int64_t n, const void* q, int nq, int kernel,
                int include_self, void* out, cudaStream_t st);

// attractive / KL / step ------------------------------------------------------------
// fold=false leaves the KL partials in ctx->part (the caller folds them)
int attractive(fitsne_ctx* ctx, const void* Yfull, const void* forces, double alpha,
               void* out, int mode, bool kl, cudaStream_t st,
               bool fold = true);  // mode 0 F_attr, 1 grad(forces), 2 grad(fused gather)
int kl_sum(fitsne_ctx* ctx, const void* Yfull, cudaStream_t st);  // -> scal[1] = sum p log1p(d2)
int compute_plogp(fitsne_ctx* ctx, cudaStream_t st);
int step_update(fitsne_ctx* ctx, void* Y, const void* grad, void* vel, void* gains, int64_t n,
                double momentum, double lr, cudaStream_t st);
int nonfinite_count(fitsne_ctx* ctx, const void* x, int64_t count, int* out_host,
                    cudaStream_t st);
int gradient_overlapped(fitsne_ctx* ctx, const void* Y, double alpha, void* grad, cudaStream_t st,
                        void* grad_host = nullptr);
int combine_rows(fitsne_ctx* ctx, const void* attr, const void* frep, int64_t n, double alpha,
                 void* out, cudaStream_t st);
int iterate_fused(fitsne_ctx* ctx, const void* Yin, void* Yout, void* vel, void* gains,
                  double alpha, double momentum, double lr, double* kl_dev, int32_t* status_dev,
                  cudaStream_t st);

// tiled attractive SpMV (tiled.cu) -------------------------------------------------
// true when the tiled kernel applies to this call (builds the tiled copy of P
// on first use)
bool tiled_usable(fitsne_ctx* ctx, const void* Y, cudaStream_t st);
// F_attr -> *fattr (zeroed buffer owned by the tiled copy; the consumer clears
// it), KL partials -> (*part)[0, *nparts)
int attract_tiled_join(fitsne_ctx* ctx, const void* Y, int ctas, cudaStream_t st, int* nparts);
int attract_tiled(fitsne_ctx* ctx, const void* Y, bool kl, cudaStream_t st, void** fattr,
                  double** part, int* nparts);
// out = F_attr (mode 0) or 4 (alpha F_attr - frep) (mode 1); clears F_attr
int tiled_finish(fitsne_ctx* ctx, const void* frep, double alpha, int mode, void* out, cudaStream_t st);
void free_tiled(fitsne_ctx* ctx);
int comm_free(fitsne_ctx* ctx);  // comm.cu
// the tiled F_attr buffer's consumer (which clears it) has been queued
void tiled_consumed(fitsne_ctx* ctx);
bool tiled_relabeled(const fitsne_ctx* ctx);  // the tiled copy runs over relabelled points
void tiled_mark_dirty(fitsne_ctx* ctx, cudaStream_t st);  // a queued consumer did not run
// error exit of a multi-stream schedule: wait for the internal streams so no
// queued work outlives the call (the next call reuses their buffers)
int join_on_error(fitsne_ctx* ctx, int rc);
// band spread (bandspread.cu): fp32, 2-D, p = 3, n_int <= 1024
bool band_spread_applies(const fitsne_ctx* ctx, int64_t n);
uint32_t* band_counters(fitsne_ctx* ctx, int64_t n, int* words);
int gather_band(fitsne_ctx* ctx, int64_t n, void* frep, cudaStream_t st);
int spread_band(fitsne_ctx* ctx, const void* Y, int64_t n, void* accum, cudaStream_t st,
                const GridArgs* gd = nullptr);
// The tiled SpMV as kTiledPieces launches over consecutive row ranges (each
// over the whole persistent grid), so a consumer can start on the rows of
// piece k while piece k + 1 runs.  Row range of piece k: [rows[k], rows[k+1]).
constexpr int kTiledPieces = 4;
int attract_tiled_piece(fitsne_ctx* ctx, const void* Y, int piece, cudaStream_t st, void** fattr);
void tiled_piece_rows(const fitsne_ctx* ctx, int64_t* rows);
// Cuthill-McKee ordering of a symmetric CSR pattern (reorder.cu):
// order[new] = old, pos_of[old] = new
int cuthill_mckee(const int64_t* rowptr, const int32_t* col, int n, int* order, int* pos_of, int num_sms,
                  cudaStream_t st);
// fitsne_gradient_host (attract.cu)
int gradient_host(fitsne_ctx* ctx, const void* Y_host, double alpha, void* grad_host, cudaStream_t st);
int tiled_stats(fitsne_ctx* ctx, const void* Y, int64_t* out, cudaStream_t st);

// four-step FFT convolution for long transforms (bigfft.cu)
bool big_fft_applies(const fitsne_ctx* ctx, int L);
int conv_big_tsne(fitsne_ctx* ctx, void* accum, int nrep, int64_t rstride, bool with_k1, int64_t n_total,
                  cudaStream_t st);
int conv_big_general(fitsne_ctx* ctx, const void* coeffs, int ncol, int kern, void* out, cudaStream_t st);

int read_scalars(fitsne_ctx* ctx, int count, cudaStream_t st);  // scal[0..count) -> h_scal
int sub_inplace(fitsne_ctx* ctx, void* out, const void* q, int64_t count, cudaStream_t st);

}  // namespace fitsne
