"""Sharded (multi-GPU) t-SNE gradient: one process per GPU, torch.distributed.

Points and CSR rows are partitioned by contiguous index range (rank r owns
[N r / R, N (r+1) / R)).  One evaluation of 4 (alpha F_attr - F_rep)
(optimizer.py:248-262) for the local rows:

  1. local bounding box on the device    fitsne_bbox_device
  2. one MIN all-reduce of {min, -max, -nonfinite} and one readback
                                         -> identical grid on every rank
     (grid formulas nbody.py:131-143, fitsne_grid_from_bbox)
  3. all-gather of Y                     (needed by the row-partitioned SpMV)
  4. spread of the local points into a private accumulator   fitsne_spread_tsne
  5. all-reduce SUM of the accumulator (4 slots x G nodes)
  6. FFT stage + Parseval Z (replicated; the grid is small)  fitsne_fft_tsne
  7. gather of F_rep at the local points                     fitsne_gather_tsne
  8. SpMV over the local rows + combine                      fitsne_attractive on a
     side stream beside 4-7 (CUDA path), then fitsne_combine_rows

The stage arithmetic is pluggable (`stages`): `LibStages` runs the CUDA
library; the multi-process CPU tests plug in an oracle-backed implementation
to exercise the partitioning and the collectives with the gloo backend.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .affinities import DeviceCSR, device_csr, n_points

__all__ = ["shard_range", "LibStages", "ShardedGradient", "NcclGradient"]


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    return n * rank // world, n * (rank + 1) // world


class LibStages:
    """Stage implementation on the CUDA library (one context per rank)."""

    # bbox, band spread (count, scan x2, scatter, reduce), FFT (rows, spectrum
    # columns, columns, rows inverse), gather, tiled SpMV + finish, combine
    launches_per_step = 14

    # Y is all-gathered into a padded layout (rank r's rows at [r m, r m +
    # count_r), m = the largest shard) so ragged shards need no per-step
    # concatenation: the local CSR's column indices are remapped to it once
    padded_columns = True

    def __init__(self, P, dims, dtype, device, min_intervals, points_per_interval,
                 intervals_per_integer, row_begin, row_end, counts=None):
        self.dims = dims
        self.dtype = dtype
        self.device = device
        self.n_total = n_points(P)
        self.ctx = _lib.Context(device, dims, dtype, points_per_interval, min_intervals,
                                intervals_per_integer)
        # the row SpMV (attract_start) runs beside the repulsion stages: the
        # context's default overlapped schedule sizes its grid to 11/12 of the SMs
        csr = device_csr(P, dtype, device, row_begin, row_end)
        counts = counts or [self.n_total]
        self.shard = max(counts)
        if min(counts) != max(counts):
            starts = torch.tensor(np.cumsum([0] + list(counts))[:-1], device=csr.col.device)
            c = csr.col.long()
            r = torch.bucketize(c, starts, right=True) - 1
            col = (r * self.shard + (c - starts[r])).to(torch.int32)
            csr = DeviceCSR(csr.rowptr, col.contiguous(), csr.val, csr.row_begin,
                            self.shard * len(counts), csr.ordered_total)
        self.csr = csr
        self.ctx.set_affinities(self.csr)
        self._acc = None
        self._acc_dirty = False
        self._f = None
        self._zh = torch.zeros(1, dtype=torch.float64).pin_memory()
        self._zev = None

    # -- collectives run on device tensors (NCCL) --------------------------
    def to_comm(self, x: np.ndarray) -> torch.Tensor:
        return torch.as_tensor(x, dtype=torch.float64, device=self.device)

    def bbox(self, y_local: torch.Tensor) -> np.ndarray:
        out = (C.c_double * (2 * self.dims))()
        _lib.check(self.ctx.lib.fitsne_bbox(self.ctx.h, _lib.ptr(y_local), y_local.shape[0], out,
                                            self.ctx.stream), "fitsne_bbox")
        return np.array(out[:], dtype=np.float64)

    def bbox_start(self, y_local: torch.Tensor) -> torch.Tensor:
        """Local bounding box on the device as {min, -max, -nonfinite} (no
        host sync; queued ahead of the SpMV so its blocks get the GPU first)."""
        buf = torch.empty(2 * self.dims + 1, dtype=torch.float64, device=self.device)
        _lib.check(self.ctx.lib.fitsne_bbox_device(self.ctx.h, _lib.ptr(y_local), y_local.shape[0],
                                                   _lib.ptr(buf), self.ctx.stream),
                   "fitsne_bbox_device")
        return buf

    def grid_finish(self, buf: torch.Tensor, group) -> None:
        """One MIN all-reduce of the packed boxes, one readback, the grid."""
        s = self.dims
        dist.all_reduce(buf, op=dist.ReduceOp.MIN, group=group)
        v = buf.cpu().numpy()
        if -v[2 * s] > 0:
            raise ValueError("points must be finite")
        self.set_grid(np.concatenate([v[:s], -v[s:2 * s]]))

    def set_grid(self, bbox: np.ndarray) -> None:
        arr = (C.c_double * (2 * self.dims))(*bbox.tolist())
        g = _lib.Grid()
        _lib.check(self.ctx.lib.fitsne_grid_from_bbox(self.ctx.h, arr, C.byref(g)),
                   "fitsne_grid_from_bbox")

    def spread(self, y_local: torch.Tensor) -> torch.Tensor:
        """Private spread into a persistent accumulator (the FFT stage
        consumes and clears it, so it is zeroed only when first made or after
        a step that failed in between); its dtype follows the grid pipeline
        (fp64 for a wide fp32 embedding, fitsne_grid_accum_dtype)."""
        n_acc = int(self.ctx.lib.fitsne_grid_accum_len(self.ctx.h))
        dt = torch.float64 if self.ctx.lib.fitsne_grid_accum_dtype(self.ctx.h) == _lib.F64 \
            else torch.float32
        if self._acc is None or self._acc.numel() < n_acc or self._acc.dtype != dt:
            self._acc = torch.zeros(max(n_acc, 1), dtype=dt, device=self.device)
        elif self._acc_dirty:
            self._acc.zero_()
        acc = self._acc[:n_acc]
        self._acc_dirty = True
        _lib.check(self.ctx.lib.fitsne_spread_tsne(self.ctx.h, _lib.ptr(y_local), y_local.shape[0],
                                                   _lib.ptr(acc), self.ctx.stream),
                   "fitsne_spread_tsne")
        return acc

    def fft(self, acc: torch.Tensor, want_z: bool = True):
        """FFT stage + Parseval Z.  Without want_z, Z is copied to pinned host
        memory behind the FFT stage (no host round trip inside the step); the
        caller checks it with check_z() once the rest of the step is queued."""
        z = C.c_double()
        _lib.check(self.ctx.lib.fitsne_fft_tsne(self.ctx.h, _lib.ptr(acc), self.n_total, 0,
                                                C.byref(z) if want_z else None, self.ctx.stream),
                   "fitsne_fft_tsne")
        self._acc_dirty = False  # consumed and cleared by the FFT stage
        if want_z:
            return float(z.value)
        _lib.check(self.ctx.lib.fitsne_read_z(self.ctx.h, _lib.ptr(self._zh), self.ctx.stream),
                   "fitsne_read_z")
        self._zev = torch.cuda.Event()
        self._zev.record(torch.cuda.current_stream(self.device))
        return None

    def check_z(self) -> None:
        """Z > 0 (optimizer.py:242-243): waits for the FFT stage only."""
        if self._zev is not None:
            self._zev.synchronize()
            z = float(self._zh[0])
            self._zev = None
            if not z > 0:
                raise ValueError("normalization Z must be positive")

    def gather(self, y_local: torch.Tensor) -> torch.Tensor:
        if self._f is None or self._f.shape != y_local.shape or self._f.dtype != y_local.dtype:
            self._f = torch.empty_like(y_local)
        f = self._f
        _lib.check(self.ctx.lib.fitsne_gather_tsne(self.ctx.h, _lib.ptr(y_local), y_local.shape[0],
                                                   _lib.ptr(f), None, None, self.ctx.stream),
                   "fitsne_gather_tsne")
        return f

    # -- SpMV concurrent with the repulsion stages ---------------------------
    def attract_start(self, y_full: torch.Tensor):
        """F_attr of the local rows on a side stream, ordered after the work
        already queued (the all-gather of Y); returns the completion event."""
        if not hasattr(self, "_side"):
            self._side = torch.cuda.Stream(device=self.device)
            self._attr = None
        n_local = self.csr.n_rows
        if self._attr is None or self._attr.shape[0] != n_local:
            self._attr = torch.empty((n_local, self.dims), dtype=self.dtype, device=self.device)
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(self.device))
        self._side.wait_event(ready)
        y_full.record_stream(self._side)
        _lib.check(self.ctx.lib.fitsne_attractive(self.ctx.h, _lib.ptr(y_full), _lib.ptr(self._attr),
                                                  C.c_void_p(self._side.cuda_stream)),
                   "fitsne_attractive")
        done = torch.cuda.Event()
        done.record(self._side)
        return done

    def attract_finish(self, done, forces_local: torch.Tensor, alpha: float) -> torch.Tensor:
        torch.cuda.current_stream(self.device).wait_event(done)
        g = torch.empty_like(forces_local)
        _lib.check(self.ctx.lib.fitsne_combine_rows(self.ctx.h, _lib.ptr(self._attr),
                                                    _lib.ptr(forces_local), forces_local.shape[0],
                                                    float(alpha), _lib.ptr(g), self.ctx.stream),
                   "fitsne_combine_rows")
        return g

    def attract_rows(self, y_full: torch.Tensor, forces_local: torch.Tensor,
                     alpha: float) -> torch.Tensor:
        g = torch.empty_like(forces_local)
        _lib.check(self.ctx.lib.fitsne_gradient_rows(self.ctx.h, _lib.ptr(y_full),
                                                     _lib.ptr(forces_local), float(alpha),
                                                     _lib.ptr(g), self.ctx.stream),
                   "fitsne_gradient_rows")
        return g


class ShardedGradient:
    """Row-partitioned gradient over a torch.distributed process group."""

    def __init__(self, P, n_dims=2, dtype=torch.float32, device=None, min_intervals=20,
                 points_per_interval=3, intervals_per_integer=1.0, group=None, stages=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.n = n_points(P)
        self.dims = n_dims
        self.row_begin, self.row_end = shard_range(self.n, self.rank, self.world)
        self.counts = [shard_range(self.n, r, self.world)[1] - shard_range(self.n, r, self.world)[0]
                       for r in range(self.world)]
        if stages is None:
            stages = LibStages(P, n_dims, dtype, device, min_intervals, points_per_interval,
                               intervals_per_integer, self.row_begin, self.row_end, self.counts)
        self.stages = stages
        self.launches_per_step = getattr(stages, "launches_per_step", 0)
        self._padded = getattr(stages, "padded_columns", False)
        self._yfull = None
        self._ypad = None

    def local(self, y_full):
        return y_full[self.row_begin:self.row_end]

    def _all_gather_rows(self, y_local):
        if self.world == 1:
            return y_local.contiguous()
        if self._padded:
            # padded layout (LibStages.padded_columns): one all-gather into a
            # persistent buffer, no per-step allocation or concatenation
            m = max(self.counts)
            if self._yfull is None or self._yfull.dtype != y_local.dtype:
                self._yfull = y_local.new_zeros((m * self.world, self.dims))
                self._ypad = y_local.new_zeros((m, self.dims))
            src = y_local.contiguous()
            if y_local.shape[0] != m:
                self._ypad[: y_local.shape[0]].copy_(y_local)
                src = self._ypad
            dist.all_gather_into_tensor(self._yfull, src, group=self.group)
            return self._yfull
        if min(self.counts) == max(self.counts):  # equal shards: gather in place
            out = y_local.new_empty((self.n, self.dims))
            dist.all_gather_into_tensor(out, y_local.contiguous(), group=self.group)
            return out
        m = max(self.counts)
        pad = y_local.new_zeros((m, self.dims))
        pad[: y_local.shape[0]] = y_local
        bufs = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(bufs, pad, group=self.group)
        return torch.cat([b[:c] for b, c in zip(bufs, self.counts)], 0).contiguous()

    def gradient(self, y_local, alpha: float = 1.0, y_full=None):
        """Gradient rows of this rank (n_local, s); y_local are its own points."""
        if alpha < 1.0:
            raise ValueError("exaggeration alpha must be >= 1")
        st = self.stages
        overlap = hasattr(st, "attract_start")
        # 3: all-gather Y (skipped when the caller already holds it)
        if y_full is None:
            y_full = self._all_gather_rows(y_local)
        elif self._padded and self.world > 1 and min(self.counts) != max(self.counts):
            m = max(self.counts)
            pad = y_full.new_zeros((m * self.world, self.dims))
            for r, c in enumerate(self.counts):
                b = shard_range(self.n, r, self.world)[0]
                pad[r * m: r * m + c] = y_full[b: b + c]
            y_full = pad
        device_box = hasattr(st, "bbox_start")
        if device_box:
            box = st.bbox_start(y_local)  # 1: queued first, so it gets the whole GPU
        if overlap:
            # 8a: the local rows' SpMV needs no grid: it runs on a side stream
            # while the host waits for the global box and 4-7 are queued
            done = st.attract_start(y_full)
        # 2: global bounding box -> identical grid everywhere
        if device_box:
            st.grid_finish(box, self.group)  # one all-reduce, one readback
        else:
            bb = st.bbox(y_local)
            s = self.dims
            lo = st.to_comm(bb[:s])
            hi = st.to_comm(bb[s:])
            dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=self.group)
            dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=self.group)
            st.set_grid(np.concatenate([lo.cpu().numpy(), hi.cpu().numpy()]))
        # 4-5: private spread + grid all-reduce
        acc = st.spread(y_local)
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=self.group)
        # 6: replicated FFT stage (Z stays on the device on the CUDA path)
        z = st.fft(acc, want_z=not overlap) if overlap else st.fft(acc)
        if z is not None and not z > 0:
            raise ValueError("normalization Z must be positive")
        # 7-8: gather local F_rep, combine with the SpMV over the local rows
        f_local = st.gather(y_local)
        if overlap:
            g = st.attract_finish(done, f_local, alpha)
            if hasattr(st, "check_z"):
                st.check_z()  # the rest of the step is already queued
            return g
        return st.attract_rows(y_full, f_local, alpha)


class NcclGradient:
    """The sharded gradient run entirely inside the library over its own NCCL
    communicator (fitsne_comm_init / fitsne_gradient_sharded): one C-ABI call
    per evaluation, the same partition and collectives as ShardedGradient.
    torch.distributed only carries the 128-byte NCCL id from rank 0."""

    def __init__(self, P, n_dims=2, dtype=torch.float32, device=None, min_intervals=20,
                 points_per_interval=3, intervals_per_integer=1.0, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.n = n_points(P)
        self.dims = n_dims
        self.dtype = dtype
        self.device = device
        self.row_begin, self.row_end = shard_range(self.n, self.rank, self.world)
        self.ctx = _lib.Context(device, n_dims, dtype, points_per_interval, min_intervals,
                                intervals_per_integer)
        self.csr = device_csr(P, dtype, device, self.row_begin, self.row_end)
        self.ctx.set_affinities(self.csr)
        uid = (C.c_char * 128)()
        if self.rank == 0:
            _lib.check(self.ctx.lib.fitsne_nccl_unique_id(uid), "fitsne_nccl_unique_id")
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0, group=group)
        uid = (C.c_char * 128).from_buffer_copy(box[0])
        _lib.check(self.ctx.lib.fitsne_comm_init(self.ctx.h, uid, self.rank, self.world, self.n),
                   "fitsne_comm_init")

    def local(self, y_full):
        return y_full[self.row_begin:self.row_end]

    def gradient(self, y_local, alpha: float = 1.0, out=None, z=None):
        """Gradient rows of this rank (n_local, s); y_local are its own points."""
        if alpha < 1.0:
            raise ValueError("exaggeration alpha must be >= 1")
        y_local = y_local.contiguous()
        g = out if out is not None else torch.empty_like(y_local)
        zc = C.c_double()
        _lib.check(self.ctx.lib.fitsne_gradient_sharded(self.ctx.h, _lib.ptr(y_local), float(alpha),
                                                        _lib.ptr(g), C.byref(zc), self.ctx.stream),
                   "fitsne_gradient_sharded")
        if z is not None:
            z.append(float(zc.value))
        return g

    def close(self):
        if getattr(self, "ctx", None) is not None:
            self.ctx.lib.fitsne_comm_destroy(self.ctx.h)
