"""Cauchy-kernel n-body sums on a B200: drop-in for ``fftsne.nbody``.

Same public names, signatures, return conventions and exceptions as the
reference module (/root/reference/pkg/src/fftsne/nbody.py).  Every array
computation runs in libfitsne_b200 (sm_100a):

  make_grid          nbody.py:118-150  -> fitsne_make_grid (device bbox + fp64 formulas)
  spread_charges     nbody.py:240-251  -> fitsne_spread
  kernel_matvec_fft  nbody.py:300-311  -> fitsne_kernel_matvec (hand-written FFT)
  kernel_matvec_direct nbody.py:314-341 -> fitsne_exact_nbody on the node coordinates
  gather_potentials  nbody.py:344-350  -> fitsne_gather
  evaluate_nbody     nbody.py:379-399  -> fitsne_evaluate_nbody
  brute_force_nbody  nbody.py:402-419  -> fitsne_exact_nbody

``kernel_eval``, ``lagrange_weights`` and ``InterpGrid`` are scalar/host
helpers of the API (closed-form formulas on a handful of values), not part of
the per-iteration path.

Extra keyword-only arguments (not in the reference): ``dtype`` ("float32" /
"float64"; default float64 for numpy inputs, the tensor's dtype for torch
inputs) and ``intervals_per_integer`` (FIt-SNE's option; 1.0 = reference).
Torch CUDA tensor inputs give CUDA tensor outputs; anything else gives float64
numpy arrays like the reference.
"""

from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _arrays as A
from . import _lib

__all__ = [
    "Kernel",
    "InterpGrid",
    "kernel_eval",
    "make_grid",
    "lagrange_weights",
    "spread_charges",
    "kernel_matvec_fft",
    "kernel_matvec_direct",
    "gather_potentials",
    "evaluate_nbody",
    "brute_force_nbody",
]


class Kernel(enum.Enum):
    """Embedding-space kernels (nbody.py:38-42)."""

    CAUCHY = "cauchy"                    # (1 + d^2)^-1
    CAUCHY_SQUARED = "cauchy_squared"    # (1 + d^2)^-2


_KCODE = {Kernel.CAUCHY: _lib.CAUCHY, Kernel.CAUCHY_SQUARED: _lib.CAUCHY_SQUARED}


def _kcode(kernel) -> int:
    if isinstance(kernel, Kernel):
        return _KCODE[kernel]
    # accept the reference's enum (same values) as well
    val = getattr(kernel, "value", kernel)
    for k, c in _KCODE.items():
        if k.value == val:
            return c
    raise ValueError(f"unknown kernel: {kernel!r}")


def kernel_eval(kernel, squared_distance):
    """Kernel value on squared distances (nbody.py:45-59); host helper."""
    code = _kcode(kernel)
    d2 = np.asarray(squared_distance, dtype=float)
    v = 1.0 / (1.0 + d2)
    if code == _lib.CAUCHY_SQUARED:
        v = v * v
    return float(v) if v.ndim == 0 else v


@dataclass(frozen=True)
class InterpGrid:
    """Equispaced interpolation grid (nbody.py:62-104)."""

    dims: int
    lo: tuple
    hi: tuple
    n_intervals: int
    points_per_interval: int

    def __post_init__(self):
        if self.dims not in (1, 2):
            raise ValueError("only 1D and 2D grids are supported")
        if self.n_intervals < 1:
            raise ValueError("n_intervals must be >= 1")
        if self.points_per_interval < 2:
            raise ValueError("points_per_interval must be >= 2")
        if len(self.lo) != self.dims or len(self.hi) != self.dims:
            raise ValueError("bounds do not match dims")
        if any(not h > l for l, h in zip(self.lo, self.hi)):
            raise ValueError("grid bounds must satisfy hi > lo")

    @property
    def nodes_per_dim(self) -> int:
        return self.n_intervals * self.points_per_interval

    @property
    def total_nodes(self) -> int:
        return self.nodes_per_dim ** self.dims

    @property
    def spacing(self) -> np.ndarray:
        return (np.asarray(self.hi, dtype=float) - np.asarray(self.lo, dtype=float)) / self.nodes_per_dim

    def nodes(self, dim: int = 0) -> np.ndarray:
        return self.lo[dim] + (np.arange(self.nodes_per_dim) + 0.5) * self.spacing[dim]

    # -- device descriptor -------------------------------------------------
    def _c(self) -> _lib.Grid:
        g = _lib.Grid()
        for d in range(self.dims):
            g.lo[d] = float(self.lo[d])
            g.hi[d] = float(self.hi[d])
        g.dims = self.dims
        g.n_intervals = int(self.n_intervals)
        g.points_per_interval = int(self.points_per_interval)
        return g


def _grid_from_c(g: _lib.Grid) -> InterpGrid:
    return InterpGrid(
        dims=int(g.dims),
        lo=tuple(float(g.lo[d]) for d in range(g.dims)),
        hi=tuple(float(g.hi[d]) for d in range(g.dims)),
        n_intervals=int(g.n_intervals),
        points_per_interval=int(g.points_per_interval),
    )


def _ctx_for_grid(grid: InterpGrid, dtype, device):
    ctx = _lib.context(device, grid.dims, dtype, grid.points_per_interval, 1)
    _lib.check(ctx.lib.fitsne_set_grid(ctx.h, C.byref(grid._c())), "fitsne_set_grid")
    return ctx


def make_grid(points, min_intervals: int = 20, points_per_interval: int = 3, *,
              intervals_per_integer: float = 1.0, dtype=None) -> InterpGrid:
    """Grid over the bounding box of ``points`` (nbody.py:118-150), on the device."""
    pts = A.as_points(points)
    if min_intervals < 1:
        raise ValueError("min_intervals must be >= 1")
    if points_per_interval < 2:
        raise ValueError("points_per_interval must be >= 2")
    dev = A.device_of(pts)
    dt = A.compute_dtype(pts, dtype)
    y = A.to_device(pts, dt, dev)
    ctx = _lib.context(dev, y.shape[1], dt, points_per_interval, min_intervals,
                       intervals_per_integer)
    g = _lib.Grid()
    rc = ctx.lib.fitsne_make_grid(ctx.h, _lib.ptr(y), y.shape[0], C.byref(g), ctx.stream)
    if rc in (_lib.ENONFINITE, _lib.EPOINTS):
        raise ValueError("points must be finite")
    _lib.check(rc, "fitsne_make_grid")
    return _grid_from_c(g)


def lagrange_weights(nodes, x):
    """Lagrange basis weights at ``x`` for arbitrary nodes (nbody.py:153-173); host helper."""
    nd = np.asarray(nodes, dtype=float)
    if nd.ndim != 1 or nd.size < 1:
        raise ValueError("nodes must be a 1D array")
    if np.unique(nd).size != nd.size:
        raise ValueError("interpolation nodes must be pairwise distinct")
    xa = np.asarray(x, dtype=float)
    out = np.empty(xa.shape + (nd.size,))
    for j in range(nd.size):
        num = np.ones(xa.shape)
        den = 1.0
        for m in range(nd.size):
            if m != j:
                num = num * (xa - nd[m])
                den = den * (nd[j] - nd[m])
        out[..., j] = num / den
    return out


def spread_charges(points, charges, grid: InterpGrid, *, dtype=None):
    """Charges -> grid-node coefficients (nbody.py:240-251)."""
    pts = A.as_points(points, grid.dims)
    n = pts.shape[0]
    q_shape = tuple(charges.shape) if isinstance(charges, torch.Tensor) else np.shape(charges)
    if q_shape != (n,):
        raise ValueError("need exactly one charge per point")
    dev = A.device_of(pts, charges)
    dt = A.compute_dtype(pts, dtype)
    y = A.to_device(pts, dt, dev)
    q = A.to_device(charges, dt, dev).reshape(n, 1)
    ctx = _ctx_for_grid(grid, dt, dev)
    out = torch.empty(grid.total_nodes, dtype=dt, device=dev)
    _lib.check(ctx.lib.fitsne_spread(ctx.h, _lib.ptr(y), n, _lib.ptr(q), 1, _lib.ptr(out),
                                     ctx.stream), "fitsne_spread")
    return A.output(out, A.is_device_input(points))


def kernel_matvec_fft(coeffs, kernel, grid: InterpGrid, workers: int = 1, *, dtype=None):
    """Toeplitz node-kernel product through the circulant FFT (nbody.py:300-311)."""
    code = _kcode(kernel)
    dev = A.device_of(coeffs)
    dt = A.compute_dtype(coeffs, dtype)
    w = A.to_device(coeffs, dt, dev).reshape(-1)
    if w.numel() != grid.total_nodes:
        raise ValueError("coefficient length does not match the grid")
    ctx = _ctx_for_grid(grid, dt, dev)
    out = torch.empty_like(w)
    _lib.check(ctx.lib.fitsne_kernel_matvec(ctx.h, code, _lib.ptr(w), 1, _lib.ptr(out), ctx.stream),
               "fitsne_kernel_matvec")
    return A.output(out, A.is_device_input(coeffs))


def _node_coordinates(grid: InterpGrid) -> np.ndarray:
    if grid.dims == 1:
        return grid.nodes(0)[:, None]
    gx, gy = np.meshgrid(grid.nodes(0), grid.nodes(1), indexing="ij")
    return np.column_stack([gx.ravel(), gy.ravel()])


def kernel_matvec_direct(coeffs, kernel, grid: InterpGrid, *, dtype=None):
    """Dense node-kernel product (nbody.py:314-341): O(G^2) on the device."""
    code = _kcode(kernel)
    dev = A.device_of(coeffs)
    dt = A.compute_dtype(coeffs, dtype)
    w = A.to_device(coeffs, dt, dev).reshape(-1)
    if w.numel() != grid.total_nodes:
        raise ValueError("coefficient length does not match the grid")
    nodes = A.to_device(_node_coordinates(grid), dt, dev)
    ctx = _lib.context(dev, grid.dims, dt, grid.points_per_interval, 1)
    out = torch.empty_like(w)
    _lib.check(ctx.lib.fitsne_exact_nbody(ctx.h, _lib.ptr(nodes), nodes.shape[0], _lib.ptr(w), 1,
                                          code, 1, _lib.ptr(out), ctx.stream), "fitsne_exact_nbody")
    return A.output(out, A.is_device_input(coeffs))


def gather_potentials(points, values, grid: InterpGrid, *, dtype=None):
    """Grid-node values -> point potentials (nbody.py:344-350)."""
    dev = A.device_of(points, values)
    dt = A.compute_dtype(values, dtype)
    v = A.to_device(values, dt, dev).reshape(-1)
    if v.numel() != grid.total_nodes:
        raise ValueError("value length does not match the grid")
    pts = A.as_points(points, grid.dims)
    y = A.to_device(pts, dt, dev)
    ctx = _ctx_for_grid(grid, dt, dev)
    out = torch.empty(y.shape[0], dtype=dt, device=dev)
    _lib.check(ctx.lib.fitsne_gather(ctx.h, _lib.ptr(y), y.shape[0], _lib.ptr(v), 1, _lib.ptr(out),
                                     ctx.stream), "fitsne_gather")
    return A.output(out, A.is_device_input(points))


def _charges_2d(charges, n, dt, dev):
    q = A.to_device(charges, dt, dev)
    if q.shape[0] != n:
        raise ValueError("charges must match point count")
    return (q.reshape(n, 1) if q.dim() == 1 else q.contiguous()), q.dim() == 1


def evaluate_nbody(points, charges, kernel, min_intervals: int = 20, points_per_interval: int = 3,
                   include_self: bool = True, workers: int = 1, *, intervals_per_integer=1.0,
                   dtype=None):
    """phi_i = sum_j K(y_i, y_j) q_j through the grid pipeline (nbody.py:379-399)."""
    code = _kcode(kernel)
    pts = A.as_points(points)
    dev = A.device_of(pts, charges)
    dt = A.compute_dtype(pts, dtype)
    y = A.to_device(pts, dt, dev)
    n = y.shape[0]
    q, single = _charges_2d(charges, n, dt, dev)
    if min_intervals < 1:
        raise ValueError("min_intervals must be >= 1")
    ctx = _lib.context(dev, y.shape[1], dt, points_per_interval, min_intervals, intervals_per_integer)
    out = torch.empty_like(q)
    rc = ctx.lib.fitsne_evaluate_nbody(ctx.h, _lib.ptr(y), n, _lib.ptr(q), q.shape[1], code,
                                       1 if include_self else 0, _lib.ptr(out), ctx.stream)
    if rc in (_lib.ENONFINITE, _lib.EPOINTS):
        raise ValueError("points must be finite")
    _lib.check(rc, "fitsne_evaluate_nbody")
    out = out[:, 0] if single else out
    return A.output(out, A.is_device_input(points))


def brute_force_nbody(points, charges, kernel, include_self: bool = True, block: int = 512, *,
                      dtype=None):
    """Exact O(N^2) sums (nbody.py:402-419) on the device; ``block`` is accepted and unused."""
    code = _kcode(kernel)
    pts = A.as_points(points)
    dev = A.device_of(pts, charges)
    dt = A.compute_dtype(pts, dtype)
    y = A.to_device(pts, dt, dev)
    n = y.shape[0]
    q, single = _charges_2d(charges, n, dt, dev)
    ctx = _lib.context(dev, y.shape[1], dt, 3, 1)
    out = torch.empty_like(q)
    _lib.check(ctx.lib.fitsne_exact_nbody(ctx.h, _lib.ptr(y), n, _lib.ptr(q), q.shape[1], code,
                                          1 if include_self else 0, _lib.ptr(out), ctx.stream),
               "fitsne_exact_nbody")
    out = out[:, 0] if single else out
    return A.output(out, A.is_device_input(points))


def point_interp(points, grid: InterpGrid, *, dtype=None):
    """Parity hook for ``nbody._point_interp`` (nbody.py:201-230): (node_index int64, weights)."""
    pts = A.as_points(points, grid.dims)
    dev = A.device_of(pts)
    dt = A.compute_dtype(pts, dtype)
    y = A.to_device(pts, dt, dev)
    n = y.shape[0]
    k = grid.points_per_interval ** grid.dims
    idx = torch.empty((n, k), dtype=torch.int64, device=dev)
    w = torch.empty((n, k), dtype=dt, device=dev)
    ctx = _ctx_for_grid(grid, dt, dev)
    _lib.check(ctx.lib.fitsne_point_interp(ctx.h, _lib.ptr(y), n, _lib.ptr(idx), _lib.ptr(w),
                                           ctx.stream), "fitsne_point_interp")
    if A.is_device_input(points):
        return idx, w
    return idx.cpu().numpy(), w.to(torch.float64).cpu().numpy()
