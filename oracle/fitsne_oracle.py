"""CPU oracle for the FIt-SNE gradient path -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) may import it.  The product path
(``paper_1712_09005_b200``) runs exclusively on the CUDA library and fails
loudly when that library is missing.

It restates, in numpy/scipy, the algorithm of the reference package
``fftsne`` (``/root/reference/pkg/src/fftsne``), function by function, with
the same arithmetic order wherever bit-exactness matters (box indices, node
indices, Lagrange weights).  The reference's third-party numerics are the
same libraries used here: ``np.bincount`` for spreading / scatter-adds and
``scipy.fft`` (pocketfft) for the circulant convolution; the reference's
numba ``fastmath`` exact loop is restated as blocked numpy.

Pinning: ``tests/test_oracle_golden.py`` checks this module against golden
vectors produced by running the reference itself (``tests/golden/make_golden.py``,
run in the build container where ``/root/reference`` is importable) and
against the closed-form known answers in the reference tests
(``pkg/tests/test_nbody.py``, ``pkg/tests/test_optimizer.py``).
"""

from __future__ import annotations

import math
from typing import NamedTuple

import numpy as np
import scipy.fft as _fft

CAUCHY = "cauchy"                 # 1/(1+d^2)      nbody.py:41
CAUCHY_SQUARED = "cauchy_squared"  # 1/(1+d^2)^2   nbody.py:42


class Grid(NamedTuple):
    """Equispaced interpolation grid (nbody.py:62-104)."""

    lo: tuple
    hi: tuple
    n_int: int
    p: int

    @property
    def dims(self):
        return len(self.lo)

    @property
    def n(self):  # nodes per dimension
        return self.n_int * self.p

    @property
    def h(self):  # node spacing per dimension, nbody.py:97-99
        return (np.asarray(self.hi) - np.asarray(self.lo)) / self.n

    def node_coords(self, d):  # nbody.py:101-104
        return self.lo[d] + (np.arange(self.n) + 0.5) * self.h[d]


def cauchy(kind, d2):
    """Kernel values on squared distances (nbody.py:45-59)."""
    base = 1.0 / (1.0 + np.asarray(d2, dtype=float))
    if kind == CAUCHY:
        return base
    if kind == CAUCHY_SQUARED:
        return base * base
    raise ValueError(kind)


def grid_for(points, min_intervals=20, p=3, intervals_per_integer=1.0):
    """Bounding-box grid of ``points`` (N, s) (nbody.py:118-150).

    The interval count is max(min_intervals, ceil(largest span)); spans below
    one are widened to unit width about their centre, others padded by 1e-6
    of the span.  ``intervals_per_integer`` generalises the reference's
    hard-coded 1 (FIt-SNE's option); 1.0 reproduces the reference exactly.
    """
    y = np.asarray(points, dtype=float)
    if y.ndim == 1:
        y = y[:, None]
    mins = y.min(axis=0)
    maxs = y.max(axis=0)
    width = maxs - mins
    widest = float(width.max())
    if intervals_per_integer == 1.0:
        n_int = max(min_intervals, int(math.ceil(widest)))
    else:
        n_int = max(min_intervals, int(math.ceil(widest * intervals_per_integer)))
    lo, hi = [], []
    for d in range(y.shape[1]):
        if width[d] < 1.0:
            mid = 0.5 * (mins[d] + maxs[d])
            lo.append(float(mid - 0.5))
            hi.append(float(mid + 0.5))
        else:
            eps = 1e-6 * width[d]
            lo.append(float(mins[d] - eps))
            hi.append(float(maxs[d] + eps))
    return Grid(tuple(lo), tuple(hi), n_int, p)


def _basis_denominators(p):
    # prod_{i != j} (j - i), nbody.py:176-180
    return np.array([np.prod([j - i for i in range(p) if i != j]) for j in range(p)],
                    dtype=float)


def _basis_values(u, p):
    # Lagrange basis on nodes 0..p-1 at offsets u, nbody.py:183-190
    den = _basis_denominators(p)
    diffs = u[:, None] - np.arange(p)[None, :]
    w = np.empty((u.size, p))
    for j in range(p):
        keep = [i for i in range(p) if i != j]
        w[:, j] = np.prod(diffs[:, keep], axis=1) / den[j]
    return w


def interp(grid, points):
    """Node indices and tensor-product weights per point (nbody.py:201-230).

    Returns (node_index (N, p^s) int64, weights (N, p^s) float64).  The
    box index follows the reference's order of operations exactly:
    t = (x - lo)/h; cell = clip(t // p, 0, n_int-1); u = t - cell*p - 0.5.
    """
    y = np.asarray(points, dtype=float)
    if y.ndim == 1:
        y = y[:, None]
    p = grid.p
    h = grid.h
    base, wts = [], []
    for d in range(y.shape[1]):
        x = y[:, d]
        if np.any(x < grid.lo[d]) or np.any(x > grid.hi[d]):
            raise ValueError("point outside grid bounds")
        t = (x - grid.lo[d]) / h[d]
        cell = np.clip((t // p).astype(np.int64), 0, grid.n_int - 1)
        u = t - cell * p - 0.5
        base.append(cell * p)
        wts.append(_basis_values(u, p))
    offs = np.arange(p, dtype=np.int64)
    if y.shape[1] == 1:
        return base[0][:, None] + offs[None, :], wts[0]
    n = grid.n
    rows = base[0][:, None, None] + offs[None, :, None]
    cols = base[1][:, None, None] + offs[None, None, :]
    idx = (rows * n + cols).reshape(y.shape[0], p * p)
    w = (wts[0][:, :, None] * wts[1][:, None, :]).reshape(y.shape[0], p * p)
    return idx, w


def spread(idx, w, charges, grid):
    """Scatter-add of weighted charges onto the nodes (nbody.py:233-237)."""
    total = grid.n ** grid.dims
    return np.bincount(idx.ravel(), weights=(w * np.asarray(charges)[:, None]).ravel(),
                       minlength=total)


def spectrum(kind, grid, workers=1):
    """Real FFT of the kernel's circulant embedding (nbody.py:262-282).

    Returns (spectrum, L) with L = next_fast_len(2n - 1).
    """
    n = grid.n
    L = _fft.next_fast_len(2 * n - 1)
    if grid.dims == 1:
        col = cauchy(kind, (np.arange(n) * grid.h[0]) ** 2)
        c = np.zeros(L)
        c[:n] = col
        c[L - n + 1:] = col[:0:-1]
        return _fft.rfft(c), L
    hx, hy = grid.h
    first = cauchy(kind, ((np.arange(n) * hx) ** 2)[:, None] + ((np.arange(n) * hy) ** 2)[None, :])
    c = np.zeros((L, L))
    c[:n, :n] = first
    c[L - n + 1:, :n] = first[:0:-1, :]
    c[:n, L - n + 1:] = first[:, :0:-1]
    c[L - n + 1:, L - n + 1:] = first[:0:-1, :0:-1]
    return _fft.rfft2(c, workers=workers), L


def toeplitz_apply(coeffs, spec, L, grid, workers=1):
    """Node-kernel matvec through the circulant FFT (nbody.py:285-297)."""
    n = grid.n
    if grid.dims == 1:
        f = _fft.rfft(coeffs, n=L, workers=workers) * spec
        return _fft.irfft(f, n=L, workers=workers)[:n]
    f = _fft.rfft2(coeffs.reshape(n, n), s=(L, L), workers=workers) * spec
    return _fft.irfft2(f, s=(L, L), workers=workers)[:n, :n].ravel()


def toeplitz_direct(coeffs, kind, grid):
    """Dense node-kernel matvec (the oracle for toeplitz_apply; nbody.py:314-341)."""
    n = grid.n
    if grid.dims == 1:
        x = grid.node_coords(0)
        return cauchy(kind, (x[:, None] - x[None, :]) ** 2) @ coeffs
    hx, hy = grid.h
    ix = np.arange(n)
    dx2 = ((ix[:, None] - ix[None, :]) * hx) ** 2
    dy2 = ((ix[:, None] - ix[None, :]) * hy) ** 2
    W = coeffs.reshape(n, n)
    out = np.zeros_like(W)
    for a in range(n):
        kern = cauchy(kind, dx2[a][:, None] + dy2)   # (n_x', n_y, n_y')
        out[a] = np.einsum("bj,bkj->k", W, kern) if False else (kern * W[:, None, :]).sum(axis=(0, 2))
    return out.ravel()


def gather(idx, w, values):
    """Interpolate node values back to the points (nbody.py:344-350)."""
    return (np.asarray(values)[idx] * w).sum(axis=1)


def nbody_fft(points, charges, kind, min_intervals=20, p=3, include_self=True, workers=1,
              intervals_per_integer=1.0):
    """Grid evaluation of phi_i = sum_j K(y_i, y_j) q_j (nbody.py:353-399)."""
    y = np.asarray(points, dtype=float)
    if y.ndim == 1:
        y = y[:, None]
    q = np.asarray(charges, dtype=float)
    grid = grid_for(y, min_intervals, p, intervals_per_integer)
    idx, w = interp(grid, y)
    spec, L = spectrum(kind, grid, workers)
    cols = q if q.ndim == 2 else q[:, None]
    out = np.empty_like(cols)
    for c in range(cols.shape[1]):
        v = toeplitz_apply(spread(idx, w, cols[:, c], grid), spec, L, grid, workers)
        out[:, c] = gather(idx, w, v)
    if not include_self:
        out -= cols
    return out if q.ndim == 2 else out[:, 0]


def nbody_exact(points, charges, kind, include_self=True, block=512):
    """O(N^2) kernel sums (nbody.py:402-419)."""
    y = np.asarray(points, dtype=float)
    if y.ndim == 1:
        y = y[:, None]
    q = np.asarray(charges, dtype=float)
    cols = q if q.ndim == 2 else q[:, None]
    out = np.empty_like(cols)
    for a in range(0, y.shape[0], block):
        b = min(a + block, y.shape[0])
        d2 = ((y[a:b, None, :] - y[None, :, :]) ** 2).sum(-1)
        out[a:b] = cauchy(kind, d2) @ cols
    if not include_self:
        out -= cols
    return out if q.ndim == 2 else out[:, 0]


# --------------------------------------------------------------------------
# optimizer.py restatement
# --------------------------------------------------------------------------

def repulsion_sums_fft(y, min_intervals, p, workers=1, intervals_per_integer=1.0):
    """k1 = K1*1 - 1, k2[:, c] = K2*y_c - y_c, k2[:, s] = K2*1 - 1 (optimizer.py:193-211)."""
    grid = grid_for(y, min_intervals, p, intervals_per_integer)
    idx, w = interp(grid, y)
    s1, L = spectrum(CAUCHY, grid, workers)
    s2, _ = spectrum(CAUCHY_SQUARED, grid, workers)

    def conv(q, s):
        return gather(idx, w, toeplitz_apply(spread(idx, w, q, grid), s, L, grid, workers))

    n, s = y.shape
    ones = np.ones(n)
    k1 = conv(ones, s1) - 1.0
    k2 = np.empty((n, s + 1))
    for c in range(s):
        k2[:, c] = conv(y[:, c], s2) - y[:, c]
    k2[:, s] = conv(ones, s2) - 1.0
    return k1, k2


def repulsion_sums_exact(y, block=256):
    """Self-excluded exact K1 / K2 sums (optimizer.py:169-190), blocked numpy."""
    n, s = y.shape
    k1 = np.empty(n)
    k2 = np.empty((n, s + 1))
    aug = np.concatenate([y, np.ones((n, 1))], axis=1)
    for a in range(0, n, block):
        b = min(a + block, n)
        d2 = ((y[a:b, None, :] - y[None, :, :]) ** 2).sum(-1)
        q = 1.0 / (1.0 + d2)
        r = np.arange(a, b)
        q[r - a, r] = 0.0
        k1[a:b] = q.sum(axis=1)
        k2[a:b] = (q * q) @ aug
    return k1, k2


def repulsion(y, min_intervals=20, p=3, method="auto", workers=1, intervals_per_integer=1.0):
    """(forces, z, k1, k2) exactly as compute_repulsive (optimizer.py:214-245)."""
    y = np.ascontiguousarray(y, dtype=float)
    n = y.shape[0]
    if method == "auto":
        method = "exact" if n <= 1000 else "fft"   # optimizer.py:37, 233-234
    if method == "exact":
        k1, k2 = repulsion_sums_exact(y)
    elif method == "fft":
        k1, k2 = repulsion_sums_fft(y, min_intervals, p, workers, intervals_per_integer)
    else:
        raise ValueError(method)
    z = float(k1.sum())
    forces = (y * k2[:, -1:] - k2[:, :-1]) / z
    return forces, z, k1, k2


def attraction(rows, cols, vals, y):
    """sum_j p_ij (1+d^2)^-1 (y_i - y_j) over upper-COO pairs, both directions
    (optimizer.py:150-166)."""
    n = y.shape[0]
    dy = y[rows] - y[cols]
    wgt = vals / (1.0 + (dy * dy).sum(axis=1))
    out = np.empty_like(y)
    for c in range(y.shape[1]):
        t = wgt * dy[:, c]
        out[:, c] = np.bincount(rows, weights=t, minlength=n) - np.bincount(cols, weights=t, minlength=n)
    return out


def grad(rows, cols, vals, y, alpha=1.0, min_intervals=20, p=3, method="auto", workers=1,
         intervals_per_integer=1.0):
    """4 (alpha F_attr - F_rep) (optimizer.py:248-262)."""
    f_rep = repulsion(y, min_intervals, p, method, workers, intervals_per_integer)[0]
    return 4.0 * (alpha * attraction(rows, cols, vals, y) - f_rep)


def kl_given_z(rows, cols, vals, y, z):
    """2 sum_{p>0} p (log p - log q), q = 1/((1+d^2) Z) (optimizer.py:265-275)."""
    dy = y[rows] - y[cols]
    d2 = (dy * dy).sum(axis=1)
    m = vals > 0
    pv, d2 = vals[m], d2[m]
    q = 1.0 / ((1.0 + d2) * z)
    return 2.0 * float(np.sum(pv * (np.log(pv) - np.log(q))))


def update(y, g, velocity, gains, lr, momentum):
    """Momentum + gains step (optimizer.py:299-323); returns (y, velocity, gains)."""
    agree = np.sign(g) == np.sign(velocity)
    v = momentum * velocity - lr * gains * g
    new_gains = np.where(agree, gains * 0.8, gains + 0.2)
    np.maximum(new_gains, 0.01, out=new_gains)
    return y + v, v, new_gains


def initial_embedding(n, dims, seed):
    """Seeded Y0 draw of run_tsne (optimizer.py:350, 378-379)."""
    seeds = np.random.SeedSequence(seed).spawn(3)
    return np.random.default_rng(seeds[1]).normal(0.0, 1e-4, size=(n, dims))


def alpha_at(it, n_iter, early_coeff=12.0, early_until=250, late_coeff=1.0, late_from=None):
    """ExaggerationSchedule.alpha (optimizer.py:63-73)."""
    if it < early_until:
        return early_coeff
    lf = late_from if late_from is not None else max(early_until, n_iter - 250)
    if late_coeff != 1.0 and it >= lf:
        return late_coeff
    return 1.0


def tsne(rows, cols, vals, n, dims=2, n_iter=1000, lr=200.0, momentum_early=0.5,
         momentum_late=0.8, momentum_switch=250, early_coeff=12.0, early_until=250,
         late_coeff=1.0, late_from=None, min_intervals=20, p=3, method="auto", seed=0,
         workers=1, y0=None):
    """The run_tsne descent loop on precomputed affinities (optimizer.py:377-415)."""
    y = initial_embedding(n, dims, seed) if y0 is None else np.array(y0, dtype=float)
    vel = np.zeros((n, dims))
    gains = np.ones((n, dims))
    kl = np.empty(n_iter)
    for it in range(n_iter):
        a = alpha_at(it, n_iter, early_coeff, early_until, late_coeff, late_from)
        attr = attraction(rows, cols, vals, y)
        f_rep, z, _, _ = repulsion(y, min_intervals, p, method, workers)
        g = 4.0 * (a * attr - f_rep)
        kl[it] = kl_given_z(rows, cols, vals, y, z)
        mom = momentum_early if it < momentum_switch else momentum_late
        y, vel, gains = update(y, g, vel, gains, lr, mom)
    return y, kl


def upper_to_csr(n, rows, cols, vals):
    """Full symmetric CSR (both triangles) from upper COO: (rowptr, col, val)."""
    r = np.concatenate([rows, cols])
    c = np.concatenate([cols, rows])
    v = np.concatenate([vals, vals])
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rowptr, r + 1, 1)
    return np.cumsum(rowptr), c, v
