"""t-SNE gradient, KL and descent on a B200: drop-in for ``fftsne.optimizer``.

Same public names, signatures, defaults, return types and exceptions as the
reference (/root/reference/pkg/src/fftsne/optimizer.py).  The arithmetic runs
in libfitsne_b200 (sm_100a):

  compute_attractive  optimizer.py:150-166 -> fitsne_attractive (warp-per-row CSR SpMV)
  compute_repulsive   optimizer.py:214-245 -> fitsne_repulsive (fft) / fitsne_repulsive_exact
  gradient            optimizer.py:248-262 -> fitsne_gradient (fft) / exact sums + fitsne_gradient_rows
  kl_divergence       optimizer.py:278-296 -> fitsne_kl (+ Z from the grid or the exact sums)
  step                optimizer.py:299-323 -> fitsne_step
  run_tsne            optimizer.py:331-415 -> fitsne_iterate (fused iteration, KL logged on device)

Extensions (keyword-only / extra config fields): ``dtype`` (float32 |
float64), ``device``, FIt-SNE's option names ``n_interpolation_points``,
``min_num_intervals`` and ``intervals_per_integer``.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _arrays as A
from . import _lib
from .affinities import SparseAffinities, device_csr, n_points, ordered_total

__all__ = [
    "ExaggerationSchedule",
    "TsneConfig",
    "OptimizerState",
    "Repulsion",
    "TsneResult",
    "compute_attractive",
    "compute_repulsive",
    "gradient",
    "kl_divergence",
    "step",
    "run_tsne",
]

EXACT_REPULSION_MAX_N = 1000   # optimizer.py:37
EXACT_KL_MAX_N = 10_000        # optimizer.py:38


@dataclass
class ExaggerationSchedule:
    """alpha = early_coeff before early_until_iter, late_coeff from late_from
    (when late_coeff != 1), else 1 (optimizer.py:41-73; including its
    validation rule that late_from defaults to max(early_until, n_iter - 250))."""

    early_coeff: float = 12.0
    early_until_iter: int = 250
    late_coeff: float = 1.0
    late_from_iter: int | None = None

    def validate(self, n_iter: int) -> None:
        if self.early_coeff < 1.0 or self.late_coeff < 1.0:
            raise ValueError("exaggeration coefficients must be >= 1")
        late_from = self.resolved_late_from(n_iter)
        if not 0 <= self.early_until_iter <= late_from <= n_iter:
            raise ValueError("need 0 <= early_until_iter <= late_from_iter <= n_iter")

    def resolved_late_from(self, n_iter: int) -> int:
        if self.late_from_iter is not None:
            return self.late_from_iter
        return max(self.early_until_iter, n_iter - 250)

    def alpha(self, iteration: int, n_iter: int) -> float:
        if iteration < self.early_until_iter:
            return self.early_coeff
        if self.late_coeff != 1.0 and iteration >= self.resolved_late_from(n_iter):
            return self.late_coeff
        return 1.0


@dataclass
class TsneConfig:
    dims: int = 2
    perplexity: float = 30.0
    n_iter: int = 1000
    learning_rate: float = 200.0
    momentum_early: float = 0.5
    momentum_late: float = 0.8
    momentum_switch_iter: int = 250
    exaggeration: ExaggerationSchedule = field(default_factory=ExaggerationSchedule)
    seed: int = 0
    knn_method: str = "auto"
    n_neighbors: int | None = None
    n_trees: int = 50
    subsample: int | None = None
    min_intervals: int = 20
    points_per_interval: int = 3
    repulsion_method: str = "auto"   # auto | exact | fft
    pca_dims: int | None = 50
    workers: int = 1
    # --- B200 extensions -------------------------------------------------
    dtype: str = "float64"           # "float32" for the fast path
    device: int | None = None
    intervals_per_integer: float = 1.0
    n_interpolation_points: int | None = None   # FIt-SNE alias of points_per_interval
    min_num_intervals: int | None = None        # FIt-SNE alias of min_intervals
    # locality relabelling of the points (Z-order of the embedding) in run_tsne
    # off by default: on the C3 synthetic data it costs more than it saves
    reorder_iters: tuple | None = None
    reorder_min_n: int = 100_000

    def __post_init__(self):
        if self.n_interpolation_points is not None:
            self.points_per_interval = int(self.n_interpolation_points)
        if self.min_num_intervals is not None:
            self.min_intervals = int(self.min_num_intervals)

    def validate(self) -> None:
        if self.dims not in (1, 2):
            raise ValueError("embedding dims must be 1 or 2")
        if self.n_iter < 1:
            raise ValueError("n_iter must be positive")
        if self.perplexity <= 0:
            raise ValueError("perplexity must be positive")
        self.exaggeration.validate(self.n_iter)


@dataclass
class OptimizerState:
    iteration: int
    velocity: object
    gains: object
    learning_rate: float

    @classmethod
    def fresh(cls, n: int, dims: int, learning_rate: float = 200.0) -> "OptimizerState":
        return cls(iteration=0, velocity=np.zeros((n, dims)), gains=np.ones((n, dims)),
                   learning_rate=learning_rate)


@dataclass
class Repulsion:
    forces: object         # (N, s)
    z: float
    k1_potential: object   # (N,)
    k2_potentials: object  # (N, s + 1): coordinate charges first, unit charge last


@dataclass
class TsneResult:
    embedding: object
    kl_log: object
    affinities: object


# -----------------------------------------------------------------------------
def _shape(x):
    return tuple(x.shape) if isinstance(x, torch.Tensor) else np.shape(x)


def _embedding(Y, dtype):
    dev = A.device_of(Y)
    dt = A.compute_dtype(Y, dtype)
    return A.to_device(Y, dt, dev), dev, dt


def _ctx_with_P(P, dev, dims, dt, p=3, min_int=20, ipi=1.0):
    csr = device_csr(P, dt, dev)
    ctx = _lib.context(dev, dims, dt, p, min_int, ipi)
    ctx.set_affinities(csr, owner=P)
    return ctx, csr


def compute_attractive(P, Y, *, dtype=None):
    """sum_j p_ij (1 + d_ij^2)^-1 (y_i - y_j) (optimizer.py:150-166)."""
    shp = _shape(Y)
    if len(shp) != 2 or shp[0] != n_points(P):
        raise ValueError("embedding shape does not match the affinities")
    y, dev, dt = _embedding(Y, dtype)
    ctx, _ = _ctx_with_P(P, dev, y.shape[1], dt)
    out = torch.empty_like(y)
    _lib.check(ctx.lib.fitsne_attractive(ctx.h, _lib.ptr(y), _lib.ptr(out), ctx.stream),
               "fitsne_attractive")
    return A.output(out, A.is_device_input(Y))


def _check_embedding(Y):
    shp = _shape(Y)
    if len(shp) != 2 or shp[1] not in (1, 2):
        raise ValueError("embedding must be (N, 1) or (N, 2)")
    if shp[0] < 2:
        raise ValueError("repulsion needs at least two points")
    return shp[0]


def _resolve_method(method, n, limit=EXACT_REPULSION_MAX_N):
    if method == "auto":
        return "exact" if n <= limit else "fft"
    if method not in ("exact", "fft"):
        raise ValueError(f"unknown repulsion method: {method!r}")
    return method


def _repulsion_device(y, dev, dt, min_intervals, points_per_interval, method, ipi=1.0,
                      check_z=True):
    n, s = y.shape
    ctx = _lib.context(dev, s, dt, points_per_interval, min_intervals, ipi)
    forces = torch.empty_like(y)
    k1 = torch.empty(n, dtype=dt, device=dev)
    k2 = torch.empty((n, s + 1), dtype=dt, device=dev)
    z = C.c_double()
    fn = ctx.lib.fitsne_repulsive if method == "fft" else ctx.lib.fitsne_repulsive_exact
    rc = fn(ctx.h, _lib.ptr(y), n, _lib.ptr(forces), C.byref(z), _lib.ptr(k1), _lib.ptr(k2),
            ctx.stream)
    if not (rc == _lib.EZ and not check_z):
        _lib.check(rc, "fitsne_repulsive")
    return forces, float(z.value), k1, k2


def compute_repulsive(Y, min_intervals: int = 20, points_per_interval: int = 3,
                      method: str = "auto", workers: int = 1, *, dtype=None,
                      intervals_per_integer: float = 1.0) -> Repulsion:
    """F_i = (y_i S_unit,i - S_coord,i) / Z (optimizer.py:214-245)."""
    n = _check_embedding(Y)
    method = _resolve_method(method, n)
    y, dev, dt = _embedding(Y, dtype)
    f, z, k1, k2 = _repulsion_device(y, dev, dt, min_intervals, points_per_interval, method,
                                     intervals_per_integer)
    on_dev = A.is_device_input(Y)
    return Repulsion(forces=A.output(f, on_dev), z=z, k1_potential=A.output(k1, on_dev),
                     k2_potentials=A.output(k2, on_dev))


def gradient(P, Y, alpha: float = 1.0, min_intervals: int = 20, points_per_interval: int = 3,
             method: str = "auto", workers: int = 1, *, dtype=None,
             intervals_per_integer: float = 1.0, out=None):
    """4 (alpha F_attr - F_rep) (optimizer.py:248-262).

    ``out`` (extension): a caller-owned tensor of Y's shape -- e.g. pinned host
    memory -- that receives the gradient in place (and is returned).
    """
    if alpha < 1.0:
        raise ValueError("exaggeration alpha must be >= 1")
    shp = _shape(Y)
    if len(shp) != 2 or shp[0] != n_points(P):
        raise ValueError("embedding shape does not match the affinities")
    n = _check_embedding(Y)
    method = _resolve_method(method, n)
    if method == "fft" and not A.is_device_input(Y) and (out is None or not out.is_cuda):
        return _gradient_host(P, Y, alpha, min_intervals, points_per_interval, dtype,
                              intervals_per_integer, out)
    y, dev, dt = _embedding(Y, dtype)
    ctx, _ = _ctx_with_P(P, dev, y.shape[1], dt, points_per_interval, min_intervals,
                         intervals_per_integer)
    if out is not None and out.is_cuda and out.dtype == dt and out.is_contiguous():
        g = out
    elif A.is_device_input(Y):
        g = torch.empty_like(y)
    else:
        g = _scratch(ctx, "grad", y)   # result leaves the device: reuse the scratch
    if method == "fft":
        _lib.check(ctx.lib.fitsne_gradient(ctx.h, _lib.ptr(y), float(alpha), _lib.ptr(g), None,
                                           ctx.stream), "fitsne_gradient")
    else:
        f, _, _, _ = _repulsion_device(y, dev, dt, min_intervals, points_per_interval, "exact")
        _lib.check(ctx.lib.fitsne_gradient_rows(ctx.h, _lib.ptr(y), _lib.ptr(f), float(alpha),
                                                _lib.ptr(g), ctx.stream), "fitsne_gradient_rows")
    if g is out:
        return out
    return A.output(g, A.is_device_input(Y) and out is None, like=Y, out=out)


def _gradient_host(P, Y, alpha, min_intervals, points_per_interval, dtype, intervals_per_integer,
                   out):
    """Host arrays in and out (the reference's numpy convention): one
    fitsne_gradient_host call copies Y in, computes, and copies the gradient
    out piece by piece while the SpMV still runs."""
    dev = A.device_of(Y)
    dt = A.compute_dtype(Y, dtype)
    yh = A.host_input(Y, dt)
    ctx, _ = _ctx_with_P(P, dev, yh.shape[1], dt, points_per_interval, min_intervals,
                         intervals_per_integer)
    gh = A.host_output(yh.shape, dt, out)
    _lib.check(ctx.lib.fitsne_gradient_host(ctx.h, _lib.ptr(yh), float(alpha), _lib.ptr(gh),
                                            ctx.stream), "fitsne_gradient_host")
    if out is not None:
        if gh is not out:
            out.copy_(gh)
        return out
    if isinstance(Y, torch.Tensor):
        return gh.clone()
    return gh.numpy().astype(np.float64)


def _scratch(ctx, name, like):
    """Per-context device scratch reused across calls (host-bound results only)."""
    store = ctx.__dict__.setdefault("_scratch", {})
    t = store.get(name)
    if t is None or t.shape != like.shape or t.dtype != like.dtype or t.device != like.device:
        t = torch.empty_like(like)
        store[name] = t
    return t


def _kl_device(ctx, y, z):
    out = C.c_double()
    _lib.check(ctx.lib.fitsne_kl(ctx.h, _lib.ptr(y), float(z), C.byref(out), ctx.stream), "fitsne_kl")
    return float(out.value)


def kl_divergence(P, Y, method: str = "auto", *, dtype=None) -> float:
    """KL(P || Q) over the stored pairs (optimizer.py:278-296)."""
    shp = _shape(Y)
    if shp[0] < 2:
        raise ValueError("KL needs at least two points")
    n = shp[0]
    if method == "auto":
        method = "exact" if n <= EXACT_KL_MAX_N else "fft"
    y, dev, dt = _embedding(Y, dtype)
    if y.dim() == 1:
        y = y.reshape(-1, 1)
    # Z: exact O(N^2) sum, or the grid's unit-charge Cauchy sum with the
    # reference's evaluate_nbody defaults (min_intervals 20, p 3)
    # (the reference checks neither Z's sign nor its finiteness here: a
    # non-finite exact Z gives a NaN KL, optimizer.py:289-296)
    _, z, _, _ = _repulsion_device(y, dev, dt, 20, 3, "exact" if method == "exact" else "fft",
                                   check_z=False)
    ctx, _ = _ctx_with_P(P, dev, y.shape[1], dt)
    return _kl_device(ctx, y, z)


def step(state: OptimizerState, Y, grad, momentum: float | None = None, *, dtype=None):
    """Momentum + gains update (optimizer.py:299-323); returns the moved embedding."""
    gs, ys, vs = _shape(grad), _shape(Y), _shape(state.velocity)
    if gs != ys or gs != vs:
        raise ValueError("gradient, embedding and state shapes must agree")
    dev = A.device_of(Y, grad, state.velocity)
    dt = A.compute_dtype(Y, dtype)
    if momentum is None:
        momentum = 0.5 if state.iteration < 250 else 0.8
    y = A.to_device(Y, dt, dev).clone()
    g = A.to_device(grad, dt, dev)
    v_dev = isinstance(state.velocity, torch.Tensor) and state.velocity.is_cuda
    vel = A.to_device(state.velocity, dt, dev).clone()
    gains = A.to_device(state.gains, dt, dev).clone()
    n = y.shape[0] if y.dim() > 0 else 0
    ctx = _lib.context(dev, y.shape[1] if y.dim() == 2 else 1, dt)
    rc = ctx.lib.fitsne_step(ctx.h, _lib.ptr(y), _lib.ptr(g), _lib.ptr(vel), _lib.ptr(gains), n,
                             float(momentum), float(state.learning_rate), ctx.stream)
    if rc == _lib.ENONFINITE:
        raise FloatingPointError(f"non-finite gradient at iteration {state.iteration}")
    _lib.check(rc, "fitsne_step")
    state.velocity = A.output(vel, v_dev)
    state.gains = A.output(gains, v_dev)
    state.iteration += 1
    return A.output(y, A.is_device_input(Y))


def _validate_affinities(P) -> None:
    if abs(ordered_total(P) - 1.0) > 1e-9:
        raise ValueError("affinity mass over ordered pairs must be 1 (within 1e-9)")


def run_tsne(data=None, affinities=None, config: TsneConfig | None = None, callback=None,
             ) -> TsneResult:
    """Seeded init + gradient descent (optimizer.py:331-415) on the device.

    Without a callback each iteration is one fused device step (grid, spread,
    FFT, Z, gather, SpMV, KL, update); the KL log stays on the device until the
    end.  With a callback the per-iteration forces are materialised and copied
    out, as the reference's callback contract requires.
    """
    cfg = config or TsneConfig()
    cfg.validate()
    if (data is None) == (affinities is None):
        raise ValueError("provide exactly one of data or affinities")
    seeds = np.random.SeedSequence(cfg.seed).spawn(3)
    if data is not None:
        # (PCA ->) affinities on the device (optimizer.py:351-372; affinity_build.py)
        from .affinity_build import AffinityConfig, affinities_from_data, pca_reduce
        x = np.asarray(data, dtype=float)
        if x.ndim != 2:
            raise ValueError("data must be (N, d)")
        dev0 = cfg.device if cfg.device is not None else A.device_of()
        if cfg.pca_dims is not None and x.shape[1] > cfg.pca_dims:
            x = pca_reduce(x, cfg.pca_dims, seed=int(seeds[2].generate_state(1)[0]), device=dev0)
        aff_cfg = AffinityConfig(perplexity=cfg.perplexity, n_neighbors=cfg.n_neighbors,
                                 method=cfg.knn_method, n_trees=cfg.n_trees,
                                 subsample=cfg.subsample,
                                 seed=int(seeds[0].generate_state(1)[0]))
        P, _ = affinities_from_data(x, aff_cfg, device=dev0)
    else:
        P = affinities
        _validate_affinities(P)
    n = n_points(P)
    rng = np.random.default_rng(seeds[1])
    y0 = rng.normal(0.0, 1e-4, size=(n, cfg.dims))          # optimizer.py:378-379
    dt = A.resolve(cfg.dtype) or torch.float64
    dev = cfg.device if cfg.device is not None else A.device_of()
    method = _resolve_method(cfg.repulsion_method, n)
    if callback is not None or method == "exact":
        return _run_unfused(P, y0, cfg, dev, dt, method, callback)
    return _run_fused(P, y0, cfg, dev, dt)


def _part1by1(x: torch.Tensor) -> torch.Tensor:
    x = x & 0xFFFF
    x = (x | (x << 8)) & 0x00FF00FF
    x = (x | (x << 4)) & 0x0F0F0F0F
    x = (x | (x << 2)) & 0x33333333
    return (x | (x << 1)) & 0x55555555


def _locality_order(y: torch.Tensor):
    """Z-order (Morton) permutation of the embedding: perm[new] = old, inv[old] = new."""
    lo = y.min(0).values
    span = (y.max(0).values - lo).clamp_min(1e-30)
    q = ((y - lo) / span * 65535.0).long().clamp_(0, 65535)
    key = q[:, 0] if y.shape[1] == 1 else (_part1by1(q[:, 0]) | (_part1by1(q[:, 1]) << 1))
    perm = torch.argsort(key)
    inv = torch.empty_like(perm)
    inv[perm] = torch.arange(perm.numel(), device=perm.device)
    return perm, inv


def _run_fused(P, y0, cfg, dev, dt) -> TsneResult:
    """Fused device iterations.  For large N the points are relabelled in the
    Z-order of the current embedding at cfg.reorder_iters: P's neighbours are
    then close in index, so the SpMV's neighbour gathers share cache lines.
    The relabelling is a symmetric permutation of P, Y and the optimiser
    state (results are unchanged up to summation order); the embedding is
    returned in the caller's order."""
    from .affinities import permute_csr
    n, s = y0.shape
    ctx, csr = _ctx_with_P(P, dev, s, dt, cfg.points_per_interval, cfg.min_intervals,
                           cfg.intervals_per_integer)
    reorder_at = set(cfg.reorder_iters or ()) if n >= cfg.reorder_min_n else set()
    order = None  # order[current label] = caller's index
    with torch.cuda.device(dev):
        ya = torch.from_numpy(y0).to(device=dev, dtype=dt)
        yb = torch.empty_like(ya)
        vel = torch.zeros_like(ya)
        gains = torch.ones_like(ya)
        kl = torch.zeros(cfg.n_iter, dtype=torch.float64, device=dev)
        status = torch.zeros(cfg.n_iter, dtype=torch.int32, device=dev)
        st = ctx.stream
        for it in range(cfg.n_iter):
            if it in reorder_at:
                perm, inv = _locality_order(ya)
                ya = ya[perm].contiguous()
                yb = torch.empty_like(ya)
                vel = vel[perm].contiguous()
                gains = gains[perm].contiguous()
                csr = permute_csr(csr, perm, inv)
                ctx.set_affinities(csr)
                order = perm if order is None else order[perm]
            alpha = cfg.exaggeration.alpha(it, cfg.n_iter)
            mom = cfg.momentum_early if it < cfg.momentum_switch_iter else cfg.momentum_late
            rc = ctx.lib.fitsne_iterate(
                ctx.h, _lib.ptr(ya), _lib.ptr(yb), _lib.ptr(vel), _lib.ptr(gains), float(alpha),
                float(mom), float(cfg.learning_rate), C.c_void_p(kl.data_ptr() + 8 * it),
                C.c_void_p(status.data_ptr() + 4 * it), st)
            if rc in (_lib.ENONFINITE, _lib.EPOINTS):
                _raise_status(status, it)
            _lib.check(rc, "fitsne_iterate")
            ya, yb = yb, ya
        torch.cuda.current_stream(dev).synchronize()
        _raise_status(status, None)
        if order is not None:
            out = torch.empty_like(ya)
            out[order] = ya
            ya = out
        return TsneResult(embedding=ya.to(torch.float64).cpu().numpy(),
                          kl_log=kl.cpu().numpy(), affinities=P)


def _raise_status(status, it_fail):
    st = status.cpu().numpy()
    bad = np.nonzero(st)[0]
    if bad.size:
        k = int(bad[0])
        if st[k] & 1:
            raise FloatingPointError(f"non-finite gradient at iteration {k}")
        raise FloatingPointError(f"embedding diverged at iteration {k}")
    if it_fail is not None:
        raise FloatingPointError(f"embedding diverged at iteration {it_fail - 1}")


def _run_unfused(P, y0, cfg, dev, dt, method, callback) -> TsneResult:
    n, s = y0.shape
    y = torch.from_numpy(y0).to(device=dev, dtype=dt)
    state = OptimizerState(0, torch.zeros_like(y), torch.ones_like(y), cfg.learning_rate)
    kl_log = np.empty(cfg.n_iter)
    ctx, _ = _ctx_with_P(P, dev, s, dt, cfg.points_per_interval, cfg.min_intervals,
                         cfg.intervals_per_integer)
    for it in range(cfg.n_iter):
        alpha = cfg.exaggeration.alpha(it, cfg.n_iter)
        attr = compute_attractive(P, y)
        f, z, k1, k2 = _repulsion_device(y, dev, dt, cfg.min_intervals, cfg.points_per_interval,
                                         method, cfg.intervals_per_integer)
        rep = Repulsion(forces=f, z=z, k1_potential=k1, k2_potentials=k2)
        ctx.set_affinities(device_csr(P, dt, dev))
        grad = torch.empty_like(y)
        _lib.check(ctx.lib.fitsne_gradient_rows(ctx.h, _lib.ptr(y), _lib.ptr(f), float(alpha),
                                                _lib.ptr(grad), ctx.stream), "fitsne_gradient_rows")
        kl_log[it] = _kl_device(ctx, y, z)
        if callback is not None:
            callback(it, y.to(torch.float64).cpu().numpy(), {
                "attractive": attr.to(torch.float64).cpu().numpy(),
                "repulsion": Repulsion(*(v.to(torch.float64).cpu().numpy()
                                         if isinstance(v, torch.Tensor) else v
                                         for v in (rep.forces, rep.z, rep.k1_potential,
                                                   rep.k2_potentials))),
                "alpha": alpha,
                "kl": kl_log[it],
            })
        mom = cfg.momentum_early if it < cfg.momentum_switch_iter else cfg.momentum_late
        y = step(state, y, grad, mom)
        if not bool(torch.isfinite(y).all()):
            raise FloatingPointError(f"embedding diverged at iteration {it}")
    return TsneResult(embedding=y.to(torch.float64).cpu().numpy(), kl_log=kl_log, affinities=P)
