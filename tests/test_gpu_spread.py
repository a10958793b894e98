"""Box-sorted spread (radix sort + segmented warp reduction) vs the direct
per-point atomic scatter and vs the oracle's np.bincount spread
(nbody.py:233-237), including the all-points-in-four-boxes case."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

from conftest import rel_inf
from oracle import fitsne_oracle as O

pytestmark = pytest.mark.gpu


def _spread(y, dtype, sorted_on, dims, mode=None, grid_f64=0):
    """Spread through fitsne_spread_tsne into a caller's accumulator.  The
    fp32 spread kernels are tested with the fp32 grid pipeline (grid_f64=0);
    grid_f64=2 routes an fp32 context through its fp64 twin (double
    accumulator, fitsne_grid_accum_dtype)."""
    from paper_1712_09005_b200 import _lib
    dt = torch.float32 if dtype == "float32" else torch.float64
    yt = torch.from_numpy(np.ascontiguousarray(y)).to(device=0, dtype=dt)
    ctx = _lib.Context(0, dims, dt, 3, 50)
    if mode is None:
        mode = 2 if sorted_on else 0
    _lib.check(ctx.lib.fitsne_set_option(ctx.h, 1, mode))
    _lib.check(ctx.lib.fitsne_set_option(ctx.h, _lib.OPT_GRID_F64, grid_f64))
    g = _lib.Grid()
    _lib.check(ctx.lib.fitsne_make_grid(ctx.h, _lib.ptr(yt), yt.shape[0], C.byref(g), ctx.stream))
    adt = torch.float64 if ctx.lib.fitsne_grid_accum_dtype(ctx.h) == _lib.F64 else torch.float32
    wide = adt != dt
    acc = torch.zeros(int(ctx.lib.fitsne_grid_accum_len(ctx.h)), dtype=adt, device=0)
    _lib.check(ctx.lib.fitsne_spread_tsne(ctx.h, _lib.ptr(yt), yt.shape[0], _lib.ptr(acc), ctx.stream))
    torch.cuda.synchronize()
    a = acc.reshape(-1, 4).cpu().numpy().astype(np.float64)
    # the y channels are spread centred on the grid (y - c, c = (lo + hi) / 2
    # in the working precision): add c * (unit channel) back for the
    # reference's bincount layout
    for d in range(dims):
        c = 0.5 * (g.lo[d] + g.hi[d])
        c = float(np.float32(c)) if dtype == "float32" and not wide else c
        a[:, 1 + d] += c * a[:, 0]
    return a, g


def _oracle(y, g, dims):
    grid = O.Grid(tuple(g.lo[d] for d in range(dims)), tuple(g.hi[d] for d in range(dims)),
                  g.n_intervals, 3)
    idx, w = O.interp(grid, y)
    cols = [O.spread(idx, w, np.ones(len(y)), grid)] + [O.spread(idx, w, y[:, d], grid)
                                                        for d in range(dims)]
    return np.stack(cols, 1)


CASES = {
    "blobs": lambda rng, d: np.concatenate([c + 1.5 * rng.standard_normal((5000, d))
                                            for c in rng.uniform(-40, 40, (20, d))]),
    "y0": lambda rng, d: rng.normal(0, 1e-4, (100_000, d)),
    "uniform": lambda rng, d: rng.uniform(-30, 30, (50_000, d)),
}


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("dims", [1, 2])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_sorted_spread_matches_bincount(cuda, case, dims, dtype):
    rng = np.random.default_rng(7)
    y = CASES[case](rng, dims)
    if dtype == "float32":
        y = y.astype(np.float32).astype(np.float64)
    a, g = _spread(y, dtype, True, dims)
    b, _ = _spread(y, dtype, False, dims)
    ref = _oracle(y, g, dims)
    tol = 1e-12 if dtype == "float64" else 1e-4
    for c in range(dims + 1):
        assert rel_inf(a[:, c], ref[:, c]) <= tol, c
        assert rel_inf(b[:, c], ref[:, c]) <= tol, c


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_sorted_spread_large_grid_radix_path(cuda, dtype):
    """> 48k boxes: the LSD-radix variant of the sorted spread."""
    rng = np.random.default_rng(9)
    y = rng.uniform(-200, 200, (60_000, 2))
    if dtype == "float32":
        y = y.astype(np.float32).astype(np.float64)
    a, g = _spread(y, dtype, True, 2)
    assert g.n_intervals ** 2 > 48 * 1024
    ref = _oracle(y, g, 2)
    tol = 1e-12 if dtype == "float64" else 5e-4
    for c in range(3):
        assert rel_inf(a[:, c], ref[:, c]) <= tol, c


def test_wide_fp32_spread_into_double_accumulator(cuda):
    """An fp32 context with the fp64 grid pipeline (FITSNE_OPT_GRID_F64 = 2)
    reports a double accumulator and fills it with the fp64 spread."""
    rng = np.random.default_rng(10)
    y = rng.uniform(-200, 200, (60_000, 2)).astype(np.float32).astype(np.float64)
    a, g = _spread(y, "float32", True, 2, mode=1, grid_f64=2)
    ref = _oracle(y, g, 2)
    for c in range(3):
        assert rel_inf(a[:, c], ref[:, c]) <= 1e-12, c


BAND_CASES = dict(CASES)
BAND_CASES.update({
    # sparse rows: sorted pieces span many box rows (direct-scatter fallback blocks)
    "uniform_sparse": lambda rng, d: rng.uniform(-60, 60, (5_000, d)),
    # power-law blob sizes, one blob holding most points (crowded boxes)
    "crowded": lambda rng, d: np.concatenate([c + s * rng.standard_normal((m, d)) for c, s, m in zip(
        rng.uniform(-80, 80, (12, d)), rng.uniform(0.05, 3, 12),
        [300_000, 1000, 5, 1, 7000, 2, 50_000, 3, 11, 900, 1, 4000])]),
    "odd_count": lambda rng, d: rng.normal(0, 5, (2049 * 3 + 17, d)),
})


@pytest.mark.parametrize("case", list(BAND_CASES))
def test_band_spread_matches_bincount(cuda, case):
    """Band spread (mode 3; the fp32 2-D p = 3 default): box-row counting sort
    + in-block box sort + per-thread box runs, vs the oracle's bincount and the
    direct scatter."""
    rng = np.random.default_rng(17)
    y = BAND_CASES[case](rng, 2).astype(np.float32).astype(np.float64)
    a, g = _spread(y, "float32", False, 2, mode=3)
    b, _ = _spread(y, "float32", False, 2, mode=0)
    ref = _oracle(y, g, 2)
    for c in range(3):
        assert rel_inf(a[:, c], ref[:, c]) <= 1e-4, c
        assert rel_inf(b[:, c], ref[:, c]) <= 1e-4, c


def test_band_spread_is_the_fp32_default(cuda):
    rng = np.random.default_rng(3)
    y = BAND_CASES["blobs"](rng, 2).astype(np.float32).astype(np.float64)
    a, g = _spread(y, "float32", False, 2, mode=1)
    ref = _oracle(y, g, 2)
    for c in range(3):
        assert rel_inf(a[:, c], ref[:, c]) <= 1e-4, c


@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("cols", [1, 2, 4])
def test_fft_columns_per_block(cuda, dtype, cols):
    """k_cols with 1, 2 or 4 adjacent columns per block (FITSNE_OPT_FFT_COLS)
    gives the reference's repulsion (forces and Z) on grids of odd and even
    FFT length."""
    from paper_1712_09005_b200 import _lib
    dt = torch.float32 if dtype == "float32" else torch.float64
    rng = np.random.default_rng(cols)
    for span in (37.0, 91.5):
        y = rng.uniform(-span / 2, span / 2, (6000, 2))
        y = y.astype(np.float32).astype(np.float64) if dtype == "float32" else y
        yt = torch.from_numpy(y).to(device=0, dtype=dt)
        ctx = _lib.Context(0, 2, dt, 3, 20)
        _lib.check(ctx.lib.fitsne_set_option(ctx.h, 11, cols))
        f = torch.empty_like(yt)
        z = C.c_double()
        _lib.check(ctx.lib.fitsne_repulsive(ctx.h, _lib.ptr(yt), yt.shape[0], _lib.ptr(f), C.byref(z),
                                            None, None, ctx.stream))
        torch.cuda.synchronize()
        fo, zo, _, _ = O.repulsion(y, 20, 3, "fft")
        tol = 1e-10 if dtype == "float64" else 1e-3
        got = f.cpu().numpy().astype(np.float64)
        assert np.linalg.norm(got - fo) <= tol * np.linalg.norm(fo)
        assert abs(z.value - zo) <= 1e-6 * zo
