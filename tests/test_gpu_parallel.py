"""Sharded-gradient stages on the CUDA library (LibStages) in a single-rank
NCCL group: every collective runs, the math must equal the oracle gradient.
(Multi-rank partitioning is covered with gloo on CPU in test_parallel_gloo.)"""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist

from oracle import fitsne_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group(cuda):
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1)
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-9), (torch.float32, 1e-3)])
def test_lib_stages_single_rank(nccl_group, dtype, tol):
    from paper_1712_09005_b200.affinities import SparseAffinities
    from paper_1712_09005_b200.parallel import ShardedGradient
    rng = np.random.default_rng(3)
    n = 20000
    c = rng.uniform(-30, 30, (10, 2))
    y = c[rng.integers(0, 10, n)] + 2 * rng.standard_normal((n, 2))
    r = np.repeat(np.arange(n), 10)
    cc = rng.integers(0, n - 1, n * 10)
    cc = cc + (cc >= r)
    key = np.unique(np.minimum(r, cc) * n + np.maximum(r, cc))
    P = SparseAffinities(n=n, rows=key // n, cols=key % n, values=np.full(key.size, 0.5 / key.size))
    sg = ShardedGradient(P, n_dims=2, dtype=dtype, device=0, min_intervals=50)
    yt = torch.from_numpy(y).to(device=0, dtype=dtype)
    g = sg.gradient(yt, alpha=12.0).double().cpu().numpy()
    ref = O.grad(P.rows, P.cols, P.values, y.astype(np.float32).astype(np.float64)
                 if dtype == torch.float32 else y, 12.0, 50, 3, "fft")
    assert np.linalg.norm(g - ref) / np.linalg.norm(ref) <= tol


def test_lib_stages_tiled_overlap_matches_fused(nccl_group):
    """The sharded flow with the tiled SpMV on a side stream beside the
    repulsion stages (fitsne_attractive + fitsne_combine_rows) equals the
    single-GPU fused gradient (to fp32 summation-order noise)."""
    from paper_1712_09005_b200 import optimizer
    from paper_1712_09005_b200.affinities import SparseAffinities
    from paper_1712_09005_b200.parallel import ShardedGradient
    rng = np.random.default_rng(8)
    n, k = 40_000, 60
    c = rng.uniform(-40, 40, (12, 2))
    y = (c[rng.integers(0, 12, n)] + 2 * rng.standard_normal((n, 2))).astype(np.float32)
    r = np.repeat(np.arange(n), k)
    cc = rng.integers(0, n - 1, n * k)
    cc = cc + (cc >= r)
    key = np.unique(np.minimum(r, cc) * n + np.maximum(r, cc))
    v = rng.exponential(1.0, key.size)
    P = SparseAffinities(n=n, rows=key // n, cols=key % n, values=v / (2 * v.sum()))
    assert 2 * key.size >= (1 << 22)  # the tiled layout applies
    sg = ShardedGradient(P, n_dims=2, dtype=torch.float32, device=0, min_intervals=50)
    yt = torch.from_numpy(y).cuda()
    g = None
    for _ in range(3):  # repeated calls: accumulators are consumed and cleared
        g = sg.gradient(yt, alpha=4.0).double().cpu().numpy()
    ref = optimizer.gradient(P, yt, 4.0, 50, 3, "fft").double().cpu().numpy()
    # both fp32: same math, different summation order (F_rep gathered inside
    # the fused combine vs. a separate gather)
    assert np.linalg.norm(g - ref) / np.linalg.norm(ref) <= 1e-4


def test_bbox_device_packed_layout(cuda):
    """fitsne_bbox_device: {min, -max, -nonfinite} on the device, matching
    fitsne_bbox; empty input gives the MIN-identity; a NaN sets the flag."""
    import ctypes as C
    from paper_1712_09005_b200 import _lib
    rng = np.random.default_rng(4)
    for dtype in (torch.float32, torch.float64):
        ctx = _lib.Context(0, 2, dtype, 3, 50)
        y = torch.from_numpy(rng.normal(3.0, 7.0, (12345, 2))).to(device=0, dtype=dtype)
        buf = torch.empty(5, dtype=torch.float64, device=0)
        _lib.check(ctx.lib.fitsne_bbox_device(ctx.h, _lib.ptr(y), y.shape[0], _lib.ptr(buf),
                                              ctx.stream), "bbox_device")
        host = (C.c_double * 4)()
        _lib.check(ctx.lib.fitsne_bbox(ctx.h, _lib.ptr(y), y.shape[0], host, ctx.stream), "bbox")
        v = buf.cpu().numpy()
        np.testing.assert_array_equal(v[:2], np.array(host[:2]))
        np.testing.assert_array_equal(-v[2:4], np.array(host[2:4]))
        assert v[4] == 0.0
        yc = y.cpu().double().numpy()
        np.testing.assert_array_equal(v[:2], yc.min(0))
        np.testing.assert_array_equal(-v[2:4], yc.max(0))
        _lib.check(ctx.lib.fitsne_bbox_device(ctx.h, _lib.ptr(y), 0, _lib.ptr(buf), ctx.stream), "e")
        v = buf.cpu().numpy()
        assert np.all(np.isinf(v[:4]) & (v[:4] > 0)) and v[4] == 0.0
        y[17, 1] = float("nan")
        _lib.check(ctx.lib.fitsne_bbox_device(ctx.h, _lib.ptr(y), y.shape[0], _lib.ptr(buf),
                                              ctx.stream), "nan")
        assert buf.cpu().numpy()[4] < 0


def test_lib_stages_wide_fp32_uses_fp64_grid(nccl_group):
    """A wide fp32 embedding (span ~600 > 256): the sharded stages switch the
    grid accumulator to fp64 (fitsne_grid_accum_dtype) and keep the 1e-3 bar."""
    from paper_1712_09005_b200.affinities import SparseAffinities
    from paper_1712_09005_b200.parallel import ShardedGradient
    rng = np.random.default_rng(5)
    n = 20000
    c = rng.uniform(0, 600, (30, 2))
    y = (c[rng.integers(0, 30, n)] + 3 * rng.standard_normal((n, 2))).astype(np.float32)
    r = np.repeat(np.arange(n), 10)
    cc = rng.integers(0, n - 1, n * 10)
    cc = cc + (cc >= r)
    key = np.unique(np.minimum(r, cc) * n + np.maximum(r, cc))
    P = SparseAffinities(n=n, rows=key // n, cols=key % n, values=np.full(key.size, 0.5 / key.size))
    sg = ShardedGradient(P, n_dims=2, dtype=torch.float32, device=0, min_intervals=50)
    yt = torch.from_numpy(y).cuda()
    for _ in range(2):
        g = sg.gradient(yt, alpha=1.0).double().cpu().numpy()
    assert sg.stages._acc.dtype == torch.float64
    ref = O.grad(P.rows, P.cols, P.values, y.astype(np.float64), 1.0, 50, 3, "fft")
    assert np.linalg.norm(g - ref) / np.linalg.norm(ref) <= 1e-3


@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-9), (torch.float32, 1e-4)])
def test_native_nccl_sharded_gradient(nccl_group, dtype, tol):
    """The library's own NCCL path (fitsne_comm_init + fitsne_gradient_sharded,
    a single-rank communicator) equals the fused single-GPU gradient and the
    oracle, with the tiled SpMV on its side stream."""
    from paper_1712_09005_b200 import optimizer
    from paper_1712_09005_b200.affinities import SparseAffinities
    from paper_1712_09005_b200.parallel import NcclGradient
    rng = np.random.default_rng(12)
    n, k = 40_000, 60
    c = rng.uniform(-40, 40, (12, 2))
    y = c[rng.integers(0, 12, n)] + 2 * rng.standard_normal((n, 2))
    r = np.repeat(np.arange(n), k)
    cc = rng.integers(0, n - 1, n * k)
    cc = cc + (cc >= r)
    key = np.unique(np.minimum(r, cc) * n + np.maximum(r, cc))
    v = rng.exponential(1.0, key.size)
    P = SparseAffinities(n=n, rows=key // n, cols=key % n, values=v / (2 * v.sum()))
    sg = NcclGradient(P, n_dims=2, dtype=dtype, device=0, min_intervals=50)
    yt = torch.from_numpy(y).to(device=0, dtype=dtype)
    zs = []
    for _ in range(3):  # repeated: accumulators consumed and cleared
        g = sg.gradient(yt, alpha=4.0, z=zs).double().cpu().numpy()
    ref = optimizer.gradient(P, yt, 4.0, 50, 3, "fft").double().cpu().numpy()
    assert np.linalg.norm(g - ref) / np.linalg.norm(ref) <= tol
    yo = y.astype(np.float32).astype(np.float64) if dtype == torch.float32 else y
    o = O.grad(P.rows, P.cols, P.values, yo, 4.0, 50, 3, "fft")
    assert np.linalg.norm(g - o) / np.linalg.norm(o) <= (1e-3 if dtype == torch.float32 else 1e-9)
    _, z_o, _, _ = O.repulsion(yo, 50, 3, "fft")
    assert abs(zs[-1] - z_o) <= 1e-5 * z_o
    sg.close()
