"""Sharded gradient (parallel.py) with world_size 2 over gloo on CPU.

The CUDA stages are replaced by an oracle-backed stage implementation, so the
test exercises the partitioning, the bbox MIN/MAX all-reduce, the Y
all-gather and the grid SUM all-reduce exactly as the GPU path runs them, and
checks the concatenated rank gradients against the single-process oracle
gradient (optimizer.py:248-262)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fitsne_oracle as O


class OracleStages:
    """numpy restatement of the library stages on one shard (test only)."""

    def __init__(self, rows, cols, vals, n, dims, lo_row, hi_row, min_int=50, p=3):
        self.rows, self.cols, self.vals, self.n = rows, cols, vals, n
        self.dims, self.lo_row, self.hi_row = dims, lo_row, hi_row
        self.min_int, self.p = min_int, p
        self.grid = None

    def to_comm(self, x):
        return torch.as_tensor(np.asarray(x, dtype=np.float64))

    def bbox(self, y_local):
        y = y_local.numpy()
        return np.concatenate([y.min(0), y.max(0)])

    def set_grid(self, bbox):
        s = self.dims
        # the grid of the union of all points: the same formulas on the global box
        corners = np.stack([bbox[:s], bbox[s:]])
        self.grid = O.grid_for(corners, self.min_int, self.p)

    def spread(self, y_local):
        y = y_local.numpy()
        idx, w = O.interp(self.grid, y)
        chans = [np.ones(len(y))] + [y[:, d] for d in range(self.dims)]
        cols = [O.spread(idx, w, q, self.grid) for q in chans]
        cols += [np.zeros(self.grid.n ** self.dims)] * (4 - len(cols))
        acc = np.stack(cols, 1)
        return torch.as_tensor(acc.reshape(-1))

    def fft(self, acc):
        a = acc.numpy().reshape(-1, 4)
        s1, L = O.spectrum(O.CAUCHY, self.grid)
        s2, _ = O.spectrum(O.CAUCHY_SQUARED, self.grid)
        self.pot = np.stack([O.toeplitz_apply(a[:, c], s2, L, self.grid) for c in range(1 + self.dims)], 1)
        k1 = O.toeplitz_apply(a[:, 0], s1, L, self.grid)
        self.z = float(a[:, 0] @ k1) - self.n
        return self.z

    def gather(self, y_local):
        y = y_local.numpy()
        idx, w = O.interp(self.grid, y)
        phi = np.stack([O.gather(idx, w, self.pot[:, c]) for c in range(1 + self.dims)], 1)
        h4 = phi[:, 0] - 1.0
        hc = phi[:, 1:] - y
        return torch.as_tensor((y * h4[:, None] - hc) / self.z)

    def attract_rows(self, y_full, f_local, alpha):
        att = O.attraction(self.rows, self.cols, self.vals, y_full.numpy())[self.lo_row:self.hi_row]
        return torch.as_tensor(4.0 * (alpha * att - f_local.numpy()))


def _problem(n=1200, dims=2, seed=0):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-15, 15, (6, dims))
    y = c[rng.integers(0, 6, n)] + rng.standard_normal((n, dims))
    r = np.repeat(np.arange(n), 8)
    cc = rng.integers(0, n - 1, n * 8)
    cc = cc + (cc >= r)
    key = np.unique(np.minimum(r, cc) * n + np.maximum(r, cc))
    rows, cols = key // n, key % n
    vals = rng.exponential(1.0, rows.size)
    vals /= 2 * vals.sum()
    return y, rows, cols, vals


def _worker(rank, world, port, dims, q, n_points=1200):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1712_09005_b200.parallel import ShardedGradient, shard_range
        y, rows, cols, vals = _problem(n=n_points, dims=dims)
        n = len(y)
        lo, hi = shard_range(n, rank, world)

        class PHolder:
            pass
        P = PHolder()
        P.n, P.rows, P.cols, P.values = n, rows, cols, vals
        st = OracleStages(rows, cols, vals, n, dims, lo, hi)
        sg = ShardedGradient(P, n_dims=dims, stages=st)
        g_local = sg.gradient(torch.as_tensor(y[lo:hi]), alpha=12.0)
        parts = [torch.zeros((shard_range(n, r, world)[1] - shard_range(n, r, world)[0], dims),
                             dtype=torch.float64) for r in range(world)]
        m = max(p.shape[0] for p in parts)
        pad = torch.zeros((m, dims), dtype=torch.float64)
        pad[: g_local.shape[0]] = g_local
        bufs = [torch.zeros_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad)
        if rank == 0:
            full = torch.cat([b[: p.shape[0]] for b, p in zip(bufs, parts)]).numpy()
            q.put(full)
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("dims,world,n_points", [(1, 2, 1200), (2, 2, 1200), (2, 3, 1201)])
def test_sharded_gradient_world2_matches_single_process(dims, world, n_points):
    """world 2 (equal shards: all_gather_into_tensor) and world 3 with a
    ragged last shard (padded all-gather)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, q, n_points))
             for r in range(world)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    y, rows, cols, vals = _problem(n=n_points, dims=dims)
    ref = O.grad(rows, cols, vals, y, 12.0, 50, 3, "fft")
    # the shard's grid is the global one, so the only differences are summation order
    assert np.linalg.norm(full - ref) / np.linalg.norm(ref) <= 1e-10


def test_shard_ranges_cover_all_points():
    from paper_1712_09005_b200.parallel import shard_range
    for n in (1, 7, 1000, 1_300_000):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
