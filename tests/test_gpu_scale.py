"""Oracle parity at the BASELINE configurations the bench measures.

The production path -- tiled attractive SpMV (3072 x 8192 tiles on the
overlapped persistent grid), band spread, hand-written FFT stage, two-stream
schedule, host-buffer entry fitsne_gradient_host -- is checked against the
oracle (the reference's algorithm, oracle/fitsne_oracle.py) on the SAME
seeded inputs the bench times:

  C3  N=1.3M 2-D (bench.py's workload): gradient rel-L2 <= 1e-3 (fp32) and
      <= 1e-5 (fp64), node indices of all 1.3M points bit-exact;
  C5  N=1M 1-D, 30-cluster kNN P: gradient, and the first 20 iterations of the
      fused run_tsne against the oracle's descent (KL log and embedding);
  C4  N=10M 2-D, random kNN P (900M stored entries): the device gradient on a
      20k-row sample against the oracle's repulsion (all 10M points) and
      exact per-row attraction.

North-star tolerances: rel-L2 <= 1e-5 in fp64 mode and <= 1e-3 in fp32 mode,
box / node indices bit-exact (optimizer.py:248-262, nbody.py:201-230).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import fitsne_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

WORKERS = os.cpu_count() or 1


def _tiled_in_use(dt, y):
    from paper_1712_09005_b200 import _lib
    ctx = _lib.context(0, 2, dt, 3, 50, 1.0)
    st = (C.c_int64 * 8)()
    _lib.check(ctx.lib.fitsne_tiled_stats(ctx.h, _lib.ptr(y), st, ctx.stream), "tiled_stats")
    return int(st[0]), int(st[1])


# ----------------------------------------------------------------------------- C3
@pytest.fixture(scope="module")
def c3(cuda):
    from tools import synth
    P, Y = synth.c3(device="cuda", n=1_300_000, seed=3)   # bench.py's inputs
    y32 = Y.astype(np.float32)
    ref = O.grad(P.rows, P.cols, P.values, y32.astype(np.float64), 1.0, 50, 3, "fft", WORKERS)
    return P, y32, ref


def test_c3_production_gradient_fp32(c3):
    """Both public entry points at C3, fp32: the host-buffer call (numpy in,
    numpy out: fitsne_gradient_host) and the device call (fitsne_gradient) --
    on the tiled SpMV + band spread + overlapped schedule the bench times."""
    from paper_1712_09005_b200 import optimizer
    P, y32, ref = c3
    g_host = optimizer.gradient(P, y32, 1.0, 50, 3, "fft")
    yd = torch.from_numpy(y32).cuda()
    g_dev = optimizer.gradient(P, yd, 1.0, 50, 3, "fft").double().cpu().numpy()
    used, ntiles = _tiled_in_use(torch.float32, yd)
    assert used == 1 and ntiles > 10_000          # the production SpMV ran
    e_host, e_dev = rel_l2(g_host, ref), rel_l2(g_dev, ref)
    print(f"C3 fp32 gradient rel-L2: host {e_host:.2e}, device {e_dev:.2e}")
    assert e_host <= 1e-3 and e_dev <= 1e-3


def test_c3_attraction_and_repulsion_separately(c3):
    from paper_1712_09005_b200 import optimizer
    P, y32, _ = c3
    yd = torch.from_numpy(y32).cuda()
    y64 = y32.astype(np.float64)
    fa = optimizer.compute_attractive(P, yd).double().cpu().numpy()
    assert rel_l2(fa, O.attraction(P.rows, P.cols, P.values, y64)) <= 1e-5
    rep = optimizer.compute_repulsive(yd, 50, 3, "fft")
    f_o, z_o, _, _ = O.repulsion(y64, 50, 3, "fft", WORKERS)
    assert abs(rep.z - z_o) / z_o <= 1e-5
    assert rel_l2(rep.forces.double().cpu().numpy(), f_o) <= 1e-3


def test_c3_gradient_fp64(c3):
    from paper_1712_09005_b200 import optimizer
    P, y32, ref = c3
    g = optimizer.gradient(P, y32.astype(np.float64), 1.0, 50, 3, "fft", dtype="float64")
    e = rel_l2(g, ref)
    print(f"C3 fp64 gradient rel-L2 {e:.2e}")
    assert e <= 1e-5


def test_c3_shuffled_relabelled(c3):
    """C3 with its points in random order (real data have no cluster order):
    the library relabels P on the device (Cuthill-McKee), the tiled SpMV runs
    on the relabelled points, and the gradient in the caller's order matches
    the oracle's; the relabelling recovers (at least) the generator order's
    locality."""
    from tools import synth
    from paper_1712_09005_b200 import _lib, optimizer
    P, y32, _ = c3
    Ps, ys = synth.shuffle(P, y32, seed=1003)
    yd = torch.from_numpy(ys).cuda()
    g = optimizer.gradient(Ps, yd, 1.0, 50, 3, "fft").double().cpu().numpy()
    ctx = _lib.context(0, 2, torch.float32, 3, 50, 1.0)
    st = (C.c_int64 * 8)()
    _lib.check(ctx.lib.fitsne_tiled_stats(ctx.h, _lib.ptr(yd), st, ctx.stream), "tiled_stats")
    print(f"C3 shuffled: segments {st[7]} -> {st[4]} (relabelled {st[6]})")
    assert st[0] == 1 and st[6] == 1
    ref = O.grad(Ps.rows, Ps.cols, Ps.values, ys.astype(np.float64), 1.0, 50, 3, "fft", WORKERS)
    e = rel_l2(g, ref)
    print(f"C3 shuffled fp32 gradient rel-L2 {e:.2e}")
    assert e <= 1e-3


def test_c3_node_indices_bit_exact(c3):
    """Node indices of all 1.3M points on the C3 grid (fp32 mode uses the
    production cell function, box_weights3_f32) equal the oracle's."""
    from paper_1712_09005_b200 import nbody
    _, y32, _ = c3
    yd = torch.from_numpy(y32).cuda()
    g = nbody.make_grid(yd, 50, 3)
    og = O.grid_for(y32.astype(np.float64), 50, 3)
    assert (g.lo, g.hi, g.n_intervals) == (og.lo, og.hi, og.n_int)
    idx, _ = nbody.point_interp(yd, g)
    oidx, _ = O.interp(og, y32.astype(np.float64))
    np.testing.assert_array_equal(idx.cpu().numpy(), oidx)


# ----------------------------------------------------------------------------- C5
@pytest.fixture(scope="module")
def c5(cuda):
    from tools import synth
    X, _ = synth.mixture(1_000_000, 50, 30, seed=5, device="cuda")
    r, c, v = synth.affinities(X, 90, 30.0)
    y = synth.pca2(X, 150.0, dims=1).cpu().numpy()       # a 1-D embedding of span ~300
    del X
    P = synth.Upper(1_000_000, r.cpu().numpy(), c.cpu().numpy(), v.cpu().numpy())
    return P, y.astype(np.float32)


def test_c5_gradient_1d(c5):
    from paper_1712_09005_b200 import optimizer
    P, y32 = c5
    y64 = y32.astype(np.float64)
    ref = O.grad(P.rows, P.cols, P.values, y64, 1.0, 50, 3, "fft", WORKERS)
    g32 = optimizer.gradient(P, y32, 1.0, 50, 3, "fft")
    g64 = optimizer.gradient(P, y64, 1.0, 50, 3, "fft", dtype="float64")
    e32, e64 = rel_l2(g32, ref), rel_l2(g64, ref)
    print(f"C5 1-D gradient rel-L2: fp32 {e32:.2e}, fp64 {e64:.2e}")
    assert e32 <= 1e-3 and e64 <= 1e-5


def test_c5_first_20_iterations_match_oracle(c5):
    """The fused device run_tsne (1-D, p = 3, min 50 intervals) against the
    oracle's descent loop from the same seeded Y0 (optimizer.py:377-415)."""
    from paper_1712_09005_b200 import optimizer as opt
    P, _ = c5
    n_iter = 20
    cfg = opt.TsneConfig(dims=1, n_iter=n_iter, learning_rate=200.0, min_intervals=50,
                         points_per_interval=3, exaggeration=opt.ExaggerationSchedule(12.0, n_iter),
                         seed=0, pca_dims=None, repulsion_method="fft", dtype="float32")
    res = opt.run_tsne(affinities=P, config=cfg)
    y_o, kl_o = O.tsne(P.rows, P.cols, P.values, P.n, dims=1, n_iter=n_iter, lr=200.0,
                       early_coeff=12.0, early_until=n_iter, min_intervals=50, p=3,
                       method="fft", seed=0, workers=WORKERS)
    kerr = np.max(np.abs(res.kl_log - kl_o) / np.abs(kl_o))
    yerr = rel_l2(res.embedding, y_o)
    print(f"C5 20 iterations: KL max rel {kerr:.2e}, embedding rel-L2 {yerr:.2e}")
    assert kerr <= 1e-4
    assert yerr <= 1e-3


# ----------------------------------------------------------------------------- C4
class _DeviceUpper:
    """Upper-COO P held on the device (900M ordered entries do not need a
    host round trip); the drop-in API accepts torch tensors for rows/cols/values."""

    def __init__(self, n, rows, cols, values):
        self.n, self.rows, self.cols, self.values = n, rows, cols, values

    @property
    def ordered_total(self):
        return 2.0 * float(self.values.sum().item())


def test_c4_sampled_rows_10m(cuda):
    from tools import synth
    from paper_1712_09005_b200 import optimizer
    n = 10_000_000
    r, c, v = synth.random_knn_graph(n, 45, seed=4, device="cuda")
    P = _DeviceUpper(n, r, c, v)
    y32 = synth.blobs2d(n, 100, 100.0, 2.0, seed=4).astype(np.float32)
    yd = torch.from_numpy(y32).cuda()
    g = optimizer.gradient(P, yd, 1.0, 50, 3, "fft")
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(n, 20_000, replace=False))
    g_s = g[torch.from_numpy(rows).cuda()].double().cpu().numpy()
    # oracle: repulsion over all 10M points, exact attraction of the sampled rows
    y64 = y32.astype(np.float64)
    f_rep = O.repulsion(y64, 50, 3, "fft", WORKERS)[0][rows]
    sel = torch.from_numpy(rows).cuda()
    mr, mc = torch.isin(r, sel), torch.isin(c, sel)
    i = torch.cat([r[mr], c[mc]]).cpu().numpy()
    j = torch.cat([c[mr], r[mc]]).cpu().numpy()
    p = torch.cat([v[mr], v[mc]]).cpu().numpy()
    dy = y64[i] - y64[j]
    w = p / (1.0 + (dy * dy).sum(1))
    pos = np.searchsorted(rows, i)
    attr = np.stack([np.bincount(pos, w * dy[:, d], minlength=rows.size) for d in range(2)], 1)
    ref = 4.0 * (attr - f_rep)
    e = rel_l2(g_s, ref)
    print(f"C4 (N=10M, {2 * r.numel()} entries) sampled-row gradient rel-L2 {e:.2e}")
    assert e <= 1e-3
