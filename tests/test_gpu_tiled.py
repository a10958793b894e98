"""Tiled attractive SpMV (csrc/tiled.cu) against the oracle and the CSR kernel.

The tiled layout is forced (FITSNE_OPT_TILED_SPMV = 2) with small tile
shapes so that the small inputs here span many row blocks, column chunks and
CTAs (row blocks split between CTAs, CTAs with no tiles, odd point counts,
partial chunks).  fp32 tolerance: rel-L2 <= 1e-5 on F_attr (the bar for the
gradient is 1e-3); the KL sum to 1e-6.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import fitsne_oracle as O

pytestmark = pytest.mark.gpu

OPT_TILED, OPT_ROWS, OPT_COLS, OPT_CTAS = 5, 6, 7, 8


def _graph(n, k, seed, clustered=True):
    """Symmetric kNN-like P (upper COO) with cluster structure, plus Y."""
    rng = np.random.default_rng(seed)
    if clustered:
        lab = np.sort(rng.integers(0, 7, n))
        rows, cols = [], []
        for i in range(n):
            same = np.flatnonzero(lab == lab[i])
            j = rng.choice(same, size=min(k, same.size), replace=False)
            rows.append(np.full(j.size, i))
            cols.append(j)
        r, c = np.concatenate(rows), np.concatenate(cols)
    else:
        r = np.repeat(np.arange(n), k)
        c = rng.integers(0, n, n * k)
    keep = r != c
    lo, hi = np.minimum(r[keep], c[keep]), np.maximum(r[keep], c[keep])
    key = np.unique(lo.astype(np.int64) * n + hi)
    rr, cc = key // n, key % n
    v = rng.random(rr.size) + 0.05
    v /= 2 * v.sum()
    Y = rng.standard_normal((n, 2)) * 10
    return rr, cc, v, Y


def _csr(n, rr, cc, v, row_begin=0, row_end=None):
    from paper_1712_09005_b200.affinities import csr_from_full
    dev = torch.device("cuda", 0)
    r = torch.from_numpy(np.concatenate([rr, cc])).to(dev)
    c = torch.from_numpy(np.concatenate([cc, rr])).to(dev)
    w = torch.from_numpy(np.concatenate([v, v])).to(dev)
    return csr_from_full(n, r, c, w, torch.float32, row_begin, n if row_end is None else row_end)


def _ctx(tiled, rows=64, cols=128, ctas=0):
    from paper_1712_09005_b200 import _lib
    ctx = _lib.Context(0, 2, torch.float32, 3, 20, 1.0)
    for opt, val in ((OPT_TILED, tiled), (OPT_ROWS, rows), (OPT_COLS, cols), (OPT_CTAS, ctas)):
        _lib.check(ctx.lib.fitsne_set_option(ctx.h, opt, val), "set_option")
    return ctx


def _attr(ctx, csr, y):
    from paper_1712_09005_b200 import _lib
    ctx.set_affinities(csr)
    out = torch.empty((csr.n_rows, 2), dtype=torch.float32, device=y.device)
    _lib.check(ctx.lib.fitsne_attractive(ctx.h, _lib.ptr(y), _lib.ptr(out), ctx.stream), "attractive")
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64)


SHAPES = [(64, 128, 0), (64, 128, 3), (2, 2, 0), (256, 1024, 7), (4096, 6144, 0), (128, 64, 5000)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("n,k,clustered", [(3001, 25, True), (1500, 40, False)])
def test_tiled_attractive_vs_oracle(cuda, shape, n, k, clustered):
    rr, cc, v, Y = _graph(n, k, seed=n + k, clustered=clustered)
    csr = _csr(n, rr, cc, v)
    y = torch.from_numpy(Y.astype(np.float32)).cuda()
    want = O.attraction(rr, cc, v, Y.astype(np.float32).astype(np.float64))
    got = _attr(_ctx(2, *shape), csr, y)
    assert rel_l2(got, want) <= 1e-5
    base = _attr(_ctx(0), csr, y)
    assert rel_l2(got, base) <= 1e-5


def test_tiled_repeat_calls_clear_accumulator(cuda):
    rr, cc, v, Y = _graph(2001, 20, seed=5)
    csr = _csr(2001, rr, cc, v)
    y = torch.from_numpy(Y.astype(np.float32)).cuda()
    ctx = _ctx(2, 64, 256, 4)
    a = _attr(ctx, csr, y)
    b = _attr(ctx, csr, y)
    assert rel_l2(a, b) <= 1e-6  # consume-and-clear: no accumulation across calls


def test_tiled_row_range(cuda):
    """Rows [a, b) of P against the full Y (the sharded multi-GPU layout)."""
    n = 2500
    rr, cc, v, Y = _graph(n, 30, seed=11)
    y = torch.from_numpy(Y.astype(np.float32)).cuda()
    full = O.attraction(rr, cc, v, Y.astype(np.float32).astype(np.float64))
    for a, b in ((0, 700), (700, 1901), (1901, n)):
        csr = _csr(n, rr, cc, v, a, b)
        got = _attr(_ctx(2, 128, 256, 6), csr, y)
        assert rel_l2(got, full[a:b]) <= 1e-5


def test_tiled_kl_and_gradient(cuda):
    from paper_1712_09005_b200 import _lib
    n = 3001
    rr, cc, v, Y = _graph(n, 25, seed=3)
    csr = _csr(n, rr, cc, v)
    y = torch.from_numpy(Y.astype(np.float32)).cuda()
    res = {}
    for mode in (0, 2):
        ctx = _ctx(mode, 128, 512, 5)
        ctx.set_affinities(csr)
        kl = C.c_double()
        _lib.check(ctx.lib.fitsne_kl(ctx.h, _lib.ptr(y), 1.0, C.byref(kl), ctx.stream), "kl")
        g = torch.empty_like(y)
        _lib.check(ctx.lib.fitsne_gradient(ctx.h, _lib.ptr(y), 12.0, _lib.ptr(g), None, ctx.stream),
                   "gradient")
        torch.cuda.synchronize()
        res[mode] = (kl.value, g.cpu().numpy().astype(np.float64))
    assert abs(res[2][0] - res[0][0]) <= 1e-6 * abs(res[0][0])
    assert rel_l2(res[2][1], res[0][1]) <= 1e-5
    Yd = Y.astype(np.float32).astype(np.float64)
    want = O.grad(rr, cc, v, Yd, 12.0, min_intervals=20, p=3)
    assert rel_l2(res[2][1], want) <= 1e-3


@pytest.mark.parametrize("ctas", [3, 7, 40])
def test_schedule_options_agree(cuda, ctas):
    """F_rep gathered beside the SpMV + streaming combine (FITSNE_OPT_SIDE_GATHER)
    and the joining SpMV launch (FITSNE_OPT_SPMV_JOIN) against the combine that
    gathers F_rep itself and a single launch: same gradient, every switch
    combination, over repeated calls (the dynamic schedule's ticket counter runs
    on), and in the fused iteration."""
    from paper_1712_09005_b200 import _lib
    n = 6007
    rr, cc, v, Y = _graph(n, 30, seed=11)
    csr = _csr(n, rr, cc, v)
    y = torch.from_numpy(Y.astype(np.float32)).cuda()
    want = O.grad(rr, cc, v, Y.astype(np.float32).astype(np.float64), 4.0, min_intervals=20, p=3)
    got = {}
    for sg in (0, 1):
        for join in (0, 1):
            ctx = _ctx(2, 128, 512, ctas)
            _lib.check(ctx.lib.fitsne_set_option(ctx.h, _lib.OPT_SIDE_GATHER, sg), "set_option")
            _lib.check(ctx.lib.fitsne_set_option(ctx.h, _lib.OPT_SPMV_JOIN, join), "set_option")
            ctx.set_affinities(csr)
            g = torch.empty_like(y)
            for _ in range(3):
                g.fill_(float("nan"))
                _lib.check(ctx.lib.fitsne_gradient(ctx.h, _lib.ptr(y), 4.0, _lib.ptr(g), None, ctx.stream),
                           "gradient")
                torch.cuda.synchronize()
                a = g.cpu().numpy().astype(np.float64)
                assert rel_l2(a, want) <= 1e-3
                got.setdefault((sg, join), a)
                assert rel_l2(a, got[(sg, join)]) <= 2e-5  # summation order of the fp32 atomics only
            # fused iteration with the KL: the joining CTAs' KL partials are counted
            yo, vel, gains = torch.empty_like(y), torch.zeros_like(y), torch.ones_like(y)
            kl = torch.zeros(1, dtype=torch.float64, device=y.device)
            st = torch.zeros(1, dtype=torch.int32, device=y.device)
            _lib.check(ctx.lib.fitsne_iterate(ctx.h, _lib.ptr(y), _lib.ptr(yo), _lib.ptr(vel), _lib.ptr(gains),
                                              4.0, 0.5, 200.0, _lib.ptr(kl), _lib.ptr(st), ctx.stream), "iterate")
            torch.cuda.synchronize()
            got[(sg, join, "kl")] = float(kl.item())
            got[(sg, join, "y")] = yo.cpu().numpy().astype(np.float64)
    base = got[(0, 0)]
    for key, a in got.items():
        if len(key) == 2:
            assert rel_l2(a, base) <= 2e-5, key
        elif key[2] == "kl":
            assert abs(a - got[(0, 0, "kl")]) <= 1e-7 * abs(got[(0, 0, "kl")]), key  # fp32 partial sums
        else:
            assert rel_l2(a, got[(0, 0, "y")]) <= 1e-5, key


@pytest.mark.parametrize("pieces", [0, 1, 2])
@pytest.mark.parametrize("shape", [(128, 512, 5), (64, 256, 0), (2048, 4096, 2)])
def test_gradient_host_pieces(cuda, shape, pieces):
    """fitsne_gradient_host (pinned host Y in, host gradient out; with pieces
    the tiled SpMV runs in row pieces with the copy-out overlapped) equals the
    device-buffer gradient up to float atomics order (rel-L2 1e-5), and the
    oracle to 1e-3."""
    from paper_1712_09005_b200 import _lib
    n = 5003
    rr, cc, v, Y = _graph(n, 30, seed=11)
    csr = _csr(n, rr, cc, v)
    y32 = Y.astype(np.float32)
    ctx = _ctx(2, *shape)
    _lib.check(ctx.lib.fitsne_set_option(ctx.h, 10, pieces), "set_option")
    ctx.set_affinities(csr)
    y = torch.from_numpy(y32).cuda()
    g = torch.empty_like(y)
    _lib.check(ctx.lib.fitsne_gradient(ctx.h, _lib.ptr(y), 4.0, _lib.ptr(g), None, ctx.stream), "grad")
    torch.cuda.synchronize()
    yh = torch.from_numpy(y32).pin_memory()
    for _ in range(2):  # the accumulator is consumed and cleared piece by piece
        gh = torch.full_like(yh, float("nan")).pin_memory()
        _lib.check(ctx.lib.fitsne_gradient_host(ctx.h, _lib.ptr(yh), 4.0, _lib.ptr(gh), ctx.stream),
                   "gradient_host")
        assert np.isfinite(gh.numpy()).all()
        assert rel_l2(gh.numpy().astype(np.float64), g.cpu().numpy().astype(np.float64)) <= 1e-5
    want = O.grad(rr, cc, v, y32.astype(np.float64), 4.0, min_intervals=20, p=3)
    assert rel_l2(gh.numpy().astype(np.float64), want) <= 1e-3


def test_public_gradient_host_arrays(cuda):
    """optimizer.gradient with numpy / CPU-tensor inputs takes the host path;
    results match the CUDA-tensor call."""
    from paper_1712_09005_b200 import optimizer, affinities
    n = 40_000
    rr, cc, v, Y = _graph(n, 60, seed=5, clustered=False)
    P = affinities.SparseAffinities(n=n, rows=rr, cols=cc, values=v)
    y32 = Y.astype(np.float32)
    dev = optimizer.gradient(P, torch.from_numpy(y32).cuda(), 2.0, 50, 3, "fft").cpu().numpy()
    host_np = optimizer.gradient(P, y32, 2.0, 50, 3, "fft", dtype="float32")
    assert host_np.dtype == np.float64
    assert rel_l2(host_np, dev.astype(np.float64)) <= 1e-5
    out = torch.empty((n, 2), dtype=torch.float32).pin_memory()
    r = optimizer.gradient(P, torch.from_numpy(y32).pin_memory(), 2.0, 50, 3, "fft", out=out)
    assert r is out
    assert rel_l2(out.numpy().astype(np.float64), dev.astype(np.float64)) <= 1e-5


def test_tiled_run_tsne_matches_csr(cuda):
    """The fused iteration (SpMV + KL + update) with the tiled kernel tracks
    the CSR kernel's trajectory over the first iterations."""
    from paper_1712_09005_b200 import _lib, optimizer
    from paper_1712_09005_b200.affinities import SparseAffinities
    n = 2000
    rr, cc, v, _ = _graph(n, 20, seed=21)
    P = SparseAffinities(n=n, rows=rr, cols=cc, values=v)
    logs = {}
    for mode in (0, 2):
        ctx = _lib.context(0, 2, torch.float32, 3, 50, 1.0)
        _lib.check(ctx.lib.fitsne_set_option(ctx.h, OPT_TILED, mode), "set_option")
        _lib.check(ctx.lib.fitsne_set_option(ctx.h, OPT_ROWS, 256), "set_option")
        _lib.check(ctx.lib.fitsne_set_option(ctx.h, OPT_COLS, 512), "set_option")
        cfg = optimizer.TsneConfig(dims=2, n_iter=30, seed=1, dtype="float32", min_intervals=50,
                                   exaggeration=optimizer.ExaggerationSchedule(12.0, 10))
        try:
            logs[mode] = np.asarray(optimizer.run_tsne(affinities=P, config=cfg).kl_log, dtype=float)
        finally:
            # the context is the cached per-thread one: put the defaults back
            for opt, val in ((OPT_TILED, 1), (OPT_ROWS, 3072), (OPT_COLS, 8192)):
                _lib.check(ctx.lib.fitsne_set_option(ctx.h, opt, val), "set_option")
    assert np.max(np.abs(logs[2] - logs[0]) / np.abs(logs[0])) <= 1e-4


def test_misaligned_y_uses_csr_kernel(cuda):
    rr, cc, v, Y = _graph(1001, 15, seed=8)
    csr = _csr(1001, rr, cc, v)
    buf = torch.zeros(2 * 1001 + 4, dtype=torch.float32, device="cuda")
    y_al = buf[4:].view(1001, 2)   # 16-byte aligned: tiled kernel
    y_al.copy_(torch.from_numpy(Y.astype(np.float32)))
    buf2 = torch.zeros(2 * 1001 + 2, dtype=torch.float32, device="cuda")
    y_mis = buf2[2:].view(1001, 2)  # 8-byte aligned only: bulk copies need 16, CSR kernel
    y_mis.copy_(torch.from_numpy(Y.astype(np.float32)))
    ctx = _ctx(2, 64, 128, 0)
    a = _attr(ctx, csr, y_al)
    b = _attr(ctx, csr, y_mis)
    assert rel_l2(a, b) <= 1e-5


def test_option_validation(cuda):
    from paper_1712_09005_b200 import _lib
    ctx = _lib.Context(0, 2, torch.float32, 3, 20, 1.0)
    for opt, val in ((OPT_TILED, 3), (OPT_ROWS, 3), (OPT_COLS, 0), (OPT_COLS, 32768), (OPT_CTAS, -1)):
        assert ctx.lib.fitsne_set_option(ctx.h, opt, val) != 0


def test_tiled_unsorted_rows(cuda):
    """A CSR whose rows are not column-sorted (a relabelled P) is re-sorted
    by the tiled build: every (row, chunk) is still one segment."""
    from paper_1712_09005_b200.affinities import permute_csr
    n = 3001
    rr, cc, v, Y = _graph(n, 25, seed=17)
    csr = _csr(n, rr, cc, v)
    perm = torch.from_numpy(np.random.default_rng(0).permutation(n)).cuda()
    inv = torch.empty_like(perm)
    inv[perm] = torch.arange(n, device="cuda")
    pcsr = permute_csr(csr, perm, inv)
    y = torch.from_numpy(Y.astype(np.float32)).cuda()[perm].contiguous()
    want = O.attraction(rr, cc, v, Y.astype(np.float32).astype(np.float64))[perm.cpu().numpy()]
    for shape in ((64, 128, 0), (512, 1024, 9)):
        got = _attr(_ctx(2, *shape), pcsr, y)
        assert rel_l2(got, want) <= 1e-5


def test_random_graph_keeps_csr_kernel(cuda):
    """Auto mode: a P without column locality (random partners, ~1 entry per
    (row, chunk) segment) stays on the CSR kernel even above 2^22 entries;
    forced tiling still works and agrees."""
    from paper_1712_09005_b200 import _lib
    n, k = 600_000, 8  # 16 entries per row over 74 chunks of 8192 points
    rr, cc, v, Y = _graph(n, k, seed=31, clustered=False)
    assert 2 * rr.size >= (1 << 22)
    csr = _csr(n, rr, cc, v)
    y = torch.from_numpy(Y.astype(np.float32)).cuda()
    st = (C.c_int64 * 8)()
    ctx = _ctx(1, 3072, 8192)
    ctx.set_affinities(csr)
    _lib.check(ctx.lib.fitsne_tiled_stats(ctx.h, _lib.ptr(y), st, ctx.stream), "stats")
    assert st[0] == 0
    auto = _attr(ctx, csr, y)
    forced = _attr(_ctx(2, 3072, 8192), csr, y)
    want = O.attraction(rr, cc, v, Y.astype(np.float32).astype(np.float64))
    assert rel_l2(auto, want) <= 1e-5
    assert rel_l2(forced, want) <= 1e-5


@pytest.mark.parametrize("dtype,tol", [("float32", 1e-3), ("float64", 1e-5)])
def test_one_dim_gradient_at_scale(cuda, dtype, tol):
    """1-D embedding (config C5's path: 1-D grid, single-block FFT), N = 200k
    clustered points, random kNN-like P: gradient vs the oracle."""
    from paper_1712_09005_b200 import optimizer
    from paper_1712_09005_b200.affinities import SparseAffinities
    rng = np.random.default_rng(41)
    n, k = 200_000, 15
    c = rng.uniform(-150, 150, 30)
    y = (c[rng.integers(0, 30, n)] + 3.0 * rng.standard_normal(n))[:, None]
    r = np.repeat(np.arange(n), k)
    cc = rng.integers(0, n - 1, n * k)
    cc = cc + (cc >= r)
    key = np.unique(np.minimum(r, cc) * n + np.maximum(r, cc))
    vals = rng.exponential(1.0, key.size)
    vals /= 2 * vals.sum()
    P = SparseAffinities(n=n, rows=key // n, cols=key % n, values=vals)
    yd = y.astype(np.float32).astype(np.float64) if dtype == "float32" else y
    g = optimizer.gradient(P, torch.from_numpy(yd).to(device=0, dtype=getattr(torch, dtype)), 12.0,
                           50, 3, "fft").double().cpu().numpy()
    want = O.grad(P.rows, P.cols, P.values, yd, 12.0, 50, 3, "fft")
    assert rel_l2(g, want) <= tol


def _shuffled(n, rr, cc, v, Y, seed):
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    r, c = inv[rr], inv[cc]
    return np.minimum(r, c), np.maximum(r, c), v, Y[perm]


@pytest.mark.parametrize("relabel", [1, 2])
@pytest.mark.parametrize("shape", [(64, 128, 0), (256, 1024, 7), (2, 2, 3)])
def test_relabelled_tiles_on_shuffled_graph(cuda, relabel, shape):
    """A clustered graph in random point order: the tiled copy built over the
    device Cuthill-McKee relabelling (FITSNE_OPT_RELABEL) gives the oracle's
    F_attr in the caller's order; auto mode takes the relabelling because it
    cuts the (row, chunk) segments."""
    from paper_1712_09005_b200 import _lib
    n = 5003
    rr, cc, v, Y = _shuffled(n, *_graph(n, 24, 11), seed=5)
    y = torch.from_numpy(Y.astype(np.float32)).cuda()
    ctx = _ctx(2, *shape)
    _lib.check(ctx.lib.fitsne_set_option(ctx.h, _lib.OPT_RELABEL, relabel), "set_option")
    got = _attr(ctx, _csr(n, rr, cc, v), y)
    st = (C.c_int64 * 8)()
    _lib.check(ctx.lib.fitsne_tiled_stats(ctx.h, _lib.ptr(y), st, ctx.stream), "stats")
    assert st[0] == 1
    if relabel == 2:
        assert st[6] == 1
    elif shape[1] >= 128:  # chunks wide enough for the clusters: relabelling pays
        assert st[6] == 1 and st[4] <= 0.5 * st[7]
    ref = O.attraction(rr, cc, v, Y.astype(np.float32).astype(np.float64))
    assert rel_l2(got, ref) <= 1e-5


def test_relabel_off_keeps_caller_order(cuda):
    from paper_1712_09005_b200 import _lib
    n = 3001
    rr, cc, v, Y = _shuffled(n, *_graph(n, 16, 12), seed=6)
    y = torch.from_numpy(Y.astype(np.float32)).cuda()
    ctx = _ctx(2, 64, 128)
    _lib.check(ctx.lib.fitsne_set_option(ctx.h, _lib.OPT_RELABEL, 0), "set_option")
    got = _attr(ctx, _csr(n, rr, cc, v), y)
    st = (C.c_int64 * 8)()
    _lib.check(ctx.lib.fitsne_tiled_stats(ctx.h, _lib.ptr(y), st, ctx.stream), "stats")
    assert st[0] == 1 and st[6] == 0
    assert rel_l2(got, O.attraction(rr, cc, v, Y.astype(np.float32).astype(np.float64))) <= 1e-5


def test_relabelled_gradient_and_iterate(cuda):
    """The overlapped gradient (tiled SpMV on relabelled points, combine in
    the caller's order) and the fused run_tsne iteration on a shuffled graph."""
    from paper_1712_09005_b200 import _lib, optimizer
    from paper_1712_09005_b200.affinities import SparseAffinities
    n = 20_000
    rr, cc, v, Y = _shuffled(n, *_graph(n, 30, 13), seed=7)
    P = SparseAffinities(n=n, rows=rr, cols=cc, values=v)
    y32 = Y.astype(np.float32)
    with _lib.option(OPT_TILED, 2), _lib.option(_lib.OPT_RELABEL, 2):
        g = optimizer.gradient(P, torch.from_numpy(y32).cuda(), 12.0, 50, 3, "fft")
        g_host = optimizer.gradient(P, y32, 12.0, 50, 3, "fft")
    ref = O.grad(rr, cc, v, y32.astype(np.float64), 12.0, 50, 3, "fft")
    assert rel_l2(g.double().cpu().numpy(), ref) <= 1e-3
    assert rel_l2(g_host, ref) <= 1e-3


@pytest.mark.parametrize("relabel", [0, 2])
@pytest.mark.parametrize("shape", [(64, 128, 0), (256, 1024, 7), (2, 2, 3), (4096, 6144, 0)])
def test_tiled_1d(cuda, shape, relabel):
    """1-D embeddings on the tiled SpMV (float chunks of twice the points):
    F_attr and the KL sum against the oracle, with and without relabelling."""
    from paper_1712_09005_b200 import _lib
    n = 5003
    rr, cc, v, Y = _graph(n, 24, 21)
    if relabel:
        rr, cc, v, Y = _shuffled(n, rr, cc, v, Y, seed=9)
    y1 = Y[:, :1].astype(np.float32)
    y = torch.from_numpy(np.ascontiguousarray(y1)).cuda()
    ctx = _lib.Context(0, 1, torch.float32, 3, 20, 1.0)
    for opt, val in ((OPT_TILED, 2), (OPT_ROWS, shape[0]), (OPT_COLS, shape[1]), (OPT_CTAS, shape[2]),
                     (_lib.OPT_RELABEL, relabel)):
        _lib.check(ctx.lib.fitsne_set_option(ctx.h, opt, val), "set_option")
    csr = _csr(n, rr, cc, v)
    ctx.set_affinities(csr)
    out = torch.empty((n, 1), dtype=torch.float32, device=y.device)
    _lib.check(ctx.lib.fitsne_attractive(ctx.h, _lib.ptr(y), _lib.ptr(out), ctx.stream), "attractive")
    st = (C.c_int64 * 8)()
    _lib.check(ctx.lib.fitsne_tiled_stats(ctx.h, _lib.ptr(y), st, ctx.stream), "stats")
    assert st[0] == 1 and st[6] == (1 if relabel else 0)
    ref = O.attraction(rr, cc, v, y1.astype(np.float64))
    assert rel_l2(out.cpu().numpy().astype(np.float64), ref) <= 1e-5
    kl = C.c_double()
    _lib.check(ctx.lib.fitsne_kl(ctx.h, _lib.ptr(y), 2.5, C.byref(kl), ctx.stream), "kl")
    assert abs(kl.value - O.kl_given_z(rr, cc, v, y1.astype(np.float64), 2.5)) <= 1e-5 * abs(kl.value)


def test_tiled_1d_gradient_and_run(cuda):
    """The 1-D production path (tiled SpMV in the overlapped schedule, the
    fused iteration) against the oracle."""
    from paper_1712_09005_b200 import _lib, optimizer
    from paper_1712_09005_b200.affinities import SparseAffinities
    n = 20_000
    rr, cc, v, Y = _graph(n, 30, 22)
    P = SparseAffinities(n=n, rows=rr, cols=cc, values=v)
    y1 = np.ascontiguousarray(Y[:, :1].astype(np.float32))
    with _lib.option(OPT_TILED, 2):
        g = optimizer.gradient(P, torch.from_numpy(y1).cuda(), 4.0, 50, 3, "fft").double().cpu().numpy()
        cfg = optimizer.TsneConfig(dims=1, n_iter=5, learning_rate=200.0, min_intervals=50,
                                   exaggeration=optimizer.ExaggerationSchedule(12.0, 5), seed=0,
                                   pca_dims=None, repulsion_method="fft", dtype="float32")
        res = optimizer.run_tsne(affinities=P, config=cfg)
    assert rel_l2(g, O.grad(rr, cc, v, y1.astype(np.float64), 4.0, 50, 3, "fft")) <= 1e-3
    _, kl_o = O.tsne(rr, cc, v, n, dims=1, n_iter=5, lr=200.0, early_coeff=12.0, early_until=5,
                     min_intervals=50, p=3, method="fft", seed=0)
    assert np.max(np.abs(res.kl_log - kl_o) / np.abs(kl_o)) <= 1e-4


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_spectrum_ahead_option(cuda, dtype):
    """FITSNE_OPT_SPEC_AHEAD (kernel spectrum on its own stream beside the
    spread): the gradient equals the default schedule's and the oracle's,
    over repeated calls with a changing grid."""
    from paper_1712_09005_b200 import _lib
    n = 4001
    rr, cc, v, Y = _graph(n, 20, seed=3)
    from paper_1712_09005_b200.affinities import SparseAffinities, device_csr
    P = SparseAffinities(n=n, rows=rr, cols=cc, values=v)
    csr = device_csr(P, dtype, 0)
    tol = 1e-3 if dtype == torch.float32 else 1e-9
    got = {}
    for opt in (0, 1):
        ctx = _lib.Context(0, 2, dtype, 3, 20, 1.0)
        _lib.check(ctx.lib.fitsne_set_option(ctx.h, _lib.OPT_SPEC_AHEAD, opt), "set_option")
        ctx.set_affinities(csr)
        for k, scale in enumerate((1.0, 1.7, 0.6)):   # the grid (and its spectrum) changes between calls
            yk = torch.from_numpy(Y * scale).to(dtype).cuda()
            g = torch.empty_like(yk)
            _lib.check(ctx.lib.fitsne_gradient(ctx.h, _lib.ptr(yk), 2.0, _lib.ptr(g), None, ctx.stream), "gradient")
            torch.cuda.synchronize()
            got[(opt, k)] = g.double().cpu().numpy()
            want = O.grad(rr, cc, v, yk.double().cpu().numpy(), 2.0, min_intervals=20, p=3)
            assert rel_l2(got[(opt, k)], want) <= tol, (opt, k)
    for k in range(3):
        assert rel_l2(got[(1, k)], got[(0, k)]) <= (2e-5 if dtype == torch.float32 else 1e-12), k
