"""How much does point ordering change the C3 SpMV?  (GPU probe, not a test.)

Builds the C3 inputs, then for several point orderings relabels P (symmetric
permutation) and Y and times the attractive SpMV (fitsne_gradient_rows) and the
whole gradient.  Orderings that need X (PCA of the data) are upper bounds for
what an ordering computed from P alone could achieve.
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from tools import synth  # noqa: E402
from paper_1712_09005_b200 import _lib  # noqa: E402
from paper_1712_09005_b200.affinities import csr_from_full, permute_csr  # noqa: E402


def morton(coords, bits=10):
    """Morton key of (n, k) float coords, `bits` per axis."""
    c = coords - coords.min(0).values
    c = c / c.max(0).values.clamp_min(1e-30)
    q = (c * ((1 << bits) - 1)).long()
    key = torch.zeros(q.shape[0], dtype=torch.long, device=q.device)
    k = q.shape[1]
    for b in range(bits):
        for a in range(k):
            key |= ((q[:, a] >> b) & 1) << (b * k + a)
    return key


def timed(fn, steps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / steps


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_300_000
    t0 = time.time()
    X, labels = synth.mixture(n, 50, 40, 3, anisotropic=True, power=1.5, device="cuda")
    rows, cols, vals = synth.affinities(X, 90, 30.0)
    Y = synth.pca2(X, 100.0).float()
    r = torch.cat([rows, cols])
    c = torch.cat([cols, rows])
    v = torch.cat([vals, vals])
    base = csr_from_full(n, r, c, v, torch.float32, 0, n)
    del r, c, v
    print(f"inputs {time.time() - t0:.1f}s nnz {base.col.numel()}", flush=True)

    Xc = X - X.mean(0, keepdim=True)
    _, _, V = torch.linalg.svd(Xc[::13].double(), full_matrices=False)
    pcs = (Xc.double() @ V[:8].T).float()
    lab = torch.from_numpy(labels).cuda()

    orders = {"identity": torch.arange(n, device="cuda"),
              "random": torch.randperm(n, device="cuda"),
              "morton_y": torch.argsort(morton(Y, 16))}
    for k in (2, 3, 4, 6):
        orders[f"morton_pc{k}"] = torch.argsort(morton(pcs[:, :k], 60 // k))
    # within-cluster ordering by local PCs (an upper bound of graph orderings)
    key = torch.zeros(n, dtype=torch.long, device="cuda")
    for cl in range(40):
        m = lab == cl
        if int(m.sum()) < 2:
            continue
        xc = X[m] - X[m].mean(0, keepdim=True)
        _, _, Vc = torch.linalg.svd(xc[:: max(1, xc.shape[0] // 20000)].double(),
                                    full_matrices=False)
        lp = (xc.double() @ Vc[:3].T).float()
        key[m] = (cl << 40) | morton(lp, 13)
    orders["cluster_localpc3"] = torch.argsort(key)
    # Morton order of a short t-SNE run from the PCA start (an ordering
    # computed from P itself: the embedding places graph neighbours together)
    for iters in (100, 300):
        ctx = _lib.Context(0, 2, torch.float32, 3, 50, 1.0)
        ctx.set_affinities(base)
        y0 = Y.clone() * 0.01
        y1 = torch.empty_like(y0)
        vel = torch.zeros_like(y0)
        gains = torch.ones_like(y0)
        kd = torch.zeros(1, dtype=torch.float64, device="cuda")
        stt = torch.zeros(1, dtype=torch.int32, device="cuda")
        tt = time.time()
        for it in range(iters):
            _lib.check(ctx.lib.fitsne_iterate(ctx.h, _lib.ptr(y0), _lib.ptr(y1), _lib.ptr(vel),
                                              _lib.ptr(gains), 12.0, 0.5, float(n) / 12.0,
                                              _lib.ptr(kd), _lib.ptr(stt), ctx.stream), "iterate")
            y0, y1 = y1, y0
        torch.cuda.synchronize()
        print(f"tsne{iters}: {time.time() - tt:.2f}s span {(y0.max(0).values - y0.min(0).values).tolist()}",
              flush=True)
        orders[f"morton_tsne{iters}"] = torch.argsort(morton(y0, 16))
        del ctx

    ctxs = {}
    for mode in (0, 2):
        c = _lib.Context(0, 2, torch.float32, 3, 50, 1.0)
        _lib.check(c.lib.fitsne_set_option(c.h, 5, mode), "opt")
        ctxs[mode] = c
    for name, perm in orders.items():
        inv = torch.empty_like(perm)
        inv[perm] = torch.arange(n, device="cuda")
        csr = permute_csr(base, perm, inv)
        y = Y[perm].contiguous()
        g = torch.empty_like(y)
        f = torch.zeros_like(y)
        line = f"{name:18s}"
        for mode, ctx in ctxs.items():
            ctx.set_affinities(csr)
            t_spmv = timed(lambda: _lib.check(ctx.lib.fitsne_gradient_rows(
                ctx.h, _lib.ptr(y), _lib.ptr(f), 1.0, _lib.ptr(g), ctx.stream), "rows"))
            t_grad = timed(lambda: _lib.check(ctx.lib.fitsne_gradient(
                ctx.h, _lib.ptr(y), 1.0, _lib.ptr(g), None, ctx.stream), "grad"))
            line += f" | {'tiled' if mode else 'csr'} spmv {t_spmv * 1e3:6.1f} us grad {t_grad * 1e3:6.1f} us"
        print(line, flush=True)
        del csr


if __name__ == "__main__":
    main()
