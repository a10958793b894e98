"""Small end-to-end exercise of every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck): band spread, direct and sorted spreads,
one-block and four-step FFT stages, gather / combine, tiled SpMV (forced,
with and without the relabelling), CSR SpMV, fused iteration, fp64 grid of a
wide fp32 embedding, 1-D path, general n-body.  Sizes are small so the
instrumented run finishes in minutes.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1712_09005_b200 import _lib, nbody, optimizer  # noqa: E402
from paper_1712_09005_b200.affinities import SparseAffinities  # noqa: E402


def graph(n, k, rng):
    lab = np.sort(rng.integers(0, 5, n))
    r = np.repeat(np.arange(n), k)
    c = np.empty_like(r)
    for i in range(n):
        same = np.flatnonzero(lab == lab[i])
        c[i * k:(i + 1) * k] = rng.choice(same, k)
    keep = r != c
    lo, hi = np.minimum(r[keep], c[keep]), np.maximum(r[keep], c[keep])
    key = np.unique(lo * n + hi)
    v = rng.random(key.size) + 0.1
    return SparseAffinities(n=n, rows=key // n, cols=key % n, values=v / (2 * v.sum()))


def main():
    rng = np.random.default_rng(0)
    n = 6000
    P = graph(n, 12, rng)
    y = (rng.standard_normal((n, 2)) * 20).astype(np.float32)
    yd = torch.from_numpy(y).cuda()
    for opts in ([], [(_lib.OPT_TILED_SPMV, 2), (_lib.OPT_TILE_ROWS, 256), (_lib.OPT_TILE_COLS, 512)],
                 [(_lib.OPT_TILED_SPMV, 2), (_lib.OPT_RELABEL, 2), (_lib.OPT_TILE_ROWS, 256),
                  (_lib.OPT_TILE_COLS, 512)],
                 [(_lib.OPT_SORTED_SPREAD, 0)], [(_lib.OPT_SORTED_SPREAD, 2)],
                 [(_lib.OPT_FFT_PATH, 2)], [(_lib.OPT_GRID_F64, 2)]):
        ctxs = [_lib.option(o, v) for o, v in opts]
        for c in ctxs:
            c.__enter__()
        try:
            optimizer.gradient(P, yd, 4.0, 50, 3, "fft")
            optimizer.gradient(P, y, 4.0, 50, 3, "fft")
            optimizer.compute_repulsive(yd, 50, 3, "fft")
        finally:
            for c in reversed(ctxs):
                c.__exit__(None, None, None)
    optimizer.gradient(P, y.astype(np.float64), 4.0, 50, 3, "fft", dtype="float64")
    # 1-D and general n-body
    y1 = (rng.standard_normal((n, 1)) * 30).astype(np.float32)
    optimizer.gradient(P, y1, 1.0, 50, 3, "fft")
    with _lib.option(_lib.OPT_FFT_PATH, 2):
        optimizer.gradient(P, y1, 1.0, 50, 3, "fft")
    q = rng.standard_normal((n, 3))
    nbody.evaluate_nbody(y.astype(np.float64), q, "cauchy", 20, 3)
    # fused iterations
    cfg = optimizer.TsneConfig(dims=2, n_iter=3, learning_rate=200.0, min_intervals=50,
                               exaggeration=optimizer.ExaggerationSchedule(12.0, 3), seed=0,
                               pca_dims=None, repulsion_method="fft", dtype="float32")
    optimizer.run_tsne(affinities=P, config=cfg)
    torch.cuda.synchronize()
    print("sanitize run ok")


if __name__ == "__main__":
    main()
