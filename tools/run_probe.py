"""Marginal cost of a fused run_tsne iteration at C3 (GPU probe): two runs of
different length on the same P; prints seconds and the per-iteration
difference, plus a CUPTI timeline of three iterations."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from tools import synth  # noqa: E402
from paper_1712_09005_b200 import optimizer  # noqa: E402


def run(P, n_iter):
    cfg = optimizer.TsneConfig(
        dims=2, n_iter=n_iter, learning_rate=200.0, min_intervals=50, points_per_interval=3,
        exaggeration=optimizer.ExaggerationSchedule(12.0, 250, 4.0, 750 if n_iter >= 750 else n_iter), seed=0, pca_dims=None,
        repulsion_method="fft", dtype="float32", device=0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = optimizer.run_tsne(affinities=P, config=cfg)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, res


P, _ = synth.c3(device="cuda")
run(P, 300)
a, _ = run(P, 300)
b, res = run(P, 1000)
print(f"300 it {a:.3f}s  1000 it {b:.3f}s  marginal {(b - a) / 700 * 1e3:.3f} ms/it  "
      f"final KL {res.kl_log[-1]:.4f} span {np.ptp(res.embedding, axis=0)}", flush=True)
