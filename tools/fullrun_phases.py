"""Where does a C3 run_tsne spend its time?  (GPU probe)"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from tools import synth  # noqa: E402
from paper_1712_09005_b200 import optimizer  # noqa: E402


def run(P, reorder, n_iter=1000):
    cfg = optimizer.TsneConfig(
        dims=2, n_iter=n_iter, learning_rate=200.0, min_intervals=50, points_per_interval=3,
        exaggeration=optimizer.ExaggerationSchedule(12.0, n_iter // 4, 4.0, 3 * n_iter // 4), seed=0,
        pca_dims=None,
        repulsion_method="fft", dtype="float32", device=0,
        reorder_iters=(100, 250, 500, 750) if reorder else None)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = optimizer.run_tsne(affinities=P, config=cfg)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, res


P, _ = synth.c3(device="cuda", n=1_300_000)
for label, reorder in (("no-reorder #1", False), ("no-reorder #2", False), ("reorder", True),
                       ("no-reorder #3", False)):
    sec, res = run(P, reorder)
    print(f"{label:14s} {sec:6.3f} s  {1000 / sec:7.1f} it/s  KL {res.kl_log[-1]:.4f}", flush=True)
sec, _ = run(P, False, n_iter=100)
print(f"100 iterations {sec:6.3f} s", flush=True)
