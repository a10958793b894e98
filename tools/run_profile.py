"""cProfile of a steady-state C3 run_tsne (second run on the same P): where the
wall time outside the fused iterations goes.  GPU probe."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tools import synth  # noqa: E402
from paper_1712_09005_b200 import optimizer  # noqa: E402

cache = sys.argv[sys.argv.index("--inputs-cache") + 1] if "--inputs-cache" in sys.argv else ""
if cache and Path(cache).exists():
    with np.load(cache) as z:
        P = synth.Upper(int(z["n"]), z["rows"], z["cols"], z["values"])
else:
    P, _ = synth.c3(device="cuda")
cfg = optimizer.TsneConfig(dims=2, n_iter=1000, learning_rate=200.0, min_intervals=50, points_per_interval=3,
                           exaggeration=optimizer.ExaggerationSchedule(12.0, 250, 4.0, 750), seed=0, pca_dims=None,
                           repulsion_method="fft", dtype="float32", device=0)
optimizer.run_tsne(affinities=P, config=cfg)
torch.cuda.synchronize()
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
optimizer.run_tsne(affinities=P, config=cfg)
torch.cuda.synchronize()
pr.disable()
print(f"second run: {time.perf_counter() - t0:.3f} s")
pstats.Stats(pr).sort_stats("cumulative").print_stats(22)
