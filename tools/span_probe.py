"""fp32 repulsion accuracy vs the oracle as the grid (FFT length) grows."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import fitsne_oracle as O  # noqa: E402
from paper_1712_09005_b200 import optimizer  # noqa: E402

for span in [float(a) for a in sys.argv[1:]] or [200.0, 428.0, 600.0, 700.0, 860.0]:
    rng = np.random.default_rng(21)
    c = rng.uniform(0, span, (40, 2))
    c[:2] = [[0.0, 0.0], [span, span]]
    y = np.clip(c[rng.integers(0, 40, 20_000)] + 3.0 * rng.standard_normal((20_000, 2)), 0, span)
    f, z, _, _ = O.repulsion(y.astype(np.float32).astype(np.float64), 50, 3, "fft")
    for dt in ("float32", "float64"):
        try:
            rep = optimizer.compute_repulsive(torch.from_numpy(y.astype(dt)).cuda(), 50, 3, "fft")
        except ValueError as e:
            print(span, dt, "error", e)
            continue
        g = rep.forces.double().cpu().numpy()
        err = np.linalg.norm(g - f) / np.linalg.norm(f)
        print(f"span {span:6.1f} {dt}: rel-L2 {err:.3e}  z rel {abs(rep.z - z) / z:.2e}", flush=True)
