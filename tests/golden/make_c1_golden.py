"""Run the REFERENCE on BASELINE config 1 and store its KL trajectory.

C1: N=10,000, d=50, 10 equal isotropic clusters with centres ~ N(0, 25 I),
affinities by exact kNN k=90 / perplexity 30 (the reference's own
affinities_from_data), 2-D run_tsne with 1000 iterations, learning rate 200,
early exaggeration 12 for 250 iterations, momentum 0.5 -> 0.8, p = 3,
min_intervals 50, fp64.  The data come from tools/synth.mixture (seeded,
torch CPU generator) so the GPU test can rebuild the same X.

    python tests/golden/make_c1_golden.py   (~3 min on 8 cores)
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(HERE))

from make_golden import import_reference  # noqa: E402
from tools import synth  # noqa: E402


def main(src="/root/reference/pkg/src"):
    nb, op, SA = import_reference(src)
    import fftsne.affinities as ra
    X, _ = synth.mixture(10_000, 50, 10, seed=1, centre_std=5.0)
    X = X.double().numpy()
    t0 = time.time()
    P, _ = ra.affinities_from_data(X, ra.AffinityConfig(perplexity=30, n_neighbors=90, method="exact"))
    t1 = time.time()
    cfg = op.TsneConfig(dims=2, n_iter=1000, learning_rate=200.0, min_intervals=50,
                        points_per_interval=3, exaggeration=op.ExaggerationSchedule(12.0, 250),
                        seed=0, pca_dims=None, repulsion_method="fft")
    res = op.run_tsne(affinities=P, config=cfg)
    t2 = time.time()
    np.savez_compressed(HERE / "c1_reference.npz", kl_log=res.kl_log,
                        nnz_upper=np.array([P.rows.size]), p_sum=np.array([P.values.sum()]),
                        affinity_s=np.array([t1 - t0]), run_s=np.array([t2 - t1]),
                        emb_span=np.ptp(res.embedding, axis=0))
    print(f"P: {P.rows.size} pairs ({t1 - t0:.1f} s); run {t2 - t1:.1f} s; final KL {res.kl_log[-1]:.6f}")


if __name__ == "__main__":
    main(*sys.argv[1:])
