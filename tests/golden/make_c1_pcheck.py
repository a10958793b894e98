"""Fingerprint of the REFERENCE's own C1 affinities (for tests/test_gpu_fullrun.py).

The C1 full-run test rebuilds P on the GPU (tools/synth.affinities: exact
kNN, the reference's perplexity bisection and symmetrisation).  To show that
both runs start from the same P without committing the 683k-pair matrix, this
script runs the reference's affinities_from_data on the same seeded X and
stores a fingerprint: a SHA-256 of the sorted (row, col) pattern and the
per-point row sums of P (both triangles, float64, 10k values).

    python tests/golden/make_c1_pcheck.py   (~15 s)
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(HERE))

from make_golden import import_reference  # noqa: E402
from tools import synth  # noqa: E402


def pattern_sha(n, rows, cols):
    key = np.sort(np.asarray(rows, np.int64) * n + np.asarray(cols, np.int64))
    return hashlib.sha256(key.tobytes()).hexdigest()


def row_sums(n, rows, cols, vals):
    return (np.bincount(rows, weights=vals, minlength=n) + np.bincount(cols, weights=vals, minlength=n))


def main(src="/root/reference/pkg/src"):
    import_reference(src)
    import fftsne.affinities as ra
    X, _ = synth.mixture(10_000, 50, 10, seed=1, centre_std=5.0)
    X = X.double().numpy()
    P, _ = ra.affinities_from_data(X, ra.AffinityConfig(perplexity=30, n_neighbors=90, method="exact"))
    sha = pattern_sha(P.n, P.rows, P.cols)
    np.savez_compressed(HERE / "c1_pcheck.npz", pattern_sha256=np.array([sha]),
                        row_sums=row_sums(P.n, P.rows, P.cols, P.values))
    print(f"{P.rows.size} pairs, pattern {sha[:16]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
