"""Full-run parity on BASELINE config 1 (north star: final KL within 1%).

The reference itself was run on C1 in the build container
(tests/golden/make_c1_golden.py -> c1_reference.npz: its affinities from
affinities_from_data, then run_tsne for 1000 iterations, fp64).  Here the
same X is regenerated (tools/synth.mixture, seeded), P is rebuilt on the GPU
with the reference's definitions (exact kNN, perplexity bisection,
symmetrisation; tools/synth.affinities) and the device run_tsne is run in fp64
and fp32.  t-SNE descent is chaotic, so the trajectory is compared pointwise
only over the first iterations and by its final value within 1%.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden" / "c1_reference.npz"


@pytest.fixture(scope="module")
def c1(cuda):
    from tools import synth
    from paper_1712_09005_b200.affinities import SparseAffinities
    X, _ = synth.mixture(10_000, 50, 10, seed=1, centre_std=5.0)
    r, c, v = synth.affinities(X.double().cuda(), 90, 30.0)
    P = SparseAffinities(n=10_000, rows=r.cpu().numpy(), cols=c.cpu().numpy(),
                         values=v.cpu().numpy())
    with np.load(GOLD) as z:
        ref = {k: z[k] for k in z.files}
    return P, ref


def _run(P, dtype):
    from paper_1712_09005_b200 import optimizer as opt
    cfg = opt.TsneConfig(dims=2, n_iter=1000, learning_rate=200.0, min_intervals=50,
                         points_per_interval=3, exaggeration=opt.ExaggerationSchedule(12.0, 250),
                         seed=0, pca_dims=None, repulsion_method="fft", dtype=dtype)
    return opt.run_tsne(affinities=P, config=cfg)


def test_c1_affinities_match_reference_structure(c1):
    P, ref = c1
    assert P.rows.size == int(ref["nnz_upper"][0])
    assert abs(P.values.sum() - float(ref["p_sum"][0])) <= 1e-12


def test_c1_affinities_identical_to_reference(c1):
    """The GPU-built P is the reference's P: the same (row, col) pattern
    (SHA-256 of the sorted pairs) and the same per-point mass to 1e-6 (the
    perplexity bisections stop at different sigmas inside their tolerance)
    (fingerprint of the reference's affinities_from_data,
    tests/golden/make_c1_pcheck.py), so both full runs start from one input."""
    import hashlib
    P, _ = c1
    with np.load(Path(__file__).resolve().parent / "golden" / "c1_pcheck.npz") as z:
        sha, rs_ref = str(z["pattern_sha256"][0]), z["row_sums"]
    key = np.sort(P.rows.astype(np.int64) * P.n + P.cols.astype(np.int64))
    assert hashlib.sha256(key.tobytes()).hexdigest() == sha
    rs = np.bincount(P.rows, weights=P.values, minlength=P.n) + np.bincount(P.cols, weights=P.values,
                                                                           minlength=P.n)
    assert np.max(np.abs(rs - rs_ref) / rs_ref) <= 1e-6


@pytest.mark.parametrize("dtype,early_tol", [("float64", 1e-6), ("float32", 1e-3)])
def test_c1_full_run_final_kl_within_1pct(c1, dtype, early_tol):
    P, ref = c1
    res = _run(P, dtype)
    kl, kref = res.kl_log, ref["kl_log"]
    assert np.all(np.isfinite(kl))
    # early iterations: same inputs, same Y0 draw -> same KL up to rounding
    assert np.max(np.abs(kl[:10] - kref[:10]) / kref[:10]) <= early_tol
    # full run: final KL within 1% (north star)
    assert abs(kl[-1] - kref[-1]) <= 0.01 * kref[-1], (kl[-1], kref[-1])
    # the embedding has the reference's extent (same dynamics).  The span of a
    # single axis depends on where the outermost cluster lands in a chaotic
    # run (measured on 10 device runs: up to -14% on one axis), so the sum of
    # both axes is compared (measured spread within +-9%)
    span = np.ptp(res.embedding, axis=0)
    assert abs(span.sum() - ref["emb_span"].sum()) <= 0.15 * ref["emb_span"].sum()
