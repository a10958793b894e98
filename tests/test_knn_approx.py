"""Approximate kNN (random-projection forest) of the affinity pipeline against
the reference's own outputs (tests/golden/make_knn_golden.py ->
knn_approx_reference.npz; affinities.py:167-206, 332-358)."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE / "golden"))

from make_knn_golden import cloud, duplicates  # noqa: E402

from paper_1712_09005_b200 import affinity_build as AB  # noqa: E402


@pytest.fixture(scope="module")
def gold():
    with np.load(HERE / "golden" / "knn_approx_reference.npz") as z:
        return {k: z[k] for k in z.files}


def _check_knn(dev, gold):
    for tag, x, k, trees, seed in (("cloud", cloud(), 15, 6, 3), ("dup", duplicates(), 40, 1, 1)):
        idx, d2 = AB.knn_approx(torch.from_numpy(x).to(dev), k, n_trees=trees, seed=seed)
        assert idx.shape == (x.shape[0], k) and idx.dtype == torch.int64
        # neighbour indexing is bit-exact: same forest, same ranking, same tie order
        np.testing.assert_array_equal(idx.cpu().numpy(), gold[tag + "_idx"])
        np.testing.assert_allclose(d2.cpu().numpy(), gold[tag + "_d2"], rtol=1e-13, atol=1e-13)


def test_knn_approx_matches_reference_cpu(gold):
    _check_knn("cpu", gold)


def test_knn_approx_argument_errors():
    x = torch.zeros(10, 3, dtype=torch.float64)
    with pytest.raises(ValueError):
        AB.knn_approx(x, 10)
    with pytest.raises(ValueError):
        AB.knn_approx(x, 3, n_trees=0)


@pytest.mark.gpu
def test_knn_approx_matches_reference_gpu(gold):
    _check_knn("cuda", gold)


@pytest.mark.gpu
def test_affinities_from_data_approx(gold):
    """method="approx" (and "auto" above exact_max_n) builds the reference's P."""
    x = cloud()
    for cfg in (AB.AffinityConfig(perplexity=5.0, n_neighbors=15, method="approx", n_trees=6, seed=3),
                AB.AffinityConfig(perplexity=5.0, n_neighbors=15, method="auto", n_trees=6, seed=3,
                                  exact_max_n=1000)):
        P, bw = AB.affinities_from_data(x, cfg)
        np.testing.assert_array_equal(P.rows, gold["cloud_rows"])
        np.testing.assert_array_equal(P.cols, gold["cloud_cols"])
        np.testing.assert_allclose(P.values, gold["cloud_vals"], rtol=1e-9, atol=1e-15)
        np.testing.assert_allclose(bw.sigma, gold["cloud_sigma"], rtol=1e-4)
