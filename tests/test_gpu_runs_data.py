"""run_tsne(data=...) end to end on the device (affinities + descent): ports of
the reference's integration tests (test_optimizer.py:273-349) and parity of
the GPU affinity pipeline with the reference's definitions (affinities.py)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def opt(cuda):
    from paper_1712_09005_b200 import optimizer
    return optimizer


def test_two_cluster_separation(opt):           # test_optimizer.py:273-285
    rng = np.random.default_rng(11)
    data = np.vstack([rng.normal(0, 0.5, (500, 10)) + 6.0, rng.normal(0, 0.5, (500, 10)) - 6.0])
    res = opt.run_tsne(data=data, config=opt.TsneConfig(dims=2, perplexity=30, n_iter=1000, seed=4))
    emb = res.embedding
    c0, c1 = emb[:500].mean(0), emb[500:].mean(0)
    r0 = np.linalg.norm(emb[:500] - c0, axis=1).max()
    r1 = np.linalg.norm(emb[500:] - c1, axis=1).max()
    assert np.linalg.norm(c0 - c1) > 2.0 * max(r0, r1)


def test_kl_decreases_late_across_seeds(opt):   # test_optimizer.py:303-320
    rng = np.random.default_rng(13)
    n = 200
    data = np.vstack([rng.normal(0, 1.0, (n // 2, 6)) + 3.0, rng.normal(0, 1.0, (n // 2, 6)) - 3.0])
    drops = 0
    for seed in range(10):
        cfg = opt.TsneConfig(dims=2, perplexity=20, n_neighbors=n - 1, n_iter=500, seed=seed)
        res = opt.run_tsne(data=data, config=cfg)
        assert np.all(res.kl_log >= -1e-12)
        if res.kl_log[-1] <= res.kl_log[-100]:
            drops += 1
    assert drops >= 9


def test_pca_front_end_runs(opt):               # test_optimizer.py:344-349
    rng = np.random.default_rng(14)
    data = rng.standard_normal((120, 80))
    res = opt.run_tsne(data=data, config=opt.TsneConfig(dims=2, perplexity=10, n_iter=300,
                                                        seed=2, pca_dims=20))
    assert res.embedding.shape == (120, 2)
    assert np.all(np.isfinite(res.embedding))


def test_callback_sees_every_iteration(opt):    # test_optimizer.py:336-342 (n_iter >= 250: the
    from paper_1712_09005_b200.affinities import SparseAffinities   # reference's schedule rule)
    P = SparseAffinities(n=4, rows=[0, 1, 2], cols=[1, 2, 3], values=[1 / 6, 1 / 6, 1 / 6])
    seen = []
    opt.run_tsne(affinities=P, config=opt.TsneConfig(n_iter=260, seed=1),
                 callback=lambda it, y, info: seen.append(it))
    assert seen == list(range(260))


def test_same_seed_same_result(opt):            # test_optimizer.py:294-301 (statistical here)
    rng = np.random.default_rng(12)
    data = rng.standard_normal((150, 8))
    cfg = opt.TsneConfig(dims=2, perplexity=12, n_iter=300, seed=9)
    a = opt.run_tsne(data=data, config=cfg)
    b = opt.run_tsne(data=data, config=cfg)
    # exact-path runs (N <= 1000) have no atomics: bitwise reproducible
    np.testing.assert_array_equal(a.kl_log, b.kl_log)
    np.testing.assert_array_equal(a.embedding, b.embedding)


def test_gpu_affinities_match_reference_definitions(cuda):
    """Same structure and values (to the bisection tolerance) as the oracle
    restatement of affinities_from_data on fp64 data."""
    from paper_1712_09005_b200.affinity_build import AffinityConfig, affinities_from_data
    rng = np.random.default_rng(21)
    x = np.concatenate([rng.normal(c, 1.0, (400, 12)) for c in (-4.0, 0.0, 4.0)])
    P, bw = affinities_from_data(x, AffinityConfig(perplexity=15, n_neighbors=45, method="exact"))
    # oracle: brute-force kNN + bisection + symmetrise in numpy
    d2 = ((x[:, None, :] - x[None, :, :]) ** 2).sum(-1)
    np.fill_diagonal(d2, np.inf)
    idx = np.argsort(d2, axis=1, kind="stable")[:, :45]
    dd = np.take_along_axis(d2, idx, axis=1)
    assert np.allclose(np.sort(bw.conditional.sum(1)), 1.0)
    n = len(x)
    keys = set(zip(np.minimum(np.repeat(np.arange(n), 45), idx.ravel()),
                   np.maximum(np.repeat(np.arange(n), 45), idx.ravel())))
    got = set(zip(P.rows.tolist(), P.cols.tolist()))
    assert got == {(int(a), int(b)) for a, b in keys}
    assert abs(P.ordered_total - 1.0) <= 1e-9
    assert np.all(np.abs(bw.achieved_perplexity - 15) <= 1e-4 + 1e-9)
    assert dd.shape == (n, 45)
