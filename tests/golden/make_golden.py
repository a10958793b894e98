"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container, where the reference package is importable:

    python tests/golden/make_golden.py [/path/to/reference/pkg/src]

It copies nothing into the repo except the small .npz fixtures it writes next
to this script: seeded inputs plus the reference's outputs for make_grid,
_point_interp, _spread, the kernel spectra / FFT matvec, gather,
compute_repulsive (fft + exact), compute_attractive, gradient, KL, step and
two short run_tsne trajectories.  The GPU box never reads /root/reference;
tests compare against these files and against oracle/fitsne_oracle.py.
"""

from __future__ import annotations

import os
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent


def import_reference(src):
    # numba caches next to the sources: import from a writable copy
    tmp = Path(tempfile.mkdtemp(prefix="fftsne_ref_"))
    shutil.copytree(src, tmp / "src")
    os.environ.setdefault("NUMBA_CACHE_DIR", str(tmp / "numba"))
    sys.path.insert(0, str(tmp / "src"))
    import fftsne.nbody as nb  # noqa: E402
    import fftsne.optimizer as op  # noqa: E402
    from fftsne.affinities import SparseAffinities  # noqa: E402
    return nb, op, SparseAffinities


def random_affinities(n, rng, density, SparseAffinities):
    # same construction as the reference tests (test_optimizer.py:21-28)
    iu = np.triu_indices(n, 1)
    vals = rng.random(iu[0].size)
    if density < 1.0:
        vals *= rng.random(vals.size) < density
    keep = vals > 0
    vals = vals[keep] / (2.0 * vals[keep].sum())
    return SparseAffinities(n=n, rows=iu[0][keep], cols=iu[1][keep], values=vals)


def knn_like_affinities(y, k, rng, SparseAffinities):
    """Sparse P on a point set: k random partners per row, Exp(1) weights."""
    n = y.shape[0]
    r = np.repeat(np.arange(n), k)
    c = rng.integers(0, n - 1, size=n * k)
    c = c + (c >= r)
    lo, hi = np.minimum(r, c), np.maximum(r, c)
    key = np.unique(lo * n + hi)
    rows, cols = key // n, key % n
    vals = rng.exponential(1.0, size=rows.size)
    vals /= 2.0 * vals.sum()
    return SparseAffinities(n=n, rows=rows, cols=cols, values=vals)


def blobs(n, dims, rng, centers=20, span=40.0, std=1.5):
    c = rng.uniform(-span, span, size=(centers, dims))
    sizes = rng.multinomial(n, rng.dirichlet(np.ones(centers)))
    return np.concatenate([c[i] + std * rng.standard_normal((s, dims)) for i, s in enumerate(sizes)])


def main(src):
    nb, op, SA = import_reference(src)
    out = {}

    # -- grid cases (test_nbody.py:60-93 + adversarial spans)
    grid_cases = [
        np.linspace(0.0, 5.0, 11)[:, None],
        np.linspace(0.0, 100.0, 7)[:, None],
        np.full((4, 1), 0.3),
        np.array([[0.0, 0.0], [40.0, 3.0]]),
        np.array([0.0, 10.0])[:, None],
        np.random.default_rng(1).normal(0, 1e-4, (500, 2)),
        np.random.default_rng(2).uniform(-37.3, 51.9, (777, 2)),
    ]
    for i, pts in enumerate(grid_cases):
        g = nb.make_grid(pts, min_intervals=20 if i != 4 else 5, points_per_interval=3)
        out[f"grid{i}_pts"] = pts
        out[f"grid{i}_desc"] = np.array([*g.lo, *g.hi, g.n_intervals, g.points_per_interval],
                                        dtype=float)

    # -- point interp + spread + gather, 1-D and 2-D, p in {2, 3, 4}
    rng = np.random.default_rng(100)
    for dims in (1, 2):
        for p in (2, 3, 4):
            pts = blobs(3000, dims, rng, centers=6, span=12.0, std=1.0)
            g = nb.make_grid(pts, min_intervals=25, points_per_interval=p)
            it = nb._point_interp(g, pts)
            q = rng.standard_normal(pts.shape[0])
            tag = f"interp_d{dims}_p{p}"
            out[tag + "_pts"] = pts
            out[tag + "_q"] = q
            out[tag + "_desc"] = np.array([*g.lo, *g.hi, g.n_intervals, p], dtype=float)
            out[tag + "_idx"] = it.node_index
            out[tag + "_w"] = it.weights
            coeffs = nb._spread(it, q, g)
            out[tag + "_spread"] = coeffs
            for kern in nb.Kernel:
                out[tag + f"_matvec_{kern.value}"] = nb.kernel_matvec_fft(coeffs, kern, g)
            vals = rng.standard_normal(g.total_nodes)
            out[tag + "_vals"] = vals
            out[tag + "_gather"] = nb.gather_potentials(pts, vals, g)

    # -- repulsion (fft + exact), config-2-like blobs, 1-D and 2-D
    for dims in (1, 2):
        y = blobs(4000, dims, np.random.default_rng(200 + dims), centers=20, span=40.0, std=1.5)
        rep = op.compute_repulsive(y, min_intervals=50, points_per_interval=3, method="fft")
        tag = f"rep_d{dims}"
        out[tag + "_y"] = y
        out[tag + "_forces"] = rep.forces
        out[tag + "_z"] = np.array([rep.z])
        out[tag + "_k1"] = rep.k1_potential
        out[tag + "_k2"] = rep.k2_potentials
        ex = op.compute_repulsive(y[:800], method="exact")
        out[tag + "_exact_forces"] = ex.forces
        out[tag + "_exact_z"] = np.array([ex.z])
        out[tag + "_exact_k1"] = ex.k1_potential
        out[tag + "_exact_k2"] = ex.k2_potentials

    # -- attractive / gradient / KL on a sparse P
    for dims in (1, 2):
        rng = np.random.default_rng(300 + dims)
        y = blobs(3000, dims, rng, centers=10, span=20.0, std=2.0)
        P = knn_like_affinities(y, 12, rng, SA)
        tag = f"grad_d{dims}"
        out[tag + "_y"] = y
        out[tag + "_rows"], out[tag + "_cols"], out[tag + "_vals"] = P.rows, P.cols, P.values
        out[tag + "_attr"] = op.compute_attractive(P, y)
        out[tag + "_grad_a1"] = op.gradient(P, y, 1.0, 50, 3, method="fft")
        out[tag + "_grad_a12"] = op.gradient(P, y, 12.0, 50, 3, method="fft")
        out[tag + "_kl_fft"] = np.array([op.kl_divergence(P, y, method="fft")])
        out[tag + "_kl_exact"] = np.array([op.kl_divergence(P, y, method="exact")])

    # -- dense small P, exact path (test_optimizer.py style)
    rng = np.random.default_rng(400)
    P = random_affinities(60, rng, 0.4, SA)
    y = rng.standard_normal((60, 2))
    out["small_rows"], out["small_cols"], out["small_vals"] = P.rows, P.cols, P.values
    out["small_y"] = y
    out["small_grad_exact"] = op.gradient(P, y, 1.0, method="exact")
    out["small_kl_exact"] = np.array([op.kl_divergence(P, y, "exact")])

    # -- step sequence
    rng = np.random.default_rng(500)
    st = op.OptimizerState.fresh(50, 2, 200.0)
    y = rng.standard_normal((50, 2))
    out["step_y0"] = y.copy()
    grads = rng.standard_normal((6, 50, 2))
    out["step_grads"] = grads
    for k in range(6):
        y = op.step(st, y, grads[k], momentum=0.5 if k < 3 else 0.8)
    out["step_y"] = y
    out["step_vel"] = st.velocity
    out["step_gains"] = st.gains

    # -- short trajectories (n_iter >= 250 because of the reference's
    #    schedule validation, optimizer.py:54-66)
    rng = np.random.default_rng(600)
    y = blobs(300, 2, rng, centers=3, span=5.0, std=1.0)
    P = knn_like_affinities(y, 10, rng, SA)
    cfg = op.TsneConfig(dims=2, n_iter=260, learning_rate=200.0, seed=3, pca_dims=None,
                        min_intervals=20)
    res = op.run_tsne(affinities=P, config=cfg)
    out["run_exact_rows"], out["run_exact_cols"], out["run_exact_vals"] = P.rows, P.cols, P.values
    out["run_exact_embedding"] = res.embedding
    out["run_exact_kl"] = res.kl_log

    rng = np.random.default_rng(700)
    y = blobs(1500, 2, rng, centers=5, span=10.0, std=1.0)
    P = knn_like_affinities(y, 15, rng, SA)
    cfg = op.TsneConfig(dims=2, n_iter=300, learning_rate=200.0, seed=5, pca_dims=None,
                        min_intervals=50, repulsion_method="fft",
                        exaggeration=op.ExaggerationSchedule(12.0, 250))
    res = op.run_tsne(affinities=P, config=cfg)
    out["run_fft_rows"], out["run_fft_cols"], out["run_fft_vals"] = P.rows, P.cols, P.values
    out["run_fft_embedding"] = res.embedding
    out["run_fft_kl"] = res.kl_log

    np.savez_compressed(HERE / "reference_golden.npz", **out)
    total = sum(v.nbytes for v in out.values())
    print(f"wrote {len(out)} arrays ({total / 1e6:.1f} MB raw) to {HERE / 'reference_golden.npz'}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src")
