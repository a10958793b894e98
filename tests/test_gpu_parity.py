"""CUDA path vs the reference (golden fixtures) and the pinned oracle.

Tolerances (north star): gradient rel-L2 <= 1e-5 in fp64 mode and <= 1e-3 in
fp32 mode; box / node indices bit-exact.  Every call goes through the C-ABI
(libfitsne_b200.so) via the drop-in Python API.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import rel_inf, rel_l2
from oracle import fitsne_oracle as O

pytestmark = pytest.mark.gpu

TOL = {"float64": 1e-5, "float32": 1e-3}
DTYPES = ["float64", "float32"]


@pytest.fixture(scope="module")
def fs(cuda):
    import paper_1712_09005_b200 as pkg
    from paper_1712_09005_b200 import nbody, optimizer, affinities
    return pkg, nbody, optimizer, affinities


def _P(affinities, r, c, v):
    n = int(max(r.max(), c.max()) + 1) if r.size else 2
    return affinities.SparseAffinities(n=n, rows=r, cols=c, values=v)


def _cast(x, dtype):
    return np.asarray(x, dtype=np.float32 if dtype == "float32" else np.float64)


# ----------------------------------------------------------------------------- a1/a2
class TestGridInterp:
    @pytest.mark.parametrize("i", range(7))
    def test_make_grid_bit_exact(self, fs, golden, i):
        _, nbody, _, _ = fs
        pts = golden[f"grid{i}_pts"]
        g = nbody.make_grid(pts, min_intervals=20 if i != 4 else 5, points_per_interval=3)
        desc = np.array([*g.lo, *g.hi, g.n_intervals, g.points_per_interval], dtype=float)
        np.testing.assert_array_equal(desc, golden[f"grid{i}_desc"])

    def test_make_grid_fp32_points(self, fs):
        _, nbody, _, _ = fs
        rng = np.random.default_rng(7)
        pts = (rng.standard_normal((20000, 2)) * 30).astype(np.float32)
        g = nbody.make_grid(torch.from_numpy(pts).cuda(), 50, 3)
        o = O.grid_for(pts.astype(np.float64), 50, 3)
        assert (g.lo, g.hi, g.n_intervals) == (o.lo, o.hi, o.n_int)

    @pytest.mark.parametrize("dims", [1, 2])
    @pytest.mark.parametrize("p", [2, 3, 4])
    def test_point_interp_bit_exact(self, fs, golden, dims, p):
        _, nbody, _, _ = fs
        tag = f"interp_d{dims}_p{p}"
        pts = golden[tag + "_pts"]
        g = nbody.make_grid(pts, 25, p)
        idx, w = nbody.point_interp(pts, g)
        np.testing.assert_array_equal(idx, golden[tag + "_idx"])
        np.testing.assert_array_equal(w, golden[tag + "_w"])

    @pytest.mark.parametrize("p", [2, 3, 4])
    def test_point_interp_fp32_indices(self, fs, p):
        _, nbody, _, _ = fs
        rng = np.random.default_rng(p)
        pts = (rng.standard_normal((200000, 2)) * 25).astype(np.float32)
        g = nbody.make_grid(torch.from_numpy(pts).cuda(), 50, p)
        idx, w = nbody.point_interp(torch.from_numpy(pts).cuda(), g)
        og = O.grid_for(pts.astype(np.float64), 50, p)
        oidx, ow = O.interp(og, pts.astype(np.float64))
        np.testing.assert_array_equal(idx.cpu().numpy(), oidx)
        # weights are computed in fp64 and rounded once to fp32
        np.testing.assert_allclose(w.cpu().numpy(), ow, rtol=6e-8, atol=1e-9)

    def test_adversarial_cell_boundaries(self, fs):
        """Points exactly on / one ulp around cell edges: indices bit-exact."""
        _, nbody, _, _ = fs
        g0 = nbody.InterpGrid(dims=1, lo=(0.0,), hi=(60.0,), n_intervals=20, points_per_interval=3)
        h = 60.0 / 60
        edges = np.arange(0, 21) * 3 * h
        pts = np.concatenate([edges, np.nextafter(edges, -1), np.nextafter(edges, 100)])
        pts = np.clip(pts, 0.0, 60.0)
        idx, w = nbody.point_interp(pts, g0)
        og = O.Grid((0.0,), (60.0,), 20, 3)
        oidx, ow = O.interp(og, pts)
        np.testing.assert_array_equal(idx, oidx)
        np.testing.assert_array_equal(w, ow)


# ----------------------------------------------------------------------------- a3-a6
class TestNbodyPieces:
    @pytest.mark.parametrize("dims", [1, 2])
    @pytest.mark.parametrize("p", [2, 3, 4])
    @pytest.mark.parametrize("dtype", DTYPES)
    def test_spread_matvec_gather(self, fs, golden, dims, p, dtype):
        _, nbody, _, _ = fs
        tag = f"interp_d{dims}_p{p}"
        pts = golden[tag + "_pts"]
        g = nbody.make_grid(pts, 25, p)
        tol = 1e-12 if dtype == "float64" else 2e-5
        coeffs = nbody.spread_charges(pts, golden[tag + "_q"], g, dtype=dtype)
        assert rel_inf(coeffs, golden[tag + "_spread"]) <= tol
        for kern in nbody.Kernel:
            v = nbody.kernel_matvec_fft(golden[tag + "_spread"], kern, g, dtype=dtype)
            assert rel_inf(v, golden[tag + f"_matvec_{kern.value}"]) <= (1e-12 if dtype == "float64" else 2e-5)
        got = nbody.gather_potentials(pts, golden[tag + "_vals"], g, dtype=dtype)
        assert rel_inf(got, golden[tag + "_gather"]) <= (1e-13 if dtype == "float64" else 2e-5)

    @pytest.mark.parametrize("dims", [1, 2])
    def test_matvec_fft_vs_direct(self, fs, dims):
        _, nbody, _, _ = fs
        rng = np.random.default_rng(5)
        pts = rng.uniform(-10, 10, size=(200, dims))
        g = nbody.make_grid(pts, 20)
        w = rng.standard_normal(g.total_nodes)
        for kern in nbody.Kernel:
            a = nbody.kernel_matvec_fft(w, kern, g)
            b = nbody.kernel_matvec_direct(w, kern, g)
            assert rel_inf(a, b) <= 1e-12

    @pytest.mark.parametrize("dims", [1, 2])
    def test_evaluate_nbody_vs_brute(self, fs, dims):
        _, nbody, _, _ = fs
        rng = np.random.default_rng(11)
        pts = rng.uniform(-5, 5, size=(2000, dims))
        q = np.ones(2000)
        a = nbody.evaluate_nbody(pts, q, nbody.Kernel.CAUCHY, include_self=False)
        b = nbody.brute_force_nbody(pts, q, nbody.Kernel.CAUCHY, include_self=False)
        ref = O.nbody_fft(pts, q, O.CAUCHY, include_self=False)
        assert rel_inf(a, b) <= 1e-3
        assert rel_inf(a, ref) <= 1e-11
        assert rel_inf(b, O.nbody_exact(pts, q, O.CAUCHY, include_self=False)) <= 1e-12

    def test_multi_column_charges(self, fs):
        _, nbody, _, _ = fs
        rng = np.random.default_rng(14)
        pts = rng.uniform(-3, 3, size=(150, 2))
        qs = rng.standard_normal((150, 5))
        stacked = nbody.evaluate_nbody(pts, qs, nbody.Kernel.CAUCHY, include_self=False)
        ref = O.nbody_fft(pts, qs, O.CAUCHY, include_self=False)
        assert rel_inf(stacked, ref) <= 1e-11


# ----------------------------------------------------------------------------- a7-a10
class TestForces:
    @pytest.mark.parametrize("dims", [1, 2])
    @pytest.mark.parametrize("dtype", DTYPES)
    def test_repulsive_fft(self, fs, golden, dims, dtype):
        _, _, opt, _ = fs
        tag = f"rep_d{dims}"
        y = golden[tag + "_y"]
        rep = opt.compute_repulsive(_cast(y, dtype) if dtype == "float32" else y, 50, 3, "fft",
                                    dtype=dtype)
        ref_f = golden[tag + "_forces"]
        if dtype == "float32":
            ref_f = O.repulsion(_cast(y, dtype).astype(np.float64), 50, 3, "fft")[0]
        assert rel_l2(rep.forces, ref_f) <= TOL[dtype] * 0.1
        assert abs(rep.z - golden[tag + "_z"][0]) <= 1e-4 * golden[tag + "_z"][0]
        if dtype == "float64":
            assert rel_l2(rep.forces, golden[tag + "_forces"]) <= 1e-11
            assert abs(rep.z - golden[tag + "_z"][0]) <= 1e-12 * golden[tag + "_z"][0]
            assert rel_l2(rep.k1_potential, golden[tag + "_k1"]) <= 1e-11
            assert rel_l2(rep.k2_potentials, golden[tag + "_k2"]) <= 1e-11

    @pytest.mark.parametrize("dims", [1, 2])
    def test_repulsive_exact(self, fs, golden, dims):
        _, _, opt, _ = fs
        tag = f"rep_d{dims}"
        y = golden[tag + "_y"][:800]
        rep = opt.compute_repulsive(y, method="exact")
        assert rel_l2(rep.forces, golden[tag + "_exact_forces"]) <= 1e-12
        assert abs(rep.z - golden[tag + "_exact_z"][0]) <= 1e-12 * rep.z
        assert rel_l2(rep.k2_potentials, golden[tag + "_exact_k2"]) <= 1e-12
        auto = opt.compute_repulsive(y, method="auto")
        np.testing.assert_array_equal(auto.forces, rep.forces)

    @pytest.mark.parametrize("dims", [1, 2])
    @pytest.mark.parametrize("dtype", DTYPES)
    def test_attractive_gradient(self, fs, golden, dims, dtype):
        _, _, opt, aff = fs
        tag = f"grad_d{dims}"
        y = golden[tag + "_y"]
        P = _P(aff, golden[tag + "_rows"], golden[tag + "_cols"], golden[tag + "_vals"])
        attr = opt.compute_attractive(P, y, dtype=dtype)
        assert rel_l2(attr, golden[tag + "_attr"]) <= (1e-12 if dtype == "float64" else 1e-5)
        for a, key in ((1.0, "_grad_a1"), (12.0, "_grad_a12")):
            g = opt.gradient(P, y, a, 50, 3, "fft", dtype=dtype)
            assert rel_l2(g, golden[tag + key]) <= TOL[dtype]
            if dtype == "float64":
                assert rel_l2(g, golden[tag + key]) <= 1e-10

    @pytest.mark.parametrize("dims", [1, 2])
    def test_kl(self, fs, golden, dims):
        _, _, opt, aff = fs
        tag = f"grad_d{dims}"
        y = golden[tag + "_y"]
        P = _P(aff, golden[tag + "_rows"], golden[tag + "_cols"], golden[tag + "_vals"])
        assert opt.kl_divergence(P, y, "fft") == pytest.approx(golden[tag + "_kl_fft"][0], rel=1e-10)
        assert opt.kl_divergence(P, y, "exact") == pytest.approx(golden[tag + "_kl_exact"][0], rel=1e-10)

    def test_small_exact_gradient(self, fs, golden):
        _, _, opt, aff = fs
        P = _P(aff, golden["small_rows"], golden["small_cols"], golden["small_vals"])
        g = opt.gradient(P, golden["small_y"], 1.0, method="exact")
        assert rel_l2(g, golden["small_grad_exact"]) <= 1e-12
        assert opt.kl_divergence(P, golden["small_y"], "exact") == pytest.approx(
            golden["small_kl_exact"][0], rel=1e-12)

    def test_step_sequence(self, fs, golden):
        _, _, opt, _ = fs
        st = opt.OptimizerState.fresh(50, 2, 200.0)
        y = golden["step_y0"].copy()
        for k, g in enumerate(golden["step_grads"]):
            y = opt.step(st, y, g, momentum=0.5 if k < 3 else 0.8)
        np.testing.assert_allclose(y, golden["step_y"], rtol=1e-14, atol=1e-12)
        np.testing.assert_allclose(st.velocity, golden["step_vel"], rtol=1e-14, atol=1e-12)
        np.testing.assert_allclose(st.gains, golden["step_gains"], rtol=1e-15)
        assert st.iteration == 6


# ----------------------------------------------------------------------------- a13
class TestRuns:
    def test_fft_run_fp64(self, fs, golden):
        _, _, opt, aff = fs
        P = _P(aff, golden["run_fft_rows"], golden["run_fft_cols"], golden["run_fft_vals"])
        cfg = opt.TsneConfig(dims=2, n_iter=300, learning_rate=200.0, seed=5, pca_dims=None,
                             min_intervals=50, repulsion_method="fft",
                             exaggeration=opt.ExaggerationSchedule(12.0, 250))
        res = opt.run_tsne(affinities=P, config=cfg)
        ref = golden["run_fft_kl"]
        assert rel_l2(res.kl_log[:20], ref[:20]) <= 1e-9
        assert abs(res.kl_log[-1] - ref[-1]) <= 0.01 * ref[-1]

    def test_fft_run_fp32(self, fs, golden):
        _, _, opt, aff = fs
        P = _P(aff, golden["run_fft_rows"], golden["run_fft_cols"], golden["run_fft_vals"])
        cfg = opt.TsneConfig(dims=2, n_iter=300, learning_rate=200.0, seed=5, pca_dims=None,
                             min_intervals=50, repulsion_method="fft", dtype="float32",
                             exaggeration=opt.ExaggerationSchedule(12.0, 250))
        res = opt.run_tsne(affinities=P, config=cfg)
        ref = golden["run_fft_kl"]
        assert rel_l2(res.kl_log[:5], ref[:5]) <= 1e-4
        assert abs(res.kl_log[-1] - ref[-1]) <= 0.02 * ref[-1]


# ----------------------------------------------------------------------------- large
class TestLargeProperties:
    def test_c2_fp32_vs_oracle(self, fs):
        """Config 2: N=100k blobs, fp32 repulsion vs the fp64 oracle (<= 1e-3)."""
        _, _, opt, _ = fs
        rng = np.random.default_rng(2)
        c = rng.uniform(-40, 40, (20, 2))
        sizes = rng.multinomial(100_000, rng.dirichlet(np.ones(20)))
        y = np.concatenate([c[i] + 1.5 * rng.standard_normal((s, 2)) for i, s in enumerate(sizes)])
        y32 = y.astype(np.float32)
        rep = opt.compute_repulsive(torch.from_numpy(y32).cuda(), 50, 3, "fft")
        f, z, _, _ = O.repulsion(y32.astype(np.float64), 50, 3, "fft")
        assert rel_l2(rep.forces.cpu().numpy(), f) <= 1e-3
        assert abs(rep.z - z) <= 1e-4 * z

    def test_c2_interpolation_error_vs_exact(self, fs):
        """Config 2 against the exact O(N^2) sums (the device k_exact kernel in
        fp64 as the accuracy oracle): the fp32 FFT path's interpolation error
        must not exceed the reference algorithm's own (oracle fp64 FFT vs the
        same exact sums) by more than 10%."""
        _, _, opt, _ = fs
        rng = np.random.default_rng(2)
        c = rng.uniform(-40, 40, (20, 2))
        sizes = rng.multinomial(100_000, rng.dirichlet(np.ones(20)))
        y = np.concatenate([c[i] + 1.5 * rng.standard_normal((s, 2)) for i, s in enumerate(sizes)])
        y = y.astype(np.float32).astype(np.float64)
        exact = opt.compute_repulsive(torch.from_numpy(y).cuda(), method="exact")
        fe = exact.forces.cpu().numpy()
        ours = opt.compute_repulsive(torch.from_numpy(y.astype(np.float32)).cuda(), 50, 3, "fft")
        f_ref, z_ref, _, _ = O.repulsion(y, 50, 3, "fft")
        err_ours = rel_l2(ours.forces.cpu().numpy(), fe)
        err_ref = rel_l2(f_ref, fe)
        assert 1e-3 < err_ref < 5e-2  # the interpolation error the reference itself makes
        assert err_ours <= 1.1 * err_ref, (err_ours, err_ref)
        assert abs(ours.z - exact.z) <= 1e-3 * exact.z

    def test_translation_invariance(self, fs):
        _, nbody, _, _ = fs
        rng = np.random.default_rng(13)
        pts = rng.uniform(-4, 4, size=(300, 2))
        q = rng.uniform(0.5, 1.5, 300)
        base = nbody.evaluate_nbody(pts, q, nbody.Kernel.CAUCHY_SQUARED, include_self=False)
        shifted = nbody.evaluate_nbody(pts + 137.25, q, nbody.Kernel.CAUCHY_SQUARED, include_self=False)
        assert rel_inf(shifted, base) <= 1e-6

    def test_iteration_zero_contention(self, fs):
        """Y0 ~ N(0, 1e-4): every point in 4 boxes (worst spread contention)."""
        _, _, opt, _ = fs
        rng = np.random.default_rng(0)
        y = rng.normal(0, 1e-4, (200_000, 2))
        rep = opt.compute_repulsive(torch.from_numpy(y.astype(np.float32)).cuda(), 50, 3, "fft")
        f, z, _, _ = O.repulsion(y.astype(np.float32).astype(np.float64), 50, 3, "fft")
        assert rel_l2(rep.forces.cpu().numpy(), f) <= 1e-3
        assert abs(rep.z - z) <= 1e-4 * z

    @pytest.mark.parametrize("dtype,span,tol", [
        ("float32", 200.0, 1e-3),   # fp32 grid pipeline
        ("float32", 430.0, 1e-3),   # fp64 grid pipeline of an fp32 context (span > 256)
        ("float32", 860.0, 1e-3),   # longest one-block fp32 transform (L = 5184)
        ("float64", 428.0, 1e-5),   # longest one-block fp64 transform (L = 2592)
        ("float64", 860.0, 1e-5),   # fp64 four-step FFT (L = 5184)
        ("float32", 2000.0, 1e-3),  # four-step FFT, L = 12288
        ("float64", 2000.0, 1e-5),
    ])
    def test_wide_grids(self, fs, dtype, span, tol):
        """Wide embeddings (late t-SNE layouts) against the reference's
        algorithm at any span (nbody.py:134, 267, 276 size every grid with
        next_fast_len).  In fp32 the repulsive force F = y_i K2*1 - K2*y
        cancels |y|-sized terms, so past span 256 an fp32 context runs its
        grid pipeline in fp64 (FITSNE_OPT_GRID_F64) and keeps the 1e-3 bar;
        transforms longer than one block's shared memory take the four-step
        path.  Z stays accurate throughout."""
        _, _, opt, _ = fs
        rng = np.random.default_rng(21)
        # 40 blobs spread over [0, span]^2 (a late-iteration t-SNE layout)
        c = rng.uniform(0, span, (40, 2))
        c[:2] = [[0.0, 0.0], [span, span]]
        y = c[rng.integers(0, 40, 20_000)] + 3.0 * rng.standard_normal((20_000, 2))
        y = np.clip(y, 0.0, span).astype(np.float32 if dtype == "float32" else np.float64)
        rep = opt.compute_repulsive(torch.from_numpy(y).cuda(), 50, 3, "fft")
        f, z, _, _ = O.repulsion(y.astype(np.float64), 50, 3, "fft")
        err = rel_l2(rep.forces.cpu().numpy(), f)
        assert err <= tol, err
        assert abs(rep.z - z) <= 1e-5 * z

    @pytest.mark.parametrize("span", [600.0, 2000.0])
    def test_wide_gradient_fp32(self, fs, span):
        """fp32 gradient through both entry points (device buffers: the
        overlapped schedule's combine reads the fp64 grid's F_rep; host
        buffers: fitsne_gradient_host) at wide spans, and the fused iteration
        (fitsne_iterate) against the oracle's update."""
        _, _, opt, aff = fs
        rng = np.random.default_rng(int(span))
        n = 20_000
        c = rng.uniform(0, span, (40, 2))
        y = (c[rng.integers(0, 40, n)] + 3.0 * rng.standard_normal((n, 2))).astype(np.float32)
        r = np.repeat(np.arange(n), 8)
        cc = rng.integers(0, n - 1, n * 8)
        cc = cc + (cc >= r)
        key = np.unique(np.minimum(r, cc) * n + np.maximum(r, cc))
        v = rng.exponential(1.0, key.size)
        P = aff.SparseAffinities(n=n, rows=key // n, cols=key % n, values=v / (2 * v.sum()))
        y64 = y.astype(np.float64)
        ref = O.grad(P.rows, P.cols, P.values, y64, 4.0, 50, 3, "fft")
        g_dev = opt.gradient(P, torch.from_numpy(y).cuda(), 4.0, 50, 3, "fft").double().cpu().numpy()
        g_host = opt.gradient(P, y, 4.0, 50, 3, "fft")
        assert rel_l2(g_dev, ref) <= 1e-3 and rel_l2(g_host, ref) <= 1e-3

    def test_grid_too_large(self, fs):
        """Only a grid whose FFT exceeds the four-step path's 65535 points is
        refused (span > ~10900 at p = 3)."""
        _, _, opt, _ = fs
        y = np.array([[0.0, 0.0], [12000.0, 1.0], [5.0, 7.0]])
        with pytest.raises(ValueError, match="FFT"):
            opt.compute_repulsive(y, 50, 3, "fft")

    @pytest.mark.parametrize("dtype", DTYPES)
    @pytest.mark.parametrize("dims", [1, 2])
    def test_four_step_path_matches_one_block_path(self, fs, dtype, dims):
        """The four-step FFT (forced at a length the one-block kernels also
        handle) gives the same repulsion, Z and nbody matvec as the one-block
        kernels and the oracle."""
        from paper_1712_09005_b200 import _lib, nbody
        _, _, opt, _ = fs
        rng = np.random.default_rng(dims)
        y = (rng.standard_normal((30_000, dims)) * 40).astype(np.float32 if dtype == "float32" else np.float64)
        yd = torch.from_numpy(y).cuda()
        f_o, z_o, _, _ = O.repulsion(y.astype(np.float64), 50, 3, "fft")
        out = {}
        q = torch.from_numpy(rng.standard_normal(y.shape[0])).to(yd)
        for path in (1, 2):
            with _lib.option(_lib.OPT_FFT_PATH, path):
                rep = opt.compute_repulsive(yd, 50, 3, "fft")
                out[path] = (rep.forces.double().cpu().numpy(), rep.z,
                             nbody.evaluate_nbody(yd, q, "cauchy", 50, 3).double().cpu().numpy(), q)
        tol = TOL[dtype]
        assert rel_l2(out[2][0], f_o) <= tol and rel_l2(out[2][0], out[1][0]) <= tol
        assert abs(out[2][1] - z_o) <= 1e-5 * z_o
        nb_o = O.nbody_fft(y.astype(np.float64), out[2][3].double().cpu().numpy(), O.CAUCHY, 50, 3)
        assert rel_l2(out[2][2], nb_o) <= (1e-4 if dtype == "float32" else 1e-10)


# ----------------------------------------------------------------------------- errors
class TestErrors:
    def test_nonfinite_points(self, fs):
        _, nbody, _, _ = fs
        with pytest.raises(ValueError):
            nbody.make_grid(np.array([[0.0, np.nan], [1.0, 2.0]]))

    def test_outside_grid(self, fs):
        _, nbody, _, _ = fs
        g = nbody.make_grid(np.array([0.0, 5.0]))
        with pytest.raises(ValueError, match="outside"):
            nbody.spread_charges([6.0], [1.0], g)

    def test_alpha_and_shapes(self, fs):
        _, _, opt, aff = fs
        P = aff.SparseAffinities(n=2, rows=[0], cols=[1], values=[0.5])
        with pytest.raises(ValueError):
            opt.gradient(P, np.zeros((2, 2)), alpha=0.5)
        with pytest.raises(ValueError):
            opt.compute_attractive(P, np.zeros((3, 2)))
        with pytest.raises(ValueError):
            opt.compute_repulsive(np.array([[0.0, 0.0]]))

    def test_nonfinite_gradient_step(self, fs):
        _, _, opt, _ = fs
        state = opt.OptimizerState.fresh(1, 2)
        with pytest.raises(FloatingPointError):
            opt.step(state, np.zeros((1, 2)), np.array([[np.nan, 0.0]]))
        assert state.iteration == 0


class TestDeviceGrid:
    """The device-grid schedule (grid computed by k_bbox, stages queued before
    the host sees it) against the host-grid schedule and the oracle, across
    calls whose span grows past the launch capacity (host fallback) and
    shrinks, for the gradient (device and host buffers) and the fused step."""

    def _P(self, n, rng):
        from paper_1712_09005_b200.affinities import SparseAffinities
        r = np.repeat(np.arange(n), 10)
        cc = rng.integers(0, n - 1, n * 10)
        cc = cc + (cc >= r)
        key = np.unique(np.minimum(r, cc) * n + np.maximum(r, cc))
        v = rng.exponential(1.0, key.size)
        return SparseAffinities(n=n, rows=key // n, cols=key % n, values=v / (2 * v.sum()))

    def test_growing_and_shrinking_spans(self, fs):
        from paper_1712_09005_b200 import _lib
        _, _, opt, _ = fs
        rng = np.random.default_rng(31)
        n = 30_000
        P = self._P(n, rng)
        base = rng.standard_normal((n, 2))
        with _lib.option(_lib.OPT_DEVICE_GRID, 1):
            for scale in (20.0, 22.0, 40.0, 41.0, 80.0, 30.0, 10.0, 0.05, 60.0, 140.0):
                y = (base * scale).astype(np.float32)
                ref = O.grad(P.rows, P.cols, P.values, y.astype(np.float64), 4.0, 50, 3, "fft")
                g_dev = opt.gradient(P, torch.from_numpy(y).cuda(), 4.0, 50, 3, "fft").double().cpu().numpy()
                g_host = opt.gradient(P, y, 4.0, 50, 3, "fft")
                assert rel_l2(g_dev, ref) <= 1e-3, scale
                assert rel_l2(g_host, ref) <= 1e-3, scale
        with _lib.option(_lib.OPT_DEVICE_GRID, 0):
            g0 = opt.gradient(P, torch.from_numpy(y).cuda(), 4.0, 50, 3, "fft").double().cpu().numpy()
        assert rel_l2(g_dev, g0) <= 1e-5

    def test_fused_run_matches_host_grid_schedule(self, fs):
        from paper_1712_09005_b200 import _lib
        _, _, opt, _ = fs
        rng = np.random.default_rng(32)
        P = self._P(20_000, rng)
        cfg = opt.TsneConfig(dims=2, n_iter=300, learning_rate=2000.0, min_intervals=50,
                             exaggeration=opt.ExaggerationSchedule(12.0, 100), seed=0, pca_dims=None,
                             repulsion_method="fft", dtype="float32")
        with _lib.option(_lib.OPT_DEVICE_GRID, 1):
            a = opt.run_tsne(affinities=P, config=cfg)
        with _lib.option(_lib.OPT_DEVICE_GRID, 0):
            b = opt.run_tsne(affinities=P, config=cfg)
        # same schedule of the same math: identical up to float atomics order
        assert np.max(np.abs(a.kl_log[:20] - b.kl_log[:20]) / b.kl_log[:20]) <= 1e-5
        assert abs(a.kl_log[-1] - b.kl_log[-1]) / b.kl_log[-1] <= 2e-2
