"""The reference's unit-test contract (pkg/tests/test_nbody.py,
pkg/tests/test_optimizer.py), re-expressed against the drop-in API so every
check runs through libfitsne_b200 on the GPU.  Each test names the reference
test it covers."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api(cuda):
    from paper_1712_09005_b200 import nbody, optimizer
    from paper_1712_09005_b200.affinities import SparseAffinities
    return nbody, optimizer, SparseAffinities


def _rinf(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


def _dense_pairs(n, rng, density=1.0, SA=None):
    iu = np.triu_indices(n, 1)
    v = rng.random(iu[0].size)
    if density < 1.0:
        v = v * (rng.random(v.size) < density)
    k = v > 0
    v = v[k] / (2.0 * v[k].sum())
    return SA(n=n, rows=iu[0][k], cols=iu[1][k], values=v)


def _node_coords(g):
    if g.dims == 1:
        return g.nodes(0)[:, None]
    gx, gy = np.meshgrid(g.nodes(0), g.nodes(1), indexing="ij")
    return np.column_stack([gx.ravel(), gy.ravel()])


# --------------------------------------------------------------- test_nbody.py
class TestGridRules:
    def test_floor_and_span(self, api):                    # test_nbody.py:61-70
        nb = api[0]
        assert nb.make_grid(np.linspace(0.0, 5.0, 11), min_intervals=20).n_intervals == 20
        assert nb.make_grid(np.linspace(0.0, 5.0, 11), min_intervals=20).nodes_per_dim == 60
        assert nb.make_grid(np.linspace(0.0, 100.0, 7), min_intervals=20).n_intervals == 100

    def test_degenerate_widening(self, api):               # test_nbody.py:71-76
        g = api[0].make_grid(np.full(4, 0.3), min_intervals=20)
        assert g.n_intervals == 20
        assert g.lo[0] == pytest.approx(-0.2) and g.hi[0] == pytest.approx(0.8)

    def test_empty_and_inside(self, api):                  # test_nbody.py:78-87
        nb = api[0]
        with pytest.raises(ValueError):
            nb.make_grid(np.empty((0, 2)))
        g = nb.make_grid(np.array([0.0, 4.0]), min_intervals=20)
        assert g.lo[0] < 0.0 < 4.0 < g.hi[0]

    def test_shared_interval_count_and_spacing(self, api):  # test_nbody.py:89-99
        nb = api[0]
        g = nb.make_grid(np.array([[0.0, 0.0], [40.0, 3.0]]), min_intervals=20)
        assert g.n_intervals == 40 and g.dims == 2
        g = nb.make_grid(np.array([0.0, 10.0]), min_intervals=5, points_per_interval=3)
        gaps = np.diff(g.nodes(0))
        np.testing.assert_allclose(gaps, gaps[0])

    def test_interp_grid_validation(self, api):            # test_nbody.py:315-327
        nb = api[0]
        with pytest.raises(ValueError):
            nb.InterpGrid(dims=1, lo=(1.0,), hi=(1.0,), n_intervals=5, points_per_interval=3)
        with pytest.raises(ValueError):
            nb.InterpGrid(dims=1, lo=(0.0,), hi=(1.0,), n_intervals=5, points_per_interval=1)


class TestKernelAndWeights:
    def test_kernel_values(self, api):                     # test_nbody.py:39-58
        nb = api[0]
        assert nb.kernel_eval(nb.Kernel.CAUCHY, 0.0) == 1.0
        assert nb.kernel_eval(nb.Kernel.CAUCHY_SQUARED, 1.0) == 0.25
        assert nb.kernel_eval(nb.Kernel.CAUCHY, 3.0) == 0.25
        np.testing.assert_allclose(nb.kernel_eval(nb.Kernel.CAUCHY, np.array([0.0, 1.0, 3.0])),
                                   [1.0, 0.5, 0.25])
        for kern in nb.Kernel:
            for d2 in (0.0, 1e-9, 1.0, 1e6, 1e12):
                assert 0.0 < nb.kernel_eval(kern, d2) <= 1.0

    def test_lagrange(self, api):                          # test_nbody.py:97-124
        nb = api[0]
        np.testing.assert_allclose(nb.lagrange_weights([0.0, 0.5, 1.0], 0.5), [0, 1, 0], atol=1e-15)
        np.testing.assert_allclose(nb.lagrange_weights([0.0, 0.5, 1.0], 0.25), [0.375, 0.75, -0.125])
        with pytest.raises(ValueError):
            nb.lagrange_weights([0.0, 0.0, 1.0], 0.5)
        rng = np.random.default_rng(0)
        for _ in range(50):
            nodes = np.sort(rng.uniform(-50, 50, rng.integers(2, 7)))
            if np.diff(nodes).min() < 1e-3:
                continue
            w = nb.lagrange_weights(nodes, rng.uniform(-60, 60))
            assert abs(w.sum() - 1.0) < 1e-6 * max(1.0, np.abs(w).sum())


class TestSpreadGather:
    def test_point_on_node(self, api):                     # test_nbody.py:128-134
        nb = api[0]
        g = nb.make_grid(np.array([0.0, 10.0]), min_intervals=10)
        c = nb.spread_charges([g.nodes(0)[7], 10.0], [5.0, 0.0], g)
        assert c[7] == pytest.approx(5.0)
        np.testing.assert_allclose(np.delete(c, 7), 0.0, atol=1e-12)

    def test_charge_conserved(self, api):                  # test_nbody.py:136-142
        nb = api[0]
        rng = np.random.default_rng(3)
        pts, q = rng.uniform(-4, 7, (80, 2)), rng.standard_normal(80)
        assert nb.spread_charges(pts, q, nb.make_grid(pts)).sum() == pytest.approx(q.sum())

    def test_spread_and_gather_vs_direct_loop(self, api):  # test_nbody.py:144-157, 223-236
        nb = api[0]
        rng = np.random.default_rng(4)
        pts, q = rng.uniform(0, 9, 50), rng.standard_normal(50)
        g = nb.make_grid(pts, min_intervals=9)
        nodes, p = g.nodes(0), g.points_per_interval
        width = (g.hi[0] - g.lo[0]) / g.n_intervals
        want = np.zeros(g.total_nodes)
        vals = rng.standard_normal(g.total_nodes)
        gat = np.empty(50)
        for k, (x, c) in enumerate(zip(pts, q)):
            cell = min(int((x - g.lo[0]) / width), g.n_intervals - 1)
            w = nb.lagrange_weights(nodes[cell * p:(cell + 1) * p], x)
            want[cell * p:(cell + 1) * p] += w * c
            gat[k] = w @ vals[cell * p:(cell + 1) * p]
        np.testing.assert_allclose(nb.spread_charges(pts, q, g), want, atol=1e-12)
        np.testing.assert_allclose(nb.gather_potentials(pts, vals, g), gat)

    def test_gather_on_node_constant_quadratic(self, api):  # test_nbody.py:214-221, 238-258
        nb = api[0]
        g = nb.make_grid(np.array([0.0, 10.0]), min_intervals=10)
        vals = np.random.default_rng(7).standard_normal(g.total_nodes)
        assert nb.gather_potentials([g.nodes(0)[13]], vals, g)[0] == pytest.approx(vals[13])
        rng = np.random.default_rng(8)
        pts = rng.uniform(-3, 3, (40, 2))
        g2 = nb.make_grid(pts)
        np.testing.assert_allclose(nb.gather_potentials(pts, np.full(g2.total_nodes, 2.5), g2), 2.5)
        x = np.random.default_rng(10).uniform(0.0, 12.0, 200)
        g3 = nb.make_grid(x, min_intervals=12, points_per_interval=3)
        poly = lambda t: 0.7 * t ** 2 - 3.1 * t + 0.25  # noqa: E731
        np.testing.assert_allclose(nb.gather_potentials(x, poly(g3.nodes(0)), g3), poly(x),
                                   rtol=1e-12, atol=1e-12)

    def test_outside_rejected(self, api):                  # test_nbody.py:159-162
        nb = api[0]
        with pytest.raises(ValueError, match="outside"):
            nb.spread_charges([6.0], [1.0], nb.make_grid(np.array([0.0, 5.0])))


class TestMatvec:
    def test_basis_vector_and_zero(self, api):             # test_nbody.py:166-180
        nb = api[0]
        g = nb.make_grid(np.array([0.0, 6.0]), min_intervals=6)
        e1 = np.zeros(g.total_nodes)
        e1[0] = 1.0
        col = nb.kernel_matvec_fft(e1, nb.Kernel.CAUCHY, g)
        x = g.nodes(0)
        np.testing.assert_allclose(col, nb.kernel_eval(nb.Kernel.CAUCHY, (x - x[0]) ** 2), atol=1e-13)
        g2 = nb.make_grid(np.random.default_rng(0).uniform(0, 5, (20, 2)))
        z = nb.kernel_matvec_fft(np.zeros(g2.total_nodes), nb.Kernel.CAUCHY_SQUARED, g2)
        np.testing.assert_allclose(z, 0.0, atol=1e-14)

    @pytest.mark.parametrize("dims", [1, 2])
    def test_direct_vs_dense_nodes(self, api, dims):       # test_nbody.py:190-200
        nb = api[0]
        rng = np.random.default_rng(6)
        g = nb.make_grid(rng.uniform(0, 8, (30, dims)), min_intervals=8)
        w = rng.standard_normal(g.total_nodes)
        c = _node_coords(g)
        dense = nb.kernel_eval(nb.Kernel.CAUCHY, ((c[:, None] - c[None]) ** 2).sum(-1)) @ w
        np.testing.assert_allclose(nb.kernel_matvec_direct(w, nb.Kernel.CAUCHY, g), dense, rtol=1e-12)
        np.testing.assert_allclose(nb.kernel_matvec_fft(w, nb.Kernel.CAUCHY, g), dense, rtol=1e-10,
                                   atol=1e-12 * np.abs(dense).max())

    def test_size_mismatch(self, api):                     # test_nbody.py:202-205
        nb = api[0]
        g = nb.make_grid(np.array([0.0, 5.0]))
        with pytest.raises(ValueError):
            nb.kernel_matvec_fft(np.ones(g.total_nodes + 1), nb.Kernel.CAUCHY, g)


class TestNbody:
    def test_small_hand_values(self, api):                 # test_nbody.py:262-272, 302-313
        nb = api[0]
        assert nb.evaluate_nbody([0.3], [1.0], nb.Kernel.CAUCHY, include_self=False)[0] == \
            pytest.approx(0.0, abs=1e-5)
        out = nb.evaluate_nbody([0.0, 1.0], [1.0, 1.0], nb.Kernel.CAUCHY, include_self=False)
        assert out[0] == pytest.approx(0.5, abs=1e-3) and out[1] == pytest.approx(0.5, abs=1e-3)
        assert nb.brute_force_nbody([1.5], [3.0], nb.Kernel.CAUCHY)[0] == pytest.approx(3.0)
        np.testing.assert_allclose(nb.brute_force_nbody([0.0, 1.0], [1.0, 1.0],
                                                        nb.Kernel.CAUCHY_SQUARED, include_self=False),
                                   [0.25, 0.25])
        pts = np.array([[-1.0, 0.0], [1.0, 0.0], [0.0, 1.0], [0.0, -1.0]])
        o = nb.brute_force_nbody(pts, np.ones(4), nb.Kernel.CAUCHY, include_self=False)
        assert o[0] == pytest.approx(o[1]) and o[2] == pytest.approx(o[3])

    def test_error_decreases_with_intervals(self, api):    # test_nbody.py:283-296
        nb = api[0]
        rng = np.random.default_rng(12)
        pts = rng.uniform(-10, 10, (1500, 2))
        q = np.ones(1500)
        ex = nb.brute_force_nbody(pts, q, nb.Kernel.CAUCHY, include_self=False)
        errs = [_rinf(nb.evaluate_nbody(pts, q, nb.Kernel.CAUCHY, min_intervals=m,
                                        include_self=False), ex) for m in (20, 40, 80)]
        assert errs[1] <= errs[0] * 1.25 and errs[2] <= errs[1] * 1.25 and errs[2] < errs[0]


# ------------------------------------------------------------ test_optimizer.py
class TestForcesContract:
    def test_attractive(self, api):                        # test_optimizer.py:57-79
        _, opt, SA = api
        P = SA(n=2, rows=[0], cols=[1], values=[0.5])
        np.testing.assert_allclose(opt.compute_attractive(P, np.array([[0.0], [1.0]])), [[-0.25], [0.25]])
        P0 = SA(n=3, rows=[0], cols=[1], values=[0.0])
        np.testing.assert_allclose(opt.compute_attractive(P0, np.random.default_rng(0)
                                                          .standard_normal((3, 2))), 0.0)
        rng = np.random.default_rng(1)
        Pd = _dense_pairs(100, rng, 0.3, SA)
        Y = rng.standard_normal((100, 2))
        full = np.zeros((100, 100))
        full[Pd.rows, Pd.cols] = Pd.values
        full += full.T
        d = Y[:, None] - Y[None]
        want = ((full / (1 + (d ** 2).sum(-1)))[:, :, None] * d).sum(1)
        np.testing.assert_allclose(opt.compute_attractive(Pd, Y), want, atol=1e-12)
        with pytest.raises(ValueError):
            opt.compute_attractive(P, np.zeros((3, 2)))

    def test_repulsive(self, api):                         # test_optimizer.py:82-125
        _, opt, _ = api
        rep = opt.compute_repulsive(np.array([[0.0], [1.0]]), method="exact")
        assert rep.z == pytest.approx(1.0)
        np.testing.assert_allclose(rep.forces, [[-0.25], [0.25]])
        np.testing.assert_allclose(rep.k2_potentials[0], [0.25, 0.25])
        with pytest.raises(ValueError):
            opt.compute_repulsive(np.array([[0.0, 0.0]]))
        rng = np.random.default_rng(3)
        pts = rng.uniform(-10, 10, (1500, 2))
        ex = opt.compute_repulsive(pts, method="exact")
        fine = opt.compute_repulsive(pts, min_intervals=100, method="fft")
        assert _rinf(fine.forces, ex.forces) <= 1e-3
        for dims in (1, 2):
            p2 = np.random.default_rng(2).uniform(-10, 10, (1500, dims))
            zf = opt.compute_repulsive(p2, method="fft").z
            ze = opt.compute_repulsive(p2, method="exact").z
            assert abs(zf - ze) / ze <= 1e-3
        p4 = np.random.default_rng(4).uniform(-10, 10, (1200, 2))
        ex4 = opt.compute_repulsive(p4, method="exact")
        errs = [_rinf(opt.compute_repulsive(p4, min_intervals=m, method="fft").forces, ex4.forces)
                for m in (20, 40, 80)]
        assert errs[2] < errs[1] < errs[0]

    def test_gradient(self, api):                          # test_optimizer.py:129-167
        _, opt, SA = api
        rng = np.random.default_rng(6)
        P = _dense_pairs(40, rng, 1.0, SA)
        Y = rng.standard_normal((40, 2))
        g1 = opt.gradient(P, Y, alpha=1.0, method="exact")
        g5 = opt.gradient(P, Y, alpha=5.0, method="exact")
        np.testing.assert_allclose(g5 - g1, 16.0 * opt.compute_attractive(P, Y), atol=1e-12)
        P2 = SA(n=2, rows=[0], cols=[1], values=[0.5])
        g = opt.gradient(P2, np.array([[-1.0, 0.0], [1.0, 0.0]]), method="exact")
        np.testing.assert_allclose(g[0], -g[1], atol=1e-12)
        with pytest.raises(ValueError):
            opt.gradient(P2, np.zeros((2, 2)), alpha=0.5)

    def test_gradient_matches_finite_differences(self, api):  # test_optimizer.py:143-161
        _, opt, SA = api
        rng = np.random.default_rng(7)
        n = 20
        P = _dense_pairs(n, rng, 1.0, SA)
        Y = rng.standard_normal((n, 2))
        g = opt.gradient(P, Y, alpha=1.0, method="exact")
        h = 1e-5
        fd = np.zeros_like(Y)
        for i in range(n):
            for c in range(2):
                yp, ym = Y.copy(), Y.copy()
                yp[i, c] += h
                ym[i, c] -= h
                fd[i, c] = (opt.kl_divergence(P, yp, "exact") - opt.kl_divergence(P, ym, "exact")) / (2 * h)
        mask = np.abs(fd) > 1e-10
        assert np.max(np.abs(g[mask] - fd[mask]) / np.abs(fd[mask])) <= 1e-5


class TestKlContract:
    def test_kl(self, api):                                # test_optimizer.py:171-199
        _, opt, SA = api
        P = SA(n=2, rows=[0], cols=[1], values=[0.5])
        assert opt.kl_divergence(P, np.zeros((2, 2))) == pytest.approx(0.0, abs=1e-12)
        rng = np.random.default_rng(8)
        P = _dense_pairs(30, rng, 1.0, SA)
        Y = rng.standard_normal((30, 2))
        c = opt.kl_divergence(P, Y, "exact")
        d2 = ((Y[P.rows] - Y[P.cols]) ** 2).sum(1)
        logq = -np.log1p(d2) - np.log(opt.compute_repulsive(Y, method="exact").z)
        assert c + 2.0 * (P.values * logq).sum() == pytest.approx(2.0 * (P.values * np.log(P.values)).sum(),
                                                                  rel=1e-12)
        rng = np.random.default_rng(10)
        P3 = _dense_pairs(60, rng, 1.0, SA)
        assert opt.kl_divergence(P3, rng.standard_normal((60, 2)) * 3, "exact") >= 0.0


class TestStepScheduleContract:
    def test_step_rules(self, api):                        # test_optimizer.py:203-241
        _, opt, _ = api
        st = opt.OptimizerState.fresh(3, 2)
        y = np.arange(6.0).reshape(3, 2)
        np.testing.assert_array_equal(opt.step(st, y, np.zeros((3, 2)), momentum=0.5), y)
        st = opt.OptimizerState.fresh(1, 1, learning_rate=200.0)
        assert opt.step(st, np.array([[0.0]]), np.array([[2.0]]), momentum=0.5)[0, 0] == pytest.approx(-400.0)
        st = opt.OptimizerState.fresh(1, 1, learning_rate=1.0)
        y = np.array([[0.0]])
        for k in range(4):
            y = opt.step(st, y, np.array([[1.0]]), momentum=0.0)
            assert st.gains[0, 0] == pytest.approx(1.0 + 0.2 * (k + 1))
        st = opt.OptimizerState.fresh(1, 1, learning_rate=1.0)
        y = opt.step(st, np.array([[0.0]]), np.array([[1.0]]), momentum=0.0)
        g1 = st.gains[0, 0]
        opt.step(st, y, np.array([[-1.0]]), momentum=0.0)
        assert st.gains[0, 0] == pytest.approx(g1 * 0.8)
        st = opt.OptimizerState.fresh(1, 1)
        st.gains[:] = 0.011
        st.velocity[:] = 1.0
        opt.step(st, np.zeros((1, 1)), np.ones((1, 1)), momentum=0.0)
        assert st.gains[0, 0] >= 0.01
        with pytest.raises(FloatingPointError):
            opt.step(opt.OptimizerState.fresh(1, 2), np.zeros((1, 2)), np.array([[np.nan, 0.0]]))

    def test_schedule(self, api):                          # test_optimizer.py:245-269
        _, opt, _ = api
        s = opt.ExaggerationSchedule(12.0, 250, 4.0, 750)
        assert [s.alpha(i, 1000) for i in (0, 249, 250, 749, 750, 999)] == [12, 12, 1, 1, 4, 4]
        s = opt.ExaggerationSchedule(late_coeff=12.0)
        assert s.resolved_late_from(1000) == 750
        assert s.alpha(700, 1000) == 1.0 and s.alpha(800, 1000) == 12.0
        with pytest.raises(ValueError):
            opt.ExaggerationSchedule(early_until_iter=500, late_coeff=2.0, late_from_iter=400).validate(1000)
        with pytest.raises(ValueError):
            opt.ExaggerationSchedule(early_coeff=0.5).validate(1000)


class TestRunContract:
    def test_run_guards_and_two_points(self, api):         # test_optimizer.py:287-334
        _, opt, SA = api
        P = SA(n=2, rows=[0], cols=[1], values=[0.5])
        res = opt.run_tsne(affinities=P, config=opt.TsneConfig(dims=2, n_iter=1000, seed=0))
        assert np.all(np.isfinite(res.embedding))
        assert np.linalg.norm(res.embedding[0] - res.embedding[1]) > 1e-8
        with pytest.raises(ValueError):
            opt.run_tsne(affinities=SA(n=3, rows=[0], cols=[1], values=[0.9]),
                         config=opt.TsneConfig(n_iter=300))
        with pytest.raises(ValueError):
            opt.run_tsne(data=np.zeros((2, 2)), affinities=P)
        with pytest.raises(ValueError):
            opt.run_tsne(data=np.zeros((10, 3)), config=opt.TsneConfig(dims=3))
