"""Pin the CPU oracle (oracle/fitsne_oracle.py) to the reference.

Every fixture in tests/golden/reference_golden.npz was produced by running the
reference package itself (tests/golden/make_golden.py).  The oracle must
reproduce it: bit-exact for grids, node indices and weights, and to rounding
(<= 1e-12) for the floating-point pipeline.  The closed-form known answers of
the reference tests (test_nbody.py, test_optimizer.py) are checked too.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import rel_inf, rel_l2
from oracle import fitsne_oracle as O


def _grid(desc, dims):
    lo = tuple(desc[:dims])
    hi = tuple(desc[dims:2 * dims])
    return O.Grid(lo, hi, int(desc[2 * dims]), int(desc[2 * dims + 1]))


class TestGridAndInterp:
    def test_grids_bit_exact(self, golden):
        for i in range(7):
            pts = golden[f"grid{i}_pts"]
            g = O.grid_for(pts, 20 if i != 4 else 5, 3)
            desc = np.array([*g.lo, *g.hi, g.n_int, g.p], dtype=float)
            np.testing.assert_array_equal(desc, golden[f"grid{i}_desc"])

    @pytest.mark.parametrize("dims", [1, 2])
    @pytest.mark.parametrize("p", [2, 3, 4])
    def test_interp_bit_exact(self, golden, dims, p):
        tag = f"interp_d{dims}_p{p}"
        pts = golden[tag + "_pts"]
        g = O.grid_for(pts, 25, p)
        np.testing.assert_array_equal(np.array([*g.lo, *g.hi, g.n_int, p], float), golden[tag + "_desc"])
        idx, w = O.interp(g, pts)
        np.testing.assert_array_equal(idx, golden[tag + "_idx"])
        np.testing.assert_array_equal(w, golden[tag + "_w"])

    @pytest.mark.parametrize("dims", [1, 2])
    @pytest.mark.parametrize("p", [2, 3, 4])
    def test_spread_matvec_gather(self, golden, dims, p):
        tag = f"interp_d{dims}_p{p}"
        pts = golden[tag + "_pts"]
        g = O.grid_for(pts, 25, p)
        idx, w = O.interp(g, pts)
        coeffs = O.spread(idx, w, golden[tag + "_q"], g)
        np.testing.assert_array_equal(coeffs, golden[tag + "_spread"])
        for kind in (O.CAUCHY, O.CAUCHY_SQUARED):
            spec, L = O.spectrum(kind, g)
            v = O.toeplitz_apply(coeffs, spec, L, g)
            assert rel_inf(v, golden[tag + f"_matvec_{kind}"]) <= 1e-13
        got = O.gather(idx, w, golden[tag + "_vals"])
        assert rel_inf(got, golden[tag + "_gather"]) <= 1e-14


class TestRepulsionAttraction:
    @pytest.mark.parametrize("dims", [1, 2])
    def test_fft_repulsion(self, golden, dims):
        tag = f"rep_d{dims}"
        y = golden[tag + "_y"]
        f, z, k1, k2 = O.repulsion(y, 50, 3, "fft")
        assert rel_l2(f, golden[tag + "_forces"]) <= 1e-12
        assert abs(z - golden[tag + "_z"][0]) <= 1e-12 * z
        assert rel_l2(k1, golden[tag + "_k1"]) <= 1e-12
        assert rel_l2(k2, golden[tag + "_k2"]) <= 1e-12

    @pytest.mark.parametrize("dims", [1, 2])
    def test_exact_repulsion(self, golden, dims):
        tag = f"rep_d{dims}"
        y = golden[tag + "_y"][:800]
        f, z, k1, k2 = O.repulsion(y, method="exact")
        assert rel_l2(f, golden[tag + "_exact_forces"]) <= 1e-12
        assert abs(z - golden[tag + "_exact_z"][0]) <= 1e-12 * z
        assert rel_l2(k2, golden[tag + "_exact_k2"]) <= 1e-12

    @pytest.mark.parametrize("dims", [1, 2])
    def test_attraction_gradient_kl(self, golden, dims):
        tag = f"grad_d{dims}"
        y = golden[tag + "_y"]
        r, c, v = golden[tag + "_rows"], golden[tag + "_cols"], golden[tag + "_vals"]
        assert rel_l2(O.attraction(r, c, v, y), golden[tag + "_attr"]) <= 1e-13
        assert rel_l2(O.grad(r, c, v, y, 1.0, 50, 3, "fft"), golden[tag + "_grad_a1"]) <= 1e-12
        assert rel_l2(O.grad(r, c, v, y, 12.0, 50, 3, "fft"), golden[tag + "_grad_a12"]) <= 1e-12
        _, z, _, _ = O.repulsion(y, 20, 3, "fft")
        kl = O.kl_given_z(r, c, v, y, z)
        assert kl == pytest.approx(golden[tag + "_kl_fft"][0], rel=1e-12)

    def test_small_exact(self, golden):
        r, c, v, y = golden["small_rows"], golden["small_cols"], golden["small_vals"], golden["small_y"]
        assert rel_l2(O.grad(r, c, v, y, 1.0, method="exact"), golden["small_grad_exact"]) <= 1e-12
        _, z, _, _ = O.repulsion(y, method="exact")
        assert O.kl_given_z(r, c, v, y, z) == pytest.approx(golden["small_kl_exact"][0], rel=1e-12)

    def test_step_sequence(self, golden):
        y = golden["step_y0"].copy()
        vel = np.zeros_like(y)
        gains = np.ones_like(y)
        for k, g in enumerate(golden["step_grads"]):
            y, vel, gains = O.update(y, g, vel, gains, 200.0, 0.5 if k < 3 else 0.8)
        np.testing.assert_array_equal(y, golden["step_y"])
        np.testing.assert_array_equal(vel, golden["step_vel"])
        np.testing.assert_array_equal(gains, golden["step_gains"])


class TestTrajectories:
    def test_exact_run(self, golden):
        r, c, v = golden["run_exact_rows"], golden["run_exact_cols"], golden["run_exact_vals"]
        n = int(max(r.max(), c.max()) + 1)
        y, kl = O.tsne(r, c, v, n, dims=2, n_iter=260, seed=3, min_intervals=20)
        # The reference's numba fastmath loop and numpy differ in the last bits.
        # Over an exaggerated descent that noise grows chaotically: perturbing
        # Y0 by 1e-13 moves the final KL at N=300 by ~2.5% (measured), so the
        # pointwise check stops after the first iterations and the final KL is
        # compared statistically.
        assert rel_l2(kl[:10], golden["run_exact_kl"][:10]) <= 1e-10
        assert abs(kl[-1] - golden["run_exact_kl"][-1]) <= 0.05 * golden["run_exact_kl"][-1]

    def test_fft_run(self, golden):
        r, c, v = golden["run_fft_rows"], golden["run_fft_cols"], golden["run_fft_vals"]
        n = int(max(r.max(), c.max()) + 1)
        y, kl = O.tsne(r, c, v, n, dims=2, n_iter=300, seed=5, min_intervals=50, method="fft")
        assert rel_l2(kl, golden["run_fft_kl"]) <= 1e-10
        assert rel_l2(y, golden["run_fft_embedding"]) <= 1e-8


class TestKnownAnswers:
    """Closed-form values from the reference tests."""

    def test_kernel_values(self):  # test_nbody.py:39-46
        assert O.cauchy(O.CAUCHY, 0.0) == 1.0
        assert O.cauchy(O.CAUCHY_SQUARED, 1.0) == 0.25
        assert O.cauchy(O.CAUCHY, 3.0) == 0.25

    def test_quarter_point_weights(self):  # test_nbody.py:102-106
        g = O.Grid((0.0,), (1.0,), 1, 3)   # nodes at 1/6, 1/2, 5/6
        x = np.array([[1.0 / 6.0 + 0.25 * (1.0 / 3.0) * 2.0]])  # u = 0.5 -> standard check below
        idx, w = O.interp(g, x)
        assert idx.tolist() == [[0, 1, 2]]
        np.testing.assert_allclose(w.sum(), 1.0)
        u = np.array([0.5])
        np.testing.assert_allclose(O._basis_values(u, 3)[0], [0.375, 0.75, -0.125])

    def test_two_point_attraction(self):  # test_optimizer.py:57-60
        f = O.attraction(np.array([0]), np.array([1]), np.array([0.5]), np.array([[0.0], [1.0]]))
        np.testing.assert_allclose(f, [[-0.25], [0.25]])

    def test_two_point_repulsion(self):  # test_optimizer.py:82-86
        f, z, k1, k2 = O.repulsion(np.array([[0.0], [1.0]]), method="exact")
        assert z == pytest.approx(1.0)
        np.testing.assert_allclose(f, [[-0.25], [0.25]])
        np.testing.assert_allclose(k2[0], [0.25, 0.25])

    def test_step_minus_400(self):  # test_optimizer.py:209-212
        y, v, g = O.update(np.array([[0.0]]), np.array([[2.0]]), np.zeros((1, 1)), np.ones((1, 1)), 200.0, 0.5)
        assert y[0, 0] == -400.0

    def test_schedule_phases(self):  # test_optimizer.py:245-253
        a = lambda it: O.alpha_at(it, 1000, 12.0, 250, 4.0, 750)
        assert [a(0), a(249), a(250), a(749), a(750), a(999)] == [12.0, 12.0, 1.0, 1.0, 4.0, 4.0]

    def test_csr_roundtrip(self):
        rng = np.random.default_rng(0)
        iu = np.triu_indices(30, 1)
        keep = rng.random(iu[0].size) < 0.3
        r, c = iu[0][keep], iu[1][keep]
        v = rng.random(r.size)
        rowptr, col, val = O.upper_to_csr(30, r, c, v)
        dense = np.zeros((30, 30))
        for i in range(30):
            dense[i, col[rowptr[i]:rowptr[i + 1]]] = val[rowptr[i]:rowptr[i + 1]]
        ref = np.zeros((30, 30))
        ref[r, c] = v
        ref += ref.T
        np.testing.assert_array_equal(dense, ref)
