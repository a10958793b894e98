"""P wire format: SparseAffinities <-> full CSR <-> .npz."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1712_09005_b200.affinities import (FORMAT_VERSION, SparseAffinities, from_csr,
                                              load_affinities, save_affinities, to_csr)


def _P(n=300, k=12, seed=0):
    rng = np.random.default_rng(seed)
    r = np.repeat(np.arange(n), k)
    c = rng.integers(0, n, n * k)
    keep = r != c
    key = np.unique(np.minimum(r[keep], c[keep]) * n + np.maximum(r[keep], c[keep]))
    v = rng.random(key.size)
    return SparseAffinities(n=n, rows=key // n, cols=key % n, values=v / (2 * v.sum()))


def test_csr_round_trip():
    P = _P()
    n, rowptr, col, val = to_csr(P)
    assert rowptr[-1] == 2 * P.rows.size and col.dtype == np.int32
    for i in (0, 17, n - 1):  # ascending columns inside every row
        assert np.all(np.diff(col[rowptr[i]:rowptr[i + 1]]) > 0)
    Q = from_csr(n, rowptr, col, val)
    o = np.lexsort((P.cols, P.rows))
    np.testing.assert_array_equal(Q.rows, P.rows[o])
    np.testing.assert_array_equal(Q.cols, P.cols[o])
    np.testing.assert_array_equal(Q.values, P.values[o])


def test_scipy_input_matches():
    sp = pytest.importorskip("scipy.sparse")
    P = _P(seed=1)
    M = sp.coo_matrix((np.r_[P.values, P.values], (np.r_[P.rows, P.cols], np.r_[P.cols, P.rows])),
                      shape=(P.n, P.n)).tocsr()
    a, b = to_csr(P), to_csr(M)
    for x, y in zip(a[1:], b[1:]):
        np.testing.assert_array_equal(x, y)


def test_file_round_trip(tmp_path):
    P = _P(seed=2)
    y0 = np.random.default_rng(3).standard_normal((P.n, 2)) * 1e-4
    f = tmp_path / "p.npz"
    save_affinities(f, P, y0)
    Q, y = load_affinities(f)
    np.testing.assert_array_equal(y, y0)
    assert Q.n == P.n and Q.ordered_total == pytest.approx(P.ordered_total, rel=1e-15)
    np.testing.assert_array_equal(to_csr(Q)[2], to_csr(P)[2])


def test_rejects_bad_files_and_asymmetry(tmp_path):
    P = _P(seed=4)
    n, rowptr, col, val = to_csr(P)
    bad = val.copy()
    bad[0] *= 2
    with pytest.raises(ValueError, match="symmetric"):
        from_csr(n, rowptr, col, bad)
    f = tmp_path / "v.npz"
    np.savez(f, format=np.array("fitsne-b200-csr"), version=np.array(FORMAT_VERSION + 1), n=n,
             rowptr=rowptr, col=col, val=val)
    with pytest.raises(ValueError, match="version"):
        load_affinities(f)
    g = tmp_path / "o.npz"
    np.savez(g, a=np.zeros(3))
    with pytest.raises(ValueError, match="not a"):
        load_affinities(g)


def test_ordered_total_is_cached_with_the_contents():
    """ordered_total sums every stored value once per contents of P: a second
    call reuses it, an in-place rescaling of the values is seen."""
    import numpy as np
    from paper_1712_09005_b200.affinities import SparseAffinities, ordered_total
    rng = np.random.default_rng(0)
    n = 500
    key = np.unique(rng.integers(0, n * n, 4000))
    r, c = key // n, key % n
    keep = r < c
    r, c = r[keep], c[keep]
    v = rng.random(r.size)
    v /= 2 * v.sum()
    P = SparseAffinities(n=n, rows=r, cols=c, values=v)
    assert abs(ordered_total(P) - 1.0) < 1e-12
    assert any(k[0] == "ordered_total" for k in P.__dict__["_fitsne_csr"] if isinstance(k, tuple))
    assert abs(ordered_total(P) - 1.0) < 1e-12          # cached
    P.values *= 2.0                                     # in-place edit: the sampled checksum changes
    assert abs(ordered_total(P) - 2.0) < 1e-12
