"""Affinity input type and its device CSR form.

``SparseAffinities`` mirrors the reference type (affinities.py:78-104): the
symmetric P stored once per unordered pair (rows < cols, int64) with float64
values whose ordered-pair total is 2 * sum(values) = 1.  The gradient kernels
read P as the FULL symmetric CSR (both triangles, int64 row pointers, int32
column indices, values in the compute dtype), built once on the device and
cached on the P object -- the "P-matrix CSR input" of the north star.

Any object with ``n``, ``rows``, ``cols``, ``values`` (e.g. the reference's
own SparseAffinities) and a symmetric ``scipy.sparse`` matrix (full, both
triangles) are accepted too.

The data -> affinities pipeline (kNN, perplexity calibration, symmetrize) of
the reference is outside this path (P is precomputed and held fixed).
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass

import numpy as np
import torch

__all__ = ["SparseAffinities", "DeviceCSR", "device_csr", "csr_from_full", "to_csr", "from_csr",
           "save_affinities", "load_affinities", "FORMAT", "FORMAT_VERSION"]

# on-disk format of P: a versioned .npz holding the full
# symmetric CSR (both triangles) so the oracle and the GPU box read the same P
FORMAT = "fitsne-b200-csr"
FORMAT_VERSION = 1


@dataclass
class SparseAffinities:
    n: int
    rows: np.ndarray
    cols: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.rows = np.asarray(self.rows, dtype=np.int64)
        self.cols = np.asarray(self.cols, dtype=np.int64)
        self.values = np.asarray(self.values, dtype=float)
        if not (self.rows.shape == self.cols.shape == self.values.shape):
            raise ValueError("rows, cols, values must share a shape")
        if np.any(self.rows >= self.cols):
            raise ValueError("entries must be stored with row < col")
        if np.any(self.values < 0):
            raise ValueError("affinities must be nonnegative")

    @property
    def ordered_total(self) -> float:
        return 2.0 * float(self.values.sum())


@dataclass
class DeviceCSR:
    """Rows [row_begin, row_begin + n_rows) of the full symmetric P."""

    rowptr: torch.Tensor   # (n_rows+1,) int64, rowptr[0] == 0
    col: torch.Tensor      # (nnz,) int32 global column indices
    val: torch.Tensor      # (nnz,) compute dtype
    row_begin: int
    n_total: int
    ordered_total: float   # sum of all stored values (both triangles)

    @property
    def n_rows(self) -> int:
        return self.rowptr.numel() - 1

    def as_tuple(self):
        return (self.rowptr, self.col, self.val, self.row_begin, self.n_total)


def _coo_full(P, device):
    """(rows, cols, vals) of the full symmetric matrix on the device."""
    if hasattr(P, "rows") and hasattr(P, "cols") and hasattr(P, "values"):
        n = int(P.n)
        if isinstance(P.rows, torch.Tensor):
            # device-resident upper COO (e.g. a P built on the GPU, too large
            # to round-trip through host memory)
            r = P.rows.to(device=device, dtype=torch.int64)
            c = P.cols.to(device=device, dtype=torch.int64)
            v = P.values.to(device=device, dtype=torch.float64)
            return n, torch.cat([r, c]), torch.cat([c, r]), torch.cat([v, v])
        r = torch.as_tensor(np.asarray(P.rows, dtype=np.int64)).to(device)
        c = torch.as_tensor(np.asarray(P.cols, dtype=np.int64)).to(device)
        v = torch.as_tensor(np.asarray(P.values, dtype=np.float64)).to(device)
        return n, torch.cat([r, c]), torch.cat([c, r]), torch.cat([v, v])
    try:
        import scipy.sparse as sp
    except ImportError:  # pragma: no cover
        sp = None
    if sp is not None and sp.issparse(P):
        coo = P.tocoo()
        if coo.shape[0] != coo.shape[1]:
            raise ValueError("affinity matrix must be square")
        n = coo.shape[0]
        return (n, torch.as_tensor(coo.row.astype(np.int64)).to(device),
                torch.as_tensor(coo.col.astype(np.int64)).to(device),
                torch.as_tensor(coo.data.astype(np.float64)).to(device))
    raise TypeError("affinities must be a SparseAffinities-like object or a scipy.sparse matrix")


def csr_from_full(n, r, c, v, dtype, row_begin=0, row_end=None) -> DeviceCSR:
    """Sort device COO (full matrix) into CSR rows [row_begin, row_end)."""
    if row_end is None:
        row_end = n
    total = float(v.sum().item()) if v.numel() else 0.0
    if row_begin != 0 or row_end != n:
        keep = (r >= row_begin) & (r < row_end)
        r, c, v = r[keep], c[keep], v[keep]
    order = torch.argsort(r * n + c)
    r, c, v = r[order], c[order], v[order]
    counts = torch.bincount(r - row_begin, minlength=row_end - row_begin)
    rowptr = torch.zeros(row_end - row_begin + 1, dtype=torch.int64, device=r.device)
    torch.cumsum(counts, 0, out=rowptr[1:])
    return DeviceCSR(rowptr.contiguous(), c.to(torch.int32).contiguous(), v.to(dtype).contiguous(),
                     int(row_begin), int(n), total)


_side_cache: dict = {}


def _cache_slot(P):
    try:
        d = P.__dict__
        return d.setdefault("_fitsne_csr", {})
    except AttributeError:
        key = id(P)
        slot = _side_cache.get(key)
        if slot is None:
            slot = {}
            _side_cache[key] = slot
            try:
                weakref.finalize(P, _side_cache.pop, key, None)
            except TypeError:
                pass
        return slot


def _addr(a):
    if isinstance(a, torch.Tensor):
        return int(a.data_ptr())
    try:
        return int(np.asarray(a).__array_interface__["data"][0])
    except Exception:  # noqa: BLE001 - not a numpy-compatible buffer
        return id(a)


def _sample_sum(a):
    """Checksum of ~256 evenly spaced entries (called on every use of P: each
    sample of a C3-sized array is a cache and TLB miss when the host caches are
    cold, so the count is what the call costs -- ~5 us warm, ~40 us cold)."""
    if isinstance(a, torch.Tensor):
        return float(a[:: max(1, a.numel() // 256)].double().sum().item()) if a.numel() else 0.0
    a = np.asarray(a)
    if a.size == 0:
        return 0.0
    return float(a[:: max(1, a.size // 256)].sum())


def _fingerprint(P):
    """Identity of P's contents for the device cache.  P is treated as
    immutable (as the reference's pure functions read it afresh on every
    call): replaced arrays are seen through their buffers, and in-place edits
    through a sampled checksum of the values (edits that miss every sampled
    entry are not detected)."""
    if hasattr(P, "rows"):
        return (int(P.n), len(P.rows), _addr(P.rows), _addr(P.cols), _addr(P.values),
                _sample_sum(P.values), _sample_sum(P.cols))
    return (P.shape, P.nnz, id(P), _sample_sum(getattr(P, "data", np.zeros(0))))


def device_csr(P, dtype: torch.dtype, device: int, row_begin: int = 0, row_end=None) -> DeviceCSR:
    """Device CSR of P in ``dtype``, built once and cached on the P object."""
    slot = _cache_slot(P)
    key = (dtype, device, row_begin, row_end, _fingerprint(P))
    hit = slot.get(key)
    if hit is not None:
        return hit
    with torch.cuda.device(device):
        n, r, c, v = _coo_full(P, torch.device("cuda", device))
        csr = csr_from_full(n, r, c, v, dtype, row_begin, n if row_end is None else row_end)
        del r, c, v
    # keep one entry per (dtype, device, rows): drop stale fingerprints
    for k in [k for k in slot if k[:4] == key[:4]]:
        del slot[k]
    slot[key] = csr
    return csr


def n_points(P) -> int:
    if hasattr(P, "n"):
        return int(P.n)
    return int(P.shape[0])


def ordered_total(P) -> float:
    """Mass of P over ordered pairs.  The sum over every stored value (63 ms
    at C3) is kept with P under the same contents fingerprint as the device
    CSR, so a second run on the same P does not pay it again."""
    try:
        slot, key = _cache_slot(P), ("ordered_total", _fingerprint(P))
    except Exception:  # noqa: BLE001 - an object the cache cannot describe: just compute
        slot, key = None, None
    if slot is not None and key in slot:
        return slot[key]
    # one evaluation: ordered_total may be a property that sums every stored
    # value (hasattr would evaluate it a first time)
    t = getattr(P, "ordered_total", None)
    if t is not None:
        total = float(t() if callable(t) else t)
    else:
        total = float(P.sum())
    if slot is not None:
        for k in [k for k in slot if k[0] == "ordered_total"]:
            del slot[k]
        slot[key] = total
    return total


def permute_csr(csr: DeviceCSR, perm: torch.Tensor, inv: torch.Tensor) -> DeviceCSR:
    """Symmetric relabelling P' = P[perm][:, perm] of a full (all-rows) CSR.

    perm[new] = old, inv[old] = new.  Row segments move with their rows and
    column indices are relabelled; entries inside a row keep their order (no
    re-sort is needed for locality: a warp's gathers touch few cache lines as
    long as the labels of a row's neighbours are close).
    """
    if csr.row_begin != 0 or csr.n_rows != csr.n_total:
        raise ValueError("permute_csr needs the full matrix")
    rowptr, col, val = csr.rowptr, csr.col, csr.val
    n = csr.n_rows
    deg = rowptr[1:] - rowptr[:-1]
    new_deg = deg[perm]
    new_rowptr = torch.zeros_like(rowptr)
    torch.cumsum(new_deg, 0, out=new_rowptr[1:])
    nnz = int(new_rowptr[-1].item())
    row_of = torch.repeat_interleave(torch.arange(n, device=rowptr.device), new_deg,
                                     output_size=nnz)
    src = torch.arange(nnz, device=rowptr.device) - new_rowptr[row_of] + rowptr[perm][row_of]
    del row_of
    new_col = inv[col[src].long()].to(torch.int32)
    new_val = val[src]
    return DeviceCSR(new_rowptr, new_col.contiguous(), new_val.contiguous(), 0, n, csr.ordered_total)


# ----------------------------------------------------------------------------- host CSR / files
def to_csr(P):
    """Full symmetric CSR on the host: (n, rowptr int64, col int32, val float64).

    Rows list their columns in ascending order (the layout fitsne_set_affinities
    and the tiled build expect)."""
    if hasattr(P, "rows") and hasattr(P, "cols") and hasattr(P, "values"):
        n = int(P.n)
        r0 = np.asarray(P.rows, dtype=np.int64)
        c0 = np.asarray(P.cols, dtype=np.int64)
        v0 = np.asarray(P.values, dtype=np.float64)
        r = np.concatenate([r0, c0])
        c = np.concatenate([c0, r0])
        v = np.concatenate([v0, v0])
    else:
        import scipy.sparse as sp
        if not sp.issparse(P):
            raise TypeError("affinities must be a SparseAffinities-like object or a scipy.sparse matrix")
        coo = P.tocoo()
        if coo.shape[0] != coo.shape[1]:
            raise ValueError("affinity matrix must be square")
        n = coo.shape[0]
        r, c, v = coo.row.astype(np.int64), coo.col.astype(np.int64), coo.data.astype(np.float64)
    order = np.lexsort((c, r))
    r, c, v = r[order], c[order], v[order]
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=rowptr[1:])
    return n, rowptr, c.astype(np.int32), v


def from_csr(n, rowptr, col, val) -> SparseAffinities:
    """SparseAffinities (upper-triangle pairs) from a full symmetric CSR.

    Raises ValueError unless the CSR is symmetric (every (i, j, p) has its
    (j, i, p)) with an empty diagonal -- the invariants of the reference type
    (affinities.py:78-104)."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    col = np.asarray(col, dtype=np.int64)
    val = np.asarray(val, dtype=np.float64)
    if rowptr.shape != (int(n) + 1,) or rowptr[0] != 0 or rowptr[-1] != col.size or col.size != val.size:
        raise ValueError("malformed CSR")
    row = np.repeat(np.arange(int(n), dtype=np.int64), np.diff(rowptr))
    if np.any(row == col):
        raise ValueError("affinities have a non-empty diagonal")
    up = row < col
    lo = ~up
    ku = np.lexsort((col[up], row[up]))
    kl = np.lexsort((row[lo], col[lo]))
    ru, cu, vu = row[up][ku], col[up][ku], val[up][ku]
    if not (np.array_equal(ru, col[lo][kl]) and np.array_equal(cu, row[lo][kl])
            and np.array_equal(vu, val[lo][kl])):
        raise ValueError("affinities are not symmetric")
    return SparseAffinities(n=int(n), rows=ru, cols=cu, values=vu)


def save_affinities(path, P, y0=None) -> None:
    """Write P (and optionally the initial embedding Y0) as a versioned .npz."""
    n, rowptr, col, val = to_csr(P)
    extra = {} if y0 is None else {"y0": np.asarray(y0, dtype=np.float64)}
    np.savez(path, format=np.array(FORMAT), version=np.array(FORMAT_VERSION, dtype=np.int64),
             n=np.array(n, dtype=np.int64), rowptr=rowptr, col=col, val=val, **extra)


def load_affinities(path):
    """(SparseAffinities, Y0 or None) from a file written by save_affinities."""
    with np.load(path, allow_pickle=False) as z:
        if "format" not in z.files or str(z["format"]) != FORMAT:
            raise ValueError(f"{path}: not a {FORMAT} file")
        if int(z["version"]) != FORMAT_VERSION:
            raise ValueError(f"{path}: format version {int(z['version'])}, expected {FORMAT_VERSION}")
        P = from_csr(int(z["n"]), z["rowptr"], z["col"], z["val"])
        y0 = np.array(z["y0"]) if "y0" in z.files else None
    return P, y0
