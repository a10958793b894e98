"""ctypes binding of libfitsne_b200.so (include/fitsne_b200.h).

The library is the only compute path: if it cannot be loaded, or no CUDA
device is visible, every call raises instead of falling back to the CPU.
Device memory and streams come from torch (plumbing only); the kernels are the
library's own sm_100a code.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
import weakref
from pathlib import Path

import torch

_PKG = Path(__file__).resolve().parent
# FITSNE_LIB selects another in-tree build of the library (A/B experiments)
LIB_PATH = _PKG / os.environ.get("FITSNE_LIB", "libfitsne_b200.so")

OK, EINVAL, ENONFINITE, EZ, ECUDA, ENOMEM, EOUTSIDE, ETOOBIG, EPOINTS, ENCCL = range(10)
# implementation switches (include/fitsne_b200.h fitsne_option)
(OPT_SORTED_SPREAD, OPT_OVERLAP, OPT_SPMV_BLOCKS_PER_SM, OPT_SPREAD_REPLICAS, OPT_TILED_SPMV,
 OPT_TILE_ROWS, OPT_TILE_COLS, OPT_TILED_CTAS, OPT_TILED_BANK_ORDER, OPT_HOST_PIECES, OPT_FFT_COLS,
 OPT_FFT_PATH, OPT_GRID_F64, OPT_RELABEL, OPT_DEVICE_GRID, OPT_SIDE_GATHER,
 OPT_SPMV_JOIN, OPT_SPEC_AHEAD) = range(1, 19)
F32, F64 = 0, 1
CAUCHY, CAUCHY_SQUARED = 0, 1


class FitsneError(RuntimeError):
    """CUDA-level failure inside libfitsne_b200 (not a user error)."""


class Grid(C.Structure):
    _fields_ = [
        ("lo", C.c_double * 2),
        ("hi", C.c_double * 2),
        ("spacing", C.c_double * 2),
        ("dims", C.c_int32),
        ("n_intervals", C.c_int32),
        ("points_per_interval", C.c_int32),
        ("nodes_per_dim", C.c_int32),
        ("fft_len", C.c_int32),
        ("status", C.c_int32),
    ]


_vp = C.c_void_p
_i64 = C.c_int64
_int = C.c_int
_dbl = C.c_double

_SIGS = {
    "fitsne_last_error": (C.c_char_p, []),
    "fitsne_abi_version": (_int, []),
    "fitsne_create": (_int, [C.POINTER(_vp), _int, _int, _int, _int, _int, _dbl]),
    "fitsne_destroy": (_int, [_vp]),
    "fitsne_set_interp": (_int, [_vp, _int, _int, _dbl]),
    "fitsne_set_option": (_int, [_vp, _int, _int]),
    "fitsne_tiled_stats": (_int, [_vp, _vp, _vp, _vp]),
    "fitsne_make_grid": (_int, [_vp, _vp, _i64, C.POINTER(Grid), _vp]),
    "fitsne_bbox": (_int, [_vp, _vp, _i64, C.POINTER(_dbl), _vp]),
    "fitsne_bbox_device": (_int, [_vp, _vp, _i64, _vp, _vp]),
    "fitsne_grid_from_bbox": (_int, [_vp, C.POINTER(_dbl), C.POINTER(Grid)]),
    "fitsne_set_grid": (_int, [_vp, C.POINTER(Grid)]),
    "fitsne_point_interp": (_int, [_vp, _vp, _i64, _vp, _vp, _vp]),
    "fitsne_spread": (_int, [_vp, _vp, _i64, _vp, _int, _vp, _vp]),
    "fitsne_kernel_matvec": (_int, [_vp, _int, _vp, _int, _vp, _vp]),
    "fitsne_gather": (_int, [_vp, _vp, _i64, _vp, _int, _vp, _vp]),
    "fitsne_evaluate_nbody": (_int, [_vp, _vp, _i64, _vp, _int, _int, _int, _vp, _vp]),
    "fitsne_exact_nbody": (_int, [_vp, _vp, _i64, _vp, _int, _int, _int, _vp, _vp]),
    "fitsne_repulsive": (_int, [_vp, _vp, _i64, _vp, C.POINTER(_dbl), _vp, _vp, _vp]),
    "fitsne_repulsive_exact": (_int, [_vp, _vp, _i64, _vp, C.POINTER(_dbl), _vp, _vp, _vp]),
    "fitsne_set_affinities": (_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i64]),
    "fitsne_attractive": (_int, [_vp, _vp, _vp, _vp]),
    "fitsne_gradient": (_int, [_vp, _vp, _dbl, _vp, C.POINTER(_dbl), _vp]),
    "fitsne_gradient_host": (_int, [_vp, _vp, _dbl, _vp, _vp]),
    "fitsne_kl": (_int, [_vp, _vp, _dbl, C.POINTER(_dbl), _vp]),
    "fitsne_step": (_int, [_vp, _vp, _vp, _vp, _vp, _i64, _dbl, _dbl, _vp]),
    "fitsne_iterate": (_int, [_vp, _vp, _vp, _vp, _vp, _dbl, _dbl, _dbl, _vp, _vp, _vp]),
    "fitsne_grid_accum_len": (_i64, [_vp]),
    "fitsne_spread_tsne": (_int, [_vp, _vp, _i64, _vp, _vp]),
    "fitsne_fft_tsne": (_int, [_vp, _vp, _i64, _int, C.POINTER(_dbl), _vp]),
    "fitsne_gather_tsne": (_int, [_vp, _vp, _i64, _vp, _vp, _vp, _vp]),
    "fitsne_gradient_rows": (_int, [_vp, _vp, _vp, _dbl, _vp, _vp]),
    "fitsne_combine_rows": (_int, [_vp, _vp, _vp, _i64, _dbl, _vp, _vp]),
    "fitsne_read_z": (_int, [_vp, _vp, _vp]),
    "fitsne_grid_accum_dtype": (_int, [_vp]),
    "fitsne_nccl_unique_id": (_int, [_vp]),
    "fitsne_comm_init": (_int, [_vp, _vp, _int, _int, _i64]),
    "fitsne_comm_destroy": (_int, [_vp]),
    "fitsne_gradient_sharded": (_int, [_vp, _vp, _dbl, _vp, C.POINTER(_dbl), _vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load(path: Path | str = LIB_PATH):
    """Load the shared library and declare every prototype (no GPU needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path)
        if not p.exists():
            raise ImportError(
                f"{p} is missing: build it with `python -m paper_1712_09005_b200.build` "
                "(there is no CPU fallback)"
            )
        lib = C.CDLL(str(p))
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def lib():
    return _lib if _lib is not None else load()


def last_error() -> str:
    msg = lib().fitsne_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map a status code to the reference's exception types."""
    if rc == OK:
        return
    msg = last_error() or what
    if rc in (EINVAL, EOUTSIDE, EZ, ETOOBIG, EPOINTS):
        raise ValueError(msg)
    if rc == ENONFINITE:
        raise FloatingPointError(msg)
    if rc == ENOMEM:
        raise MemoryError(msg)
    raise FitsneError(f"{what}: {msg}" if what else msg)


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1712_09005_b200 runs only on a CUDA (sm_100a) device; none is visible "
            "and there is no CPU fallback"
        )


def ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def stream_handle(device: int | None = None):
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class Context:
    """One libfitsne context: (device, dims, dtype, interpolation options)."""

    def __init__(self, device: int, dims: int, dtype: torch.dtype, p: int, min_intervals: int,
                 intervals_per_integer: float = 1.0):
        require_cuda()
        self.lib = lib()
        self.device = device
        self.dims = dims
        self.dtype = dtype
        self.code = F64 if dtype == torch.float64 else F32
        self.p = p
        self.min_intervals = min_intervals
        self.ipi = float(intervals_per_integer)
        h = C.c_void_p()
        with torch.cuda.device(device):
            check(self.lib.fitsne_create(C.byref(h), device, dims, self.code, p, min_intervals,
                                         self.ipi), "fitsne_create")
        self.h = h
        self._P_ref = None  # the registered DeviceCSR
        for opt, val in _default_options.items():
            check(self.lib.fitsne_set_option(self.h, opt, val), "fitsne_set_option")

    def __del__(self):
        try:
            if getattr(self, "h", None) and _lib is not None:
                _lib.fitsne_destroy(self.h)
                self.h = None
        except Exception:
            pass

    @property
    def stream(self):
        return stream_handle(self.device)

    def set_affinities(self, csr, owner=None):
        """Register a DeviceCSR with this context (no-op if it is already the
        registered one).  The context keeps the CSR alive while it is
        registered; with `owner` (the caller's P, which caches the CSR), the
        registration is dropped -- and the library frees its tiled copy of P
        -- once that P is garbage-collected."""
        if csr is self._P_ref:
            return
        check(self.lib.fitsne_set_affinities(self.h, ptr(csr.rowptr), ptr(csr.col), ptr(csr.val),
                                             csr.n_rows, csr.row_begin, csr.n_total,
                                             csr.col.numel()),
              "fitsne_set_affinities")
        self._P_ref = csr
        if owner is not None:
            try:
                weakref.finalize(owner, self._released, weakref.ref(csr))
            except TypeError:  # owner not weak-referenceable: keep the CSR
                pass

    def _released(self, csr_ref):
        csr = csr_ref()
        if csr is None or self._P_ref is not csr or not getattr(self, "h", None) or _lib is None:
            return
        self._P_ref = None
        try:
            with torch.cuda.device(self.device):
                _lib.fitsne_set_affinities(self.h, None, None, None, 0, 0, 0, 0)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


_contexts: dict = {}
_default_options: dict = {}


class option:
    """Context manager (A/B tests): set an implementation switch on every
    existing context and on the contexts created inside the block; restored
    to `restore` (the library default unless given) on exit."""

    _DEFAULTS = {OPT_FFT_PATH: 0, OPT_GRID_F64: 1, OPT_TILED_SPMV: 1, OPT_SORTED_SPREAD: 1, OPT_RELABEL: 1,
                 OPT_DEVICE_GRID: 0, OPT_SIDE_GATHER: 1, OPT_SPMV_JOIN: 1, OPT_SPEC_AHEAD: 0,
                 OPT_OVERLAP: 1, OPT_HOST_PIECES: 0}

    def __init__(self, opt: int, value: int, restore: int | None = None):
        self.opt, self.value = opt, value
        self.restore = self._DEFAULTS.get(opt) if restore is None else restore

    def _apply(self, value):
        for ctx in list(_contexts.values()):
            check(ctx.lib.fitsne_set_option(ctx.h, self.opt, value), "fitsne_set_option")

    def __enter__(self):
        _default_options[self.opt] = self.value
        self._apply(self.value)
        return self

    def __exit__(self, *exc):
        _default_options.pop(self.opt, None)
        if self.restore is not None:
            self._apply(self.restore)
        return False


def context(device: int, dims: int, dtype: torch.dtype, p: int = 3, min_intervals: int = 20,
            intervals_per_integer: float = 1.0) -> Context:
    key = (device, dims, dtype, p, min_intervals, float(intervals_per_integer),
           threading.get_ident())
    ctx = _contexts.get(key)
    if ctx is None:
        ctx = Context(device, dims, dtype, p, min_intervals, intervals_per_integer)
        _contexts[key] = ctx
    return ctx
