"""Host/device array plumbing for the drop-in API.

Inputs may be numpy arrays / array-likes (the reference's convention: float64
in, new float64 numpy arrays out) or torch tensors (CPU tensors are copied to
the device; CUDA tensors are used in place and results stay on the device).
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _lib

_DTYPES = {
    None: None,
    "float32": torch.float32, "f32": torch.float32, "fp32": torch.float32,
    "float64": torch.float64, "f64": torch.float64, "fp64": torch.float64,
    np.float32: torch.float32, np.float64: torch.float64,
    torch.float32: torch.float32, torch.float64: torch.float64,
}

_default_dtype = torch.float64


def set_default_dtype(dtype) -> None:
    """Precision used for numpy inputs when a call does not pass ``dtype``."""
    global _default_dtype
    _default_dtype = resolve(dtype)


def resolve(dtype):
    try:
        d = _DTYPES[dtype]
    except (KeyError, TypeError):
        d = _DTYPES.get(np.dtype(dtype).type) if dtype is not None else None
        if d is None:
            raise ValueError(f"unsupported dtype {dtype!r}: use float32 or float64")
    return d


def compute_dtype(x, dtype=None) -> torch.dtype:
    d = resolve(dtype)
    if d is not None:
        return d
    if isinstance(x, torch.Tensor) and x.dtype in (torch.float32, torch.float64):
        return x.dtype
    return _default_dtype


def is_device_input(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def device_of(*xs) -> int:
    for x in xs:
        if isinstance(x, torch.Tensor) and x.is_cuda:
            return x.device.index
    _lib.require_cuda()
    return torch.cuda.current_device()


def host_array(x, ndmin_points=False) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        x = x.detach().cpu().numpy()
    return np.asarray(x, dtype=float)


def to_device(x, dtype: torch.dtype, device: int) -> torch.Tensor:
    """Contiguous device tensor of ``dtype`` (no copy when already there)."""
    if isinstance(x, torch.Tensor):
        t = x.detach()
        if t.is_cuda and t.device.index == device and t.dtype == dtype and t.is_contiguous():
            return t
        if t.is_cuda:
            return t.to(device=device, dtype=dtype).contiguous()
        if t.is_pinned():
            t = t.to(device=device, non_blocking=True)
            return t.to(dtype).contiguous()
        return t.to(dtype=dtype).contiguous().to(device=device)
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64 if dtype == torch.float64 else np.float32))
    return torch.from_numpy(a).to(device=device)


def as_points(x, dims=None):
    """Shape rules of nbody._as_points (nbody.py:107-115), without copying."""
    if isinstance(x, torch.Tensor):
        shape = tuple(x.shape)
    else:
        x = np.asarray(x, dtype=float)
        shape = x.shape
    if len(shape) == 1:
        x = x[:, None] if isinstance(x, np.ndarray) else x.reshape(-1, 1)
        shape = (shape[0], 1)
    if len(shape) != 2 or shape[0] == 0:
        raise ValueError("points must be a non-empty (N,) or (N, dims) array")
    if dims is not None and shape[1] != dims:
        raise ValueError(f"expected {dims}-dimensional points, got {shape[1]}")
    return x


_pinned: dict = {}


def _pinned_buffer(shape, dtype, tag="in"):
    """Reusable pinned staging buffer (cudaHostAlloc is far too slow per call).
    Keyed per thread like the library contexts (_lib.context), so concurrent
    callers never share a staging buffer."""
    n = 1
    for s in shape:
        n *= int(s)
    key = (tag, dtype, threading.get_ident())
    buf = _pinned.get(key)
    if buf is None or buf.numel() < n:
        buf = torch.empty(max(n, 1), dtype=dtype, pin_memory=True)
        _pinned[key] = buf
    return buf[:n].view(shape)


def host_input(x, dtype: torch.dtype) -> torch.Tensor:
    """Contiguous CPU tensor of ``dtype`` holding ``x`` (a host array): the
    caller's own tensor when it already qualifies, else a pinned staging copy."""
    if isinstance(x, torch.Tensor):
        t = x.detach()
        if t.dtype == dtype and t.is_contiguous():
            return t
        buf = _pinned_buffer(tuple(t.shape), dtype, "in")
        buf.copy_(t)
        return buf
    a = np.asarray(x)
    buf = _pinned_buffer(a.shape, dtype, "in")
    buf.numpy()[...] = a
    return buf


def host_output(shape, dtype: torch.dtype, out=None) -> torch.Tensor:
    """Where a host-bound result is written: ``out`` when it is a contiguous
    CPU tensor of ``dtype``, else a pinned staging buffer."""
    if out is not None:
        if tuple(out.shape) != tuple(shape):
            raise ValueError("out has the wrong shape")
        if not out.is_cuda and out.dtype == dtype and out.is_contiguous():
            return out
    return _pinned_buffer(tuple(shape), dtype, "out")


def output(t: torch.Tensor, device_result, like=None, out=None):
    """Result in the caller's convention: ``out`` (a caller-owned tensor, e.g.
    pinned host memory, filled in place), else a device tensor for device
    callers, a CPU tensor for CPU-tensor callers, float64 numpy otherwise."""
    if out is not None:
        if tuple(out.shape) != tuple(t.shape):
            raise ValueError("out has the wrong shape")
        out.copy_(t, non_blocking=True)
        if not out.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()
        return out
    if device_result:
        return t
    if isinstance(like, torch.Tensor):
        return t.cpu()
    return t.to(torch.float64).cpu().numpy()
