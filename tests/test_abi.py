"""C-ABI checks that need no GPU: the library builds/loads, exports every
symbol declared in include/fitsne_b200.h, and rejects bad arguments with the
documented status codes before touching the device."""

from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "fitsne_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fitsne_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_1712_09005_b200 import _lib, build
    build.build()
    return _lib.load()


def test_library_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_python_binding_covers_header():
    from paper_1712_09005_b200 import _lib
    assert set(declared_symbols()) == set(_lib.EXPORTED)


def test_abi_version(lib):
    assert lib.fitsne_abi_version() == 1


def test_create_rejects_bad_arguments_without_gpu(lib):
    from paper_1712_09005_b200 import _lib
    h = C.c_void_p()
    assert lib.fitsne_create(C.byref(h), 0, 3, _lib.F32, 3, 20, 1.0) == _lib.EINVAL
    assert b"dims" in lib.fitsne_last_error()
    assert lib.fitsne_create(C.byref(h), 0, 2, 7, 3, 20, 1.0) == _lib.EINVAL
    assert lib.fitsne_create(C.byref(h), 0, 2, _lib.F32, 1, 20, 1.0) == _lib.EINVAL
    assert lib.fitsne_create(C.byref(h), 0, 2, _lib.F32, 3, 0, 1.0) == _lib.EINVAL
    assert lib.fitsne_create(C.byref(h), 0, 2, _lib.F32, 3, 20, 0.0) == _lib.EINVAL
    assert h.value is None


def test_null_context_is_rejected(lib):
    from paper_1712_09005_b200 import _lib
    assert lib.fitsne_make_grid(None, None, 10, None, None) == _lib.EINVAL
    assert lib.fitsne_grid_accum_len(None) == 0


def test_status_mapping():
    from paper_1712_09005_b200 import _lib
    with pytest.raises(ValueError):
        _lib.check(_lib.EINVAL, "x")
    with pytest.raises(ValueError):
        _lib.check(_lib.EZ, "x")
    with pytest.raises(FloatingPointError):
        _lib.check(_lib.ENONFINITE, "x")
    with pytest.raises(_lib.FitsneError):
        _lib.check(_lib.ECUDA, "x")


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_1712_09005_b200 import optimizer
    import numpy as np
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        optimizer.compute_repulsive(np.random.default_rng(0).standard_normal((100, 2)), method="fft")


def test_sass_is_sm100a():
    import subprocess, shutil
    from paper_1712_09005_b200 import build
    lib = build.build()
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "--list-elf", str(lib)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
