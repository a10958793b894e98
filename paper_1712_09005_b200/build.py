"""Build libfitsne_b200.so in-tree with nvcc for sm_100a.

Usage: python -m paper_1712_09005_b200.build  (or __graft_entry__.build()).
The library statically links the CUDA runtime so it does not depend on the
libcudart that torch ships; device pointers and streams are shared through the
driver's primary context.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libfitsne_b200.so"
SOURCES = ["api.cu", "repulsion.cu", "attract.cu", "sortspread.cu", "bandspread.cu", "tiled.cu",
           "bigfft.cu", "reorder.cu", "comm.cu"]
HEADERS = ["common.cuh", "fft.cuh", "interp.cuh", "internal.h", "twiddles.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-Xptxas", "-v",
    "-shared", "-cudart", "static",
]


def nvcc() -> str:
    cand = [os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"]
    for c in cand:
        if c and Path(c).exists():
            return c
    raise RuntimeError("nvcc not found: the FIt-SNE CUDA library cannot be built")


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [PKG.parent / "include" / "fitsne_b200.h"]
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: str, obj: Path, defines=()) -> tuple[int, str]:
    flags = [f for f in NVCC_FLAGS if f not in ("-shared",)] + [f"-D{d}" for d in defines]
    cmd = [nvcc(), *flags, "-c", "-o", str(obj), str(CSRC / src)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    return res.returncode, f"== {src}\n" + (res.stdout or "") + (res.stderr or "")


def build(force: bool = False, verbose: bool = False, variant: str | None = None,
          defines=()) -> Path:
    """Build the library.  `variant` + `defines` build an A/B copy
    (libfitsne_b200_<variant>.so, selected at run time with FITSNE_LIB)."""
    lib = LIB if variant is None else PKG / f"libfitsne_b200_{variant}.so"
    if variant is None and not force and not stale():
        return LIB
    # one nvcc per translation unit, in parallel, then one link
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    tmp = lib.with_suffix(".so.tmp")
    with tempfile.TemporaryDirectory(prefix="fitsne_build_") as td:
        objs = [Path(td) / (Path(s).stem + ".o") for s in SOURCES]
        with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
            results = list(ex.map(lambda a: _compile(a[0], a[1], defines), zip(SOURCES, objs)))
        log = "".join(r[1] for r in results)
        rc = max(r[0] for r in results)
        if rc == 0:
            cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                   "-o", str(tmp), *[str(o) for o in objs]]
            res = subprocess.run(cmd, capture_output=True, text=True)
            log += "== link\n" + (res.stdout or "") + (res.stderr or "")
            rc = res.returncode
    (PKG / "build.log").write_text(log)
    if rc != 0:
        sys.stderr.write(log)
        raise RuntimeError("nvcc failed building libfitsne_b200.so (see build.log)")
    if verbose:
        sys.stdout.write(log)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    var = next((a.split("=", 1)[1] for a in args if a.startswith("--variant=")), None)
    defs = [a[2:] for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose="-v" in args, variant=var, defines=defs))
