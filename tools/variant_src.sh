#!/bin/bash
# build libfitsne_b200_<name>.so with csrc/tiled.cu replaced by another source: tools/variant_src.sh name path [flags]
set -e
cd /root/repo
name=$1; src=$2; shift 2
cp "$src" paper_1712_09005_b200/csrc/_variant_tiled.cu
python - "$name" "$@" <<'PY'
import subprocess, sys
from paper_1712_09005_b200 import build as B
name, flags = sys.argv[1], sys.argv[2:]
srcs = [str(B.CSRC / s) for s in B.SOURCES if s != "tiled.cu"] + [str(B.CSRC / "_variant_tiled.cu")]
out = B.LIB.with_name(f"libfitsne_b200_{name}.so")
r = subprocess.run([B.nvcc(), *B.NVCC_FLAGS, *flags, "-o", str(out), *srcs], capture_output=True, text=True)
if r.returncode:
    print(r.stderr[-3000:]); sys.exit(1)
print(out)
PY
rm -f paper_1712_09005_b200/csrc/_variant_tiled.cu
