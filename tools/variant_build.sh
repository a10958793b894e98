#!/bin/bash
# build libfitsne_b200 variants with extra -D flags into /tmp copies (A/B probes on the GPU box)
set -e
cd /root/repo
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  python - "$name" "$flags" <<'PY'
import subprocess, sys
from paper_1712_09005_b200 import build as B
name, flags = sys.argv[1], sys.argv[2].split()
out = B.LIB.with_name(f"libfitsne_b200_{name}.so")
cmd = [B.nvcc(), *B.NVCC_FLAGS, *flags, "-o", str(out), *[str(B.CSRC / s) for s in B.SOURCES]]
subprocess.run(cmd, check=True, capture_output=True)
print(out)
PY
done
