#!/bin/bash
# build locally (sm_100a cross-compile), then run a command on the B200 box
set -e
cd /root/repo
python -m paper_1712_09005_b200.build > /dev/null
exec timeout $(( ${GPU_TIMEOUT:-1200} + 900 )) /usr/local/graft/bin/gpurun --timeout ${GPU_TIMEOUT:-1200} -- "$@"
