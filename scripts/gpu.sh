#!/bin/bash
# build locally (nvcc cross-compiles sm_100a), then run a command on the B200 box
set -e
cd /root/repo
python paper_2401_06747_b200/build.py > /dev/null
python -c "from oracle import oracle; oracle.build()" > /dev/null
T=${GPU_TIMEOUT:-900}
exec /usr/local/graft/bin/gpurun --timeout $T -- "$@"
