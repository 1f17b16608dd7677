#!/bin/bash
# Round evidence on one B200 (run under gpurun from the repo root):
#   1. the bench line                          -> gpurun_out/bench_$TAG.json
#   2. ncu launch list of one bench step       -> gpurun_out/launches_$TAG.csv
#   3. ncu --set full of the finest-level ORAS local-CG sweep and the
#      residual stencil sweep (warm 4K RGB V-cycle) -> gpurun_out/prof_*_$TAG.ncu-rep
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
L=$(python -c "import json;print(json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1])['gpu_launches'])")
# warm-up launches: 3 steps of L plus the setup; skip 3L, list one step
ncu --metrics gpu__time_duration.sum --clock-control none -s $((3 * L)) -c $L --csv \
    --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "warm/" \
    -k regex:k_oras_local32 -c 1 -o gpurun_out/prof_oras_$TAG -f \
    python scripts/probe_vcycle.py 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "warm/" \
    -k regex:k4_residual -c 1 -o gpurun_out/prof_resid_$TAG -f \
    python scripts/probe_vcycle.py 1 > /dev/null 2>&1
ls -la gpurun_out
