#!/bin/bash
# Round evidence on one B200 (run under gpurun from the repo root):
#   1. the bench line                              -> gpurun_out/bench_$TAG.json
#   2. CUPTI per-kernel breakdown of one step      -> gpurun_out/kprof_$TAG.txt
#   3. ncu launch list of one bench step           -> gpurun_out/launches_$TAG.csv
#      (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)
#   4. ncu --set full of the finest-level V-cycle kernels (warm 4K RGB V-cycle)
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python scripts/kprof.py > gpurun_out/kprof_$TAG.txt 2>&1
L=$(python -c "import json;print(json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1])['gpu_launches'])")
# warm-up launches: 3 steps of L plus the setup; skip 3L, list one step
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s $((3 * L)) -c $L --csv \
    --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-strips > gpurun_out/launches_bench_$TAG.log 2>&1
# in the warm V-cycle the first k_ws_resid is the finest residual + norms,
# the second the finest residual + restriction; the TMA prolongations run
# coarse to fine over the levels >= 300,000 px (three at 4K)
bash scripts/ncu_kernels.sh $TAG k_oras_warp k_ws_resid:0 k_ws_resid:1:k_ws_resid_restrict \
    k_oras_blend k_ws_prolong:2

# fused RAS block kernels (tilesolve.cu) on the 4K block set
for K in k_tv_down k_tv_close; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
    -o gpurun_out/prof_${K}_$TAG -f python scripts/probe_tiles.py 2160,3840,3 1 \
    > gpurun_out/ncu_${K}_$TAG.log 2>&1
done
ls -la gpurun_out
