#!/bin/bash
# ncu --set full of the finest-level ORAS local CG, blend and residual sweeps
# (warm 4K RGB V-cycle); run under gpurun from the repo root.
TAG=${1:-r01}
mkdir -p gpurun_out
for K in k_oras_local32 k4_residual k_oras_blend; do
  timeout 300 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "warm/" \
    -k regex:$K -c 1 -o gpurun_out/prof_${K}_$TAG -f \
    python scripts/probe_vcycle.py 1 > gpurun_out/ncu_${K}_$TAG.log 2>&1
done
ls -la gpurun_out
