#!/bin/bash
# ncu --set full of finest-level V-cycle kernels (warm 4K RGB V-cycle,
# scripts/probe_vcycle.py); run under gpurun from the repo root.
#   bash scripts/ncu_kernels.sh TAG kernel_regex[:launch_skip[:name]] ...
# (launch_skip: matching launches to skip inside the warm range, e.g. the
# prolongation runs coarse-to-fine, so its finest launch is the last one)
TAG=${1:-r01}; shift
KS=${@:-k_oras_rows k_resid_tma k_oras_blend}
mkdir -p gpurun_out
for KK in $KS; do
  # kernel_regex[:launch_skip[:name]]
  IFS=: read -r K S N <<< "$KK"
  S=${S:-0}; N=${N:-$K}
  timeout 300 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "warm/" \
    -k regex:$K -s $S -c 1 -o gpurun_out/prof_${N}_$TAG -f \
    python scripts/probe_vcycle.py 1 > gpurun_out/ncu_${N}_$TAG.log 2>&1
done
