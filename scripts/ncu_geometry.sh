#!/bin/bash
# ncu --set full of the densification / dither / tonal kernels of one 4K RGB
# pipeline run (scripts/pipeline_once.py); run under gpurun from the repo root.
#   bash scripts/ncu_geometry.sh TAG [kernel[:skip] ...]
TAG=${1:-r02}; shift
KS=${@:-k_gauss_axis k_coin k_jfa_pass_key4:20 k_jfa_pass_key:20 k_jfa_key_finish:19 k_corner_scan:19 k_raster_tiles:19 k_reduce_tris_small:18 k_error_map:19 k_vi_step k_tv_down k_tv_close}
mkdir -p gpurun_out
for KK in $KS; do
  K=${KK%%:*}; S=0
  [[ "$KK" == *:* ]] && S=${KK##*:}
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:"^${K}\$" -s $S -c 1 \
    -o gpurun_out/prof_${K}_$TAG -f python scripts/pipeline_once.py > gpurun_out/ncu_${K}_$TAG.log 2>&1
done
