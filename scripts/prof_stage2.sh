#!/bin/bash
# ncu --set full captures of the stage-2 kernels (tower3c full pipeline, fp32)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_solve_al|k_ik_group" -s 2 -c 2 \
  -o gpurun_out/prof_s2_c2 -f python scripts/time_pipeline.py tower3c fp32 1 > gpurun_out/ncu_s2.log 2>&1
echo done
