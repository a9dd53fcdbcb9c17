#!/bin/bash
# ncu --set full of k_solve_al and k_ik_group on the C2 pipeline. Usage: bash scripts/gpu_prof_al.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_solve_al" -s 2 -c 1 \
  -o gpurun_out/prof_al_c2_$TAG -f python bench.py --steps 1 --warmup 3 --workload c2 --no-cpu --no-sub > gpurun_out/ncu_al_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ik_group" -s 2 -c 1 \
  -o gpurun_out/prof_ik_c2_$TAG -f python bench.py --steps 1 --warmup 3 --workload c2 --no-cpu --no-sub > gpurun_out/ncu_ik_$TAG.log 2>&1
echo done
