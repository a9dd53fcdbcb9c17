#!/bin/bash
TAG=${1:-r2k}
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err
timeout 300 python scripts/al_phases.py tetris5 3 > gpurun_out/al_phases_c3p_$TAG.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_solve_al" -s 1 -c 1 \
  -o gpurun_out/prof_al_c3p_$TAG -f python bench.py --steps 1 --warmup 3 --workload c3p --no-cpu --no-sub > gpurun_out/ncu_al_c3p_$TAG.log 2>&1
echo done
