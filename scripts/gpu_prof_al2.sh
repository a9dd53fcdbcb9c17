#!/bin/bash
# fine-grained warp-state sampling (every 32 cycles) of k_solve_al on C2 and C3p
TAG=${1:-x}
mkdir -p gpurun_out
for w in c2 c3p; do
timeout 900 ncu --section SourceCounters --section WarpStateStats --section SchedulerStats --warp-sampling-interval 0 --warp-sampling-buffer-size 268435456 \
  --clock-control none --import-source on -k regex:"k_solve_al" -s 2 -c 1 \
  -o gpurun_out/prof_al_${w}_$TAG -f python bench.py --steps 1 --warmup 3 --workload $w --no-cpu --no-sub > gpurun_out/ncu_al_${w}_$TAG.log 2>&1
done
echo done
