#!/bin/bash
# Launch lists (ncu, kernel durations) of the C2 and C1 pipelines. Usage: bash scripts/gpu_launch_s2.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
for w in c2 c1; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${w}_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --workload $w --no-cpu > /dev/null 2>&1
done
echo done
