#!/bin/bash
# per-kernel launch times (ncu, cold/serialised) of the working tree and the _ab_old copy on C2
TAG=${1:-lab}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/lab_new_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-sub > /dev/null 2>&1
(cd _ab_old && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ../gpurun_out/lab_old_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-sub > /dev/null 2>&1)
echo done
