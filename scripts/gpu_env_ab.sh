#!/bin/bash
# A/B of one environment toggle (EXP_VAR) on the same box: bench lines + lift counters
TAG=${1:-envab}
VAR=${2:-SPASM_EXP_NO_POLISHER}
mkdir -p gpurun_out
for rep in 1 2; do
  for w in ${WORKLOADS:-c2 c1 c3p}; do
    timeout 400 python bench.py --steps 20 --warmup 3 --workload $w --no-cpu --no-sub > gpurun_out/env_off_${w}_${rep}_$TAG.json 2>&1
    env $VAR=1 timeout 400 python bench.py --steps 20 --warmup 3 --workload $w --no-cpu --no-sub > gpurun_out/env_on_${w}_${rep}_$TAG.json 2>&1
  done
done
echo done
