#!/bin/bash
# A/B of the working tree against a HEAD copy in _ab_old/ on the same box (interleaved runs)
TAG=${1:-ab}
mkdir -p gpurun_out
for rep in 1 2; do
  for w in ${WORKLOADS:-c1 c3p c2}; do
    timeout 400 python bench.py --steps 20 --warmup 3 --workload $w --no-cpu --no-sub > gpurun_out/ab_new_${w}_${rep}_$TAG.json 2>&1
    (cd _ab_old && timeout 400 python bench.py --steps 20 --warmup 3 --workload $w --no-cpu --no-sub > ../gpurun_out/ab_old_${w}_${rep}_$TAG.json 2>&1)
  done
done
echo done
