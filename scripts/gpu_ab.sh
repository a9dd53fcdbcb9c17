#!/bin/bash
# A/B of the working tree against a HEAD copy in _ab_old/ on the same box (interleaved
# runs), then the GPU suite and the lift / AL diagnostics of the working tree.
TAG=${1:-ab}
mkdir -p gpurun_out
for rep in 1 2; do
  for w in ${WORKLOADS:-c2 c1 c3p}; do
    timeout 400 python bench.py --steps 20 --warmup 3 --workload $w --no-cpu --no-sub > gpurun_out/ab_new_${w}_${rep}_$TAG.json 2>&1
    (cd _ab_old && timeout 400 python bench.py --steps 20 --warmup 3 --workload $w --no-cpu --no-sub > ../gpurun_out/ab_old_${w}_${rep}_$TAG.json 2>&1)
  done
done
if [ "$2" = "tests" ]; then
  timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu_$TAG.txt
  timeout 300 python scripts/ik_profile.py tower3c 5 > gpurun_out/ik_prof_c2_$TAG.txt 2>&1
  timeout 300 python scripts/ik_profile.py tetris5 3 > gpurun_out/ik_prof_c3p_$TAG.txt 2>&1
  timeout 300 python scripts/al_phases.py tower3c 5 > gpurun_out/al_phases_c2_$TAG.txt 2>&1
fi
echo done
