#!/bin/bash
# quick AL experiment: C2 / C1 / C3p bench lines + C2 per-warp phases (+ optional GPU suite)
TAG=${1:-exp}
mkdir -p gpurun_out
for w in c2 c1 c3p; do
  timeout 400 python bench.py --steps 20 --warmup 3 --workload $w --no-cpu --no-sub > gpurun_out/bench_${w}_$TAG.json 2>&1
done
timeout 300 python scripts/al_phases.py tower3c 5 > gpurun_out/al_phases_c2_$TAG.txt 2>&1
if [ "$2" = "tests" ]; then
  timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu_$TAG.txt
fi
echo done
