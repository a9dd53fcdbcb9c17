#!/bin/bash
# Stage-2 iteration: GPU tests, C2/C1 bench lines, AL phase timer. Usage: bash scripts/gpu_s2.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu_$TAG.txt
for w in c2 c1; do
  timeout 300 python bench.py --steps 10 --warmup 3 --workload $w --no-cpu > gpurun_out/bench_${w}_$TAG.json 2>&1
done
timeout 300 python scripts/al_phases.py tower3c 5 > gpurun_out/al_phases_c2_$TAG.txt 2>&1
echo done
