#!/bin/bash
# FK experiment: microbench + stage-2 parity tests + C2/C1/C3p bench lines + phases.
TAG=${1:-fk}
mkdir -p gpurun_out
./scripts/microbench/fk_latency > gpurun_out/mb_fk_$TAG.txt 2>&1
for w in c2 c1 c3p c1f; do
  timeout 400 python bench.py --steps 20 --warmup 3 --workload $w --no-cpu --no-sub > gpurun_out/bench_${w}_$TAG.json 2>&1
done
timeout 300 python scripts/al_phases.py tower3c 5 > gpurun_out/al_phases_c2_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu_$TAG.txt
echo done
