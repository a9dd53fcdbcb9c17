#!/bin/bash
# GPU suite + bench lines for c2, c3, c5, c1 + launch list of c3/c5. Usage: bash scripts/gpu_quick.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu_$TAG.txt
for w in c2 c3 c5 c1; do
  timeout 300 python bench.py --steps 10 --warmup 3 --workload $w --no-cpu > gpurun_out/bench_${w}_$TAG.json 2>&1
done
for w in c3 c5; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${w}_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --workload $w --no-cpu > /dev/null 2>&1
done
echo done
