#!/bin/bash
# GPU tests + C4/C2 bench lines (stage-1 tower kernel iteration). Usage: bash scripts/gpu_s1t.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu_$TAG.txt
for w in c4 c2; do
  timeout 300 python bench.py --steps 10 --warmup 3 --workload $w --no-cpu > gpurun_out/bench_${w}_$TAG.json 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --workload c4 --no-cpu > /dev/null 2>&1
echo done
