#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench lines (c2 default, c1, c3, c5), launch list
# of the default workload and one ncu --set full capture of the dominant stage-2 kernel.
# Usage: bash scripts/gpu_round.sh TAG   (outputs -> gpurun_out/)
TAG=${1:-x}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 > gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
for w in c2 c1 c3 c5; do
  timeout 600 python bench.py --steps 10 --warmup 3 --workload $w > gpurun_out/bench_${w}_$TAG.json 2> gpurun_out/bench_${w}_$TAG.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --workload c2 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_solve_al" -s 2 -c 1 \
  -o gpurun_out/prof_al_c2_$TAG -f python bench.py --steps 1 --warmup 3 --workload c2 --no-cpu > gpurun_out/ncu_al_$TAG.log 2>&1
echo done
