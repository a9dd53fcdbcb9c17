#!/bin/bash
# Round-2 evidence: GPU suite, smoke, default bench (C2 + sub-records + cpu_baseline), the other
# workloads, the reference arm, launch lists and ncu --set full of the dominant kernels.
# Usage: bash scripts/gpu_final_r2.sh TAG
TAG=${1:-final}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
timeout 1500 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err
for w in c1 c1f c3 c3p c4 c5; do
  timeout 900 python bench.py --steps 10 --warmup 3 --workload $w --no-sub > gpurun_out/bench_${w}_$TAG.json 2> gpurun_out/bench_${w}_$TAG.err
done
timeout 1200 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference_$TAG.json 2> gpurun_out/bench_reference_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-sub > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --workload c5 --no-cpu --no-sub > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_solve_al" -s 2 -c 1 \
  -o gpurun_out/prof_al_c2_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu --no-sub > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_schedule_tile" -s 3 -c 1 \
  -o gpurun_out/prof_tile_c5_$TAG -f python bench.py --steps 1 --warmup 3 --workload c5 --no-cpu --no-sub > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_ik_group" -s 2 -c 1 \
  -o gpurun_out/prof_ik_c2_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu --no-sub > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_solve_al" -s 1 -c 1 \
  -o gpurun_out/prof_al_c3p_$TAG -f python bench.py --steps 1 --warmup 3 --workload c3p --no-cpu --no-sub > /dev/null 2>&1
echo done
