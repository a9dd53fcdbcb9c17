#!/bin/bash
# GPU tests + ncu full capture of the dominant kernel (k_schedule) for C5 and C3.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_schedule -s 3 -c 1 \
  -o gpurun_out/prof_c5 -f python bench.py --steps 1 --warmup 3 --workload c5 --no-cpu > gpurun_out/ncu_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_schedule -s 3 -c 1 \
  -o gpurun_out/prof_c3 -f python bench.py --steps 1 --warmup 3 --workload c3 --no-cpu > gpurun_out/ncu_c3.log 2>&1
echo done
