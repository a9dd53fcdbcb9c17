#!/bin/bash
# full GPU suite, smoke, default bench (C2 + sub-records + cpu_baseline), c3p, reference arm
TAG=${1:-r2j}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -25 > gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
timeout 1200 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err
timeout 600 python bench.py --steps 10 --warmup 3 --workload c3p --no-cpu > gpurun_out/bench_c3p_$TAG.json 2> gpurun_out/bench_c3p_$TAG.err
timeout 1200 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference_$TAG.json 2> gpurun_out/bench_reference_$TAG.err
echo done
