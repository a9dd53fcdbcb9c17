#!/bin/bash
# trace / c3p / bench sub-records check
TAG=${1:-r2d}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_trace.py tests/test_pipeline_parity_gpu.py tests/test_stage2_gpu.py -m gpu -q -s -rf 2>&1 | grep -E "fp32 AL gradient|fp32 vs reference|passed|failed|FAILED|Error" | head -80 > gpurun_out/pytest_r2d_$TAG.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c2_$TAG.json 2> gpurun_out/bench_c2_$TAG.err
timeout 600 python bench.py --steps 10 --warmup 3 --workload c3p --no-cpu > gpurun_out/bench_c3p_$TAG.json 2> gpurun_out/bench_c3p_$TAG.err
echo done
