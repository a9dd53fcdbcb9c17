#!/bin/bash
# AL restructure check: stage-2 + pipeline parity tests, phase timer, benches c2/c1/c3p
TAG=${1:-r2e}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stage2_gpu.py tests/test_pipeline_parity_gpu.py tests/test_variant_a_gpu.py tests/test_dropin_gpu.py tests/test_full_size_gpu.py -m gpu -q -x 2>&1 | tail -25 > gpurun_out/pytest_$TAG.txt
timeout 300 python scripts/al_phases.py tower3c 5 > gpurun_out/al_phases_c2_$TAG.txt 2>&1
for w in c2 c1 c3p; do
  timeout 600 python bench.py --steps 10 --warmup 3 --workload $w --no-cpu --no-sub > gpurun_out/bench_${w}_$TAG.json 2> gpurun_out/bench_${w}_$TAG.err
done
echo done
