#!/bin/bash
# Round-2 parity batch: new pipeline/variant-A/tilings/drop-in/step-cap tests (verbose, all
# failures listed), then the whole GPU suite and smoke.
TAG=${1:-r2b}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_pipeline_parity_gpu.py tests/test_variant_a_gpu.py tests/test_tilings.py \
  tests/test_dropin_gpu.py tests/test_step_cap.py tests/test_stage1_tile_gpu.py tests/test_stage2_gpu.py \
  -m gpu -q -s -rf 2>&1 | grep -v "^$" | tail -150 > gpurun_out/pytest_new_$TAG.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
echo done
