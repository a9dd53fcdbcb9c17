#!/bin/bash
# Tile-kernel checks: tile GPU tests, full GPU suite, C5/C3 bench per tile variant, ncu of k_schedule_tile.
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stage1_tile_gpu.py -x -q 2>&1 | tail -30 > gpurun_out/pytest_tile_$TAG.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu_$TAG.txt
for v in ${VARIANTS:-0 4}; do
  SPASM_STAGE1_TILE=$v timeout 300 python bench.py --steps 5 --warmup 3 --workload c5 --no-cpu > gpurun_out/bench_c5_t${v}_$TAG.json 2>&1
  SPASM_STAGE1_TILE=$v timeout 300 python bench.py --steps 5 --warmup 3 --workload c3 --no-cpu > gpurun_out/bench_c3_t${v}_$TAG.json 2>&1
done
timeout 300 python bench.py --steps 10 --warmup 3 --workload c1 --no-cpu > gpurun_out/bench_c1_$TAG.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_schedule -s 3 -c 1 \
  -o gpurun_out/prof_tile_c5_$TAG -f python bench.py --steps 1 --warmup 3 --workload c5 --no-cpu > gpurun_out/ncu_tile_c5_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_schedule -s 3 -c 1 \
  -o gpurun_out/prof_tile_c3_$TAG -f python bench.py --steps 1 --warmup 3 --workload c3 --no-cpu > gpurun_out/ncu_tile_c3_$TAG.log 2>&1
echo done
