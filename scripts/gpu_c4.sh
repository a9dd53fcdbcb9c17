#!/bin/bash
TAG=${1:-x}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_replan.py tests/test_sharded_gpu.py -x -q 2>&1 | tail -5 > gpurun_out/pytest_c4_$TAG.txt
timeout 600 python bench.py --steps 20 --warmup 3 --workload c4 > gpurun_out/bench_c4_$TAG.json 2> gpurun_out/bench_c4_$TAG.err
SPASM_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29535 bench.py --gpus 2 --steps 5 --warmup 3 --workload c4 > gpurun_out/bench_c4_g2_$TAG.json 2> gpurun_out/bench_c4_g2_$TAG.err
echo done
