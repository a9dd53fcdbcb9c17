#!/bin/bash
# Sharded stage-1 checks on one GPU: GPU tests, 2 ranks sharing cuda:0 over gloo through
# bench.py, and the N=1 bench lines.
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_sharded_gpu.py -x -q 2>&1 | tail -30 > gpurun_out/pytest_shard_$TAG.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu_$TAG.txt
SPASM_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --workload c3 > gpurun_out/bench_c3_g2gloo_$TAG.json 2> gpurun_out/bench_c3_g2gloo_$TAG.err
SPASM_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29534 bench.py --gpus 2 --steps 5 --warmup 3 --workload c2 > gpurun_out/bench_c2_g2gloo_$TAG.json 2> gpurun_out/bench_c2_g2gloo_$TAG.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_c2_$TAG.json 2> gpurun_out/bench_c2_$TAG.err
echo done
