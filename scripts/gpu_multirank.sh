#!/bin/bash
# bench.py under torchrun with 2 ranks sharing one GPU (gloo collectives): the N>1 code path
# (sharded stage 1, max-over-ranks timing, rank-0 JSON line) and the reference arm.
TAG=${1:-mr}
mkdir -p gpurun_out
export SPASM_DIST_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_g2_$TAG.json 2> gpurun_out/bench_g2_$TAG.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 2 --steps 3 --warmup 3 --workload c5 > gpurun_out/bench_g2_c5_$TAG.json 2> gpurun_out/bench_g2_c5_$TAG.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench_g2_ref_$TAG.json 2> gpurun_out/bench_g2_ref_$TAG.err
echo done
