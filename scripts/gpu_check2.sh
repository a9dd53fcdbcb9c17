#!/bin/bash
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu_$TAG.txt
bash scripts/gpu_sanitize.sh $TAG
