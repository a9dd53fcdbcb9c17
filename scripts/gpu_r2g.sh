#!/bin/bash
# device restart loop + one-sync pipeline: full GPU suite, smoke, benches c2 / c1 / c3p, C2 launch list
TAG=${1:-r2g}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -25 > gpurun_out/pytest_gpu_$TAG.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
for w in c2 c1 c3p; do
  timeout 600 python bench.py --steps 10 --warmup 3 --workload $w --no-cpu --no-sub > gpurun_out/bench_${w}_$TAG.json 2> gpurun_out/bench_${w}_$TAG.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-sub > /dev/null 2>&1
echo done
