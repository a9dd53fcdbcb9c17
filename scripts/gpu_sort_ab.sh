#!/bin/bash
# Sort change A/B: the working tree against a HEAD copy in _ab_old/ (sort timing per n, the
# sort + stage-1 GPU tests, interleaved C2 / C4 benches)
TAG=${1:-sort}
mkdir -p gpurun_out
timeout 300 python scripts/sort_timing.py > gpurun_out/sort_new_$TAG.txt 2>&1
(cd _ab_old && timeout 300 python ../scripts/sort_timing.py > ../gpurun_out/sort_old_$TAG.txt 2>&1)
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_$TAG.txt
for rep in 1 2; do for w in ${WORKLOADS:-c2 c4}; do
 timeout 400 python bench.py --steps 20 --warmup 3 --workload $w --no-cpu --no-sub > gpurun_out/ab_new_${w}_${rep}_$TAG.json 2>&1
 (cd _ab_old && timeout 400 python bench.py --steps 20 --warmup 3 --workload $w --no-cpu --no-sub > ../gpurun_out/ab_old_${w}_${rep}_$TAG.json 2>&1)
done; done
