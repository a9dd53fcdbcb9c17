timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_tail.txt
timeout 300 python scripts/host_gaps.py tower3c 20 > gpurun_out/host_gaps_tail.txt 2>&1
for rep in 1 2; do for w in c2 c1; do
 timeout 400 python bench.py --steps 20 --warmup 3 --workload $w --no-cpu --no-sub > gpurun_out/ab_new_${w}_${rep}_t.json 2>&1
 (cd _ab_old && timeout 400 python bench.py --steps 20 --warmup 3 --workload $w --no-cpu --no-sub > ../gpurun_out/ab_old_${w}_${rep}_t.json 2>&1)
done; done
