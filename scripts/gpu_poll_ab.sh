TAG=${1:-poll}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_$TAG.txt
for s in tower3c single1 tetris5; do
 timeout 300 python scripts/ik_profile.py $s 5 > gpurun_out/ikp_${s}_$TAG.txt 2>&1
 (cd _ab_old && timeout 300 python scripts/ik_profile.py $s 5 > ../gpurun_out/ikp_${s}_old_$TAG.txt 2>&1)
done
for rep in 1 2; do for w in c2 c1 c3p; do
 timeout 400 python bench.py --steps 20 --warmup 3 --workload $w --no-cpu --no-sub > gpurun_out/ab_new_${w}_${rep}_$TAG.json 2>&1
 (cd _ab_old && timeout 400 python bench.py --steps 20 --warmup 3 --workload $w --no-cpu --no-sub > ../gpurun_out/ab_old_${w}_${rep}_$TAG.json 2>&1)
done; done
