TAG=${1:-settle}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_$TAG.txt
timeout 300 python scripts/ik_profile.py tower3c 5 > gpurun_out/ikp_c2_$TAG.txt 2>&1
timeout 300 python scripts/ik_profile.py tetris5 3 > gpurun_out/ikp_c3p_$TAG.txt 2>&1
(cd _ab_old && timeout 300 python scripts/ik_profile.py tetris5 3 > ../gpurun_out/ikp_c3p_old_$TAG.txt 2>&1)
timeout 300 python scripts/al_phases.py tower3c 5 > gpurun_out/al_phases_c2_$TAG.txt 2>&1
for rep in 1 2; do for w in c2 c1 c3p; do
 timeout 400 python bench.py --steps 20 --warmup 3 --workload $w --no-cpu --no-sub > gpurun_out/ab_new_${w}_${rep}_$TAG.json 2>&1
 (cd _ab_old && timeout 400 python bench.py --steps 20 --warmup 3 --workload $w --no-cpu --no-sub > ../gpurun_out/ab_old_${w}_${rep}_$TAG.json 2>&1)
done; done
