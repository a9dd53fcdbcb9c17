mkdir -p gpurun_out
./scripts/microbench/fp32_pipes > gpurun_out/mb_fp32.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_schedule -s 3 -c 1 \
  -o gpurun_out/prof_sched_c5_v2 -f python bench.py --steps 1 --warmup 3 --workload c5 --no-cpu > gpurun_out/ncu_sched_c5.log 2>&1
echo done
