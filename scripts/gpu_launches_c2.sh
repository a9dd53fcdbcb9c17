mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_s6.csv python bench.py --steps 2 --warmup 3 --workload c2 --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c1_s6.csv python bench.py --steps 2 --warmup 3 --workload c1 --no-cpu > /dev/null 2>&1
