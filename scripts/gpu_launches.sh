mkdir -p gpurun_out
for w in c3 c5 c1; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${w}_v9.csv \
  python bench.py --steps 2 --warmup 3 --workload $w --no-cpu > /dev/null 2>&1
done
echo done
