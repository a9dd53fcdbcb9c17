#!/bin/bash
# ncu --set full of the dominant kernel of C1, C3, C4 (DRAM traffic per launch for the bench roofline)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:"k_solve_al" -s 2 -c 1 -o gpurun_out/prof_al_c1_t -f \
  python bench.py --steps 1 --warmup 3 --workload c1 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_schedule_tile" -s 3 -c 1 -o gpurun_out/prof_tile_c3_t -f \
  python bench.py --steps 1 --warmup 3 --workload c3 --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_schedule_tower_tile" -s 3 -c 1 -o gpurun_out/prof_tower_c4_t -f \
  python bench.py --steps 1 --warmup 3 --workload c4 --no-cpu > /dev/null 2>&1
echo done
