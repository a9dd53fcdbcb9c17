#!/bin/bash
# AL + IK profiling pass: phase timer on C2 and C1, ncu --set full (source) of k_solve_al and k_ik_group.
TAG=${1:-r2c}
mkdir -p gpurun_out
timeout 300 python scripts/al_phases.py tower3c 5 > gpurun_out/al_phases_c2_$TAG.txt 2>&1
timeout 300 python scripts/al_phases.py single1 5 > gpurun_out/al_phases_c1_$TAG.txt 2>&1
bash scripts/gpu_prof_al.sh $TAG
python scripts/ncu_lines.py gpurun_out/prof_al_c2_$TAG.ncu-rep 60 > gpurun_out/lines_al_$TAG.txt 2>&1
python scripts/ncu_lines.py gpurun_out/prof_ik_c2_$TAG.ncu-rep 40 > gpurun_out/lines_ik_$TAG.txt 2>&1
echo done
