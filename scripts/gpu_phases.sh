timeout 300 python scripts/al_phases.py tower3c 5 > gpurun_out/al_phases_c2_g4.txt 2>&1
