for la in 1 2 4 8; do timeout 300 python scripts/tower_lanes.py $la; done > gpurun_out/tower_lanes.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/pytest_tl.txt
