#!/bin/bash
# compute-sanitizer racecheck / synccheck of one C2 pipeline solve (AL engine named barrier,
# tile warp-mask shuffles). Usage: bash scripts/gpu_sanitize.sh TAG
TAG=${1:-x}
mkdir -p gpurun_out
cat > /tmp/one_solve.py <<'PY'
import sys
sys.path.insert(0, ".")
from paper_2510_07674_b200.bench_api import solve_scene
from paper_2510_07674_b200.problems import load_scene
sol = solve_scene(load_scene(sys.argv[1]), seed=0)
print("success", sol.success)
PY
for tool in synccheck racecheck memcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python /tmp/one_solve.py tower3c > gpurun_out/sanitize_${tool}_$TAG.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitize_${tool}_$TAG.txt
done
echo done
