#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of one C2 and one C3p-scene pipeline solve
# (AL engine named barriers 1 and 2, device restart-loop graph, in-place stage-1 rows).
TAG=${1:-x}
mkdir -p gpurun_out
cat > /tmp/one_solve.py <<'PY'
import sys
sys.path.insert(0, ".")
from paper_2510_07674_b200.bench_api import solve_scene
from paper_2510_07674_b200.problems import load_scene
name = sys.argv[1]
sc = load_scene(name)
for seed in range(2):  # the second solve of a shape runs the restart-loop graph
    sol = solve_scene(sc, seed=seed)
    print(name, "seed", seed, "success", sol.success)
PY
for scene in tower3c tetris5; do
  for tool in synccheck racecheck memcheck; do
    timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python /tmp/one_solve.py $scene > gpurun_out/sanitize_${tool}_${scene}_$TAG.txt 2>&1
    echo "exit $?" >> gpurun_out/sanitize_${tool}_${scene}_$TAG.txt
  done
done
echo done
