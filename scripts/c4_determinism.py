"""C4 replanning: run the same warm-started tick sequence twice and compare per-tick restarts,
placements and solve times (diagnostic for run-to-run variance)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2510_07674_b200.replan import replan_loop  # noqa: E402

runs = []
for r in range(3):
    ticks, _ = replan_loop(13, seed=0)
    runs.append(ticks)
    print("run", r, "restarts", [t.restarts for t in ticks])
    print("      solve_ms", [round(t.solve_ms, 2) for t in ticks])
    print("      tick_ms ", [round(t.tick_ms, 2) for t in ticks])
same = all(np.array_equal(a.placement, b.placement) for a, b in zip(runs[0], runs[1]))
print("placements identical across runs:", same)
