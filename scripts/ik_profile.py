"""k_ik_group timeline counters on a pipeline workload (diagnostic).
Usage: python scripts/ik_profile.py [scene] [solves]"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2510_07674_b200 import _native as nat  # noqa: E402
from paper_2510_07674_b200.bench_api import solve_scene  # noqa: E402
from paper_2510_07674_b200.problems import as_cost_model, load_scene  # noqa: E402

scene_name = sys.argv[1] if len(sys.argv) > 1 else "tower3c"
solves = int(sys.argv[2]) if len(sys.argv) > 2 else 5
scene = load_scene(scene_name)
model = as_cost_model(scene.problem, precision="fp32")
lib = nat.load()
solve_scene(scene, seed=99, model=model)
out = np.zeros(12)
lib.spasm_ik_profile(1, None)
lib.spasm_ik_profile(1, out.ctypes.data)  # reset
for s in range(solves):
    solve_scene(scene, seed=s, model=model)
lib.spasm_ik_profile(0, out.ctypes.data)
n = max(1.0, out[0])
print(f"scene {scene_name}: {solves} solves, {out[0]:.0f} lift CTAs (groups); per CTA:")
print(f"  cycles to the last restart's IK {out[1] / n:10.0f}   to the end {out[2] / n:10.0f}")
print(f"  IK iterations: max over restarts {out[3] / n:.1f}, winner {out[4] / n:.1f}, mean {out[7] / n / 16:.1f}")
print(f"  winner polish iterations (speculative + after IK) {out[5] / n:.1f}; polished speculatively to completion {out[6] / n * 100:.0f} %")
print(f"  max over CTAs: cycles to the last restart's IK {out[8]:.0f}, to the end {out[9]:.0f}; "
      f"IK iterations {out[11]:.0f}, winner polish iterations {out[10]:.0f}")
