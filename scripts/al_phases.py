"""Per-phase cycle breakdown of the fp32 AL kernel on a pipeline workload (diagnostic).
Usage: python scripts/al_phases.py [scene] [solves]"""
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
out = np.zeros(28)
lib.spasm_al_profile(1, None)
lib.spasm_al_profile(1, out.ctypes.data)  # reset
outers = 0
for s in range(solves):
    sol = solve_scene(scene, seed=s, model=model)
    outers += sol.stats.get("stage2_outers", 0)
lib.spasm_al_profile(0, out.ctypes.data)
names = {0: "A/P1 FK/spheres (+ placed-pose sync)", 1: "A/P2 leg/start/fixed obstacles", 2: "A/P3 placed + J^T (+ CTA barrier)",
         3: "(unused)", 4: "B totals + assemble + step", 8: "pick polish", 9: "re-eval + validate"}
tot = out.sum()
print(f"scene {scene_name}: {solves} solves, {outers} outers; cycles by phase (thread 0, summed over CTAs):")
tot = out[:12].sum()
for k, n in names.items():
    line = f"  {n:28s} {out[k] / tot * 100:6.1f}%  {out[k] / max(1, outers):14.0f} cycles/outer"
    if k < 5:
        line += f"   own work: tile t0 {out[12 + k] / max(1, outers):12.0f}  aux {out[20 + k] / max(1, outers):12.0f}"
    print(line)
print(f"  tile t0 sub-marks: leg+start done at {out[17] / max(1, outers):.0f}, B totals+pgsum done at "
      f"{out[19] / max(1, outers):.0f} cycles/outer (since the phase's start)")
print(f"  aux P2 split: placed poses done at {out[25] / max(1, outers):.0f}, twin done at {out[26] / max(1, outers):.0f} cycles/outer")
wp_all = np.zeros(32 * 8 + 4)
lib.spasm_al_profile_warps(wp_all.ctypes.data)
wp = wp_all[:256].reshape(32, 8) / max(1, outers)
pol = wp_all[256:]
print("per-warp own work (cycles/outer, summed over CTAs; since each phase's start):")
print("  warp        P1        P2   (leg/start)       P3         B")
for w in range(32):
    if wp[w].sum() == 0:
        continue
    print(f"  {w:4d} {wp[w, 0]:9.0f} {wp[w, 1]:9.0f} {wp[w, 5]:9.0f} {wp[w, 2]:12.0f} {wp[w, 4]:9.0f}")
print(f"pick polish: {pol[1]:.0f} calls, {pol[0] / max(1, pol[1]):.1f} iterations per call (max {pol[3]:.0f}), "
      f"{pol[2]:.0f} at the {1000}-iteration cap")
