"""Pipeline-level golden fixtures: the REFERENCE's own ``bench.solve_scene`` composition
(reference bench.py:168-268) run on every BASELINE scene, with its intermediate decisions
recorded.

Runs in the build container only (the reference is importable read-only there):

    python tests/golden/make_golden_pipeline.py

Stage 2 needs the test-pinned "variant B" patch, so the reference package is
copied to a temp dir and patched exactly as in make_golden_stage2.py. The stock
``seqplace.bench.solve_scene`` is then called unchanged; the names it binds at import
(``solve``, ``lift_placements``, ``solve_al``; bench.py:28-51) are wrapped so every call's
result is recorded on the way through:

  stage 1   success, report.restarts, SolveResult.indices (the returned batch rows) and costs
  lift      LiftResult.kept
  AL        AlResult.particle_index / objective, accepted outer (= len(report.outers) - 1),
            or TrajOptFailure.best_violation
  scene     SceneSolution.success / restarts / final_cost

The scenes are this repo's BASELINE mappings (paper_2510_07674_b200/problems/scenes.py),
loaded through the REFERENCE's loader (single1's non-tight packing is built through the
reference Python API, tetris.py:88,107, which its loader does not expose).

Also records, for 20 seeds per config, the stage-1-only outcome (success, restarts, returned
indices and costs) that the fp32 outcome-statistics test compares against.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)

# (scene, seeds of the full pipeline)
PIPELINE = {"single1": range(20), "tower4": range(20), "tower3c": range(20), "tetris5": range(10),
            "single1f": range(5)}
# BASELINE C3 at its stated size (64k particles, M = 8192) through the full pipeline:
# key -> (scene, solver overrides, seeds)
PIPELINE_SIZED = {"tetris5@64k": ("tetris5", {"n": 65536, "m": 8192}, range(10))}
# stage-1-only configs (scenes without a robot, or no_trajopt): seeds 0..19
STAGE1 = ["single1", "tower4", "tower3c", "tower6r", "tetris4", "tetris5", "tetris6"]
STAGE1_SEEDS = range(20)


def ref_scene(name):
    from oracle.refscene import ref_scene as build

    return build(name)


def main():
    from make_golden_stage2 import patched_reference

    patched_reference()
    from seqplace import bench

    rec = {}
    orig = {k: getattr(bench, k) for k in ("solve", "lift_placements", "solve_al")}

    def w_solve(*a, **k):
        r = orig["solve"](*a, **k)
        rec["stage1"] = r
        return r

    def w_lift(*a, **k):
        r = orig["lift_placements"](*a, **k)
        rec["lift"] = r
        return r

    def w_al(*a, **k):
        try:
            r = orig["solve_al"](*a, **k)
        except bench.TrajOptFailure as exc:
            rec["al_fail"] = exc
            raise
        rec["al"] = r
        return r

    bench.solve, bench.lift_placements, bench.solve_al = w_solve, w_lift, w_al

    path = os.path.join(HERE, "pipeline_reference.json")
    only = sys.argv[1:]  # optional: regenerate just these keys (e.g. tetris5@64k), merged into the file
    out = {"pipeline": {}, "stage1": {}}
    if only and os.path.exists(path):
        out = json.load(open(path))
    cases = [(name, name, {}, seeds) for name, seeds in PIPELINE.items()]
    cases += [(key, name, over, seeds) for key, (name, over, seeds) in PIPELINE_SIZED.items()]
    for key, name, over, seeds in cases:
        if only and key not in only:
            continue
        scene = ref_scene(name)
        for seed in seeds:
            rec.clear()
            sol = bench.solve_scene(scene, seed=seed, solver_overrides=over or None)
            s1 = rec["stage1"]
            entry = {"success": bool(sol.success), "restarts": int(sol.restarts),
                     "stage1_success": bool(s1.success), "stage1_indices": [int(i) for i in s1.indices],
                     "stage1_costs": [float(c) for c in s1.costs], "final_cost": float(sol.final_cost),
                     "lift_failed": "stage1" in rec and s1.success and "lift" not in rec,
                     "kept": [int(i) for i in rec["lift"].kept] if "lift" in rec else None,
                     "accepted_outer": len(rec["al"].report.outers) - 1 if "al" in rec else -1,
                     "al_particle": int(rec["al"].particle_index) if "al" in rec else -1,
                     "objective": float(rec["al"].objective) if "al" in rec else None,
                     "least_violation": float(rec["al_fail"].best_violation) if "al_fail" in rec else None}
            out["pipeline"][f"{key}/{seed}"] = entry
            print(key, seed, {k: v for k, v in entry.items() if k not in ("stage1_indices", "stage1_costs", "kept")},
                  flush=True)
    for name in STAGE1:
        if only and name not in only:
            continue
        scene = ref_scene(name)
        for seed in STAGE1_SEEDS:
            rec.clear()
            sol = bench.solve_scene(scene, seed=seed, no_trajopt=True)
            s1 = rec["stage1"]
            out["stage1"][f"{name}/{seed}"] = {
                "success": bool(sol.success), "restarts": int(sol.restarts),
                "stage1_indices": [int(i) for i in s1.indices], "stage1_costs": [float(c) for c in s1.costs]}
        print(name, "stage1", sum(v["success"] for k, v in out["stage1"].items() if k.startswith(name + "/")),
              "successes", flush=True)
    with open(path, "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print("wrote", path)


if __name__ == "__main__":
    main()
