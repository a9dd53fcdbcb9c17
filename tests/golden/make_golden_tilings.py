"""Exhaustive grid-tiling oracle fixtures from the REFERENCE (its tests/_oracles.py:18-70
sweep, tests/test_problems.py:425-446: domino2 has exactly 2 tilings, tetris5 exactly 4),
extended to this repo's C3 scenes tetris4 / tetris6. Every grid-aligned assignment of block
origins is evaluated by the reference's TetrisCostModel in QUADRATIC mode; the satisfying set
(cost < 1e-9) is frozen into tests/golden/tilings.json.

    python tests/golden/make_golden_tilings.py
"""
from __future__ import annotations

import itertools
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")


def grid_placements(problem):  # tests/_oracles.py:18-27
    c = problem.cell_size
    out = []
    for block in problem.blocks:
        nx = int(round((problem.box.max[0] - problem.box.min[0] - block.width) / c))
        ny = int(round((problem.box.max[1] - problem.box.min[1] - block.height) / c))
        out.append([(i, j) for i in range(nx + 1) for j in range(ny + 1)])
    return out


def main():
    from seqplace.geometry import Pose
    from seqplace.problems import as_cost_model

    from oracle.refscene import ref_scene

    out = {}
    for name in ("domino2", "tetris4", "tetris5", "tetris6"):
        problem = ref_scene(name).problem
        model = as_cost_model(problem)
        per = grid_placements(problem)
        combos = list(itertools.product(*[range(len(p)) for p in per]))
        hits = []
        c = problem.cell_size
        for chunk in range(0, len(combos), 8192):
            part = combos[chunk:chunk + 8192]
            rows = np.array([model.row_from_poses([Pose(problem.box.min[0] + per[b][k][0] * c,
                                                        problem.box.min[1] + per[b][k][1] * c, problem.z_star, 0.0)
                                                   for b, k in enumerate(a)]) for a in part])
            hit = np.flatnonzero(model.evaluate(rows, "quadratic") < 1e-9)
            hits += [[int(v) for v in part[h]] for h in hit]
        out[name] = {"placements": [[list(cell) for cell in p] for p in per], "tilings": hits,
                     "assignments": len(combos)}
        print(name, len(combos), "assignments,", len(hits), "tilings", flush=True)
    with open(os.path.join(HERE, "tilings.json"), "w") as f:
        json.dump(out, f)


if __name__ == "__main__":
    main()
