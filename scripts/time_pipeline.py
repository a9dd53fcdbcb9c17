"""Time the full two-stage pipeline (solve_scene) per scene and precision on cuda:0."""
import json
import statistics
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2510_07674_b200.bench_api import solve_scene
from paper_2510_07674_b200.problems import load_scene

scenes = sys.argv[1].split(",") if len(sys.argv) > 1 else ["tower4", "tower3c", "tetris5", "single1", "corridor3"]
precs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fp32", "fp64"]
trials = int(sys.argv[3]) if len(sys.argv) > 3 else 5
for name in scenes:
    sc = load_scene(name)
    for prec in precs:
        solve_scene(sc, seed=1000, precision=prec)  # warm-up
        torch.cuda.synchronize()
        ts, ok, viol = [], 0, []
        for s in range(trials):
            t0 = time.perf_counter()
            sol = solve_scene(sc, seed=s, precision=prec)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
            ok += int(sol.success)
            viol.append(sol.max_violation if sol.max_violation is not None else float("nan"))
        print(json.dumps({"scene": name, "precision": prec, "success": f"{ok}/{trials}",
                          "p50_wall_ms": statistics.median(ts), "min_ms": min(ts), "max_ms": max(ts),
                          "viol": [round(v, 5) for v in viol]}), flush=True)
