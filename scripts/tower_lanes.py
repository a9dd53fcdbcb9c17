"""Stage-1 tower tile kernel: lanes per particle (spasm_set_option "tower_lanes") against
stage-1 device time and outcome (diagnostic). One process per setting (the option is read at
launch; the restart graph is keyed on it).
Usage: python scripts/tower_lanes.py LANES"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2510_07674_b200 import _native as nat  # noqa: E402
from paper_2510_07674_b200 import particle_opt as po  # noqa: E402
from paper_2510_07674_b200.problems import as_cost_model, load_scene  # noqa: E402

la = int(sys.argv[1])
lib = nat.load()
nat.check(lib.spasm_set_option(b"tower_lanes", la), "option")
for name in ("tower3c", "tower6r", "tower4"):
    sc = load_scene(name)
    m = as_cost_model(sc.problem, precision="fp32")
    over = {**sc.solver_overrides, "n": 16384, "m": 2048}
    ts, out = [], []
    for seed in range(-3, 30):
        cfg = po.OptimizerConfig(**{**over, "seed": max(seed, 0) + 1000 * (seed < 0)})
        r = po.solve(m, cfg)
        if seed >= 0:
            ts.append(r.report.device_ms)
            out.append((r.success, r.report.restarts, tuple(r.indices.tolist())))
    print(f"lanes={la} {name}: stage-1 device p50 {np.median(ts):.3f} ms; outcome hash {hash(tuple(out)) & 0xffffffff:08x}; "
          f"success {sum(o[0] for o in out)}/{len(out)}, restarts {sum(o[1] for o in out)}")
