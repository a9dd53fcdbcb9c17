"""Lift kernel cluster size (spasm_set_option "ik_cluster") against the lift counters and the
pipeline solve time (diagnostic). Usage: python scripts/ik_cluster_sweep.py CS [scene]"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2510_07674_b200 import _native as nat  # noqa: E402
from paper_2510_07674_b200.bench_api import solve_scene  # noqa: E402
from paper_2510_07674_b200.problems import as_cost_model, load_scene  # noqa: E402

cs = int(sys.argv[1])
name = sys.argv[2] if len(sys.argv) > 2 else "tower3c"
lib = nat.load()
nat.check(lib.spasm_set_option(b"ik_cluster", cs), "option")
sc = load_scene(name)
model = as_cost_model(sc.problem, precision="fp32")
for s in range(3):
    solve_scene(sc, seed=100 + s, model=model)
out = np.zeros(12)
lib.spasm_ik_profile(1, None)
lib.spasm_ik_profile(1, out.ctypes.data)
ts = []
for s in range(10):
    ts.append(solve_scene(sc, seed=s, model=model).time_ms)
lib.spasm_ik_profile(0, out.ctypes.data)
n = max(1.0, out[0])
print(f"CS={cs} {name}: p50 {np.median(ts):.3f} ms; spec complete {out[6] / n * 100:.0f} %; mean end {out[2] / n:.0f}, "
      f"max end {out[9]:.0f} cycles; max polish {out[10]:.0f}")
