"""BASELINE configs[4] (C5): particle-count scaling sweep on the 8-object skeleton (tetris8),
N = 2^10 ... 2^22, M = N / 8, one GPU. Prints one JSON line per N: p50 solve time,
particle-iterations/s over device time, success rate. Usage: python scripts/sweep_c5.py [solves]"""
import json
import statistics
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2510_07674_b200.bench_api import solve_scene  # noqa: E402
from paper_2510_07674_b200.problems import as_cost_model, load_scene  # noqa: E402

solves = int(sys.argv[1]) if len(sys.argv) > 1 else 5
scene = load_scene("tetris8")
model = as_cost_model(scene.problem, precision="fp32")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for e in range(10, 23):
    n = 1 << e
    over = {"n": n, "m": max(1, n // 8)}
    solve_scene(scene, seed=10_000, solver_overrides=over, no_trajopt=True, model=model)  # warm-up
    dev, wall, its, ok = [], [], 0, 0
    stream = torch.cuda.current_stream()
    for s in range(solves):
        flush.fill_(s & 0xFF)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        sol = solve_scene(scene, seed=s, solver_overrides=over, no_trajopt=True, model=model)
        e1.record(stream)
        e1.synchronize()
        wall.append((time.perf_counter() - t0) * 1e3)
        dev.append(e0.elapsed_time(e1))
        its += sol.stats["stage1_iterations"]
        ok += int(sol.success)
    print(json.dumps({"n": n, "m": over["m"], "p50_solve_ms": statistics.median(wall),
                      "particle_iterations_per_s": its / (sum(dev) * 1e-3), "success_rate": ok / solves}))
