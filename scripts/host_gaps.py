"""How much of a solve_scene's wall time is host-induced idle GPU time (diagnostic).
Times p50 wall per solve, then the same solves behind a GPU spin (torch.cuda._sleep) so that
every launch is enqueued before the GPU reaches it: the event span from the spin's end to
an event recorded after solve_scene returns is then GPU work plus the post-sync host tail.
Usage: python scripts/host_gaps.py [scene] [solves]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_2510_07674_b200.bench_api import solve_scene  # noqa: E402
from paper_2510_07674_b200.problems import as_cost_model, load_scene  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tower3c"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
scene = load_scene(name)
model = as_cost_model(scene.problem, precision="fp32")
for s in range(3):
    solve_scene(scene, seed=100 + s, model=model)
torch.cuda.synchronize()
wall, primed, tails = [], [], []
for s in range(n):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sol = solve_scene(scene, seed=s, model=model)
    wall.append((time.perf_counter() - t0) * 1e3)
for s in range(n):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(4_000_000)  # ~2 ms spin: the host enqueues the whole pipeline meanwhile
    e0.record()
    sol = solve_scene(scene, seed=s, model=model)
    e1.record()
    torch.cuda.synchronize()
    primed.append(e0.elapsed_time(e1))
print(f"{name}: wall p50 {np.median(wall):.3f} ms; primed (GPU work + post-sync host tail) p50 "
      f"{np.median(primed):.3f} ms; host-induced idle ~{np.median(wall) - np.median(primed):.3f} ms")

# per-stage GPU spans (primed): events recorded as each stage is enqueued
from paper_2510_07674_b200 import particle_opt as _po  # noqa: E402
from paper_2510_07674_b200 import trajopt as _to  # noqa: E402

marks = {}


def _wrap(mod, fname, tag):
    f = getattr(mod, fname)

    def g(*a, **k):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        marks[tag] = ev
        return f(*a, **k)

    setattr(mod, fname, g)


_wrap(_to, "_lift_async", "lift")
_wrap(_to, "_init_async", "init")
_wrap(_to, "_solve_al_device", "al")
rows = []
for s in range(n):
    torch.cuda.synchronize()
    marks.clear()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(4_000_000)
    e0.record()
    t0 = time.perf_counter()
    sol = solve_scene(scene, seed=s, model=model)
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    if "al" not in marks:
        continue
    rows.append((e0.elapsed_time(marks["lift"]), marks["lift"].elapsed_time(marks["init"]),
                 marks["init"].elapsed_time(marks["al"]), marks["al"].elapsed_time(e1)))
if rows:
    r = np.median(np.array(rows), axis=0)
    print(f"  primed spans p50 (ms): stage 1 {r[0]:.3f}  lift {r[1]:.3f}  init {r[2]:.3f}  "
          f"AL + finalize + validate + post-sync host tail {r[3]:.3f}")

# host time after the AL solve's sync until solve_scene returns
from paper_2510_07674_b200 import _native as _nat  # noqa: E402

lib = _nat.load()
_orig = lib.spasm_solve_al
t_al = {}


def _al(*a):
    r = _orig(*a)
    t_al["t"] = time.perf_counter()
    return r


lib.spasm_solve_al = _al
tails, devs = [], []
for s in range(n):
    torch.cuda.synchronize()
    sol = solve_scene(scene, seed=s, model=model)
    t1 = time.perf_counter()
    if "t" in t_al:
        tails.append((t1 - t_al.pop("t")) * 1e3)
print(f"  host tail after spasm_solve_al returns p50 {np.median(tails):.3f} ms (solve_scene time_ms p50 of the "
      f"last solve {sol.time_ms:.3f})")
