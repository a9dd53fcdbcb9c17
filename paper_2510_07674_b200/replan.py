"""Reactive replanning (BASELINE configs[3], C4): a 6-block rearrangement whose one sphere
obstacle moves every tick, re-solved each tick warm-started from the previous tick's
placement.

The reference has no moving obstacles; its reactive mechanism is warm-start injection
(``inject_warm_start``, reference particle_opt.py:250-263, reached through
``bench.solve_scene(warm_seeds=...)``, bench.py:177,191). Each tick here rebuilds the scene
with the obstacle at its new centre (the scene/model construction is host work and is
timed as part of the tick), then calls ``bench_api.solve_scene`` with the previous tick's
best placement as the warm seed. The replan-rate sweep reports, for each target rate, the
fraction of ticks whose whole tick time met the deadline 1/rate.
"""
from __future__ import annotations

import math
import statistics
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .bench_api import solve_scene
from .problems import as_cost_model, load_scene
from .problems.scenes import tower6r

RATES_HZ = (10, 30, 100, 200)


def obstacle_center(tick: int, *, center=(0.45, -0.05, 0.28), radius=0.08, step_m=0.03):
    """Obstacle centre at `tick`: a horizontal circle of `radius` around `center`, advancing
    `step_m` of arc per tick (BASELINE C4: 1-5 cm per tick)."""
    phase = tick * step_m / radius
    return (center[0] + radius * math.cos(phase), center[1] + radius * math.sin(phase), center[2])


@dataclass
class Tick:
    tick: int
    success: bool
    tick_ms: float       # scene + model rebuild + solve (the replan latency)
    solve_ms: float      # bench.solve_scene's own span (stage 1 start to result)
    restarts: int
    warm: bool
    placement: Optional[np.ndarray] = None
    stats: dict = field(default_factory=dict)


def replan_loop(ticks: int, *, seed: int = 0, first_tick: int = 0, solver_overrides: Optional[dict] = None,
                precision: str = "fp32", step_m: float = 0.03, warm=None, comm=None):
    """Run `ticks` replanning ticks; returns (list of Tick, last placement)."""
    out = []
    for k in range(first_tick, first_tick + ticks):
        t0 = time.perf_counter()
        scene = load_scene(tower6r(obstacle_center=obstacle_center(k, step_m=step_m)))
        model = as_cost_model(scene.problem, precision=precision)
        sol = solve_scene(scene, seed=seed + k, solver_overrides=solver_overrides, precision=precision, model=model,
                          warm_seeds=None if warm is None else np.atleast_2d(warm), comm=comm)
        tick_ms = (time.perf_counter() - t0) * 1e3
        out.append(Tick(k, bool(sol.success), tick_ms, sol.time_ms, sol.restarts, warm is not None,
                        None if sol.placement is None else sol.placement.copy(), sol.stats))
        if sol.success:  # warm-start the next tick from every returned placement
            warm = (sol.particles if sol.particles is not None else sol.placement[None, :]).copy()
    return out, warm


def rate_sweep(tick_ms, rates=RATES_HZ):
    """Fraction of ticks meeting each replan deadline, plus the highest sustainable rate
    (1 / p99 tick time)."""
    t = np.asarray(tick_ms, dtype=float)
    p99 = float(np.percentile(t, 99)) if len(t) else math.inf
    return {"deadline_met": {str(r): float(np.mean(t <= 1000.0 / r)) for r in rates},
            "tick_ms_p50": float(statistics.median(t)) if len(t) else None, "tick_ms_p99": p99,
            "max_rate_hz": 1000.0 / p99 if p99 > 0 else None}
