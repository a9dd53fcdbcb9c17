"""CPU ORACLE of the reference's solve_scene composition -- test/bench infrastructure only.

Used by bench.py's cpu_baseline and --impl reference legs (the reference package itself is
pure Python and cannot travel to the GPU box; this is its float64 numpy restatement) and by
tests. Restates bench.solve_scene (reference bench.py:168-268): stage 1 -> lift_placements
-> init_trajectories -> solve_al, timed from the start of stage 1 to the result.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import stage1, stage2

STEP_CAP = 30000  # bench.py:74


@dataclass
class OracleSceneResult:
    success: bool
    time_ms: float
    stage1_iterations: int
    stage2_iterations: int
    max_violation: float
    # bookkeeping the pipeline-parity tests compare (bench.py:168-268 intermediates)
    restarts: int = -1
    stage1_indices: Optional[np.ndarray] = None
    kept: Optional[np.ndarray] = None
    accepted_outer: int = -1
    al_particle: int = -1
    objective: float = math.nan
    lift_failed: bool = False


def effective_max_restarts(cfg):  # bench.py:80-85
    per = cfg.k_lin + cfg.k_quad
    return cfg.max_restarts if per == 0 else min(cfg.max_restarts, max(1, STEP_CAP // per))


def solve_scene(scene, seed=0, threads=1, solver_overrides=None, no_trajopt=False, max_restarts=None,
                place_mode=None):
    o = stage1.oracle_model(scene.problem)
    cfg = stage1.OracleConfig(**{**scene.solver_overrides, **(solver_overrides or {})})
    cfg.seed = seed
    cfg.max_restarts = effective_max_restarts(cfg) if max_restarts is None else max_restarts
    t0 = time.perf_counter()
    res = stage1.solve(o, cfg, threads=threads)
    it1 = (res.restarts + 1 if res.success else cfg.max_restarts) * cfg.m * (cfg.k_lin + cfg.k_quad)
    rec = dict(restarts=int(res.restarts), stage1_indices=np.asarray(res.indices))
    if not res.success or scene.chain is None or no_trajopt:
        return OracleSceneResult(bool(res.success), (time.perf_counter() - t0) * 1e3, it1, 0, math.nan, **rec)
    tcfg = stage2.TrajConfig(**scene.trajopt_overrides)
    kept = None
    try:
        ends, kept = stage2.lift_placements(scene.problem, res.particles, scene.chain, scene.grasp, seed=seed,
                                            static_centers=scene.obstacle_centers,
                                            static_radii=scene.obstacle_radii)
        vals = stage2.init_trajectories(ends, scene.chain, tcfg, stage2.trajectory_stream(seed))
        al = stage2.solve_al(vals, scene.problem, scene.chain, tcfg, scene.grasp, scene.obstacle_centers,
                             scene.obstacle_radii, place_mode=place_mode)
    except stage2.LiftFailure:
        return OracleSceneResult(False, (time.perf_counter() - t0) * 1e3, it1, 0, math.nan, lift_failed=True, **rec)
    except stage2.TrajOptFailure as exc:
        it2 = len(exc.report) * len(vals) * tcfg.inner_steps
        return OracleSceneResult(False, (time.perf_counter() - t0) * 1e3, it1, it2, exc.best_violation,
                                 kept=np.asarray(kept), accepted_outer=-1, **rec)
    time_ms = (time.perf_counter() - t0) * 1e3
    it2 = len(al.outers) * len(vals) * tcfg.inner_steps
    g = stage2.build_geometry(scene.problem, scene.chain, scene.grasp, scene.obstacle_centers, scene.obstacle_radii)
    ok, worst = stage2.validate(al.values, g, tcfg.validation_epsilon)
    return OracleSceneResult(bool(ok), time_ms, it1, it2, float(worst), kept=np.asarray(kept),
                             accepted_outer=len(al.outers) - 1, al_particle=int(al.particle_index),
                             objective=float(al.objective), **rec)
