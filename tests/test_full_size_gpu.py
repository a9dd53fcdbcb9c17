"""BASELINE configs at their full sizes, checked through size-independent properties (the
CPU oracle cannot replay a 1M-particle schedule): every returned placement satisfies the
fp64 oracle's quadratic cost < epsilon; returned rows are distinct batch indices in
ascending cost order (the stable satisfying order); the full two-stage C1/C2 pipelines
return trajectories the fp64 oracle's independent validate accepts (trajopt.py:1071-1153)."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import stage1 as orc
from oracle import stage2 as orc2
from paper_2510_07674_b200 import particle_opt as po
from paper_2510_07674_b200.bench_api import solve_scene
from paper_2510_07674_b200.problems import as_cost_model, load_scene

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,over", [("tetris8", {"n": 1 << 20, "m": 1 << 17}),     # C5
                                       ("tetris5", {"n": 1 << 16, "m": 1 << 13}),     # C3
                                       ("tower3c", {}),                                # C2 stage 1
                                       ("tower6r", {"n": 16384, "m": 2048})])          # C4 stage 1
def test_full_size_stage1_placements_satisfy_fp64_oracle(name, over):
    scene = load_scene(name)
    model = as_cost_model(scene.problem, precision="fp32")
    o = orc.oracle_model(scene.problem)
    for seed in (0, 1):
        cfg = po.OptimizerConfig(**{**scene.solver_overrides, **over, "seed": seed, "max_restarts": 4})
        res = po.solve(model, cfg)
        assert res.success
        assert len(np.unique(res.indices)) == len(res.indices)
        assert np.all(np.diff(res.costs) >= 0)  # ascending satisfying order
        assert np.all(o.evaluate(res.particles, "quadratic") < cfg.epsilon * 1.01)
        assert np.all(res.particles >= o.lower - 1e-6) and np.all(res.particles <= o.upper + 1e-6)


@pytest.mark.parametrize("name", ["tower3c", "single1"])  # C2, C1 full pipelines
def test_full_pipeline_trajectory_passes_fp64_validate(name):
    scene = load_scene(name)
    model = as_cost_model(scene.problem, precision="fp32")
    g = orc2.build_geometry(scene.problem, scene.chain, scene.grasp, scene.obstacle_centers, scene.obstacle_radii)
    for seed in (0, 1):
        sol = solve_scene(scene, seed=seed, model=model)
        assert sol.success
        ok, worst = orc2.validate(sol.trajectory.segments, g)
        assert ok, (name, seed, worst)
