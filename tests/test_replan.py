"""C4 reactive replanning (replan.py): the moving-obstacle tick schedule and the rate sweep
on CPU; the warm-started replan loop on the GPU (every tick's placement satisfies the fp64
oracle for that tick's obstacle position)."""
from __future__ import annotations

import math

import numpy as np
import pytest

from oracle import stage1 as orc
from paper_2510_07674_b200.problems import load_scene
from paper_2510_07674_b200.problems.scenes import tower6r
from paper_2510_07674_b200.replan import obstacle_center, rate_sweep


@pytest.mark.parametrize("step", [0.01, 0.03, 0.05])
def test_obstacle_moves_step_per_tick(step):
    for k in range(5):
        a, b = np.array(obstacle_center(k, step_m=step)), np.array(obstacle_center(k + 1, step_m=step))
        chord = np.linalg.norm(b - a)
        assert chord == pytest.approx(step, rel=0.02)  # arc ~ chord for small steps
        assert a[2] == b[2]


def test_rate_sweep():
    r = rate_sweep([4.0, 6.0, 12.0, 40.0], rates=(10, 100))
    assert r["deadline_met"] == {"10": 1.0, "100": 0.5}
    assert r["tick_ms_p50"] == 9.0
    assert r["max_rate_hz"] == pytest.approx(1000.0 / np.percentile([4, 6, 12, 40], 99))


def test_tower6r_scene_tracks_the_obstacle():
    c = obstacle_center(3)
    scene = load_scene(tower6r(obstacle_center=c))
    np.testing.assert_allclose(scene.problem.obstacle_centers[0], c)


@pytest.mark.gpu
def test_replan_loop_warm_started_ticks_are_valid():
    from paper_2510_07674_b200.replan import replan_loop

    ticks, warm = replan_loop(4, seed=5, solver_overrides={"n": 8192, "m": 1024})
    assert all(t.success for t in ticks)
    assert [t.warm for t in ticks] == [False, True, True, True]
    for t in ticks:
        scene = load_scene(tower6r(obstacle_center=obstacle_center(t.tick)))
        o = orc.oracle_model(scene.problem)
        eps = scene.solver_overrides["epsilon"]
        assert o.evaluate(t.placement[None, :], "quadratic")[0] < eps * 1.01
    assert warm is not None and math.isfinite(ticks[-1].tick_ms)
