"""STEP_CAP (reference bench.py:74-85) and the restart-exhaustion path, mirroring the
reference's tests/test_bench.py:156-163 (`test_trials_enforce_total_step_cap`) on its
unsatisfiable blocked-tower fixture (tests/test_bench.py:51-69)."""
from __future__ import annotations

import pytest

from paper_2510_07674_b200.bench_api import STEP_CAP, effective_max_restarts
from paper_2510_07674_b200.particle_opt import OptimizerConfig
from paper_2510_07674_b200.problems import load_scene


def blocked_tower_scene(**solver):
    overrides = {"n": 16, "m": 8, "epsilon": 1e-6}
    overrides.update(solver)
    return load_scene({
        "problem_type": "tower", "name": "blocked",
        "blocks": [{"name": "c1", "cells": [[0, 0]], "cell_size": 0.1},
                   {"name": "c2", "cells": [[0, 0]], "cell_size": 0.1}],
        "box": {"min": [0.35, 0.1, 0.08], "max": [0.6, 0.35, 0.5]}, "table_height": 0.05,
        "obstacles": [{"centers": [[0.475, 0.225, 0.3]], "radii": [5.0]}],
        "solver": overrides})


def test_effective_max_restarts_caps_total_steps():
    assert STEP_CAP == 30000
    assert effective_max_restarts(OptimizerConfig(k_lin=25, k_quad=5, max_restarts=5000)) == 1000
    assert effective_max_restarts(OptimizerConfig(k_lin=25, k_quad=40, max_restarts=64)) == 64
    assert effective_max_restarts(OptimizerConfig(k_lin=25, k_quad=40, max_restarts=5000)) == 30000 // 65
    # a schedule longer than the cap still gets one restart
    assert effective_max_restarts(OptimizerConfig(k_lin=40000, k_quad=0, max_restarts=7)) == 1
    # no steps at all: the cap does not apply
    assert effective_max_restarts(OptimizerConfig(k_lin=0, k_quad=0, max_restarts=9)) == 9


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_solve_scene_enforces_total_step_cap(precision):
    from paper_2510_07674_b200.bench_api import solve_scene
    from paper_2510_07674_b200.reporting import run_trials

    scene = blocked_tower_scene(k_lin=25, k_quad=5, max_restarts=5000)
    sol = solve_scene(scene, seed=0, precision=precision)
    assert not sol.success
    assert sol.restarts == STEP_CAP // 30
    assert sol.steps == STEP_CAP
    records, summary = run_trials(scene, 1, seed=0, precision=precision)
    (r,) = records
    assert not r.success and r.restarts == STEP_CAP // 30 and r.steps == STEP_CAP
    assert summary.successes == 0
