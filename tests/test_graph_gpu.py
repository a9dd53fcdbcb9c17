"""The stage-1 restart as a CUDA graph (capi.cu solve_impl; spasm_set_option("graphs")):
identical results to the stream-launched path, across seeds (one cached graph, new restart
inputs through device memory), multi-restart solves, warm starts and both precisions."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2510_07674_b200 import _native as nat
from paper_2510_07674_b200 import particle_opt as po
from paper_2510_07674_b200.problems import as_cost_model, load_scene

pytestmark = pytest.mark.gpu


def _graphs(v):
    nat.check(nat.load().spasm_set_option(b"graphs", v), "set_option")


@pytest.fixture(autouse=True)
def _reset():
    yield
    _graphs(1)


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("name,over", [("tetris5", {"n": 2048, "m": 256, "max_restarts": 4}),
                                       ("tower4", {"n": 3000, "m": 700, "max_restarts": 3}),
                                       ("tetris8", {"n": 16384, "m": 2048, "max_restarts": 2})])
def test_graph_matches_stream_path(precision, name, over):
    scene = load_scene(name)
    m = as_cost_model(scene.problem, precision=precision)
    for seed in range(4):
        cfg = po.OptimizerConfig(**{**scene.solver_overrides, **over, "seed": seed})
        _graphs(0)
        a = po.solve(m, cfg)
        _graphs(1)
        b = po.solve(m, cfg)
        assert a.success == b.success and a.report.restarts == b.report.restarts
        assert a.report.n_satisfying == b.report.n_satisfying
        assert a.report.steps == b.report.steps and a.report.flagged == b.report.flagged
        np.testing.assert_array_equal(a.indices, b.indices)
        np.testing.assert_array_equal(a.particles, b.particles)
        np.testing.assert_array_equal(a.costs, b.costs)


def test_graph_with_warm_seeds_and_rejected_option():
    scene = load_scene("tower4")
    m = as_cost_model(scene.problem, precision="fp32")
    cfg = po.OptimizerConfig(**{**scene.solver_overrides, "n": 2000, "m": 300, "seed": 9, "max_restarts": 2})
    warm = po.solve(m, po.OptimizerConfig(**{**scene.solver_overrides, "n": 4096, "m": 512, "seed": 1})).particles[:3]
    _graphs(0)
    a = po.solve(m, cfg, warm_seeds=warm)
    _graphs(1)
    b = po.solve(m, cfg, warm_seeds=warm)
    np.testing.assert_array_equal(a.indices, b.indices)
    assert nat.load().spasm_set_option(b"graphs", 2) == nat.SPASM_ERR_USAGE


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_device_restart_loop_runs_every_restart(precision):
    """The graph path's restart loop is a conditional WHILE node with the stop test on the
    device: an unsatisfiable scene must run exactly max_restarts restarts and report failure
    (particle_opt.py:385-400), and a scene that needs several restarts must stop at the same
    restart as the host-driven loop, with the same rows."""
    from test_step_cap import blocked_tower_scene

    scene = blocked_tower_scene()
    m = as_cost_model(scene.problem, precision=precision)
    cfg = po.OptimizerConfig(**{**scene.solver_overrides, "seed": 0, "max_restarts": 5})
    _graphs(1)
    for _ in range(3):  # the graph is captured on the second solve of a shape
        r = po.solve(m, cfg)
        assert not r.success and r.report.restarts == 5 and r.report.steps == 5 * (cfg.k_lin + cfg.k_quad)
    # tetris5 with a tiny batch: success usually needs restarts
    scene = load_scene("tetris5")
    m = as_cost_model(scene.problem, precision=precision)
    multi = 0
    for seed in range(6):
        cfg = po.OptimizerConfig(**{**scene.solver_overrides, "n": 64, "m": 8, "seed": seed, "max_restarts": 40})
        _graphs(0)
        a = po.solve(m, cfg)
        _graphs(1)
        po.solve(m, cfg)
        b = po.solve(m, cfg)
        assert a.success == b.success and a.report.restarts == b.report.restarts and a.report.steps == b.report.steps
        np.testing.assert_array_equal(a.indices, b.indices)
        np.testing.assert_array_equal(a.particles, b.particles)
        multi += a.report.restarts > 0
    assert multi > 0
