"""Handle lifetimes around the process-wide caches: the pinned result-staging
pool (capi.cu pinned_get / pinned_put, spasm_trim) and the shape-keyed solve workspace
(particle_opt._Workspace). Models and trajectory handles of different shapes (D, p_return)
are created, solved, destroyed and recreated in alternation -- with spasm_trim in between --
and every result must equal the first solve of that configuration bit for bit. Also checks
the launch / device-rows / collect split of spasm_solve against spasm_solve itself."""
from __future__ import annotations

import gc

import numpy as np
import pytest
import torch

from paper_2510_07674_b200 import _native as nat
from paper_2510_07674_b200 import particle_opt as po
from paper_2510_07674_b200.bench_api import solve_scene
from paper_2510_07674_b200.problems import as_cost_model, load_scene

pytestmark = pytest.mark.gpu

CONFIGS = [("tetris5", {"n": 2048, "m": 256, "p_return": 4}), ("tower4", {"n": 1000, "m": 300, "p_return": 7}),
           ("tetris8", {"n": 4096, "m": 512, "p_return": 2}), ("single1", {"n": 512, "m": 128, "p_return": 16})]


def _solve(name, over, seed):
    scene = load_scene(name)
    model = as_cost_model(scene.problem, precision="fp32")
    cfg = po.OptimizerConfig(**{**scene.solver_overrides, **over, "seed": seed, "max_restarts": 3})
    a = po.solve(model, cfg)
    b = po.solve(model, cfg)  # second solve of the shape: the restart-loop graph
    del model
    gc.collect()
    return a, b


def test_models_of_alternating_shapes_reuse_pinned_pool_and_workspace():
    first = {}
    for rnd in range(3):
        for name, over in CONFIGS:
            a, b = _solve(name, over, seed=rnd % 2)
            for r in (a, b):
                key = (name, rnd % 2)
                ref = first.setdefault(key, r)
                assert r.success == ref.success and r.report.restarts == ref.report.restarts
                np.testing.assert_array_equal(r.indices, ref.indices)
                np.testing.assert_array_equal(r.particles, ref.particles)
                np.testing.assert_array_equal(r.costs, ref.costs)
        assert nat.load().spasm_trim() == nat.SPASM_OK


def test_pipelines_with_trajectory_handles_repeat_exactly():
    runs = {}
    for rnd in range(2):
        for name in ("tower4", "single1", "tower3c"):
            sol = solve_scene(load_scene(name), seed=1)
            prev = runs.setdefault(name, sol)
            assert sol.success == prev.success
            np.testing.assert_array_equal(sol.trajectory.segments, prev.trajectory.segments)
        nat.load().spasm_trim()


def test_launch_device_rows_collect_match_solve():
    scene = load_scene("tetris5")
    model = as_cost_model(scene.problem, precision="fp32")
    cfg = po.OptimizerConfig(**{**scene.solver_overrides, "n": 2048, "m": 256, "seed": 5, "max_restarts": 4})
    ref = po.solve(model, cfg)
    for _ in range(2):  # host-loop path, then the graph path
        pend = po.solve_launch(model, cfg)
        rows_ptr, count_ptr = pend.device_rows()
        res = pend.collect()
        count = torch.empty(1, dtype=torch.int32, device="cuda")
        rows = torch.empty((cfg.p_return, model.dimension), dtype=torch.float64, device="cuda")
        # read the device rows: device-to-device copies from the raw pointers
        nat.check(_d2d(rows.data_ptr(), rows_ptr, rows.numel() * 8), "d2d")
        nat.check(_d2d(count.data_ptr(), count_ptr, 4), "d2d")
        k = int(count.item())
        assert k == len(res.indices) == len(ref.indices)
        np.testing.assert_array_equal(rows[:k].cpu().numpy(), res.particles)
        np.testing.assert_array_equal(res.indices, ref.indices)
        np.testing.assert_array_equal(res.particles, ref.particles)


def _d2d(dst, src, nbytes):
    import ctypes

    lib = ctypes.CDLL("libcudart.so.12") if _d2d.lib is None else _d2d.lib
    _d2d.lib = lib
    lib.cudaMemcpy.restype = ctypes.c_int
    lib.cudaMemcpy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    return lib.cudaMemcpy(ctypes.c_void_p(dst), ctypes.c_void_p(src), nbytes, 3)  # cudaMemcpyDeviceToDevice


_d2d.lib = None
