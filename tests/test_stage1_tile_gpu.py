"""fp32 tetris tile kernel (stage1_tile.cuh) against the fp64 oracle and the generic
fp32 kernel (4 lanes per particle), tetris and tower scenes (stage1_tower_tile.cuh).

Tolerances (north_star: per-particle costs and gradients within rtol 1e-4 in fp32):
  * 0 steps: the kernel's final QUADRATIC cost vs the oracle on the same fp32-rounded rows,
    rtol 1e-4 / atol 1e-6;
  * one linear step (k_lin = 2: rates eta/2 then 0) and one quadratic step: the stepped
    state vs clip(x - rate * oracle_gradient(x)) on kink-free rows (margin > 1e-4), error
    <= 1e-4 x rate x max|g| per row; flags identical;
  * full schedules: the solve outcome (success, restart) matches the generic kernel and
    every returned placement satisfies the fp64 oracle.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import stage1 as orc
from paper_2510_07674_b200 import _native as nat
from paper_2510_07674_b200 import particle_opt as po
from paper_2510_07674_b200.problems import as_cost_model, load_scene

pytestmark = pytest.mark.gpu

SCENES = ["tetris4", "tetris5", "tetris6", "tetris8", "single1", "tower4", "tower3c", "tower6r"]
VARIANTS = [4]


def _set_tile(v):
    nat.check(nat.load().spasm_set_option(b"stage1_tile", v), "set_option")


@pytest.fixture(autouse=True)
def _reset_tile():
    yield
    _set_tile(-1)


def _schedule(model, x, k_lin, k_quad, eta, alpha):
    lib = nat.load()
    src = torch.as_tensor(x, device="cuda", dtype=torch.float32)
    P = src.shape[0]
    out_v = torch.empty_like(src)
    out_c = torch.empty(P, dtype=torch.float32, device="cuda")
    fl = torch.zeros(P, dtype=torch.uint8, device="cuda")
    nat.check(lib.spasm_descent_schedule(model.handle, model.dtype_id, nat.ptr(src), None, P, k_lin, k_quad, eta, alpha,
                                         1e-3, nat.ptr(out_v), nat.ptr(out_c), nat.ptr(fl), None, None, None, 0,
                                         nat.stream_handle()), "schedule")
    return out_v.double().cpu().numpy(), out_c.double().cpu().numpy(), fl.cpu().numpy().astype(bool)


def _rows(o, n, seed):
    x = np.random.default_rng(seed).uniform(o.lower, o.upper, size=(n, o.dimension))
    return x.astype(np.float32).astype(np.float64)


def test_set_option_rejects_bad_values():
    lib = nat.load()
    assert lib.spasm_set_option(b"stage1_tile", 9) == nat.SPASM_ERR_USAGE
    assert lib.spasm_set_option(b"tower_lanes", 3) == nat.SPASM_ERR_USAGE
    assert lib.spasm_set_option(b"no_such_option", 0) == nat.SPASM_ERR_USAGE


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("name", SCENES)
def test_tile_quadratic_cost_matches_oracle(name, variant):
    scene = load_scene(name)
    m = as_cost_model(scene.problem, precision="fp32")
    o = orc.oracle_model(scene.problem)
    x = _rows(o, 3001, 5)
    _set_tile(variant)
    v, c, fl = _schedule(m, x, 0, 0, 0.02, 0.1)
    np.testing.assert_array_equal(v, x)
    np.testing.assert_allclose(c, o.evaluate(x, "quadratic"), rtol=1e-4, atol=1e-6)
    assert not fl.any()


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("name", SCENES)
@pytest.mark.parametrize("mode", ["linear", "quadratic"])
def test_tile_one_step_matches_oracle_gradient(name, variant, mode):
    scene = load_scene(name)
    m = as_cost_model(scene.problem, precision="fp32")
    o = orc.oracle_model(scene.problem)
    x = _rows(o, 2048, 7)
    eta, alpha = 0.05, 0.1
    _set_tile(variant)
    if mode == "linear":
        v, _, fl = _schedule(m, x, 2, 0, eta, alpha)
        rate = eta / 2
    else:
        v, _, fl = _schedule(m, x, 0, 1, eta, alpha)
        rate = alpha
    g = o.gradient(x, mode)
    ref = np.clip(x - rate * g, o.lower, o.upper)
    ok = o.kink_margin(x) > 1e-4
    assert ok.mean() > 0.5
    scale = rate * np.maximum(np.abs(g[ok]).max(axis=1, keepdims=True), 1e-3)
    assert np.max(np.abs(v[ok] - ref[ok]) / scale) < 1e-4
    assert not fl.any()


@pytest.mark.parametrize("variant", VARIANTS)
def test_tile_full_schedule_tracks_generic_kernel(variant):
    scene = load_scene("tetris5")
    m = as_cost_model(scene.problem, precision="fp32")
    o = orc.oracle_model(scene.problem)
    x = _rows(o, 4096, 9)
    cfg = po.OptimizerConfig(**scene.solver_overrides)
    _set_tile(0)
    v0, c0, _ = _schedule(m, x, cfg.k_lin, cfg.k_quad, cfg.eta_init, cfg.alpha)
    _set_tile(variant)
    v1, c1, _ = _schedule(m, x, cfg.k_lin, cfg.k_quad, cfg.eta_init, cfg.alpha)
    # fp32 rounding differs between the two kernels; 22 steps keep most rows together
    close = np.all(np.abs(v1 - v0) < 1e-4, axis=1)
    assert close.mean() > 0.9
    sat0, sat1 = c0 < cfg.epsilon, c1 < cfg.epsilon
    assert abs(int(sat0.sum()) - int(sat1.sum())) <= max(2, 0.1 * sat0.sum())


@pytest.mark.parametrize("name", ["tetris4", "tetris5", "tetris6", "tetris8"])
def test_tile_solve_outcome_matches_generic(name):
    scene = load_scene(name)
    m = as_cost_model(scene.problem, precision="fp32")
    o = orc.oracle_model(scene.problem)
    over = {"n": 8192, "m": 1024} if name == "tetris8" else {}
    wins = [0, 0]
    for seed in range(8):
        cfg = po.OptimizerConfig(**{**scene.solver_overrides, **over, "seed": seed, "max_restarts": 3})
        for k, mode in enumerate((0, -1)):
            _set_tile(mode)
            res = po.solve(m, cfg)
            wins[k] += int(res.success)
            if res.success:
                assert np.all(o.evaluate(res.particles, "quadratic") < cfg.epsilon * 1.01)
    print(name, "successes generic / tile over 8 seeds:", wins)
    assert wins[0] == wins[1]


def _key_to_cost(keys):
    """Inverse of common.cuh order_key for fp32 keys."""
    k = keys.astype(np.uint32)
    b = np.where(k & np.uint32(0x80000000), k & np.uint32(0x7FFFFFFF), ~k)
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


@pytest.mark.parametrize("name", SCENES)
def test_tile_sample_eval_matches_generic_and_oracle(name):
    scene = load_scene(name)
    m = as_cost_model(scene.problem, precision="fp32")
    o = orc.oracle_model(scene.problem)
    lib = nat.load()
    n = 5000
    out = {}
    for mode in (0, -1):
        _set_tile(mode)
        vals = torch.empty((n, m.dimension), dtype=torch.float32, device="cuda")
        keys = torch.empty(n, dtype=torch.int32, device="cuda")
        idx = torch.empty(n, dtype=torch.int32, device="cuda")
        nat.check(lib.spasm_sample_eval(m.handle, m.dtype_id, 7, 3, nat.SAMPLER_PCG64, 100, n, None, 0, nat.ptr(vals),
                                        nat.ptr(keys), nat.ptr(idx), nat.stream_handle()), "sample_eval")
        out[mode] = (vals.double().cpu().numpy(), keys.cpu().numpy().view(np.uint32), idx.cpu().numpy())
    np.testing.assert_array_equal(out[0][0], out[-1][0])  # identical draws
    np.testing.assert_array_equal(out[-1][2], np.arange(100, 100 + n))
    c_tile = _key_to_cost(out[-1][1])
    np.testing.assert_allclose(c_tile, _key_to_cost(out[0][1]), rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(c_tile, o.evaluate(out[-1][0], "linear"), rtol=1e-4, atol=1e-6)


@pytest.mark.parametrize("name", ["tower4", "tower3c", "tower6r"])
def test_tower_lane_counts_agree(name):
    """The tower tile kernel with 1 / 2 / 4 / 8 lanes per particle (spasm_set_option
    "tower_lanes"; auto picks by obstacle count) differs only in the order of the
    cube-obstacle partial sums: one descent step agrees to fp32 rounding, and the full
    schedule's flags are identical."""
    lib = nat.load()
    scene = load_scene(name)
    m = as_cost_model(scene.problem, precision="fp32")
    o = orc.oracle_model(scene.problem)
    x = _rows(o, 2048, 11)
    over = scene.solver_overrides
    try:
        runs = {}
        for la in (1, 2, 4, 8):
            nat.check(lib.spasm_set_option(b"tower_lanes", la), "set_option")
            one = _schedule(m, x, 1, 0, over["eta_init"], over["alpha"])
            full = _schedule(m, x, over["k_lin"], over["k_quad"], over["eta_init"], over["alpha"])
            runs[la] = (one, full)
        v4, c4 = runs[4][0][0], runs[4][0][1]
        for la, ((v, c, _), (_, _, fl)) in runs.items():
            np.testing.assert_allclose(v, v4, rtol=1e-5, atol=1e-6)
            np.testing.assert_allclose(c, c4, rtol=1e-4, atol=1e-6)
            np.testing.assert_array_equal(fl, runs[4][1][2])
    finally:
        nat.check(lib.spasm_set_option(b"tower_lanes", 0), "set_option")
