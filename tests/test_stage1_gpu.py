"""Stage-1 parity on the GPU: CUDA path (through the C-ABI) vs the reference's golden
outputs and the CPU oracle.

Tolerances:
  fp64 (parity precision): costs/gradients rtol 1e-10 vs the reference's own numbers;
      schedules, draws, selections and full solves identical (indices, flags, restarts).
  fp32 (perf precision, north_star): per-particle costs and gradients within rtol 1e-4
      of the fp64 oracle evaluated on the same fp32-rounded inputs, gradients compared on
      rows whose nearest hinge kink is > 1e-4 away (the reference's own kink filter idea,
      tests/test_problems.py:348-379).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import golden
from oracle import stage1 as orc
from paper_2510_07674_b200 import particle_opt as po
from paper_2510_07674_b200.problems import as_cost_model, load_scene
from scenes_util import CASES, case_problem

pytestmark = pytest.mark.gpu


def _random_rows(model, n, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(model.lower, model.upper, size=(n, model.dimension))


@pytest.mark.parametrize("case", sorted(CASES))
def test_fp64_costs_gradients_match_reference_golden(case):
    g = golden(f"stage1_{case}.npz")
    _, problem = case_problem(case)
    m = as_cost_model(problem, precision="fp64")
    for mode in ("linear", "quadratic"):
        np.testing.assert_allclose(m.evaluate(g["values"], mode), g[f"cost_{mode}"], rtol=1e-10, atol=1e-14)
        np.testing.assert_allclose(m.gradient(g["values"], mode), g[f"grad_{mode}"], rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("case", sorted(CASES))
def test_fp32_costs_gradients_within_rtol_1e4(case):
    _, problem = case_problem(case)
    m = as_cost_model(problem, precision="fp32")
    o = orc.oracle_model(problem)
    x = _random_rows(o, 4096, 11).astype(np.float32).astype(np.float64)
    margin = o.kink_margin(x)
    for mode in ("linear", "quadratic"):
        ref_c = o.evaluate(x, mode)
        got_c = m.evaluate(torch.as_tensor(x, device="cuda", dtype=torch.float32), mode).double().cpu().numpy()
        np.testing.assert_allclose(got_c, ref_c, rtol=1e-4, atol=1e-6)
        ref_g = o.gradient(x, mode)
        got_g = m.gradient(torch.as_tensor(x, device="cuda", dtype=torch.float32), mode).double().cpu().numpy()
        ok = margin > 1e-4
        assert ok.mean() > 0.5
        scale = np.maximum(np.abs(ref_g[ok]).max(axis=1, keepdims=True), 1e-3)
        assert np.max(np.abs(got_g[ok] - ref_g[ok]) / scale) < 1e-4


def test_fp32_wall_tangent_rows_stay_inactive():
    """Clamped rows sit exactly tangent to the huge wall spheres: no spurious hinge."""
    scene = load_scene("tetris5")
    m = as_cost_model(scene.problem, precision="fp32")
    rows = np.array([m.lower, m.upper, np.where(np.arange(15) % 2, m.lower, m.upper)])
    o = orc.oracle_model(scene.problem)
    for mode in ("linear", "quadratic"):
        np.testing.assert_allclose(m.evaluate(rows, mode), o.evaluate(rows, mode), rtol=1e-5, atol=1e-7)


@pytest.mark.parametrize("case", sorted(CASES))
def test_sampler_is_bit_exact_with_numpy_stream(case):
    g = golden(f"stage1_{case}.npz")
    _, problem = case_problem(case)
    m = as_cost_model(problem, precision="fp64")
    batch = po.sample_uniform(m, 24, po.restart_stream(7, 3))
    np.testing.assert_array_equal(batch.values.cpu().numpy(), g["draw_seed7_restart3"])


def test_sampler_shards_reproduce_the_centralized_draw():
    m = as_cost_model(load_scene("tetris8").problem, precision="fp64")
    full = np.random.default_rng(np.random.SeedSequence(entropy=5, spawn_key=(2,))).uniform(
        m.lower, m.upper, size=(3000, m.dimension))
    for off, n in ((0, 1000), (1000, 1000), (2000, 1000), (1234, 777)):
        s = po.RestartStream(5, 2, row_offset=off).uniform(m.lower, m.upper, (n, m.dimension))
        np.testing.assert_array_equal(s.cpu().numpy(), full[off:off + n])


def test_select_topk_matches_reference_stable_order():
    g = golden("stage1_engine.npz")
    b = po.ParticleBatch(values=np.zeros((300, 1)), costs=g["tie_costs"])
    np.testing.assert_array_equal(po.select_topk(b, 300), g["tie_order"])
    b = po.ParticleBatch(values=np.zeros((5000, 1)), costs=g["cont_costs"])
    np.testing.assert_array_equal(po.select_topk(b, 700), g["cont_top"])
    b = po.ParticleBatch(values=np.zeros((3, 1)), costs=np.array([1.0, 1.0, 0.0]))
    np.testing.assert_array_equal(po.select_topk(b, 2), [2, 0])


# the single-CTA variants' boundaries (512 x ITEMS keys), the cluster form's CTA-count and
# ITEMS boundaries (256 x ITEMS keys per CTA, up to 16 CTAs) and the multi-CTA path
@pytest.mark.parametrize("n", [1, 2, 31, 511, 512, 513, 1024, 1025, 2047, 2048, 2049, 4097, 8192, 8193, 16383, 16384,
                               16385, 32769, 61440, 65536, 65537, 100000])
def test_device_sort_large_with_ties(n):
    rng = np.random.default_rng(n)
    for dt in (torch.float32, torch.float64):
        c = np.floor(rng.uniform(0, 50, size=n)) * 0.125
        got = po._sort_indices(torch.as_tensor(c, device="cuda", dtype=dt), n).cpu().numpy()
        np.testing.assert_array_equal(got, np.argsort(c, kind="stable"))


@pytest.mark.parametrize("case", sorted(CASES))
def test_fp64_fused_schedule_replays_reference(case):
    g = golden(f"stage1_{case}.npz")
    _, problem = case_problem(case)
    m = as_cost_model(problem, precision="fp64")
    k_lin, k_quad, eta, alpha, eps = g["sched_cfg"]
    cfg = po.OptimizerConfig(n=64, m=16, k_lin=int(k_lin), k_quad=int(k_quad), eta_init=eta, alpha=alpha,
                             epsilon=eps)
    x = g["sched_in"].copy()
    x, fl, steps = po.run_descent_schedule(m, x, cfg)
    assert steps == int(k_lin) + int(k_quad)
    # 65-step tetris8 replays amplify 1e-16 summation-order differences to ~1e-11
    np.testing.assert_allclose(x, g["sched_out"], rtol=1e-8, atol=1e-9)
    np.testing.assert_array_equal(fl, g["sched_flagged"])


@pytest.mark.parametrize("case", ["domino2", "tetris5", "tower4", "tower4_free", "tetris8", "tetris5_free"])
def test_fp64_solve_matches_reference(case):
    g = golden(f"stage1_{case}.npz")
    _, problem = case_problem(case)
    m = as_cost_model(problem, precision="fp64")
    for seed in (0, 1):
        c = g[f"solve{seed}_cfg"]
        cfg = po.OptimizerConfig(n=int(c[0]), m=int(c[1]), k_lin=int(c[2]), k_quad=int(c[3]), eta_init=c[4],
                                 alpha=c[5], epsilon=c[6], p_return=int(c[7]), max_restarts=int(c[8]), seed=int(c[9]))
        res = po.solve(m, cfg)
        assert res.success == bool(g[f"solve{seed}_success"])
        np.testing.assert_array_equal(res.indices, g[f"solve{seed}_indices"])
        np.testing.assert_allclose(res.costs, g[f"solve{seed}_costs"], rtol=1e-6, atol=1e-12)
        np.testing.assert_allclose(res.particles, g[f"solve{seed}_particles"], rtol=1e-7, atol=1e-9)
        r = res.report
        np.testing.assert_array_equal([r.restarts, r.steps, r.n_satisfying, r.flagged], g[f"solve{seed}_report"])


def test_fp32_solve_tetris5_outcome_matches_oracle():
    scene = load_scene("tetris5")
    m = as_cost_model(scene.problem, precision="fp32")
    o = orc.oracle_model(scene.problem)
    for seed in range(3):
        cfg = po.OptimizerConfig(**{**scene.solver_overrides, "seed": seed, "max_restarts": 2})
        res = po.solve(m, cfg)
        ref = orc.solve(o, orc.OracleConfig(**{**scene.solver_overrides, "seed": seed, "max_restarts": 2}))
        assert res.success == ref.success
        assert res.report.restarts == ref.restarts
        # every returned placement is independently satisfying under the fp64 oracle
        assert np.all(o.evaluate(res.particles, "quadratic") < cfg.epsilon * 1.01)
        if res.success:
            assert res.indices[0] in set(ref.indices) or abs(res.costs[0] - ref.costs[0]) < 1e-6


def test_native_trace_matches_generic_trace():
    scene = load_scene("domino2")
    m = as_cost_model(scene.problem, precision="fp64")
    cfg = po.OptimizerConfig(n=256, m=32, k_lin=4, k_quad=3, eta_init=0.03, alpha=0.1, epsilon=2e-5, seed=3,
                             max_restarts=1)
    r = po.solve(m, cfg, trace=True)
    tr = r.report.trace
    assert tr.costs.shape == (7, 32) and tr.particle_ids.shape == (32,)
    o = orc.oracle_model(scene.problem)
    vals = orc.sample_uniform(o, 256, orc.restart_stream(3, 0))
    top = orc.select_topk(o.evaluate(vals, "linear"), 32)
    np.testing.assert_array_equal(tr.particle_ids, top)
    rows = []
    x = vals[top].copy()
    ocfg = orc.OracleConfig(n=256, m=32, k_lin=4, k_quad=3, eta_init=0.03, alpha=0.1, epsilon=2e-5)
    orc.run_descent_schedule(o, x, ocfg, trace_sink=lambda s, md, c, sat: rows.append((c.copy(), sat.copy())))
    np.testing.assert_allclose(tr.costs, np.array([c for c, _ in rows]), rtol=1e-9, atol=1e-13)
    np.testing.assert_array_equal(tr.satisfied, np.array([s for _, s in rows]))


def test_warm_start_survives_selection_native():
    scene = load_scene("tetris5")
    m = as_cost_model(scene.problem, precision="fp64")
    o = orc.oracle_model(scene.problem)
    cfg = po.OptimizerConfig(**{**scene.solver_overrides, "seed": 4})
    base = po.solve(m, cfg)
    assert base.success
    warm = base.particles[:1]
    res = po.solve(m, cfg, warm_seeds=warm)
    assert res.success and res.report.restarts == 0
    ref = orc.solve(o, orc.OracleConfig(**{**scene.solver_overrides, "seed": 4}), warm_seeds=warm)
    np.testing.assert_array_equal(res.indices, ref.indices)
    assert 0 in set(res.indices.tolist())


# ---- engine semantics with torch toy models (reference tests/test_particle_opt.py:30-89) ----
class AbsModel(po.CostModel):
    def __init__(self, center=0.3, lo=0.0, hi=1.0):
        super().__init__(1, np.array([lo]), np.array([hi]))
        self.center = center

    def evaluate(self, values, mode):
        r = (values[:, 0] - self.center).abs()
        return r * r if mode == "quadratic" else r

    def gradient(self, values, mode):
        d = values[:, 0] - self.center
        return (2.0 * d if mode == "quadratic" else torch.sign(d))[:, None]


class NeverModel(po.CostModel):
    def __init__(self):
        super().__init__(1, np.zeros(1), np.ones(1))

    def evaluate(self, values, mode):
        return 1.0 + values[:, 0] ** 2

    def gradient(self, values, mode):
        return 2.0 * values

    def satisfaction(self, values, epsilon=1e-3):
        return torch.zeros(len(values), dtype=torch.bool, device=values.device)


class NanGradModel(po.CostModel):
    def __init__(self, dim=2):
        super().__init__(dim, np.zeros(dim), np.ones(dim))

    def evaluate(self, values, mode):
        return values.sum(dim=1)

    def gradient(self, values, mode):
        g = torch.ones_like(values)
        g[values[:, 0] > 0.5, 0] = float("nan")
        return g


def small_config(**kw):
    d = dict(n=64, m=16, k_lin=5, k_quad=3, eta_init=0.1, alpha=0.05, epsilon=1e-3, p_return=8, max_restarts=4, seed=0)
    d.update(kw)
    return po.OptimizerConfig(**d)


def test_generic_solve_convex_1d_matches_oracle():
    model = AbsModel(0.3)
    res = po.solve(model, small_config(k_lin=20, k_quad=10))
    assert res.success and np.all(res.costs < 1e-3)

    class OAbs(orc.OracleModel):
        dimension, lower, upper = 1, np.array([0.0]), np.array([1.0])

        def evaluate(self, v, mode):
            r = np.abs(v[:, 0] - 0.3)
            return r * r if mode == "quadratic" else r

        def gradient(self, v, mode):
            d = v[:, 0] - 0.3
            return (2 * d if mode == "quadratic" else np.sign(d))[:, None]

    ref = orc.solve(OAbs(), orc.OracleConfig(n=64, m=16, k_lin=20, k_quad=10, eta_init=0.1, alpha=0.05, epsilon=1e-3,
                                              p_return=8, max_restarts=4, seed=0))
    np.testing.assert_array_equal(res.indices, ref.indices)
    np.testing.assert_allclose(res.particles, ref.particles, rtol=1e-12)


def test_generic_failure_is_normal_return():
    res = po.solve(NeverModel(), small_config(max_restarts=3))
    assert not res.success and len(res.particles) == 0
    assert res.report.restarts == 3 and res.report.steps == 3 * 8


def test_descend_freezes_nonfinite_gradient():
    model = NanGradModel(2)
    b = po.ParticleBatch(values=np.array([[0.2, 0.2], [0.8, 0.2]]), costs=np.full(2, np.inf))
    po.descend(b, model, "linear", 0.1)
    np.testing.assert_allclose(b.values[0], [0.1, 0.1])
    np.testing.assert_allclose(b.values[1], [0.8, 0.2])
    assert b.flagged[1] and not b.flagged[0]


def test_descend_clamps_and_unit_step():
    b = po.ParticleBatch(values=np.array([[0.5]]), costs=np.array([np.inf]))
    po.descend(b, AbsModel(0.3), "linear", 0.1)
    assert b.values[0, 0] == pytest.approx(0.4) and b.costs[0] == pytest.approx(0.1)
    b = po.ParticleBatch(values=np.array([[0.05]]), costs=np.array([np.inf]))
    po.descend(b, AbsModel(-5.0), "linear", 0.2)
    assert b.values[0, 0] == 0.0


def test_native_failure_report_counts_steps():
    # tetris8 with a tiny budget never satisfies: failure is a normal return
    scene = load_scene("tetris8")
    m = as_cost_model(scene.problem)
    cfg = po.OptimizerConfig(n=64, m=8, k_lin=2, k_quad=1, eta_init=0.03, alpha=0.1, epsilon=1e-12, max_restarts=3)
    res = po.solve(m, cfg)
    assert not res.success and res.report.restarts == 3 and res.report.steps == 9
