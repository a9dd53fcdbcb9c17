"""Stage-2 parity on the GPU: the CUDA trajectory path (through the C-ABI) vs the
(variant-B patched) reference's golden outputs and the CPU oracle (oracle/stage2.py).

Tolerances:
  fp64: FK/yaw-Jacobian rtol 1e-12; AL value/constraints rtol 1e-10, gradients rtol 1e-9
      (relative to the gradient scale); validation exact flags, violation rtol 1e-10; IK /
      polish identical success flags and solutions within 1e-8; init_trajectories bit-exact;
      whole AL solves: identical accepted outer, particle index and feasibility flags,
      objective rtol 1e-6 (hundreds of chained descent steps, as the oracle's own pin).
  fp32 (throughput path): costs and constraints rtol 1e-4 (atol 1e-5) vs the fp64 oracle on
      the same fp32-rounded inputs; gradients per particle within relative norm error 1e-4
      (north_star's rtol 1e-4, measured as the reference's AL-gradient tests measure it).
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import golden, rel_err
from oracle import stage2 as o2
from paper_2510_07674_b200 import trajopt as tj
from paper_2510_07674_b200.problems import load_scene
from paper_2510_07674_b200.robot import planar_arm, spatial_arm_7dof

pytestmark = pytest.mark.gpu
G = golden("stage2.npz")


def _cfg(sc):
    return tj.TrajOptConfig(**sc.trajopt_overrides)


def _kw(sc, name):
    return {} if name == "corridor3" else dict(grasp=sc.grasp, static_centers=sc.obstacle_centers,
                                               static_radii=sc.obstacle_radii)


@pytest.mark.parametrize("name,chain", [("spatial7", spatial_arm_7dof(1.3)), ("planar3", planar_arm())])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_fk_and_yaw_jacobian(name, chain, precision):
    q = G[f"fk_{name}_q"]
    if precision == "fp32":
        q = q.astype(np.float32).astype(np.float64)
    ee, rot, org, axs, yj = tj.fk_batch_device(chain, q, precision=precision)
    f = o2.fk(chain, q)
    tol = dict(rtol=1e-12, atol=1e-13) if precision == "fp64" else dict(rtol=1e-4, atol=2e-6)
    np.testing.assert_allclose(ee, f.ee, **tol)
    np.testing.assert_allclose(rot, f.rot, **tol)
    np.testing.assert_allclose(org, f.origins, **tol)
    np.testing.assert_allclose(axs, f.axes, **tol)
    np.testing.assert_allclose(yj, o2.yaw_jac(f.rot, f.axes), **(tol if precision == "fp64" else dict(atol=1e-4)))
    if precision == "fp64":
        np.testing.assert_allclose(ee, G[f"fk_{name}_ee"], rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(yj, G[f"fk_{name}_yawjac"], rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("scene_name", ["tower4", "tetris5"])
def test_ik_and_polish_match_reference(scene_name):
    sc = load_scene(scene_name)
    tp, ty = G[f"ik_{scene_name}_tpos"], G[f"ik_{scene_name}_tyaw"]
    sol, ok, score = tj.ik_solve_batch(sc.chain, (tp, ty), seed=3)
    np.testing.assert_array_equal(ok, G[f"ik_{scene_name}_ok"])
    np.testing.assert_allclose(sol, G[f"ik_{scene_name}_sol"], rtol=1e-8, atol=1e-8)
    np.testing.assert_allclose(score, G[f"ik_{scene_name}_score"], rtol=1e-4, atol=1e-9)
    pol, pok = tj.polish_tool_down(sc.chain, G[f"ik_{scene_name}_sol"], tp, ty)
    np.testing.assert_array_equal(pok, G[f"polish_{scene_name}_ok"])
    np.testing.assert_allclose(pol, G[f"polish_{scene_name}_sol"], rtol=1e-7, atol=1e-8)


@pytest.mark.parametrize("scene_name", ["tower4", "tetris5", "corridor3"])
@pytest.mark.parametrize("mode", ["linear", "quadratic"])
def test_al_value_and_gradient_match_reference_fp64(scene_name, mode):
    sc = load_scene(scene_name)
    vals, lam, mu = G[f"al_{scene_name}_values"], G[f"al_{scene_name}_lam"], G[f"al_{scene_name}_mu"]
    obj, cons = tj.trajectory_cost(vals, sc.problem, sc.chain, _cfg(sc), mode=mode, **_kw(sc, scene_name))
    np.testing.assert_allclose(obj, G[f"al_{scene_name}_{mode}_obj"], rtol=1e-10)
    np.testing.assert_allclose(cons, G[f"al_{scene_name}_{mode}_cons"], rtol=1e-10, atol=1e-13)
    lag, grad = tj.al_value_and_gradient(vals, sc.problem, sc.chain, _cfg(sc), lam, mu, mode=mode,
                                         **_kw(sc, scene_name))
    np.testing.assert_allclose(lag, G[f"al_{scene_name}_{mode}_lag"], rtol=1e-10)
    ref = G[f"al_{scene_name}_{mode}_grad"]
    scale = np.abs(ref).max()
    assert np.abs(grad - ref).max() <= 1e-9 * scale


@pytest.mark.parametrize("scene_name", ["tower4", "tetris5", "corridor3", "single1", "tower3c"])
def test_al_value_and_gradient_vs_oracle_near_feasible(scene_name):
    """Trajectories near a feasible plan (small random perturbations of the oracle's lifted
    interpolations) exercise active contacts and placement terms, not only far-off rows."""
    sc = load_scene(scene_name)
    cfg = _cfg(sc)
    kw = _kw(sc, scene_name)
    B = 1 if scene_name == "corridor3" else len(sc.problem.initial_poses)
    T = cfg.waypoints_per_segment
    rng = np.random.default_rng(5)
    lo, hi = sc.chain.lower, sc.chain.upper
    base = rng.uniform(lo, hi, size=(1, B, 1, sc.chain.dof))
    vals = np.clip(base + 0.3 * rng.standard_normal((6, B, T, sc.chain.dof)), lo, hi)
    lam = rng.uniform(0, 2, size=(6, 3))
    mu = rng.uniform(5, 20, size=6)
    g = o2.build_geometry(sc.problem, sc.chain, sc.grasp, kw.get("static_centers"), kw.get("static_radii"))
    for mode in ("linear", "quadratic"):
        ro, rc, rl, rg = o2.evaluate(vals, g, o2.TrajConfig(**sc.trajopt_overrides), mode, lam, mu, True)
        lag, grad = tj.al_value_and_gradient(vals, sc.problem, sc.chain, cfg, lam, mu, mode=mode, **kw)
        obj, cons = tj.trajectory_cost(vals, sc.problem, sc.chain, cfg, mode=mode, **kw)
        np.testing.assert_allclose(obj, ro, rtol=1e-10)
        rc0 = o2.evaluate(vals, g, o2.TrajConfig(**sc.trajopt_overrides), mode, 0 * lam, 0 * mu, False)[1]
        np.testing.assert_allclose(cons, rc0, rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(lag, rl, rtol=1e-10)
        assert np.abs(grad - rg).max() <= 1e-9 * max(np.abs(rg).max(), 1.0)
        # fp32 throughput path on the same rounded inputs
        v32 = vals.astype(np.float32).astype(np.float64)
        ro, rc, rl, rg = o2.evaluate(v32, g, o2.TrajConfig(**sc.trajopt_overrides), mode, lam, mu, True)
        lag32, grad32 = tj.al_value_and_gradient(v32, sc.problem, sc.chain, cfg, lam, mu, mode=mode, precision="fp32",
                                                 **kw)
        np.testing.assert_allclose(lag32, rl, rtol=1e-4, atol=1e-4)
        # north_star: per-particle gradients within rtol 1e-4 (fp32), as the per-particle
        # relative norm error the reference's own AL-gradient tests use (conftest.rel_err)
        per = [rel_err(grad32[p], rg[p]) for p in range(len(rg))]
        print(scene_name, mode, "fp32 AL gradient per-particle rel err max", max(per),
              "elementwise max / scale", np.abs(grad32 - rg).max() / max(np.abs(rg).max(), 1.0))
        assert max(per) <= 1e-4, per


@pytest.mark.parametrize("scene_name", ["tower4", "tetris5", "corridor3"])
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_validate_matches_reference(scene_name, precision):
    sc = load_scene(scene_name)
    vals = G[f"al_{scene_name}_values"]
    kw = _kw(sc, scene_name)
    feas, viol = tj.validate_batch(vals, sc.problem, sc.chain, epsilon=_cfg(sc).validation_epsilon,
                                   precision=precision, **kw)
    ref = G[f"val_{scene_name}"]
    np.testing.assert_array_equal(feas, ref[:, 0].astype(bool))
    np.testing.assert_allclose(viol, ref[:, 1], rtol=1e-10 if precision == "fp64" else 1e-4)


def test_init_trajectories_bit_exact():
    sc = load_scene("tower4")
    cfg = _cfg(sc)
    ends = G["pipe_tower4_endpoints"]
    got = tj.init_trajectories(ends, sc.chain, cfg, tj.trajectory_stream(0))
    np.testing.assert_array_equal(got, G["pipe_tower4_init"])
    cfg2 = tj.TrajOptConfig(**{**sc.trajopt_overrides, "k_waypoint": 2, "k_interp": 3})
    rng_ref, rng_dev = tj.trajectory_stream(7), tj.trajectory_stream(7)
    ref = o2.init_trajectories(ends, sc.chain, cfg2, rng_ref)
    got = tj.init_trajectories(ends, sc.chain, cfg2, rng_dev)
    np.testing.assert_array_equal(got, ref)
    # the caller's generator advanced exactly as numpy's would
    assert rng_ref.bit_generator.state == rng_dev.bit_generator.state


def test_lift_placements_tower4_matches_reference():
    sc = load_scene("tower4")
    res = tj.lift_placements(sc.problem, G["pipe_tower4_placements"], sc.chain, sc.grasp, seed=0,
                             static_centers=sc.obstacle_centers, static_radii=sc.obstacle_radii)
    np.testing.assert_array_equal(res.kept, G["pipe_tower4_kept"])
    np.testing.assert_allclose(res.endpoints, G["pipe_tower4_endpoints"], rtol=1e-7, atol=1e-8)


def test_solve_al_tower4_matches_reference():
    sc = load_scene("tower4")
    res = tj.solve_al(G["pipe_tower4_init"], sc.problem, sc.chain, _cfg(sc), grasp=sc.grasp,
                      static_centers=sc.obstacle_centers, static_radii=sc.obstacle_radii)
    assert len(res.report.outers) == int(G["pipe_tower4_al_outers"])
    assert res.particle_index == int(G["pipe_tower4_al_index"])
    np.testing.assert_allclose(res.objective, G["pipe_tower4_al_objective"], rtol=1e-6)
    np.testing.assert_allclose(res.report.outers[0].constraints, G["pipe_tower4_outer0_cons"], rtol=1e-5,
                               atol=1e-9)
    np.testing.assert_allclose(res.trajectory.segments, G["pipe_tower4_al_values"], rtol=1e-5, atol=1e-7)


def test_solve_al_corridor3_matches_reference():
    sc = load_scene("corridor3")
    res = tj.solve_al(G["motion_corridor3_init"], sc.problem, sc.chain, _cfg(sc))
    assert len(res.report.outers) == int(G["motion_corridor3_outers"])
    np.testing.assert_allclose(res.objective, G["motion_corridor3_objective"], rtol=1e-8)
    np.testing.assert_allclose(res.trajectory.segments, G["motion_corridor3_values"], rtol=1e-7, atol=1e-9)


def test_solve_al_bookkeeping_matches_oracle():
    """OuterRecord bookkeeping: lam+ = lam + mu c exactly; mu grows by beta iff the max
    violation did not shrink 10x (trajopt.py:1051-1054)."""
    sc = load_scene("tower4")
    cfg = tj.TrajOptConfig(**{**sc.trajopt_overrides, "outer_iters": 3, "inner_steps": 5})
    try:
        res = tj.solve_al(G["pipe_tower4_init"], sc.problem, sc.chain, cfg, grasp=sc.grasp,
                          static_centers=sc.obstacle_centers, static_radii=sc.obstacle_radii)
        outers = res.report.outers
    except tj.TrajOptFailure as exc:
        outers = exc.report.outers
    for r in outers:
        np.testing.assert_array_equal(r.updated_multipliers, r.multipliers + r.mu[:, None] * r.constraints)
    for a, b in zip(outers, outers[1:]):
        np.testing.assert_array_equal(b.multipliers, a.updated_multipliers)


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_solve_scene_tower4_end_to_end(precision):
    from paper_2510_07674_b200.bench_api import solve_scene

    sol = solve_scene(load_scene("tower4"), seed=0, precision=precision)
    assert sol.success
    assert sol.trajectory is not None and sol.max_violation < 0.02


def test_solve_scene_motion_corridor3():
    from paper_2510_07674_b200.bench_api import solve_scene

    sol = solve_scene(load_scene("corridor3"), seed=0, precision="fp64")
    assert sol.success


@pytest.mark.parametrize("name,precision", [("tower3c", "fp32"), ("single1", "fp32"), ("tower4", "fp64"),
                                            ("tetris5", "fp32")])
def test_device_recheck_equals_validate(name, precision):
    """solve_scene's independent float64 re-check (bench.py:249) runs on the device behind the
    AL solve (spasm_solve_al checked_*); it must equal trajopt.validate on the returned
    trajectory, bit for bit."""
    from paper_2510_07674_b200.bench_api import solve_scene

    sc = load_scene(name)
    for seed in (0, 4):
        sol = solve_scene(sc, seed=seed, precision=precision)
        if sol.trajectory is None:
            continue
        ok, worst = tj.validate(sol.trajectory, sc.problem, sc.chain, grasp=sc.grasp, static_centers=sc.obstacle_centers,
                                static_radii=sc.obstacle_radii, epsilon=_cfg(sc).validation_epsilon, precision="fp64")
        assert sol.success == ok and sol.max_violation == worst


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_al_best_host_equals_device_result(precision):
    """The accepted trajectory staged in pinned memory by spasm_solve_al's one D2H copy
    (spasm_al_best_host) equals the device result widened to float64, bit for bit; a handle
    with nothing staged refuses."""
    sc = load_scene("tower4")
    geo = tj._geometry(sc.problem, sc.chain, sc.grasp, sc.obstacle_centers, sc.obstacle_radii)
    with pytest.raises(Exception):
        tj._best_host(geo, torch.empty((geo.n_segments, 1, 1)))
    v, _ = tj._device(G["pipe_tower4_init"], precision)
    status, res, best, _ = tj._solve_al_device(geo, v.clone(), _cfg(sc), None, precision, want_report=False)
    assert status == 0
    np.testing.assert_array_equal(tj._best_host(geo, best), best.double().cpu().numpy())


@pytest.mark.parametrize("name", ["tower3c", "tetris5", "single1"])
def test_lift_invariant_to_cluster_size(name):
    """The lift kernel deals each group's restarts over a thread-block cluster (selection
    slots in rank 0's shared memory); the winners, their polished solutions and the kept set
    must not depend on the cluster size (spasm_set_option "ik_cluster")."""
    from paper_2510_07674_b200 import _native as nat
    from paper_2510_07674_b200 import particle_opt as po
    from paper_2510_07674_b200.problems import as_cost_model

    lib = nat.load()
    sc = load_scene(name)
    model = as_cost_model(sc.problem, precision="fp32")
    res = po.solve(model, po.OptimizerConfig(**{**sc.solver_overrides, "seed": 3}))
    assert res.success
    outs = {}
    try:
        for cs in (1, 2, 4, 8):
            nat.check(lib.spasm_set_option(b"ik_cluster", cs), "set_option")
            for seed in range(4):
                r = tj.lift_placements(sc.problem, res.particles, sc.chain, sc.grasp, seed=seed,
                                       static_centers=sc.obstacle_centers, static_radii=sc.obstacle_radii,
                                       precision="fp32")
                outs[cs, seed] = (r.kept, r.endpoints)
    finally:
        nat.check(lib.spasm_set_option(b"ik_cluster", 0), "set_option")
    for (cs, seed), (kept, ends) in outs.items():
        np.testing.assert_array_equal(kept, outs[1, seed][0])
        np.testing.assert_array_equal(ends, outs[1, seed][1])
