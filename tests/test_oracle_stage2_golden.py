"""Pin the stage-2 CPU oracle (oracle/stage2.py) to the (variant-B patched) reference's
own outputs frozen in tests/golden/stage2.npz."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from oracle import stage2 as o2
from paper_2510_07674_b200.problems import load_scene
from paper_2510_07674_b200.robot import planar_arm, spatial_arm_7dof

G = golden("stage2.npz")


@pytest.mark.parametrize("name,chain", [("spatial7", spatial_arm_7dof(1.3)), ("planar3", planar_arm())])
def test_fk_and_yaw_jacobian(name, chain):
    f = o2.fk(chain, G[f"fk_{name}_q"])
    for key, got in (("ee", f.ee), ("rot", f.rot), ("origins", f.origins), ("axes", f.axes), ("lpos", f.lpos),
                     ("lrot", f.lrot)):
        np.testing.assert_allclose(got, G[f"fk_{name}_{key}"], rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(o2.yaw_jac(f.rot, f.axes), G[f"fk_{name}_yawjac"], rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("scene_name", ["tower4", "tetris5"])
def test_ik_and_polish(scene_name):
    sc = load_scene(scene_name)
    tp, ty = G[f"ik_{scene_name}_tpos"], G[f"ik_{scene_name}_tyaw"]
    sol, ok, score = o2.ik_solve_batch(sc.chain, tp, ty, seed=3)
    np.testing.assert_array_equal(ok, G[f"ik_{scene_name}_ok"])
    np.testing.assert_allclose(sol, G[f"ik_{scene_name}_sol"], rtol=1e-9, atol=1e-10)
    pol, pok = o2.polish_tool_down(sc.chain, sol, tp, ty)
    np.testing.assert_array_equal(pok, G[f"polish_{scene_name}_ok"])
    np.testing.assert_allclose(pol, G[f"polish_{scene_name}_sol"], rtol=1e-8, atol=1e-9)


def _cfg(sc):
    return o2.TrajConfig(**sc.trajopt_overrides)


@pytest.mark.parametrize("scene_name", ["tower4", "tetris5", "corridor3"])
@pytest.mark.parametrize("mode", ["linear", "quadratic"])
def test_al_value_and_gradient(scene_name, mode):
    sc = load_scene(scene_name)
    kw = {} if scene_name == "corridor3" else dict(static_centers=sc.obstacle_centers, static_radii=sc.obstacle_radii)
    g = o2.build_geometry(sc.problem, sc.chain, sc.grasp, **kw)
    vals = G[f"al_{scene_name}_values"]
    obj, cons, lag, grad = o2.evaluate(vals, g, _cfg(sc), mode, G[f"al_{scene_name}_lam"], G[f"al_{scene_name}_mu"],
                                       True)
    np.testing.assert_allclose(obj, G[f"al_{scene_name}_{mode}_obj"], rtol=1e-12)
    np.testing.assert_allclose(cons, G[f"al_{scene_name}_{mode}_cons"], rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(lag, G[f"al_{scene_name}_{mode}_lag"], rtol=1e-11)
    np.testing.assert_allclose(grad, G[f"al_{scene_name}_{mode}_grad"], rtol=1e-10, atol=1e-9)


@pytest.mark.parametrize("scene_name", ["tower4", "tetris5", "corridor3"])
def test_validate(scene_name):
    sc = load_scene(scene_name)
    kw = {} if scene_name == "corridor3" else dict(static_centers=sc.obstacle_centers, static_radii=sc.obstacle_radii)
    g = o2.build_geometry(sc.problem, sc.chain, sc.grasp, **kw)
    vals = G[f"al_{scene_name}_values"]
    for p in range(3):
        ok, worst = o2.validate(vals[p], g, _cfg(sc).validation_epsilon)
        assert ok == bool(G[f"val_{scene_name}"][p, 0])
        assert worst == pytest.approx(G[f"val_{scene_name}"][p, 1], rel=1e-12)


def test_tower4_pipeline_lift_init_and_al():
    sc = load_scene("tower4")
    ends, kept = o2.lift_placements(sc.problem, G["pipe_tower4_placements"], sc.chain, sc.grasp, seed=0,
                                    static_centers=sc.obstacle_centers, static_radii=sc.obstacle_radii)
    np.testing.assert_array_equal(kept, G["pipe_tower4_kept"])
    np.testing.assert_allclose(ends, G["pipe_tower4_endpoints"], rtol=1e-8, atol=1e-9)
    cfg = _cfg(sc)
    vals = o2.init_trajectories(G["pipe_tower4_endpoints"], sc.chain, cfg, o2.trajectory_stream(0))
    np.testing.assert_array_equal(vals, G["pipe_tower4_init"])
    res = o2.solve_al(G["pipe_tower4_init"], sc.problem, sc.chain, cfg, sc.grasp, sc.obstacle_centers,
                      sc.obstacle_radii)
    assert len(res.outers) == int(G["pipe_tower4_al_outers"])
    assert res.particle_index == int(G["pipe_tower4_al_index"])
    np.testing.assert_allclose(res.objective, G["pipe_tower4_al_objective"], rtol=1e-7)
    np.testing.assert_allclose(res.outers[0].constraints, G["pipe_tower4_outer0_cons"], rtol=1e-6, atol=1e-10)
    np.testing.assert_allclose(res.values, G["pipe_tower4_al_values"], rtol=1e-6, atol=1e-8)


def test_corridor3_motion_al():
    sc = load_scene("corridor3")
    cfg = _cfg(sc)
    vals = o2.init_trajectories(np.stack([sc.problem.start, sc.problem.goal])[None, None], sc.chain, cfg,
                                o2.trajectory_stream(0))
    np.testing.assert_array_equal(vals, G["motion_corridor3_init"])
    res = o2.solve_al(vals, sc.problem, sc.chain, cfg)
    assert len(res.outers) == int(G["motion_corridor3_outers"])
    np.testing.assert_allclose(res.objective, G["motion_corridor3_objective"], rtol=1e-9)
    np.testing.assert_allclose(res.values, G["motion_corridor3_values"], rtol=1e-9, atol=1e-11)
