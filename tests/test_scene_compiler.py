"""Scene compiler: this repo's loader against the REFERENCE's loader
on every bundled scene (tests/golden/scenes_reference.npz, tests/golden/make_golden_scenes.py):
obstacle sphere tables (including the cuboid obstacle type, compiled to sphere grids),
explicit and builtin chains (the Franka-like 7-DOF chain of single1f), link spheres, tool,
grasp, staged poses, box and overrides -- all exactly equal. Plus the schema checks of the
cuboid extension."""
from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import golden
from paper_2510_07674_b200.problems import SceneError, load_scene
from paper_2510_07674_b200.problems.loader import cuboid_spheres
from paper_2510_07674_b200.problems.scenes import BUNDLED, cuboid_obstacle

G = golden("scenes_reference.npz")


@pytest.mark.parametrize("name", sorted(BUNDLED))
def test_loader_matches_reference_loader(name):
    sc = load_scene(name)
    key = f"{name}/obstacle_centers"
    if key in G:
        np.testing.assert_array_equal(sc.obstacle_centers, G[key])
        np.testing.assert_array_equal(sc.obstacle_radii, G[f"{name}/obstacle_radii"])
    else:
        assert sc.obstacle_centers is None or len(sc.obstacle_centers) == 0
    if f"{name}/axes" in G:
        ch = sc.chain
        np.testing.assert_array_equal(np.array([j.axis for j in ch.joints]), G[f"{name}/axes"])
        np.testing.assert_array_equal(np.array([j.offset for j in ch.joints]), G[f"{name}/offsets"])
        np.testing.assert_array_equal(np.array([[j.lower, j.upper] for j in ch.joints]), G[f"{name}/limits"])
        centers, radii, link = ch.sphere_table()
        np.testing.assert_array_equal(np.asarray(centers), G[f"{name}/sphere_centers"])
        np.testing.assert_array_equal(np.asarray(radii), G[f"{name}/sphere_radii"])
        np.testing.assert_array_equal(np.asarray(link), G[f"{name}/sphere_link"])
        np.testing.assert_array_equal(ch.tool_translation, G[f"{name}/tool_translation"])
        np.testing.assert_array_equal(ch.tool_rotation, np.eye(3))
    if f"{name}/grasp" in G:
        np.testing.assert_array_equal([*sc.grasp.offset, sc.grasp.yaw_offset], G[f"{name}/grasp"])
    if f"{name}/initial_poses" in G:
        np.testing.assert_array_equal([p.to_array() for p in sc.problem.initial_poses], G[f"{name}/initial_poses"])
    if f"{name}/box" in G:
        np.testing.assert_array_equal([sc.problem.box.min, sc.problem.box.max], G[f"{name}/box"])
    ref = json.loads(G[f"{name}/overrides"].tobytes().decode())
    assert sc.solver_overrides == ref["solver"] and sc.trajopt_overrides == ref["trajopt"]


def test_cuboid_grid_and_pose():
    c, r = cuboid_spheres([0.2, 0.2, 0.3], 0.05)
    assert c.shape == (2 * 2 * 3, 3) and np.all(r == 0.05)
    np.testing.assert_allclose(c.min(0), [-0.05, -0.05, -0.1])
    np.testing.assert_allclose(c.max(0), [0.05, 0.05, 0.1])
    d = BUNDLED["tower4"]()
    d["obstacles"] = [cuboid_obstacle([0.5, 0.0, 0.2], [0.2, 0.1, 0.1], 0.05, yaw=np.pi / 2)]
    sc = load_scene(d)
    # rotated a quarter turn: the 2 x 1 x 1 grid lies along y
    np.testing.assert_allclose(sorted(sc.obstacle_centers[:, 1]), [-0.05, 0.05], atol=1e-12)
    np.testing.assert_allclose(sc.obstacle_centers[:, 0], 0.5, atol=1e-12)


@pytest.mark.parametrize("bad,msg", [({"size": [0.1, 0.1], "sphere_radius": 0.05}, "size"),
                                     ({"size": [0.1, 0.1, -1], "sphere_radius": 0.05}, "strictly positive"),
                                     ({"size": [0.1, 0.1, 0.1]}, "sphere_radius")])
def test_cuboid_schema_errors_carry_json_path(bad, msg):
    d = BUNDLED["tower4"]()
    d["obstacles"] = [{"cuboid": bad, "pose": [0.5, 0, 0.2, 0]}]
    with pytest.raises(SceneError, match=r"\$\.obstacles\[0\]"):
        load_scene(d)
