"""Scene-compiler golden fixtures: every bundled scene of this repo (including the BASELINE
mappings, the cuboid obstacles and the Franka-like explicit chain) loaded by the REFERENCE's
own loader (loader.py:291-455; cuboids expanded by oracle/refscene.py into the sphere sets
the reference schema takes), frozen into tests/golden/scenes_reference.npz: obstacle
spheres, chain joints / limits / link spheres / tool, grasp, staged poses and the overrides.
tests/test_scene_compiler.py checks this repo's loader against it.

    python tests/golden/make_golden_scenes.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")


def main():
    from oracle.refscene import ref_scene
    from paper_2510_07674_b200.problems.scenes import BUNDLED

    out = {}
    for name in BUNDLED:
        sc = ref_scene(name)
        p = sc.problem
        if sc.obstacle_centers is not None and len(sc.obstacle_centers):
            out[f"{name}/obstacle_centers"] = np.asarray(sc.obstacle_centers, float)
            out[f"{name}/obstacle_radii"] = np.asarray(sc.obstacle_radii, float)
        if sc.chain is not None:
            ch = sc.chain
            out[f"{name}/axes"] = np.array([j.axis for j in ch.joints], float)
            out[f"{name}/offsets"] = np.array([j.offset for j in ch.joints], float)
            out[f"{name}/limits"] = np.array([[j.lower, j.upper] for j in ch.joints], float)
            cs, rs, link = [], [], []
            for k, ss in enumerate(ch.link_spheres):
                if ss is None:
                    continue
                cs.append(np.asarray(ss.centers, float))
                rs.append(np.asarray(ss.radii, float))
                link += [k] * len(ss.radii)
            out[f"{name}/sphere_centers"] = np.concatenate(cs)
            out[f"{name}/sphere_radii"] = np.concatenate(rs)
            out[f"{name}/sphere_link"] = np.array(link)
            out[f"{name}/tool_translation"] = np.asarray(ch.tool_translation, float)
        if sc.grasp is not None:
            out[f"{name}/grasp"] = np.array([*sc.grasp.offset, sc.grasp.yaw_offset], float)
        if getattr(p, "initial_poses", None):
            out[f"{name}/initial_poses"] = np.array([pp.to_array() for pp in p.initial_poses], float)
        if hasattr(p, "box"):
            out[f"{name}/box"] = np.array([p.box.min, p.box.max], float)
        out[f"{name}/overrides"] = np.frombuffer(
            json.dumps({"solver": sc.solver_overrides, "trajopt": sc.trajopt_overrides}, sort_keys=True).encode(),
            dtype=np.uint8)
        print(name, "ok")
    np.savez_compressed(os.path.join(HERE, "scenes_reference.npz"), **out)


if __name__ == "__main__":
    main()
