"""Build a BASELINE scene (paper_2510_07674_b200/problems/scenes.py) as a REFERENCE scene
object -- test / baseline infrastructure only (bench.py's reference arm, the golden
generators). The scene dict goes through the reference's own loader (loader.py:291-455);
single1's non-tight packing, which that loader does not expose (loader.py:374-381), is built
through the reference Python API (tetris.py:88,107)."""
from __future__ import annotations

import dataclasses

import numpy as np


def ref_scene(name_or_dict):
    from seqplace.geometry import Aabb
    from seqplace.problems import TetrisProblem, load_scene

    if isinstance(name_or_dict, str):
        from paper_2510_07674_b200.problems import scenes as our_scenes

        d = our_scenes.BUNDLED[name_or_dict]()
    else:
        d = dict(name_or_dict)
    if "obstacles" in d:
        # this repo's cuboid entries -> the reference schema's explicit sphere sets (same
        # local grid, same pose transform, loader.py:157-177)
        from paper_2510_07674_b200.problems.loader import cuboid_spheres

        obs = []
        for e in d["obstacles"]:
            if "cuboid" in e:
                c, r = cuboid_spheres(e["cuboid"]["size"], e["cuboid"]["sphere_radius"])
                e = {"centers": c.tolist(), "radii": r.tolist(), "pose": list(e["pose"])}
            obs.append(e)
        d["obstacles"] = obs
    tight = d.pop("tight_packing", True)
    if tight:
        return load_scene(d)
    box = d["box"]
    area = sum(len(b["cells"]) * b["cell_size"] ** 2 for b in d["blocks"])
    side = float(np.sqrt(area))
    d["box"] = {"min": box["min"], "max": [box["min"][0] + side, box["min"][1] + side, box["max"][2]]}
    scene = load_scene(d)
    p = scene.problem
    return dataclasses.replace(scene, problem=TetrisProblem(
        blocks=p.blocks, box=Aabb(np.array(box["min"], float), np.array(box["max"], float)), z_star=p.z_star,
        yaw_mode=p.yaw_mode, weights=p.weights, initial_poses=p.initial_poses, tight_packing=False))
