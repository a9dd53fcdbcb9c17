"""Build the golden cases' problems with the product package (no reference needed)."""
from __future__ import annotations

from paper_2510_07674_b200.problems import TetrisProblem, TowerProblem, load_scene

CASES = {
    "domino2": ("domino2", None),
    "tetris5": ("tetris5", None),
    "tetris8": ("tetris8", None),
    "tower4": ("tower4", None),
    "tetris5_free": ("tetris5", "quantized-free"),
    "tower4_free": ("tower4", "quantized-free"),
}


def case_problem(case):
    name, yaw = CASES[case]
    scene = load_scene(name)
    p = scene.problem
    if yaw is None:
        return scene, p
    if isinstance(p, TetrisProblem):
        return scene, TetrisProblem(blocks=p.blocks, box=p.box, z_star=p.z_star, yaw_mode=yaw, weights=p.weights,
                                    initial_poses=p.initial_poses, tight_packing=p.tight_packing)
    return scene, TowerProblem(n_blocks=p.n_blocks, side=p.side, box=p.box, obstacle_centers=p.obstacle_centers,
                               obstacle_radii=p.obstacle_radii, yaw_mode=yaw, weights=p.weights,
                               footprint_halfwidth=p.footprint_halfwidth, table_height=p.table_height,
                               initial_poses=p.initial_poses)
