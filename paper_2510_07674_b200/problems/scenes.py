"""Bundled benchmark scenes, built as schema dicts.

The first six reproduce the reference's bundled scenes (domino2, tetris5, tetris8,
tower4, corridor3, empty3: reference scenes/*.scene.json) so parity runs load the same
problems by name; the rest are the BASELINE.json configurations mapped onto the
reference's problem families:

  single1      C1  1 block, 7-DOF arm, stage 1 + stage 2 with T = 32 waypoints
  single1f     C1  the same with the Franka-like explicit 7-DOF chain (franka_like_robot)
  tower3c      C2  3-block stacking with cuboid obstacles (cuboids as sphere grids)
  tetris4/6    C3  4- and 6-tetromino tight packings (tetris5 is the 5-block case)
  tower6r      C4  6-block rearrangement with a moving sphere obstacle (reactive)
  tetris8      C5  8-object skeleton for the particle-count scaling sweep
"""
from __future__ import annotations

import numpy as np

CELL = 0.08
BAR_H = [[0, 0], [1, 0], [2, 0], [3, 0]]
BAR_V = [[0, 0], [0, 1], [0, 2], [0, 3]]
ELL = [[0, 0], [0, 1], [0, 2], [1, 0]]
JAY = [[0, 0], [1, 0], [1, 1], [1, 2]]
SQUARE = [[0, 0], [1, 0], [0, 1], [1, 1]]
JAY_FLAT = [[0, 0], [1, 0], [2, 0], [0, 1]]
DOMINO = [[0, 0], [1, 0]]


def _blk(name, cells, c=CELL):
    return {"name": name, "cells": cells, "cell_size": c}


def _box(x0, y0, x1, y1, half_z=0.04):
    return {"min": [x0, y0, -half_z], "max": [x1, y1, half_z]}


_STAGE1_TETRIS = {"eta_init": 0.03, "alpha": 0.1, "epsilon": 2e-05, "k_lin": 25, "k_quad": 40}


def domino2():
    return {"problem_type": "tetris", "name": "domino2",
            "blocks": [_blk("domino_a", DOMINO), _blk("domino_b", DOMINO)],
            "box": _box(0.0, 0.0, 0.16, 0.16), "z_star": 0.0, "yaw_mode": "fixed", "solver": dict(_STAGE1_TETRIS)}


def tetris5():
    return {
        "problem_type": "tetris", "name": "tetris5",
        "blocks": [_blk("bar_h", BAR_H), _blk("bar_v", BAR_V), _blk("ell", ELL), _blk("jay", JAY),
                   _blk("square", SQUARE)],
        "box": _box(0.28, -0.2, 0.68, 0.12), "z_star": 0.0, "yaw_mode": "fixed",
        "initial_poses": [[0.3, 0.3, 0.0, 0.0], [-0.55, 0.25, 0.0, 0.0], [-0.45, 0.42, 0.0, 0.0],
                          [0.12, 0.48, 0.0, 0.0], [-0.15, 0.55, 0.0, 0.0]],
        "robot": {"builtin": "spatial7", "scale": 1.3},
        "grasp": {"offset": [0.04, 0.04, 0.1], "yaw_offset": 0.0},
        "solver": {"eta_init": 0.02, "alpha": 0.1, "epsilon": 2e-05, "k_lin": 12, "k_quad": 10, "p_return": 4},
        "trajopt": {"k_waypoint": 1, "w_start": 200, "lr_init": 0.003, "lr_final": 0.0005, "inner_steps": 100,
                    "outer_iters": 10},
    }


def tetris8():
    return {
        "problem_type": "tetris", "name": "tetris8",
        "blocks": [_blk("square_a", SQUARE), _blk("bar_h", BAR_H), _blk("bar_v", BAR_V), _blk("ell", ELL),
                   _blk("jay_a", JAY), _blk("square_b", SQUARE), _blk("jay_b", JAY), _blk("jay_flat", JAY_FLAT)],
        "box": _box(-0.32, -0.16, 0.32, 0.16), "z_star": 0.0, "yaw_mode": "fixed", "solver": dict(_STAGE1_TETRIS),
    }


def tetris4():
    """C3, 4 objects: 2 squares + 2 horizontal bars tile a 4x4-cell box."""
    return {"problem_type": "tetris", "name": "tetris4",
            "blocks": [_blk("square_a", SQUARE), _blk("bar_a", BAR_H), _blk("square_b", SQUARE), _blk("bar_b", BAR_H)],
            "box": _box(0.32, -0.16, 0.64, 0.16), "z_star": 0.0, "yaw_mode": "fixed",
            "solver": {"eta_init": 0.02, "alpha": 0.1, "epsilon": 2e-05, "k_lin": 12, "k_quad": 10, "p_return": 4}}


def tetris6():
    """C3, 6 objects: the tetris5 multiset plus a vertical bar tiles a 6x4-cell box."""
    return {"problem_type": "tetris", "name": "tetris6",
            "blocks": [_blk("bar_h", BAR_H), _blk("bar_v", BAR_V), _blk("ell", ELL), _blk("jay", JAY),
                       _blk("square", SQUARE), _blk("bar_v2", BAR_V)],
            "box": _box(0.24, -0.2, 0.72, 0.12), "z_star": 0.0, "yaw_mode": "fixed",
            "solver": {"eta_init": 0.02, "alpha": 0.1, "epsilon": 2e-05, "k_lin": 25, "k_quad": 40, "p_return": 4}}


def tower4():
    return {
        "problem_type": "tower", "name": "tower4",
        "blocks": [_blk(f"cube{i + 1}", [[0, 0]], 0.1) for i in range(4)],
        "box": {"min": [0.35, 0.1, 0.08], "max": [0.6, 0.35, 0.5]}, "table_height": 0.05,
        "obstacles": [{"centers": [[0.45, -0.05, 0.28]], "radii": [0.16]}],
        "initial_poses": [[0.3, -0.3, 0.1, 0.0], [0.45, -0.32, 0.1, 0.0], [0.6, -0.3, 0.1, 0.0],
                          [0.38, -0.45, 0.1, 0.0]],
        "robot": {"builtin": "spatial7", "scale": 1.3},
        "grasp": {"offset": [0.0, 0.0, 0.1], "yaw_offset": 0.0},
        "solver": {"eta_init": 0.03, "alpha": 0.1, "epsilon": 1e-05, "k_lin": 25, "k_quad": 40, "p_return": 4},
        "trajopt": {"k_waypoint": 0, "w_start": 200, "lr_init": 0.004, "lr_final": 0.0005, "inner_steps": 100,
                    "outer_iters": 15, "beta": 1.5},
    }


def cuboid_obstacle(center, size, radius, yaw=0.0):
    """A cuboid obstacle entry of the scene schema (loader: ``{"cuboid": {"size",
    "sphere_radius"}, "pose"}``), compiled by the loader to a grid of spheres."""
    return {"cuboid": {"size": [float(v) for v in size], "sphere_radius": float(radius)},
            "pose": [float(center[0]), float(center[1]), float(center[2]), float(yaw)]}


def franka_like_robot():
    """Explicit 7-DOF chain with the Franka Panda's link offsets (0.333 / 0.316 / 0.0825 /
    0.384 / 0.088 m), joint limits and z-y-z-(-y)-z-y-z axis pattern in the reference's
    translate-then-rotate model (robot.py:120-141; the loader's explicit-chain schema,
    loader.py:209-251, identity tool rotation), a 0.21 m flange + hand tool along the last
    link's z, and 11 collision spheres (BASELINE configs[0]: "Franka Panda 7-DOF")."""
    joints = [
        ([0, 0, 1], [0, 0, 0.333], [-2.8973, 2.8973]),
        ([0, 1, 0], [0, 0, 0], [-1.7628, 1.7628]),
        ([0, 0, 1], [0, 0, 0.316], [-2.8973, 2.8973]),
        ([0, -1, 0], [0.0825, 0, 0], [-3.0718, -0.0698]),
        ([0, 0, 1], [-0.0825, 0, 0.384], [-2.8973, 2.8973]),
        ([0, 1, 0], [0, 0, 0], [-0.0175, 3.7525]),
        ([0, 0, 1], [0.088, 0, 0], [-2.8973, 2.8973]),
    ]
    spheres = [
        [([0, 0, -0.18], 0.08)],                                  # base column
        [([0, 0, 0.12], 0.07), ([0, 0, 0.24], 0.07)],             # upper arm
        [([0.04, 0, 0.0], 0.07)],                                 # elbow
        [([-0.04, 0, 0.12], 0.06), ([-0.08, 0, 0.26], 0.06)],     # forearm
        [([0, 0, 0.0], 0.06)],                                    # wrist 1
        [([0.044, 0, 0.0], 0.06)],                                # wrist 2
        [([0, 0, 0.07], 0.055), ([0, 0, 0.13], 0.05)],            # flange + hand
    ]
    return {"joints": [{"axis": a, "offset": o, "limits": l} for a, o, l in joints],
            "link_spheres": [[{"center": c, "radius": r} for c, r in link] for link in spheres],
            "tool": {"translation": [0.0, 0.0, 0.2104]}}


def tower3c():
    """C2: 3-block stacking with two cuboid obstacles (0.2 x 0.2 x 0.3 m as 3x3x4 r=0.05 spheres... reduced grid)."""
    return {
        "problem_type": "tower", "name": "tower3c",
        "blocks": [_blk(f"cube{i + 1}", [[0, 0]], 0.1) for i in range(3)],
        "box": {"min": [0.3, -0.2, 0.08], "max": [0.7, 0.3, 0.45]}, "table_height": 0.05,
        "obstacles": [cuboid_obstacle([0.45, -0.05, 0.15], [0.2, 0.2, 0.3], 0.05),
                      cuboid_obstacle([0.62, 0.22, 0.1], [0.1, 0.1, 0.2], 0.05)],
        "initial_poses": [[0.3, -0.35, 0.1, 0.0], [0.45, -0.38, 0.1, 0.0], [0.6, -0.35, 0.1, 0.0]],
        "robot": {"builtin": "spatial7", "scale": 1.3},
        "grasp": {"offset": [0.0, 0.0, 0.1], "yaw_offset": 0.0},
        "solver": {"n": 16384, "m": 2048, "eta_init": 0.03, "alpha": 0.1, "epsilon": 1e-05, "k_lin": 25,
                   "k_quad": 40, "p_return": 4},
        "trajopt": {"k_waypoint": 0, "w_start": 200, "lr_init": 0.004, "lr_final": 0.0005, "inner_steps": 100,
                    "outer_iters": 15, "beta": 1.5},
    }


def tower6r(obstacle_center=(0.45, -0.05, 0.28)):
    """C4: 6-cube rearrangement with one sphere obstacle whose centre moves per replan tick."""
    return {
        "problem_type": "tower", "name": "tower6r",
        "blocks": [_blk(f"cube{i + 1}", [[0, 0]], 0.1) for i in range(6)],
        "box": {"min": [0.35, 0.1, 0.08], "max": [0.6, 0.35, 0.7]}, "table_height": 0.05,
        "obstacles": [{"centers": [list(obstacle_center)], "radii": [0.12]}],
        "solver": {"eta_init": 0.03, "alpha": 0.1, "epsilon": 1e-05, "k_lin": 25, "k_quad": 40, "p_return": 4},
    }


def single1():
    """C1: one 2x2 block placed on a table region by the 7-DOF arm, T = 32 waypoints."""
    return {
        "problem_type": "tetris", "name": "single1",
        "blocks": [_blk("square", SQUARE)],
        "box": _box(0.32, -0.16, 0.64, 0.16), "z_star": 0.0, "yaw_mode": "fixed", "tight_packing": False,
        "initial_poses": [[0.3, 0.35, 0.0, 0.0]],
        "robot": {"builtin": "spatial7", "scale": 1.3},
        "grasp": {"offset": [0.08, 0.08, 0.1], "yaw_offset": 0.0},
        "solver": {"n": 1024, "m": 1024, "eta_init": 0.02, "alpha": 0.1, "epsilon": 2e-05, "k_lin": 12,
                   "k_quad": 10, "p_return": 32},
        "trajopt": {"k_waypoint": 0, "k_interp": 31, "w_start": 200, "lr_init": 0.003, "lr_final": 0.0005,
                    "inner_steps": 100, "outer_iters": 10},
    }


def single1f():
    """C1 with the Franka-like explicit 7-DOF chain (franka_like_robot) instead of the
    builtin spatial arm; same block, table region and T = 32 waypoints."""
    d = single1()
    d["name"] = "single1f"
    d["robot"] = franka_like_robot()
    return d


def corridor3():
    return {"problem_type": "motion", "name": "corridor3", "robot": {"builtin": "planar3"},
            "start": [-1.1, 0.6, 0.3], "goal": [1.1, -0.6, -0.3],
            "obstacles": [{"centers": [[1.05, 0.0, 0.0]], "radii": [0.22]}], "trajopt": {"k_waypoint": 0}}


def empty3():
    return {"problem_type": "motion", "name": "empty3", "robot": {"builtin": "planar3"},
            "start": [-1.1, 0.6, 0.3], "goal": [1.1, -0.6, -0.3], "trajopt": {"k_waypoint": 0}}


BUNDLED = {
    "domino2": domino2, "tetris5": tetris5, "tetris8": tetris8, "tower4": tower4, "corridor3": corridor3,
    "empty3": empty3, "tetris4": tetris4, "tetris6": tetris6, "tower3c": tower3c, "tower6r": tower6r,
    "single1": single1, "single1f": single1f,
}
