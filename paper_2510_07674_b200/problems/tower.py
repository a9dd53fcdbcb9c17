"""Stacking problem and its GPU cost model (reference problems/tower.py).

Cubes are single inscribed spheres; the cost pulls cube i to height (i+1)*side, keeps
the centre of mass of everything above each cube over that cube's (yawed) square
footprint, and penalizes cube-cube and cube-obstacle overlap. Batched cost/gradient:
libspasm TowerEval (csrc/stage1_models.cuh).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from .. import _native as nat
from ..geometry import Aabb, Pose
from ..particle_opt import NativeCostModel
from .tetris import YAW_FIXED, YAW_FREE, YAW_MODES


@dataclass(frozen=True)
class TowerWeights:
    stability: float = 1.0
    height: float = 1.0
    collision: float = 1.0

    def __post_init__(self) -> None:
        if min(self.stability, self.height, self.collision) < 0:
            raise ValueError("tower weights must be nonnegative")


@dataclass
class TowerProblem:
    """Stack ``n_blocks`` cubes of edge ``side`` inside a workspace box (tower.py:46-102)."""

    n_blocks: int
    side: float
    box: Aabb
    obstacle_centers: np.ndarray | None = None
    obstacle_radii: np.ndarray | None = None
    yaw_mode: str = YAW_FIXED
    weights: TowerWeights = field(default_factory=TowerWeights)
    footprint_halfwidth: float | None = None
    table_height: float = 0.0
    initial_poses: tuple | None = None

    def __post_init__(self) -> None:
        if self.n_blocks < 2:
            raise ValueError("TowerProblem needs at least two blocks")
        if self.side <= 0:
            raise ValueError("cube side must be positive")
        if self.yaw_mode not in YAW_MODES:
            raise ValueError(f"yaw_mode must be one of {YAW_MODES}")
        if self.box.min.shape != (3,):
            raise ValueError("box must be three-dimensional")
        if self.obstacle_centers is None:
            self.obstacle_centers = np.zeros((0, 3))
            self.obstacle_radii = np.zeros(0)
        else:
            self.obstacle_centers = np.asarray(self.obstacle_centers, dtype=float).reshape(-1, 3)
            self.obstacle_radii = np.asarray(self.obstacle_radii, dtype=float).reshape(-1)
            if len(self.obstacle_centers) != len(self.obstacle_radii):
                raise ValueError("obstacle centers/radii length mismatch")
        if self.footprint_halfwidth is None:
            self.footprint_halfwidth = 0.5 * self.side
        if self.footprint_halfwidth <= 0:
            raise ValueError("footprint_halfwidth must be positive")
        if self.initial_poses is not None:
            self.initial_poses = tuple(self.initial_poses)
            if len(self.initial_poses) != self.n_blocks:
                raise ValueError("initial_poses length must match n_blocks")

    @property
    def sphere_radius(self) -> float:
        return 0.5 * self.side

    def height_target(self, index: int) -> float:
        return (index + 1) * self.side


class TowerCostModel(NativeCostModel):
    """Batched stacking cost over block-major rows (x, y, z[, yaw]) on the GPU."""

    def __init__(self, problem: TowerProblem, precision: str = "fp32"):
        self.problem = problem
        self.free_yaw = problem.yaw_mode == YAW_FREE
        self.per_block = 4 if self.free_yaw else 3
        n = problem.n_blocks
        lower = np.empty(n * self.per_block)
        upper = np.empty(n * self.per_block)
        for b in range(n):
            o = b * self.per_block
            lower[o : o + 3] = problem.box.min
            upper[o : o + 3] = problem.box.max
            if self.free_yaw:
                lower[o + 3], upper[o + 3] = -np.pi, np.pi
        targets = np.array([problem.height_target(b) for b in range(n)])
        oc = np.ascontiguousarray(problem.obstacle_centers, dtype=float)
        orr = np.ascontiguousarray(problem.obstacle_radii, dtype=float)
        w = problem.weights
        h = ctypes.c_void_p()
        nat.check(nat.load().spasm_tower_model_create(
            ctypes.byref(h), n, problem.side, problem.footprint_halfwidth, nat.ptr(targets), len(orr), nat.ptr(oc),
            nat.ptr(orr), w.stability, w.height, w.collision, int(self.free_yaw), nat.ptr(lower), nat.ptr(upper)),
            "tower model")
        super().__init__(n * self.per_block, lower, upper, h, precision)

    def split(self, values):
        v = np.asarray(values, dtype=float)
        per = v.reshape(v.shape[0], self.problem.n_blocks, self.per_block)
        return per[..., :3], (per[..., 3] if self.free_yaw else None)

    def poses_from_row(self, row) -> list:
        pos, yaw = self.split(np.asarray(row, dtype=float)[None, :])
        return [Pose(*pos[0, b], yaw=float(yaw[0, b]) if yaw is not None else 0.0) for b in range(self.problem.n_blocks)]

    def row_from_poses(self, poses) -> np.ndarray:
        if len(poses) != self.problem.n_blocks:
            raise ValueError("need one pose per block")
        per = np.empty((self.problem.n_blocks, self.per_block))
        for b, p in enumerate(poses):
            per[b, :3] = (p.x, p.y, p.z)
            if self.free_yaw:
                per[b, 3] = p.yaw
        return per.reshape(-1)
