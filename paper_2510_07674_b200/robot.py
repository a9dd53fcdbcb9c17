"""Serial-manipulator description types and grasp maps (reference robot.py).

Chains are ordered revolute joints, each a fixed translation followed by a rotation
about a fixed body axis (reference robot.py:29-68). The batched FK, Jacobians and DLS
IK run on the GPU (csrc/stage2_kernels.cuh; exposed through ``trajopt``); this module
holds the host-side chain description, the bundled arms and the scalar grasp maps.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Optional, Sequence

import numpy as np

from .geometry import Pose, SphereSet

IK_POS_TOL = 1e-4
IK_YAW_TOL = 1e-3
IK_DAMPING = 1e-3
IK_MAX_ITERS = 200
IK_STEP_CLAMP = 0.5


@dataclass
class Joint:
    axis: np.ndarray
    offset: np.ndarray
    lower: float
    upper: float

    def __post_init__(self):
        self.axis = np.asarray(self.axis, dtype=float)
        self.offset = np.asarray(self.offset, dtype=float)
        if abs(np.linalg.norm(self.axis) - 1.0) > 1e-9:
            raise ValueError("joint axis must be unit norm")
        if not self.lower < self.upper:
            raise ValueError("joint limits must satisfy lower < upper")


@dataclass
class KinematicChain:
    joints: List[Joint]
    link_spheres: List[Optional[SphereSet]]
    tool_translation: np.ndarray
    tool_rotation: np.ndarray

    def __post_init__(self):
        self.tool_translation = np.asarray(self.tool_translation, dtype=float)
        self.tool_rotation = np.asarray(self.tool_rotation, dtype=float)
        if len(self.link_spheres) != len(self.joints):
            raise ValueError("need one link_spheres entry (possibly None) per joint")

    @property
    def dof(self) -> int:
        return len(self.joints)

    @property
    def lower(self) -> np.ndarray:
        return np.array([j.lower for j in self.joints])

    @property
    def upper(self) -> np.ndarray:
        return np.array([j.upper for j in self.joints])

    def sphere_table(self):
        """Flattened link-sphere table: (local centres (S,3), radii (S,), owning link (S,))."""
        cs, rs, ls = [], [], []
        for i, sp in enumerate(self.link_spheres):
            if sp is None:
                continue
            cs.append(sp.centers)
            rs.append(sp.radii)
            ls.extend([i] * len(sp))
        if not cs:
            return np.zeros((0, 3)), np.zeros(0), np.zeros(0, dtype=np.int32)
        return np.concatenate(cs), np.concatenate(rs), np.asarray(ls, dtype=np.int32)


@dataclass
class GraspSpec:
    """Top-down grasp: EE at a fixed offset in the object's yaw frame (robot.py:310-322)."""

    offset: np.ndarray
    yaw_offset: float = 0.0

    def __post_init__(self):
        self.offset = np.asarray(self.offset, dtype=float)
        if self.offset.shape != (3,):
            raise ValueError("grasp offset must be a 3-vector")
        if self.offset[2] <= 0:
            raise ValueError("grasp offset must approach from above (z > 0)")


def grasp_pose(object_pose: Pose, grasp: GraspSpec) -> Pose:
    """End-effector target realizing a grasp of an object at a pose (robot.py:325-334)."""
    c, s = math.cos(object_pose.yaw), math.sin(object_pose.yaw)
    ox, oy, oz = grasp.offset
    return Pose(object_pose.x + c * ox - s * oy, object_pose.y + s * ox + c * oy, object_pose.z + oz,
                object_pose.yaw + grasp.yaw_offset)


def inverse_grasp(ee_pose: Pose, grasp: GraspSpec) -> Pose:
    """Object pose implied by an end-effector pose holding the grasp (robot.py:337-347)."""
    yaw = ee_pose.yaw - grasp.yaw_offset
    c, s = math.cos(yaw), math.sin(yaw)
    ox, oy, oz = grasp.offset
    return Pose(ee_pose.x - (c * ox - s * oy), ee_pose.y - (s * ox + c * oy), ee_pose.z - oz, yaw)


def planar_arm(link_lengths: Sequence[float] = (0.5, 0.5, 0.5), sphere_radius: float = 0.06,
               spheres_per_link: int = 2) -> KinematicChain:
    """Planar arm, every joint about z, links along local x (robot.py:362-382)."""
    joints, spheres = [], []
    prev = np.zeros(3)
    for L in link_lengths:
        joints.append(Joint(axis=np.array([0.0, 0.0, 1.0]), offset=prev.copy(), lower=-math.pi, upper=math.pi))
        xs = (np.arange(1, spheres_per_link + 1) / (spheres_per_link + 1)) * L
        c = np.zeros((spheres_per_link, 3))
        c[:, 0] = xs
        spheres.append(SphereSet(c, np.full(spheres_per_link, sphere_radius)))
        prev = np.array([L, 0.0, 0.0])
    return KinematicChain(joints=joints, link_spheres=spheres, tool_translation=prev, tool_rotation=np.eye(3))


# (axis, offset along z, lower, upper, link segment length) of the z-y-z-y-z-y-z arm
_SPATIAL7 = (
    ("z", 0.30, -math.pi, math.pi, 0.05),
    ("y", 0.05, -2.2, 2.2, 0.15),
    ("z", 0.15, -math.pi, math.pi, 0.15),
    ("y", 0.15, -2.6, 2.6, 0.15),
    ("z", 0.15, -math.pi, math.pi, 0.15),
    ("y", 0.15, -3.0, 3.0, 0.08),
    ("z", 0.08, -math.pi, math.pi, 0.07),
)


def spatial_arm_7dof(scale: float = 1.0) -> KinematicChain:
    """7-DOF spatial arm, links along local z, wrist roll about the tool axis (robot.py:385-420)."""
    axes = {"z": np.array([0.0, 0.0, 1.0]), "y": np.array([0.0, 1.0, 0.0])}
    joints, spheres = [], []
    for ax, off, lo, hi, seg in _SPATIAL7:
        joints.append(Joint(axis=axes[ax], offset=np.array([0.0, 0.0, off]) * scale, lower=lo, upper=hi))
        spheres.append(SphereSet(np.array([[0.0, 0.0, seg * scale * 0.5]]), np.array([0.055 * scale])))
    return KinematicChain(joints=joints, link_spheres=spheres, tool_translation=np.array([0.0, 0.0, 0.07]) * scale,
                          tool_rotation=np.eye(3))
