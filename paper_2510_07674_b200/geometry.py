"""Host-side geometric types shared by the problem definitions.

Mirrors the public names of the reference's ``seqplace.geometry`` (geometry.py:23-128)
that the problem/scene layer needs: cost modes, yaw wrapping, 4-DOF poses, sphere
sets and boxes. The penetration arithmetic itself lives in the CUDA kernels
(csrc/stage1_models.cuh, csrc/stage2_kernels.cuh); nothing here is on the hot path.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

LINEAR = "linear"
QUADRATIC = "quadratic"
MODES = (LINEAR, QUADRATIC)


def _check_mode(mode: str) -> None:
    if mode not in MODES:
        raise ValueError(f"unknown cost mode {mode!r}, expected one of {MODES}")


def mode_id(mode: str) -> int:
    _check_mode(mode)
    return 0 if mode == LINEAR else 1


def normalize_yaw(yaw):
    """Wrap angle(s) into (-pi, pi] (reference geometry.py:31-38)."""
    a = np.asarray(yaw, dtype=float)
    w = np.remainder(a + np.pi, 2.0 * np.pi) - np.pi
    w = np.where(w <= -np.pi, w + 2.0 * np.pi, w)
    return float(w) if np.ndim(yaw) == 0 else w


@dataclass
class Pose:
    """World translation plus yaw about +z; yaw is wrapped on construction."""

    x: float
    y: float
    z: float
    yaw: float = 0.0

    def __post_init__(self):
        for name in ("x", "y", "z", "yaw"):
            if not math.isfinite(getattr(self, name)):
                raise ValueError(f"Pose.{name} must be finite")
        self.yaw = normalize_yaw(self.yaw)

    @property
    def translation(self) -> np.ndarray:
        return np.array([self.x, self.y, self.z])

    def to_array(self) -> np.ndarray:
        return np.array([self.x, self.y, self.z, self.yaw])

    @staticmethod
    def from_array(v) -> "Pose":
        v = np.asarray(v, dtype=float)
        return Pose(float(v[0]), float(v[1]), float(v[2]), float(v[3]))


@dataclass
class SphereSet:
    """Spheres in a body frame: centres (n, 3), radii (n,), all radii > 0."""

    centers: np.ndarray
    radii: np.ndarray

    def __post_init__(self):
        self.centers = np.atleast_2d(np.asarray(self.centers, dtype=float))
        self.radii = np.atleast_1d(np.asarray(self.radii, dtype=float))
        if self.centers.shape[0] == 0:
            raise ValueError("SphereSet must be nonempty")
        if self.centers.shape[1] != 3:
            raise ValueError("SphereSet centers must be (n, 3)")
        if self.radii.shape[0] != self.centers.shape[0]:
            raise ValueError("SphereSet radii length must match centers")
        if np.any(self.radii <= 0.0):
            raise ValueError("SphereSet radii must be strictly positive")

    def __len__(self) -> int:
        return self.centers.shape[0]


@dataclass
class Aabb:
    """Axis-aligned box with min <= max componentwise."""

    min: np.ndarray
    max: np.ndarray

    def __post_init__(self):
        self.min = np.asarray(self.min, dtype=float)
        self.max = np.asarray(self.max, dtype=float)
        if self.min.shape != self.max.shape:
            raise ValueError("Aabb min/max shape mismatch")
        if np.any(self.min > self.max):
            raise ValueError("Aabb requires min <= max componentwise")

    def clamp(self, points):
        return np.clip(points, self.min, self.max)

    def contains(self, points, atol: float = 0.0):
        p = np.asarray(points, dtype=float)
        return np.all((p >= self.min - atol) & (p <= self.max + atol), axis=-1)


def rotation_z(yaw: float) -> np.ndarray:
    c, s = math.cos(yaw), math.sin(yaw)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def transform(sphere_set: SphereSet, pose: Pose) -> np.ndarray:
    """World centres of a sphere set under a pose."""
    return sphere_set.centers @ rotation_z(pose.yaw).T + pose.translation
