"""Stage 2 on the B200: lifting placements into joint space and the augmented-Lagrangian
trajectory optimizer (the reference's ``seqplace.trajopt``, trajopt.py:1-1179).

Same public API and error behaviour as the reference:

  trajectory_cost / al_value_and_gradient   trajopt.py:664-723   (spasm_traj_evaluate)
  lift_placements                           trajopt.py:795-876   (spasm_lift)
  motion_endpoints / init_trajectories      trajopt.py:879-923   (spasm_init_trajectories)
  solve_al                                  trajopt.py:936-1063  (spasm_solve_al)
  validate                                  trajopt.py:1071-1153 (spasm_traj_validate)
  trajectory_path_length / save_trajectory  trajopt.py:1161-1179 (host)

Every numeric stage is a libspasm kernel (csrc/stage2_kernels.cuh). There is no CPU
fallback. ``precision`` selects "fp64" (the reference's float64 op order; the parity path)
or "fp32" (the throughput path).

Placement mode inside ``solve_al``: as shipped, the reference's ``_evaluate`` ignores the
``place_mode=QUADRATIC`` that ``solve_al`` passes ("variant B", the
semantics its own tests pin): the placement term uses the collision mode (LINEAR). That is
the default here (``place_mode=None``); ``place_mode=QUADRATIC`` gives the docstring's
intent ("variant A").
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field, replace
from pathlib import Path as _Path
from typing import List, Optional, Tuple

import numpy as np

from . import _native as nat
from .geometry import LINEAR, MODES, QUADRATIC
from .robot import GraspSpec, KinematicChain

DEFAULT_VALIDATION_EPSILON = 0.02
INNER_STEP_CLAMP = 0.1
LIFT_CANDIDATES = 4
DEFAULT_PRECISION = "fp64"
_TRAJ_STREAM = 1 << 20


class LiftFailure(RuntimeError):
    """Raised when no stage-1 particle survives grasp IK."""


class TrajOptFailure(RuntimeError):
    """Raised when no particle passes validation within the outer budget."""

    def __init__(self, best_violation: float, report: "AlReport"):
        super().__init__(f"no feasible trajectory found (best violation {best_violation:.4g})")
        self.best_violation = best_violation
        self.report = report


@dataclass(frozen=True)
class TrajOptConfig:
    """Trajectory initialization + AL settings (reference trajopt.py:118-177)."""

    k_waypoint: int = 1
    k_interp: int = 5
    w_start: float = 50.0
    w_arm: float = 1.0
    w_block: float = 1.0
    w_place: float = 1.0
    mu0: float = 10.0
    beta: float = 2.0
    outer_iters: int = 20
    inner_steps: int = 50
    lr_init: float = 0.05
    lr_final: float = 0.005
    validation_epsilon: float = DEFAULT_VALIDATION_EPSILON

    def __post_init__(self):
        if int(self.k_waypoint) != self.k_waypoint or self.k_waypoint < 0:
            raise ValueError("k_waypoint must be a nonnegative integer")
        if int(self.k_interp) != self.k_interp or self.k_interp < 1:
            raise ValueError("k_interp must be a positive integer")
        for name in ("w_start", "w_arm", "w_block", "w_place"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be nonnegative")
        if self.mu0 <= 0:
            raise ValueError("mu0 must be positive")
        if self.beta <= 1:
            raise ValueError("beta must exceed 1")
        if int(self.outer_iters) != self.outer_iters or self.outer_iters < 1:
            raise ValueError("outer_iters must be a positive integer")
        if int(self.inner_steps) != self.inner_steps or self.inner_steps < 1:
            raise ValueError("inner_steps must be a positive integer")
        if self.lr_init <= 0 or self.lr_final <= 0:
            raise ValueError("learning rates must be positive")
        if self.validation_epsilon <= 0:
            raise ValueError("validation_epsilon must be positive")

    @property
    def waypoints_per_segment(self) -> int:
        return self.k_interp * (self.k_waypoint + 1) + 1


@dataclass
class Trajectory:
    """One particle's motion plan: a waypoint matrix per pick-place segment."""

    segments: np.ndarray  # (n_segments, T, dof)
    attached: Tuple[Optional[int], ...]

    def __post_init__(self):
        self.segments = np.asarray(self.segments, dtype=float)
        if self.segments.ndim != 3:
            raise ValueError("segments must have shape (n_segments, T, dof)")
        if len(self.attached) != self.segments.shape[0]:
            raise ValueError("one attached-object entry per segment required")
        self.attached = tuple(self.attached)


@dataclass
class LiftResult:
    endpoints: np.ndarray  # (particles, n_segments, 2, dof): pick and place
    kept: np.ndarray       # indices into the input placement rows that survived IK


@dataclass
class OuterRecord:
    index: int
    mu: np.ndarray
    multipliers: np.ndarray
    constraints: np.ndarray
    updated_multipliers: np.ndarray
    objective: np.ndarray
    feasible: np.ndarray
    violation: np.ndarray


@dataclass
class AlReport:
    outers: List[OuterRecord] = field(default_factory=list)
    accepted_objectives: List[float] = field(default_factory=list)
    device_ms: float = 0.0
    launches: int = 0


@dataclass
class AlResult:
    trajectory: Trajectory
    objective: float
    particle_index: int
    report: AlReport


# ---------------------------------------------------------------------------
# device geometry (the reference's _Geometry, trajopt.py:235-367) behind spasm_traj
# ---------------------------------------------------------------------------
def _torch():
    import torch

    return torch


def _check_precision(precision):
    if precision not in ("fp32", "fp64"):
        raise ValueError("precision must be 'fp32' or 'fp64'")
    return nat.F32 if precision == "fp32" else nat.F64


def _tdtype(precision):
    torch = _torch()
    return torch.float32 if precision == "fp32" else torch.float64


def _as_obstacles(centers, radii):
    if centers is None:
        return np.zeros((0, 3)), np.zeros(0)
    c = np.asarray(centers, dtype=float).reshape(-1, 3)
    r = np.asarray(radii, dtype=float).reshape(-1)
    if len(c) != len(r):
        raise ValueError("obstacle centers and radii length mismatch")
    return c, r


def _is_motion(problem):
    from .problems import MotionProblem

    return isinstance(problem, MotionProblem)


def _free_yaw_twin(problem):
    """The same placement problem with yaw as a live coordinate (trajopt.py:281-302)."""
    from .problems import YAW_FREE

    return replace(problem, yaw_mode=YAW_FREE)


def _block_sphere_table(problem):
    from .problems import TowerProblem

    if isinstance(problem, TowerProblem):
        return ([np.zeros((1, 3)) for _ in range(problem.n_blocks)],
                [np.array([problem.sphere_radius]) for _ in range(problem.n_blocks)])
    return ([b.sphere_set.centers.copy() for b in problem.blocks], [b.sphere_set.radii.copy() for b in problem.blocks])


class _Geometry:
    """Owns one spasm_traj handle (+ the placement twin it references)."""

    def __init__(self, problem, chain: KinematicChain, grasp: Optional[GraspSpec], statics_c, statics_r):
        from .problems import YAW_FIXED, as_cost_model

        self._lib = nat.load()
        self.problem = problem
        self.chain = chain
        self.grasp = grasp
        self.manipulation = not _is_motion(problem) if problem is not None else False
        self.dof = chain.dof
        self.twin = None
        self._keep = []
        loc, rad, link = chain.sphere_table()
        ch = nat.spasm_chain()
        arrs = {
            "axes": np.ascontiguousarray(np.stack([j.axis for j in chain.joints]), dtype=float),
            "offsets": np.ascontiguousarray(np.stack([j.offset for j in chain.joints]), dtype=float),
            "lower": np.ascontiguousarray(chain.lower, dtype=float),
            "upper": np.ascontiguousarray(chain.upper, dtype=float),
            "tool_translation": np.ascontiguousarray(chain.tool_translation, dtype=float),
            "tool_rotation": np.ascontiguousarray(chain.tool_rotation, dtype=float).reshape(9),
            "sphere_centers": np.ascontiguousarray(loc, dtype=float).reshape(-1),
            "sphere_radii": np.ascontiguousarray(rad, dtype=float),
            "sphere_link": np.ascontiguousarray(link, dtype=np.int32),
        }
        self._keep.append(arrs)
        ch.dof = chain.dof
        ch.n_spheres = len(rad)
        for k, v in arrs.items():
            setattr(ch, k, v.ctypes.data)
        d = nat.spasm_traj_desc()
        sc = np.ascontiguousarray(statics_c, dtype=float).reshape(-1)
        sr = np.ascontiguousarray(statics_r, dtype=float)
        self._keep += [sc, sr]
        d.n_static = len(sr)
        d.static_centers = sc.ctypes.data if len(sr) else None
        d.static_radii = sr.ctypes.data if len(sr) else None
        if self.manipulation:
            if grasp is None:
                raise ValueError("manipulation problems need a grasp specification")
            if problem.initial_poses is None:
                raise ValueError("manipulation problems need staged initial poses")
            locs, rads = _block_sphere_table(problem)
            self.n_segments = len(locs)
            self.block_counts = [len(r) for r in rads]
            spb = np.asarray(self.block_counts, dtype=np.int32)
            bc = np.ascontiguousarray(np.concatenate(locs), dtype=float).reshape(-1)
            br = np.ascontiguousarray(np.concatenate(rads), dtype=float)
            staged = np.ascontiguousarray([[p.x, p.y, p.z, p.yaw] for p in problem.initial_poses], dtype=float)
            goff = np.ascontiguousarray(grasp.offset, dtype=float)
            self.twin = as_cost_model(_free_yaw_twin(problem), precision="fp64")
            self._keep += [spb, bc, br, staged, goff]
            d.manipulation = 1
            d.n_blocks = self.n_segments
            d.spheres_per_block = spb.ctypes.data
            d.block_centers = bc.ctypes.data
            d.block_radii = br.ctypes.data
            d.staged_poses = staged.ctypes.data
            d.grasp_offset = goff.ctypes.data
            d.grasp_yaw_offset = float(grasp.yaw_offset)
            d.place_model = self.twin.handle
            d.anchor_yaw = int(problem.yaw_mode == YAW_FIXED)
            d.rows_have_yaw = int(problem.yaw_mode != YAW_FIXED)
            self.row_dim = self.n_segments * (4 if d.rows_have_yaw else 3)
        else:
            self.n_segments = 1
            start = np.ascontiguousarray(problem.start if problem is not None else np.zeros(chain.dof), dtype=float)
            goal = np.ascontiguousarray(problem.goal if problem is not None else np.zeros(chain.dof), dtype=float)
            self._keep += [start, goal]
            d.manipulation = 0
            d.n_blocks = 1
            d.start = start.ctypes.data
            d.goal = goal.ctypes.data
        h = ctypes.c_void_p()
        nat.check(self._lib.spasm_traj_create(ctypes.byref(h), ctypes.byref(ch), ctypes.byref(d)),
                  "spasm_traj_create")
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and getattr(self, "_lib", None) is not None:
            self._lib.spasm_traj_destroy(h)


_GEO_CACHE: dict = {}
_GEO_CACHE_MAX = 32


def _geometry(problem, chain, grasp, static_centers, static_radii, *, default_statics=True) -> _Geometry:
    """_build_geometry (trajopt.py:305-367), cached per (problem, chain, grasp, statics)."""
    if default_statics and static_centers is None and problem is not None:
        static_centers = getattr(problem, "obstacle_centers", None)
        static_radii = getattr(problem, "obstacle_radii", None)
    sc, sr = _as_obstacles(static_centers, static_radii)
    key = (id(problem), id(chain), id(grasp), sc.tobytes(), sr.tobytes())
    hit = _GEO_CACHE.get(key)
    if hit is not None and hit[0] is problem and hit[1] is chain and hit[2] is grasp:
        return hit[3]
    geo = _Geometry(problem, chain, grasp, sc, sr)
    if len(_GEO_CACHE) >= _GEO_CACHE_MAX:
        _GEO_CACHE.pop(next(iter(_GEO_CACHE)))
    _GEO_CACHE[key] = (problem, chain, grasp, geo)
    return geo


def _al_config(config: TrajOptConfig, T: int, place_mode) -> "nat.spasm_al_config":
    c = nat.spasm_al_config()
    c.w_start = config.w_start
    c.w_arm = config.w_arm
    c.w_block = config.w_block
    c.w_place = config.w_place
    c.mu0 = config.mu0
    c.beta = config.beta
    c.lr_init = config.lr_init
    c.lr_final = config.lr_final
    c.validation_epsilon = config.validation_epsilon
    c.outer_iters = int(config.outer_iters)
    c.inner_steps = int(config.inner_steps)
    c.place_mode = nat.QUADRATIC_ID if place_mode == QUADRATIC else nat.LINEAR_ID
    c.waypoints = int(T)
    return c


def _check_values(values, geo: _Geometry) -> np.ndarray:
    """trajopt.py:375-388 (numpy or CUDA tensors accepted)."""
    shape = tuple(values.shape)
    if len(shape) != 4:
        raise ValueError("trajectory batch must have shape (P, segments, T, dof)")
    P, B, T, dof = shape
    if P < 1:
        raise ValueError("empty trajectory batch")
    if B != geo.n_segments:
        raise ValueError(f"expected {geo.n_segments} segments, got {B}")
    if dof != geo.chain.dof:
        raise ValueError("configuration dimension mismatch")
    if T < 2:
        raise ValueError("segments need at least two waypoints")
    return values


def _is_tensor(x) -> bool:
    return type(x).__module__.startswith("torch")


def _device(values, precision):
    """(tensor on cuda, was_numpy)."""
    torch = _torch()
    nat.require_cuda()
    dt = _tdtype(precision)
    if not _is_tensor(values):
        return torch.as_tensor(np.asarray(values, dtype=float)).to(device="cuda", dtype=dt).contiguous(), True
    return values.to(device="cuda", dtype=dt).contiguous(), False


def _out(t, was_numpy):
    return t.double().cpu().numpy() if was_numpy else t


def _stream():
    return nat.stream_handle()


# ---------------------------------------------------------------------------
# cost evaluation (trajopt.py:416-723)
# ---------------------------------------------------------------------------
def _evaluate(values, geo, config, mode, lam, mu, want_grad, place_mode, precision):
    torch = _torch()
    dt = _check_precision(precision)
    v, was_np = _device(values, precision)
    P, B, T, dof = v.shape
    tdt = _tdtype(precision)
    lam_t = torch.as_tensor(lam if _is_tensor(lam) else np.broadcast_to(np.asarray(lam, dtype=float), (P, 3)).copy(),
                            dtype=tdt, device="cuda").contiguous()
    mu_t = torch.as_tensor(mu if _is_tensor(mu) else np.broadcast_to(np.asarray(mu, dtype=float), (P,)).copy(),
                           dtype=tdt, device="cuda").contiguous()
    obj = torch.empty(P, dtype=tdt, device="cuda")
    cons = torch.empty((P, 3), dtype=tdt, device="cuda")
    lag = torch.empty(P, dtype=tdt, device="cuda")
    grad = torch.empty_like(v) if want_grad else None
    pm = mode if place_mode is None else place_mode
    cfg = _al_config(config, T, None)
    nat.check(geo._lib.spasm_traj_evaluate(
        geo.handle, dt, ctypes.byref(cfg), nat.ptr(v), P, nat.LINEAR_ID if mode == LINEAR else nat.QUADRATIC_ID,
        nat.LINEAR_ID if pm == LINEAR else nat.QUADRATIC_ID, nat.ptr(lam_t), nat.ptr(mu_t), int(want_grad),
        nat.ptr(obj), nat.ptr(cons), nat.ptr(lag), nat.ptr(grad), _stream()), "spasm_traj_evaluate")
    return (_out(obj, was_np), _out(cons, was_np), _out(lag, was_np),
            _out(grad, was_np) if grad is not None else None)


def trajectory_cost(values, problem, chain: KinematicChain, config: TrajOptConfig, *, grasp: Optional[GraspSpec] = None,
                    static_centers=None, static_radii=None, mode: str = LINEAR, place_mode=None,
                    precision: str = DEFAULT_PRECISION):
    """Per-particle objective and constraint vector (trajopt.py:664-689)."""
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}")
    geo = _geometry(problem, chain, grasp, static_centers, static_radii)
    _check_values(values, geo)
    P = values.shape[0]
    obj, cons, _, _ = _evaluate(values, geo, config, mode, np.zeros((P, 3)), np.zeros(P), False, place_mode,
                                precision)
    return obj, cons


def al_value_and_gradient(values, problem, chain: KinematicChain, config: TrajOptConfig, lam, mu, *,
                          grasp: Optional[GraspSpec] = None, static_centers=None, static_radii=None,
                          mode: str = LINEAR, place_mode=None, precision: str = DEFAULT_PRECISION):
    """AL value and exact gradient per particle (trajopt.py:692-723)."""
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}")
    geo = _geometry(problem, chain, grasp, static_centers, static_radii)
    _check_values(values, geo)
    _, _, lag, grad = _evaluate(values, geo, config, mode, lam, mu, True, place_mode, precision)
    return lag, grad


# ---------------------------------------------------------------------------
# kinematics entry points (robot.fk_batch / ik_solve_batch / _polish_tool_down)
# ---------------------------------------------------------------------------
def fk_batch_device(chain: KinematicChain, Q, precision: str = DEFAULT_PRECISION):
    """Batched FK on the device: (ee (n,3), rot (n,3,3), origins (n,J,3), axes (n,J,3), yaw_jac (n,J))."""
    torch = _torch()
    geo = _geometry(None, chain, None, None, None, default_statics=False)
    dt = _check_precision(precision)
    q, was_np = _device(Q if _is_tensor(Q) else np.asarray(Q), precision)
    lead = tuple(q.shape[:-1])
    q = q.reshape(-1, chain.dof).contiguous()
    n = q.shape[0]
    tdt = _tdtype(precision)
    ee = torch.empty((n, 3), dtype=tdt, device="cuda")
    rot = torch.empty((n, 3, 3), dtype=tdt, device="cuda")
    org = torch.empty((n, chain.dof, 3), dtype=tdt, device="cuda")
    axs = torch.empty((n, chain.dof, 3), dtype=tdt, device="cuda")
    yj = torch.empty((n, chain.dof), dtype=tdt, device="cuda")
    nat.check(geo._lib.spasm_fk(geo.handle, dt, nat.ptr(q), n, nat.ptr(ee), nat.ptr(rot), nat.ptr(org), nat.ptr(axs),
                                nat.ptr(yj), _stream()), "spasm_fk")
    return tuple(_out(t.reshape(lead + tuple(t.shape[1:])), was_np) for t in (ee, rot, org, axs, yj))


def ik_solve_batch(chain: KinematicChain, targets, restarts: int = 16, seed: int = 0, max_iters: int = 200,
                   damping: float = 1e-3, precision: str = DEFAULT_PRECISION):
    """robot.ik_solve_batch (robot.py:227-302) on the device. targets: Poses or (pos (n,3), yaw (n,))."""
    torch = _torch()
    nat.require_cuda()
    if isinstance(targets, tuple) and len(targets) == 2 and not hasattr(targets[0], "x"):
        tp = np.asarray(targets[0], dtype=float).reshape(-1, 3)
        ty = np.asarray(targets[1], dtype=float).reshape(-1)
    else:
        tp = np.array([t.translation for t in targets], dtype=float).reshape(-1, 3)
        ty = np.array([t.yaw for t in targets], dtype=float)
    n = len(ty)
    if n == 0:
        return np.zeros((0, chain.dof)), np.zeros(0, dtype=bool), np.zeros(0)
    geo = _geometry(None, chain, None, None, None, default_statics=False)
    dt = _check_precision(precision)
    tdt = _tdtype(precision)
    tp_d = torch.as_tensor(tp, device="cuda").contiguous()
    ty_d = torch.as_tensor(ty, device="cuda").contiguous()
    sol = torch.empty((n, chain.dof), dtype=tdt, device="cuda")
    ok = torch.empty(n, dtype=torch.uint8, device="cuda")
    err = torch.empty(n, dtype=tdt, device="cuda")
    nat.check(geo._lib.spasm_ik_solve(geo.handle, dt, nat.ptr(tp_d), nat.ptr(ty_d), n, int(seed), int(restarts),
                                      int(max_iters), float(damping), nat.ptr(sol), nat.ptr(ok), nat.ptr(err),
                                      _stream()), "spasm_ik_solve")
    return sol.double().cpu().numpy(), ok.cpu().numpy().astype(bool), err.double().cpu().numpy()


def polish_tool_down(chain: KinematicChain, Q, target_pos, target_yaw, precision: str = DEFAULT_PRECISION):
    """_polish_tool_down (trajopt.py:726-776) on the device. Returns (Q, ok)."""
    torch = _torch()
    Q = np.array(Q, dtype=float)
    n = len(Q)
    if n == 0:
        return Q, np.zeros(0, dtype=bool)
    geo = _geometry(None, chain, None, None, None, default_statics=False)
    dt = _check_precision(precision)
    q = torch.as_tensor(Q, dtype=_tdtype(precision), device="cuda").contiguous()
    tp = torch.as_tensor(np.asarray(target_pos, dtype=float).reshape(-1, 3), device="cuda").contiguous()
    ty = torch.as_tensor(np.asarray(target_yaw, dtype=float).reshape(-1), device="cuda").contiguous()
    ok = torch.empty(n, dtype=torch.uint8, device="cuda")
    nat.check(geo._lib.spasm_polish_tool_down(geo.handle, dt, nat.ptr(q), nat.ptr(tp), nat.ptr(ty), n, nat.ptr(ok),
                                              _stream()), "spasm_polish_tool_down")
    return q.double().cpu().numpy(), ok.cpu().numpy().astype(bool)


# ---------------------------------------------------------------------------
# lifting (trajopt.py:795-876)
# ---------------------------------------------------------------------------
class _LiftDevice:
    """Device outputs of one asynchronous lift: endpoints, kept indices, status[2]."""

    def __init__(self, endpoints, kept, status, P):
        self.endpoints = endpoints
        self.kept = kept
        self.status = status
        self.P = P


def _lift_async(geo: _Geometry, placements_dev, seed: int, candidates: int, precision: str, *,
                device_rows=None) -> _LiftDevice:
    """Enqueue lift_placements. ``placements_dev`` is a (P, D) float64 CUDA tensor, or None
    with ``device_rows = (rows pointer, count pointer, P)``: the stage-1 result read in place
    (particle_opt.PendingSolve.device_rows), only its first *count rows exist."""
    torch = _torch()
    dt = _check_precision(precision)
    if device_rows is not None:
        rows_ptr, n_rows_ptr, P = device_rows
        D = geo.row_dim
    else:
        P, D = placements_dev.shape
        rows_ptr, n_rows_ptr = nat.ptr(placements_dev), None
    if D != geo.row_dim:
        raise ValueError(f"placement rows have dimension {D}, expected {geo.row_dim}")
    B, J = geo.n_segments, geo.dof
    ws_bytes = geo._lib.spasm_lift_workspace_bytes(geo.handle, dt, P, int(candidates))
    ws = torch.empty(max(int(ws_bytes), 1), dtype=torch.uint8, device="cuda")
    ends = torch.empty((P, B, 2, J), dtype=_tdtype(precision), device="cuda")
    kept = torch.empty(max(P, 1), dtype=torch.int32, device="cuda")
    status = torch.empty(2, dtype=torch.int32, device="cuda")
    nat.check(geo._lib.spasm_lift(geo.handle, dt, rows_ptr, P, n_rows_ptr, D, int(seed), int(candidates),
                                  nat.ptr(ws), ws_bytes, nat.ptr(ends), nat.ptr(kept), nat.ptr(status), _stream()),
              "spasm_lift")
    return _LiftDevice(ends, kept, status, P)


def lift_placements(problem, placements, chain: KinematicChain, grasp: GraspSpec, *, seed: int = 0,
                    static_centers=None, static_radii=None, candidates: int = LIFT_CANDIDATES,
                    precision: str = DEFAULT_PRECISION) -> LiftResult:
    """Grasp IK over staged and placed poses for each stage-1 particle (trajopt.py:795-876)."""
    torch = _torch()
    if _is_motion(problem):
        raise TypeError("point-to-point problems carry their own endpoints")
    # the branch score uses exactly the statics passed in (trajopt.py:835-836)
    geo = _geometry(problem, chain, grasp, static_centers, static_radii, default_statics=False)
    pl = np.atleast_2d(np.asarray(placements, dtype=float))
    if pl.shape[1] != geo.row_dim:
        raise ValueError(f"placement rows have dimension {pl.shape[1]}, expected {geo.row_dim}")
    nat.require_cuda()
    dev = _lift_async(geo, torch.as_tensor(pl, device="cuda").contiguous(), seed, candidates, precision)
    st = dev.status.cpu().numpy()
    if st[0] >= 0:
        raise LiftFailure(f"staged pose {int(st[0])} is not reachable tool-down")
    nk = int(st[1])
    if nk == 0:
        raise LiftFailure("every particle contains an unreachable placement")
    return LiftResult(endpoints=dev.endpoints[:nk].double().cpu().numpy(), kept=dev.kept[:nk].cpu().numpy().astype(int))


def motion_endpoints(problem, particles: int = 1) -> np.ndarray:
    if not _is_motion(problem):
        raise TypeError("motion_endpoints needs a point-to-point problem")
    ends = np.stack([problem.start, problem.goal])[None, None]
    return np.tile(ends, (particles, 1, 1, 1))


# ---------------------------------------------------------------------------
# initialization (trajopt.py:892-923)
# ---------------------------------------------------------------------------
def _pcg_state(rng) -> np.ndarray:
    st = rng.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise TypeError("init_trajectories needs a PCG64-backed numpy Generator")
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m = (1 << 64) - 1
    return np.array([s >> 64, s & m, inc >> 64, inc & m], dtype=np.uint64)


def trajectory_stream(seed: int):
    """bench._trajectory_stream (bench.py:88-91)."""
    return np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(_TRAJ_STREAM,)))


def _init_async(geo, endpoints_dev, n_active, config: TrajOptConfig, state: np.ndarray, precision: str):
    torch = _torch()
    dt = _check_precision(precision)
    P, B = endpoints_dev.shape[:2]
    T = config.waypoints_per_segment
    out = torch.empty((P, B, T, geo.dof), dtype=_tdtype(precision), device="cuda")
    st = (ctypes.c_uint64 * 4)(*[int(x) for x in state])
    nat.check(geo._lib.spasm_init_trajectories(geo.handle, dt, nat.ptr(endpoints_dev), P, B, nat.ptr(n_active),
                                               int(config.k_waypoint), int(config.k_interp), st, nat.ptr(out),
                                               _stream()), "spasm_init_trajectories")
    return out


def init_trajectories(endpoints, chain: KinematicChain, config: TrajOptConfig, rng,
                      precision: str = DEFAULT_PRECISION) -> np.ndarray:
    """Piecewise-linear seeds through uniform waypoints (trajopt.py:892-923). Consumes
    exactly the draws numpy would from ``rng`` (its state is advanced accordingly)."""
    was_np = not _is_tensor(endpoints)
    e = np.asarray(endpoints, dtype=float) if was_np else endpoints
    if e.ndim != 4 or e.shape[2] != 2:
        raise ValueError("endpoints must have shape (P, segments, 2, dof)")
    if e.shape[3] != chain.dof:
        raise ValueError("configuration dimension mismatch")
    P, B = e.shape[:2]
    geo = _geometry(None, chain, None, None, None, default_statics=False)
    ed, _ = _device(e, precision)
    state = _pcg_state(rng)
    out = _init_async(geo, ed, None, config, state, precision)
    if config.k_waypoint:
        rng.bit_generator.advance(P * B * config.k_waypoint * chain.dof)
    return _out(out, was_np)


# ---------------------------------------------------------------------------
# the augmented-Lagrangian solve (trajopt.py:936-1063)
# ---------------------------------------------------------------------------
def _particle_trajectory(values_p, geo: _Geometry) -> Trajectory:
    att = tuple(range(geo.n_segments)) if geo.manipulation else (None,) * geo.n_segments
    return Trajectory(segments=np.array(values_p, dtype=float), attached=att)


def _best_host(geo, best):
    """The accepted trajectory (B,T,J) as float64 host values, from the pinned staging the
    AL solve's one D2H copy filled (spasm_al_best_host)."""
    out = np.empty(tuple(best.shape), dtype=np.float64)
    nat.check(geo._lib.spasm_al_best_host(geo.handle, out.ctypes.data, out.size), "spasm_al_best_host")
    return out


_PINNED = {}


def _pinned_like(t):
    """A cached pinned host tensor of t's shape and dtype (reused across solves: the caller
    has read the previous contents by the time the next solve enqueues a copy into it)."""
    torch = _torch()
    key = (tuple(t.shape), t.dtype)
    h = _PINNED.get(key)
    if h is None:
        if len(_PINNED) >= 16:
            _PINNED.clear()
        h = _PINNED[key] = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    return h


def _solve_al_device(geo, values_dev, config: TrajOptConfig, place_mode, precision, *, n_active=None,
                     lift_status=None, want_report=True):
    """Launch the persistent AL solve; returns (status, result struct, best (B,T,J) tensor, report)."""
    torch = _torch()
    dt = _check_precision(precision)
    P, B, T, J = values_dev.shape
    cfg = _al_config(config, T, place_mode)
    ws_bytes = geo._lib.spasm_al_workspace_bytes(geo.handle, dt, P, ctypes.byref(cfg))
    ws = torch.empty(int(ws_bytes), dtype=torch.uint8, device="cuda")
    best = torch.empty((B, T, J), dtype=values_dev.dtype, device="cuda")
    res = nat.spasm_al_result()
    status = nat.check(geo._lib.spasm_solve_al(geo.handle, dt, ctypes.byref(cfg), nat.ptr(values_dev), P,
                                               nat.ptr(n_active), nat.ptr(lift_status), nat.ptr(ws), ws_bytes,
                                               nat.ptr(best), ctypes.byref(res), _stream()), "spasm_solve_al")
    report = AlReport(device_ms=res.device_ms, launches=2)
    if want_report and status != nat.SPASM_LIFT_FAILURE:
        report = _read_report(geo, dt, cfg, ws, P, res, precision)
    return status, res, best, report


def _read_report(geo, dt, cfg, ws, P, res, precision) -> AlReport:
    torch = _torch()
    ptrs = (ctypes.c_void_p * 10)()
    nat.check(geo._lib.spasm_al_records(geo.handle, dt, P, ctypes.byref(cfg), nat.ptr(ws), ptrs), "spasm_al_records")
    O = int(cfg.outer_iters)
    n_act = int(res.n_particles)
    n_out = int(res.n_outers)
    esz = 4 if precision == "fp32" else 8
    base = ws.data_ptr()
    host = ws.cpu().numpy()
    fdt = np.float32 if precision == "fp32" else np.float64

    def arr(i, width, dtype, count):
        off = ptrs[i] - base
        a = host[off:off + count * np.dtype(dtype).itemsize].view(dtype)
        return a

    mu = arr(0, 1, fdt, O * P).reshape(O, P)
    lam = arr(1, 3, fdt, 3 * O * P).reshape(O, P, 3)
    cons = arr(2, 3, fdt, 3 * O * P).reshape(O, P, 3)
    upd = arr(3, 3, fdt, 3 * O * P).reshape(O, P, 3)
    obj = arr(4, 1, fdt, O * P).reshape(O, P)
    viol = arr(5, 1, fdt, O * P).reshape(O, P)
    feas = arr(6, 1, np.uint8, O * P).reshape(O, P)
    rep = AlReport(device_ms=res.device_ms, launches=2)
    for o in range(n_out):
        rep.outers.append(OuterRecord(
            index=o, mu=mu[o, :n_act].astype(float), multipliers=lam[o, :n_act].astype(float),
            constraints=cons[o, :n_act].astype(float), updated_multipliers=upd[o, :n_act].astype(float),
            objective=obj[o, :n_act].astype(float), feasible=feas[o, :n_act].astype(bool),
            violation=viol[o, :n_act].astype(float)))
    if res.status == nat.SPASM_OK:
        best = math.inf
        last = rep.outers[-1]
        for p in np.flatnonzero(last.feasible):
            if last.objective[p] < best:
                best = float(last.objective[p])
                rep.accepted_objectives.append(best)
    del esz
    return rep


def solve_al(values, problem, chain: KinematicChain, config: TrajOptConfig, *, grasp: Optional[GraspSpec] = None,
             static_centers=None, static_radii=None, place_mode=None,
             precision: str = DEFAULT_PRECISION) -> AlResult:
    """Optimize a trajectory batch and return the best validated particle (trajopt.py:936-1063).

    One persistent kernel: each CTA owns a particle (inner steps, pick retraction,
    re-evaluation, validation and multiplier updates in shared memory); the first outer
    iteration with any feasible particle stops the solve, exactly as the reference's
    ``break`` does.
    """
    geo = _geometry(problem, chain, grasp, static_centers, static_radii)
    _check_values(values, geo)
    v, _ = _device(values, precision)
    v = v.clone()
    status, res, best, report = _solve_al_device(geo, v, config, place_mode, precision)
    if status == nat.SPASM_AL_FAILURE:
        raise TrajOptFailure(float(res.least_violation), report)
    return AlResult(trajectory=_particle_trajectory(best.double().cpu().numpy(), geo), objective=float(res.objective),
                    particle_index=int(res.particle_index), report=report)


# ---------------------------------------------------------------------------
# validation (trajopt.py:1071-1153)
# ---------------------------------------------------------------------------
def validate_batch(values, problem, chain: KinematicChain, *, grasp: Optional[GraspSpec] = None, static_centers=None,
                   static_radii=None, epsilon: float = DEFAULT_VALIDATION_EPSILON, precision: str = DEFAULT_PRECISION):
    """validate() for a (P, B, T, dof) batch: (feasible (P,), violation (P,))."""
    torch = _torch()
    geo = _geometry(problem, chain, grasp, static_centers, static_radii)
    _check_values(values, geo)
    dt = _check_precision(precision)
    v, was_np = _device(values, precision)
    P, B, T, J = v.shape
    cfg = _al_config(TrajOptConfig(validation_epsilon=epsilon), T, None)
    feas = torch.empty(P, dtype=torch.uint8, device="cuda")
    viol = torch.empty(P, dtype=v.dtype, device="cuda")
    nat.check(geo._lib.spasm_traj_validate(geo.handle, dt, ctypes.byref(cfg), nat.ptr(v), P, nat.ptr(feas),
                                           nat.ptr(viol), _stream()), "spasm_traj_validate")
    return feas.cpu().numpy().astype(bool), viol.double().cpu().numpy()


def validate(trajectory: Trajectory, problem, chain: KinematicChain, *, grasp: Optional[GraspSpec] = None,
             static_centers=None, static_radii=None, epsilon: float = DEFAULT_VALIDATION_EPSILON,
             precision: str = DEFAULT_PRECISION):
    """Recompute every feasibility quantity for one trajectory; (feasible, max violation)."""
    geo = _geometry(problem, chain, grasp, static_centers, static_radii)
    segs = np.asarray(trajectory.segments, dtype=float)
    if segs.shape[0] != geo.n_segments or segs.shape[2] != chain.dof:
        raise ValueError("trajectory does not match the problem layout")
    f, w = validate_batch(segs[None], problem, chain, grasp=grasp, static_centers=static_centers,
                          static_radii=static_radii, epsilon=epsilon, precision=precision)
    return bool(f[0]), float(w[0])


# ---------------------------------------------------------------------------
# export (trajopt.py:1161-1179)
# ---------------------------------------------------------------------------
def trajectory_path_length(trajectory: Trajectory) -> float:
    segs = trajectory.segments
    return float(np.sum(np.linalg.norm(np.diff(segs, axis=1), axis=-1)))


def save_trajectory(trajectory: Trajectory, path, *, max_violation: float) -> None:
    segs = trajectory.segments
    B, T, dof = segs.shape
    lines = [f"# path_length={trajectory_path_length(trajectory):.9g}", f"# max_violation={max_violation:.9g}",
             f"# columns: segment_index, t, q1..q{dof}"]
    for b in range(B):
        for t in range(T):
            lines.append(f"{b}, {t}, " + ", ".join(f"{v:.12g}" for v in segs[b, t]))
    _Path(path).write_text("\n".join(lines) + "\n")


# ---------------------------------------------------------------------------
# pipeline pieces used by bench_api.solve_scene (reference bench.py:136-268)
# ---------------------------------------------------------------------------
def _trajopt_config(scene, overrides) -> TrajOptConfig:
    merged = dict(scene.trajopt_overrides)
    if overrides:
        merged.update(overrides)
    return TrajOptConfig(**merged)


def solve_stage2(scene, result, config, seed, trajopt_overrides, t0, precision: str = "fp32", *, pending=None):
    """lift -> init -> AL solve with device-resident intermediates and one host sync (the AL
    result block); then the independent validation outside the timed span.

    With ``pending`` (a launched, uncollected stage-1 solve: particle_opt.PendingSolve) the
    lift reads the stage-1 rows in place on the device, the whole chain is enqueued behind
    the stage-1 graph, and stage 1 is collected only after the AL result: one host sync for
    the whole pipeline. Returns (SceneSolution or None, stage-1 SolveResult); None when
    stage 1 found nothing (the caller reports that failure)."""
    import time

    from .bench_api import SceneSolution

    torch = _torch()
    tcfg = _trajopt_config(scene, trajopt_overrides)
    lift_geo = _geometry(scene.problem, scene.chain, scene.grasp, scene.obstacle_centers, scene.obstacle_radii,
                         default_statics=False)
    geo = _geometry(scene.problem, scene.chain, scene.grasp, scene.obstacle_centers, scene.obstacle_radii)
    if pending is not None:
        rows_ptr, n_ptr = pending.device_rows()
        lift = _lift_async(lift_geo, None, seed, LIFT_CANDIDATES, precision,
                           device_rows=(rows_ptr, n_ptr, config.p_return))
    else:
        pl = torch.as_tensor(np.ascontiguousarray(result.particles, dtype=float)).to("cuda", non_blocking=True)
        lift = _lift_async(lift_geo, pl, seed, LIFT_CANDIDATES, precision)
    state = _pcg_state(trajectory_stream(seed))
    values = _init_async(geo, lift.endpoints, lift.status[1:], tcfg, state, precision)
    # the kept-row list reaches pinned host memory in stream order ahead of the AL solve, and
    # the accepted trajectory rides the AL solve's one D2H copy (spasm_al_best_host): no
    # further round trip after the sync
    kept_host = _pinned_like(lift.kept)
    kept_host.copy_(lift.kept, non_blocking=True)
    status, res, best, report = _solve_al_device(geo, values, tcfg, None, precision, n_active=lift.status[1:],
                                                 lift_status=lift.status, want_report=False)
    if pending is not None:
        result = pending.collect()  # already complete: the AL result came after it in stream order
        if not result.success:
            return None, result
    time_ms = (time.perf_counter() - t0) * 1e3
    n_lift = lift.P * geo.n_segments + geo.n_segments
    stats = {"stage2_particles": int(res.n_particles), "stage2_outers": int(res.n_outers),
             "stage2_iterations": int(res.n_particles) * int(res.n_outers) * int(tcfg.inner_steps),
             "stage2_launches": 6, "al_device_ms": float(res.device_ms), "lift_targets": n_lift}
    if status == nat.SPASM_LIFT_FAILURE:
        return SceneSolution(False, time_ms, result.report.restarts, result.report.steps, math.nan, stats=stats,
                             bookkeeping={"lift_failed": True}), result
    kept = kept_host[:int(res.n_particles)].numpy().copy()
    book = {"kept": kept, "accepted_outer": int(res.accepted_outer), "al_particle": int(res.particle_index),
            "objective": float(res.objective), "lift_failed": False}
    if status == nat.SPASM_AL_FAILURE:
        w = float(res.least_violation)
        return SceneSolution(False, time_ms, result.report.restarts, result.report.steps, w, max_violation=w,
                             stats=stats, bookkeeping=book), result
    traj = _particle_trajectory(_best_host(geo, best), geo)
    # the independent float64 validate of the accepted trajectory (bench.py:249) ran on the
    # device behind the AL solve (spasm_solve_al: checked_feasible / checked_violation)
    feasible, worst = bool(res.checked_feasible), float(res.checked_violation)
    return SceneSolution(bool(feasible), time_ms, result.report.restarts, result.report.steps, worst,
                         placement=np.asarray(result.particles)[int(kept[res.particle_index])].copy(),
                         trajectory=traj, path_length=trajectory_path_length(traj), max_violation=worst, stats=stats,
                         bookkeeping=book), result


def solve_motion_scene(scene, seed, trajopt_overrides, precision: str = "fp32"):
    """_solve_motion (bench.py:136-165)."""
    import time

    from .bench_api import SceneSolution

    torch = _torch()
    tcfg = _trajopt_config(scene, trajopt_overrides)
    geo = _geometry(scene.problem, scene.chain, None, None, None)
    t0 = time.perf_counter()
    ends = torch.as_tensor(motion_endpoints(scene.problem)).to(device="cuda", dtype=_tdtype(precision))
    values = _init_async(geo, ends, None, tcfg, _pcg_state(trajectory_stream(seed)), precision)
    status, res, best, report = _solve_al_device(geo, values, tcfg, None, precision, want_report=False)
    time_ms = (time.perf_counter() - t0) * 1e3
    stats = {"stage2_particles": 1, "stage2_outers": int(res.n_outers),
             "stage2_iterations": int(res.n_outers) * int(tcfg.inner_steps), "stage2_launches": 4,
             "al_device_ms": float(res.device_ms)}
    if status == nat.SPASM_AL_FAILURE:
        w = float(res.least_violation)
        return SceneSolution(False, time_ms, 0, 0, w, max_violation=w, stats=stats)
    traj = _particle_trajectory(_best_host(geo, best), geo)
    feasible, worst = bool(res.checked_feasible), float(res.checked_violation)  # device float64 validate
    return SceneSolution(bool(feasible), time_ms, 0, 0, worst, trajectory=traj,
                         path_length=trajectory_path_length(traj), max_violation=worst, stats=stats)
