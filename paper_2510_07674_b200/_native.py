"""ctypes binding of libspasm.so (the C-ABI in include/spasm.h).

There is deliberately no CPU fallback: if the shared library is missing, or a call is
made without a CUDA device, this module raises. The library is built in-tree by
``__graft_entry__.build()`` (``make -C paper_2510_07674_b200/csrc``).
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, byref, c_char_p, c_double, c_int, c_int32, c_int64, c_uint8, c_uint32, c_uint64, c_void_p

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspasm.so")

SPASM_OK = 0
SPASM_NO_SOLUTION = 1
SPASM_LIFT_FAILURE = 2
SPASM_AL_FAILURE = 3
SPASM_ERR_USAGE = 100
SPASM_ERR_CUDA = 101

F32 = 0
F64 = 1
LINEAR_ID = 0
QUADRATIC_ID = 1
SAMPLER_PCG64 = 0
SAMPLER_PHILOX = 1


class NativeError(RuntimeError):
    """A CUDA or internal failure reported by libspasm."""


class spasm_solve_config(ctypes.Structure):
    _fields_ = [
        ("n", c_int64),
        ("m", c_int64),
        ("k_lin", c_int32),
        ("k_quad", c_int32),
        ("eta_init", c_double),
        ("alpha", c_double),
        ("epsilon", c_double),
        ("p_return", c_int32),
        ("max_restarts", c_int32),
        ("seed", c_uint64),
        ("sampler", c_int32),
        ("n_traced", c_int32),
        ("update", c_int32),
        ("adam_beta1", ctypes.c_float),
        ("adam_beta2", ctypes.c_float),
        ("adam_eps", ctypes.c_float),
        ("noise_sigma", ctypes.c_float),
    ]


class spasm_solve_report(ctypes.Structure):
    _fields_ = [
        ("success", c_int32),
        ("restarts", c_int32),
        ("steps", c_int32),
        ("n_satisfying", c_int32),
        ("flagged", c_int32),
        ("n_chosen", c_int32),
        ("launches", c_int32),
        ("reserved", c_int32),
        ("device_ms", c_double),
    ]


class spasm_chain(ctypes.Structure):
    _fields_ = [
        ("dof", c_int32),
        ("n_spheres", c_int32),
        ("axes", c_void_p),
        ("offsets", c_void_p),
        ("lower", c_void_p),
        ("upper", c_void_p),
        ("tool_translation", c_void_p),
        ("tool_rotation", c_void_p),
        ("sphere_centers", c_void_p),
        ("sphere_radii", c_void_p),
        ("sphere_link", c_void_p),
    ]


class spasm_traj_desc(ctypes.Structure):
    _fields_ = [
        ("manipulation", c_int32),
        ("n_blocks", c_int32),
        ("spheres_per_block", c_void_p),
        ("block_centers", c_void_p),
        ("block_radii", c_void_p),
        ("staged_poses", c_void_p),
        ("grasp_offset", c_void_p),
        ("grasp_yaw_offset", c_double),
        ("n_static", c_int32),
        ("static_centers", c_void_p),
        ("static_radii", c_void_p),
        ("place_model", c_void_p),
        ("anchor_yaw", c_int32),
        ("rows_have_yaw", c_int32),
        ("start", c_void_p),
        ("goal", c_void_p),
    ]


class spasm_al_config(ctypes.Structure):
    _fields_ = [
        ("w_start", c_double),
        ("w_arm", c_double),
        ("w_block", c_double),
        ("w_place", c_double),
        ("mu0", c_double),
        ("beta", c_double),
        ("lr_init", c_double),
        ("lr_final", c_double),
        ("validation_epsilon", c_double),
        ("outer_iters", c_int32),
        ("inner_steps", c_int32),
        ("place_mode", c_int32),
        ("waypoints", c_int32),
    ]


class spasm_al_result(ctypes.Structure):
    _fields_ = [
        ("status", c_int32),
        ("accepted_outer", c_int32),
        ("particle_index", c_int32),
        ("n_outers", c_int32),
        ("n_particles", c_int32),
        ("lift_pick_fail", c_int32),
        ("objective", c_double),
        ("least_violation", c_double),
        ("device_ms", c_double),
        ("checked_violation", c_double),
        ("checked_feasible", c_int32),
        ("reserved", c_int32),
    ]


# name -> (restype, argtypes); the full exported surface of include/spasm.h
SIGNATURES = {
    "spasm_last_error": (c_char_p, []),
    "spasm_version": (c_int, []),
    "spasm_abi_sizeof": (c_int64, [c_char_p]),
    "spasm_trim": (c_int, []),
    "spasm_fp32_peak": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "spasm_set_option": (c_int, [c_char_p, c_int]),
    "spasm_al_profile": (c_int, [c_int, c_void_p]),
    "spasm_al_profile_warps": (c_int, [c_void_p]),
    "spasm_ik_profile": (c_int, [c_int, c_void_p]),
    "spasm_selftest_math": (c_int, [c_int64, c_uint64, c_void_p]),
    "spasm_tetris_model_create": (
        c_int,
        [POINTER(c_void_p), c_int, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
         c_double, c_double, c_double, c_double, c_int, c_void_p, c_void_p],
    ),
    "spasm_tower_model_create": (
        c_int,
        [POINTER(c_void_p), c_int, c_double, c_double, c_void_p, c_int, c_void_p, c_void_p, c_double, c_double,
         c_double, c_int, c_void_p, c_void_p],
    ),
    "spasm_model_destroy": (None, [c_void_p]),
    "spasm_model_dimension": (c_int, [c_void_p]),
    "spasm_evaluate": (c_int, [c_void_p, c_int, c_void_p, c_int64, c_int, c_void_p, c_void_p]),
    "spasm_gradient": (c_int, [c_void_p, c_int, c_void_p, c_int64, c_int, c_void_p, c_void_p]),
    "spasm_pcg64_state": (c_int, [c_uint64, c_uint64, POINTER(c_uint64)]),
    "spasm_sample": (
        c_int,
        [c_int, c_int, c_void_p, c_void_p, c_uint64, c_uint64, c_int, c_int64, c_int64, c_void_p, c_int64,
         c_void_p, c_void_p],
    ),
    "spasm_sample_eval": (
        c_int,
        [c_void_p, c_int, c_uint64, c_uint64, c_int, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
         c_void_p, c_void_p],
    ),
    "spasm_step": (
        c_int,
        [c_int, c_void_p, c_void_p, c_int64, c_int, c_double, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "spasm_descent_schedule": (
        c_int,
        [c_void_p, c_int, c_void_p, c_void_p, c_int64, c_int, c_int, c_double, c_double, c_double, c_void_p,
         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p],
    ),
    "spasm_sort_workspace_bytes": (c_int64, [c_int, c_int64]),
    "spasm_sort_pairs": (c_int, [c_int, c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "spasm_cost_keys": (c_int, [c_int, c_void_p, c_int64, c_double, c_void_p, c_void_p, c_void_p, c_void_p]),
    "spasm_solve_workspace_bytes": (c_int64, [c_void_p, c_int, POINTER(spasm_solve_config), c_int64]),
    "spasm_solve": (
        c_int,
        [c_void_p, c_int, POINTER(spasm_solve_config), c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_void_p,
         c_void_p, POINTER(spasm_solve_report), c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "spasm_solve_launch": (
        c_int, [c_void_p, c_int, POINTER(spasm_solve_config), c_void_p, c_int64, c_void_p, c_int64, c_void_p]),
    "spasm_solve_collect": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, POINTER(spasm_solve_report)]),
    "spasm_solve_device_rows": (c_int, [c_void_p, POINTER(c_void_p), POINTER(c_void_p)]),
    "spasm_shard_workspace_bytes": (c_int64, [c_void_p, c_int, POINTER(spasm_solve_config), c_int64, c_int64]),
    "spasm_shard_select": (
        c_int,
        [c_void_p, c_int, POINTER(spasm_solve_config), c_int, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_int64,
         c_void_p, c_void_p, c_void_p],
    ),
    "spasm_shard_descend": (
        c_int,
        [c_void_p, c_int, POINTER(spasm_solve_config), c_int, c_void_p, c_int, c_int64, c_int64, c_int64, c_void_p,
         c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p],
    ),
    "spasm_shard_topm_state_bytes": (c_int64, []),
    "spasm_shard_topm_init": (c_int, [c_int, c_int64, c_void_p, c_void_p]),
    "spasm_shard_topm_hist": (
        c_int, [c_void_p, c_int, POINTER(spasm_solve_config), c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "spasm_shard_topm_pick": (c_int, [c_void_p, c_void_p, c_void_p]),
    "spasm_shard_topm_local": (
        c_int, [c_void_p, c_int, POINTER(spasm_solve_config), c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "spasm_shard_topm_contrib": (
        c_int, [c_void_p, c_int, POINTER(spasm_solve_config), c_int64, c_void_p, c_int64, c_int64, c_void_p,
                c_void_p]),
    "spasm_traj_create": (c_int, [POINTER(c_void_p), POINTER(spasm_chain), POINTER(spasm_traj_desc)]),
    "spasm_traj_destroy": (None, [c_void_p]),
    "spasm_traj_segments": (c_int, [c_void_p]),
    "spasm_fk": (c_int, [c_void_p, c_int, c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                         c_void_p]),
    "spasm_ik_solve": (
        c_int,
        [c_void_p, c_int, c_void_p, c_void_p, c_int64, c_uint64, c_int, c_int, c_double, c_void_p, c_void_p,
         c_void_p, c_void_p],
    ),
    "spasm_polish_tool_down": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "spasm_traj_evaluate": (
        c_int,
        [c_void_p, c_int, POINTER(spasm_al_config), c_void_p, c_int64, c_int, c_int, c_void_p, c_void_p, c_int,
         c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    ),
    "spasm_traj_validate": (
        c_int, [c_void_p, c_int, POINTER(spasm_al_config), c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "spasm_lift_workspace_bytes": (c_int64, [c_void_p, c_int, c_int64, c_int]),
    "spasm_lift": (
        c_int,
        [c_void_p, c_int, c_void_p, c_int64, c_void_p, c_int, c_uint64, c_int, c_void_p, c_int64, c_void_p, c_void_p,
         c_void_p, c_void_p],
    ),
    "spasm_trajectory_stream_state": (c_int, [c_uint64, POINTER(c_uint64)]),
    "spasm_init_trajectories": (
        c_int,
        [c_void_p, c_int, c_void_p, c_int64, c_int, c_void_p, c_int, c_int, POINTER(c_uint64), c_void_p, c_void_p],
    ),
    "spasm_al_workspace_bytes": (c_int64, [c_void_p, c_int, c_int64, POINTER(spasm_al_config)]),
    "spasm_al_records": (c_int, [c_void_p, c_int, c_int64, POINTER(spasm_al_config), c_void_p, POINTER(c_void_p)]),
    "spasm_solve_al": (
        c_int,
        [c_void_p, c_int, POINTER(spasm_al_config), c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int64,
         c_void_p, POINTER(spasm_al_result), c_void_p],
    ),
    "spasm_al_best_host": (c_int, [c_void_p, c_void_p, c_int64]),
}

_lib = None


def load() -> ctypes.CDLL:
    """Load libspasm.so once; raise loudly if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
            "(make -C paper_2510_07674_b200/csrc). There is no CPU fallback."
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    tile = os.environ.get("SPASM_STAGE1_TILE")  # tuning/profiling switch, see spasm_set_option
    if tile is not None:
        check(lib.spasm_set_option(b"stage1_tile", int(tile)), "SPASM_STAGE1_TILE")
    return lib


def last_error() -> str:
    msg = load().spasm_last_error()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> int:
    """Map a C status to the reference's exception conventions."""
    if status in (SPASM_OK, SPASM_NO_SOLUTION, SPASM_LIFT_FAILURE, SPASM_AL_FAILURE):
        return status
    msg = last_error()
    if status == SPASM_ERR_USAGE:
        raise ValueError(f"{what}: {msg}" if what else msg)
    raise NativeError(f"{what}: {msg} (status {status})" if what else f"{msg} (status {status})")


def ptr(t) -> int:
    """Raw data pointer of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def stream_handle(device=None) -> int:
    import torch

    return torch.cuda.current_stream(device).cuda_stream


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise NativeError("no CUDA device: the SPaSM B200 kernels have no CPU fallback")
