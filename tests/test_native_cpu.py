"""The C-ABI library loads, exports every symbol include/spasm.h declares, and its
host-only entry points behave (no GPU needed: no compute calls here)."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2510_07674_b200 import _native as nat


def declared_functions():
    names = set()
    for h in os.listdir(os.path.join(ROOT, "include")):
        if h.endswith(".h"):
            src = open(os.path.join(ROOT, "include", h)).read()
            names |= set(re.findall(r"\b(spasm_[a-z0-9_]+)\s*\(", src))
    return sorted(names)


def test_library_exports_every_declared_symbol():
    lib = nat.load()
    names = declared_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(lib, n), n
    # the ctypes signature table covers the whole header
    assert set(names) <= set(nat.SIGNATURES)


@pytest.mark.parametrize("seed,restart", [(0, 0), (0, 1), (12345, 7), (2**40 + 3, 1 << 20), (99, 63)])
def test_seedsequence_restatement_matches_numpy(seed, restart):
    out = (ctypes.c_uint64 * 4)()
    assert nat.load().spasm_pcg64_state(seed, restart, out) == 0
    st = np.random.PCG64(np.random.SeedSequence(entropy=seed, spawn_key=(restart,))).state["state"]
    assert (out[0] << 64) | out[1] == st["state"]
    assert (out[2] << 64) | out[3] == st["inc"]


def test_model_create_rejects_bad_input():
    lib = nat.load()
    h = ctypes.c_void_p()
    spb = np.array([1], dtype=np.int32)
    c = np.zeros((1, 3))
    r = np.ones(1)
    lo = np.array([1.0, 0.0, 0.0])
    hi = np.array([0.0, 1.0, 1.0])  # lower > upper
    st = lib.spasm_tetris_model_create(ctypes.byref(h), 1, nat.ptr(spb), nat.ptr(c), nat.ptr(r), 0, None, None, None,
                                       1.0, 1.0, 1.0, 0.0, 0, nat.ptr(lo), nat.ptr(hi))
    assert st == nat.SPASM_ERR_USAGE
    assert "lower bound" in nat.last_error()
    with pytest.raises(ValueError):
        nat.check(st, "create")


def test_model_dimension_and_destroy():
    from paper_2510_07674_b200.problems import as_cost_model, load_scene

    for name, d in (("tetris5", 15), ("tetris8", 24), ("tower4", 12), ("domino2", 6)):
        m = as_cost_model(load_scene(name).problem)
        assert nat.load().spasm_model_dimension(m.handle) == d == m.dimension


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2510_07674_b200.problems import as_cost_model, load_scene

    m = as_cost_model(load_scene("tetris5").problem)
    with pytest.raises(nat.NativeError):
        m.evaluate(np.zeros((2, 15)), "linear")


def test_traj_handles_build_without_gpu():
    """spasm_traj_create is host-only (device tables upload lazily): every robot scene's
    _Geometry builds here, and malformed descriptions are rejected with SPASM_ERR_USAGE."""
    from paper_2510_07674_b200 import trajopt as tj
    from paper_2510_07674_b200.problems import load_scene

    for name in ("tower4", "tetris5", "single1", "tower3c", "corridor3"):
        sc = load_scene(name)
        geo = tj._geometry(sc.problem, sc.chain, sc.grasp, None, None)
        assert nat.load().spasm_traj_segments(geo.handle) == geo.n_segments
    lib = nat.load()
    ch = nat.spasm_chain()
    ch.dof = 9  # > 8 joints
    d = nat.spasm_traj_desc()
    h = ctypes.c_void_p()
    assert lib.spasm_traj_create(ctypes.byref(h), ctypes.byref(ch), ctypes.byref(d)) == nat.SPASM_ERR_USAGE
    assert "dof" in nat.last_error()


def test_trajectory_stream_state_matches_numpy():
    for seed in (0, 1, 77, 2**33 + 5):
        out = (ctypes.c_uint64 * 4)()
        assert nat.load().spasm_trajectory_stream_state(seed, out) == 0
        st = np.random.PCG64(np.random.SeedSequence(entropy=seed, spawn_key=(1 << 20,))).state["state"]
        assert (out[0] << 64) | out[1] == st["state"]
        assert (out[2] << 64) | out[3] == st["inc"]


def test_trajopt_config_validation_mirrors_reference():
    from paper_2510_07674_b200.trajopt import TrajOptConfig

    assert TrajOptConfig(k_waypoint=1, k_interp=5).waypoints_per_segment == 11
    for bad in ({"k_waypoint": -1}, {"k_interp": 0}, {"w_start": -1.0}, {"mu0": 0.0}, {"beta": 1.0},
                {"outer_iters": 0}, {"inner_steps": 0}, {"lr_init": 0.0}, {"validation_epsilon": 0.0}):
        with pytest.raises(ValueError):
            TrajOptConfig(**bad)


ABI_STRUCTS = ["spasm_solve_config", "spasm_solve_report", "spasm_chain", "spasm_traj_desc", "spasm_al_config",
               "spasm_al_result"]


@pytest.mark.parametrize("name", ABI_STRUCTS)
def test_abi_struct_sizes_match_ctypes_mirrors(name):
    lib = nat.load()
    assert lib.spasm_abi_sizeof(name.encode()) == ctypes.sizeof(getattr(nat, name))


def test_abi_sizeof_unknown_type():
    assert nat.load().spasm_abi_sizeof(b"no_such_struct") == -1


def test_integration_doc_ctypes_stub_matches_library():
    """Execute INTEGRATION.md's reference-side ctypes stub against the built library: every
    argtypes line binds an exported symbol and the documented SolveConfig has the library's
    size (a short mirror would make spasm_solve read past the caller's struct)."""
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", doc, re.S)
    stub = next(b for b in blocks if "class SolveConfig" in b)
    stub = stub.replace('ctypes.CDLL("paper_2510_07674_b200/libspasm.so")', "ctypes.CDLL(LIBPATH)")
    ns = {"LIBPATH": nat.load()._name}
    exec(compile(stub, "INTEGRATION.md", "exec"), ns)
    assert ctypes.sizeof(ns["SolveConfig"]) == ctypes.sizeof(nat.spasm_solve_config)
    assert [f[0] for f in ns["SolveConfig"]._fields_] == [f[0] for f in nat.spasm_solve_config._fields_]
