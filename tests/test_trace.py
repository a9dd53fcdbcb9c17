"""Trace path (reference bench.py:518-630): trace_solve, export_trace, selection_efficacy,
against the reference's own outputs frozen in tests/golden/trace.npz
(tests/golden/make_golden_trace.py).

CPU: export_trace is byte-identical to the reference's writer on the same TraceData.
GPU (fp64): trace_solve picks the identical traced rows (ids, selected flags) and
satisfied flags; per-step costs rtol 1e-8 (the fused fp64 schedule);
selection_efficacy returns the reference's exact fractions (same rejected subset).
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from conftest import golden
from paper_2510_07674_b200.particle_opt import TraceData
from paper_2510_07674_b200.problems import load_scene
from paper_2510_07674_b200.reporting import export_trace, selection_efficacy, trace_solve

G = golden("trace.npz")


def _golden_trace(name):
    c = G[f"{name}_costs"]
    return TraceData(steps=np.arange(1, c.shape[0] + 1), particle_ids=G[f"{name}_ids"], selected=G[f"{name}_selected"],
                     costs=c, satisfied=G[f"{name}_satisfied"])


@pytest.mark.parametrize("name", ["tetris5", "tower4"])
def test_export_trace_bytes_match_reference_writer(name, tmp_path):
    p = tmp_path / "t.csv"
    export_trace(_golden_trace(name), p)
    assert p.read_bytes() == G[f"{name}_csv"].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["tetris5", "tower4"])
def test_trace_solve_matches_reference(name, tmp_path):
    tr = trace_solve(load_scene(name), seed=3, precision="fp64")
    np.testing.assert_array_equal(tr.particle_ids, G[f"{name}_ids"])
    np.testing.assert_array_equal(tr.selected, G[f"{name}_selected"])
    np.testing.assert_array_equal(tr.satisfied, G[f"{name}_satisfied"])
    np.testing.assert_allclose(tr.costs, G[f"{name}_costs"], rtol=1e-8, atol=1e-14)
    p = tmp_path / "t.csv"
    export_trace(tr, p)
    ours = p.read_text().splitlines()
    ref = G[f"{name}_csv"].tobytes().decode().splitlines()
    assert len(ours) == len(ref) and ours[0] == ref[0]
    # every column but the cost text is identical
    for a, b in zip(ours[1:], ref[1:]):
        fa, fb = a.split(","), b.split(",")
        assert fa[:2] == fb[:2] and fa[3:] == fb[3:]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["tetris5", "domino2"])
def test_selection_efficacy_matches_reference(name):
    s, r, trials, n, m = G[f"eff_{name}"]
    got = selection_efficacy(load_scene(name), trials=int(trials), seed=1, solver_overrides={"n": int(n), "m": int(m)},
                             precision="fp64")
    assert got == (s, r)
