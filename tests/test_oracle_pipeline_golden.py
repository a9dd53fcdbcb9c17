"""Pins oracle/pipeline.py (the CPU restatement of bench.solve_scene, bench.py:168-268) to the
reference's own pipeline decisions frozen in tests/golden/pipeline_reference.json
(tests/golden/make_golden_pipeline.py). A bounded subset keeps the CPU suite in minutes;
the GPU suite compares every case (tests/test_pipeline_parity_gpu.py)."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from oracle import pipeline
from paper_2510_07674_b200.problems import load_scene

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "pipeline_reference.json")))


@pytest.mark.parametrize("case", ["single1/0", "tower4/1", "tower3c/0", "tetris5/0"])
def test_oracle_pipeline_matches_reference(case):
    name, seed = case.split("/")
    ref = GOLD["pipeline"][case]
    r = pipeline.solve_scene(load_scene(name), seed=int(seed), threads=4)
    assert r.success == ref["success"]
    assert r.restarts == ref["restarts"]
    np.testing.assert_array_equal(r.stage1_indices, ref["stage1_indices"])
    if ref["kept"] is not None:
        np.testing.assert_array_equal(r.kept, ref["kept"])
    assert r.accepted_outer == ref["accepted_outer"]
    if ref["accepted_outer"] >= 0:
        assert r.al_particle == ref["al_particle"]
        np.testing.assert_allclose(r.objective, ref["objective"], rtol=1e-10)
        np.testing.assert_allclose(r.max_violation, ref["final_cost"], rtol=1e-10)
    else:
        np.testing.assert_allclose(r.max_violation, ref["least_violation"], rtol=1e-10)


@pytest.mark.parametrize("case", ["tower6r/0", "tetris4/0", "tetris4/1", "tetris6/0", "single1/3", "tower3c/2"])
def test_oracle_stage1_matches_reference(case):
    name, seed = case.split("/")
    ref = GOLD["stage1"][case]
    r = pipeline.solve_scene(load_scene(name), seed=int(seed), threads=4, no_trajopt=True)
    assert r.success == ref["success"]
    assert r.restarts == ref["restarts"]
    np.testing.assert_array_equal(r.stage1_indices, ref["stage1_indices"])
