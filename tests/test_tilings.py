"""Exhaustive grid-enumeration oracle (reference tests/_oracles.py:18-70,
tests/test_problems.py:425-446): every grid-aligned assignment of block origins is evaluated
in QUADRATIC mode; the set with cost < 1e-9 must equal the reference's
(tests/golden/tilings.json: domino2 2, tetris4 12, tetris5 exactly 4, tetris6 12 tilings out
of up to 648,000 assignments). Exact set equality: the CPU oracle (float64) here, the GPU
model in fp64 and in fp32 (the fp32 path's cancellation-free wall form keeps the wall-tangent
rows of a tight packing exactly inactive)."""
from __future__ import annotations

import itertools
import json
import os

import numpy as np
import pytest

from oracle import stage1 as orc
from paper_2510_07674_b200.problems import as_cost_model, load_scene

T = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "tilings.json")))


def _rows(name):
    p = load_scene(name).problem
    per = T[name]["placements"]
    combos = np.array(list(itertools.product(*[range(len(c)) for c in per])), dtype=np.int64)
    c = p.cell_size
    rows = np.empty((len(combos), 3 * len(per)))
    for b, cells in enumerate(per):
        cells = np.asarray(cells, float)
        rows[:, 3 * b] = p.box.min[0] + cells[combos[:, b], 0] * c
        rows[:, 3 * b + 1] = p.box.min[1] + cells[combos[:, b], 1] * c
        rows[:, 3 * b + 2] = p.z_star
    return combos, rows


def _hits(combos, costs):
    return sorted(tuple(int(v) for v in combos[i]) for i in np.flatnonzero(costs < 1e-9))


@pytest.mark.parametrize("name", ["domino2", "tetris4", "tetris5"])
def test_oracle_tilings_match_reference(name):
    combos, rows = _rows(name)
    assert len(combos) == T[name]["assignments"]
    costs = orc.oracle_model(load_scene(name).problem).evaluate(rows, "quadratic")
    assert _hits(combos, costs) == sorted(tuple(t) for t in T[name]["tilings"])


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("name", ["domino2", "tetris4", "tetris5", "tetris6"])
def test_gpu_tilings_match_reference(name, precision):
    combos, rows = _rows(name)
    model = as_cost_model(load_scene(name).problem, precision=precision)
    costs = np.concatenate([np.asarray(model.evaluate(rows[i:i + 65536], "quadratic"))
                            for i in range(0, len(rows), 65536)])
    hits = _hits(combos, costs)
    assert hits == sorted(tuple(t) for t in T[name]["tilings"])
    if name == "tetris5":
        assert len(hits) == 4
