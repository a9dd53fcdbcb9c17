"""INTEGRATION.md section 1, executed: the maintainer's rebinding applied to the REFERENCE
package staged in baseline/_ref (scripts/stage_reference.py; git-ignored, it travels to the
GPU box with the repo snapshot), then the reference's stock ``seqplace.bench.solve_scene``
and ``run_trials`` run end to end on the GPU path. Outcomes are compared with the
reference's own decisions for the same seeds (tests/golden/pipeline_reference.json) and the
returned trajectories with the reference's own ``validate`` (its float64 numpy code)."""
from __future__ import annotations

import json
import os
import re
import sys

import numpy as np
import pytest

from conftest import ROOT

REF = os.path.join(ROOT, "baseline", "_ref")
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "pipeline_reference.json")))
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "seqplace")),
                                 reason="reference not staged (python scripts/stage_reference.py)")]


@pytest.fixture(scope="module")
def ref_bench():
    sys.path.insert(0, REF)
    import seqplace.bench as rb

    from paper_2510_07674_b200 import dropin

    originals = {n: getattr(rb, n) for n in ("solve", "solve_al", "validate", "lift_placements")}
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    block = next(b for b in re.findall(r"```python\n(.*?)```", doc, re.S) if "dropin import enable" in b)
    ns = {}
    exec(compile(block, "INTEGRATION.md", "exec"), ns)
    yield rb, originals
    dropin.disable(rb, ns["previous"])


def test_rebinding_routes_reference_names_to_the_gpu(ref_bench):
    rb, originals = ref_bench
    for n, fn in originals.items():
        assert getattr(rb, n) is not fn
        assert getattr(rb, n).__wrapped__.__module__.startswith("paper_2510_07674_b200") or \
            getattr(rb, n).__wrapped__.func.__module__.startswith("paper_2510_07674_b200")


@pytest.mark.parametrize("case", ["tower4/1", "tower3c/0", "single1/2", "tetris5/4", "tetris5/0"])
def test_stock_solve_scene_runs_on_gpu(ref_bench, case):
    rb, originals = ref_bench
    from oracle.refscene import ref_scene

    name, seed = case.split("/")
    gold = GOLD["pipeline"][case]
    scene = ref_scene(name)
    sol = rb.solve_scene(scene, seed=int(seed))
    assert sol.success == gold["success"], (case, sol.final_cost)
    assert sol.restarts == gold["restarts"]
    if sol.success:
        # the reference's own float64 validate accepts the GPU trajectory
        ok, worst = originals["validate"](sol.trajectory, scene.problem, scene.chain, grasp=scene.grasp,
                                          static_centers=scene.obstacle_centers, static_radii=scene.obstacle_radii)
        assert ok, worst
        assert np.isfinite(sol.path_length) and sol.time_ms > 0


def test_stock_run_trials_stage1_on_gpu(ref_bench):
    rb, _ = ref_bench
    from oracle.refscene import ref_scene

    records, summary = rb.run_trials(ref_scene("tetris5"), 4, seed=0, no_trajopt=True)
    assert summary.successes == 4
    for r in records:
        gold = GOLD["stage1"][f"tetris5/{r.seed}"]
        assert r.success == gold["success"] and r.restarts == gold["restarts"]
