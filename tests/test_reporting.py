"""Trial / sweep reporting (reporting.py) keeps the reference's record semantics and CSV
formats (reference bench.py:297-510): checked against the reference's own writers, imported
from /root/reference in this container when present (skipped elsewhere), plus the summary
statistics and a sweep CSV round trip. A GPU test runs real trials."""
from __future__ import annotations

import math
import os
import sys

import numpy as np
import pytest

from paper_2510_07674_b200 import reporting as rp

REF = "/root/reference/pkg/src"


def _records():
    return [rp.TrialRecord(0, 7, True, 12.5, 0, 22, 1.25e-05, None),
            rp.TrialRecord(1, 8, False, 99.0, 3, 88, math.nan, None),
            rp.TrialRecord(2, 9, True, 10.0, 1, 44, 3e-06, 2.75)]


def test_summarize_counts_successful_trials_only():
    s = rp.summarize(_records())
    assert (s.trials, s.successes) == (3, 2)
    assert s.success_rate == pytest.approx(2 / 3)
    assert s.mean_ms == pytest.approx(11.25)
    assert s.ci95_ms == pytest.approx(1.96 * np.std([12.5, 10.0], ddof=1) / math.sqrt(2))
    one = rp.summarize(_records()[:1])
    assert (one.mean_ms, one.ci95_ms) == (12.5, 0.0)
    assert math.isnan(rp.summarize(_records()[1:2]).mean_ms)


def _grid():
    return rp.SweepGrid([64, 128], [32, 128], 3,
                        [rp.SweepCell(64, 32, 3, 1.0, 1.5, 0.25), rp.SweepCell(128, 32, 3, 2 / 3, 2.0, 0.1),
                         rp.SweepCell(128, 128, 3, 0.0, math.nan, math.nan)], [(64, 128)])


def test_sweep_csv_round_trip(tmp_path):
    p = tmp_path / "sweep.csv"
    rp.write_sweep_csv(_grid(), p)
    text = p.read_text()
    assert text.splitlines()[0] == "n,m,trials,success_rate,mean_ms,ci95_ms"
    assert "# skipped n=64 m=128: need m <= n" in text
    back = rp.read_sweep_csv(p)
    assert back.skipped == [(64, 128)] and back.n_values == [64, 128] and back.m_values == [32, 128]
    assert [c.n for c in back.cells] == [64, 128, 128] and back.cells[1].success_rate == 2 / 3


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_csv_bytes_match_the_reference_writers(tmp_path):
    pytest.importorskip("numpy")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    try:
        from seqplace import bench as rb
    except Exception as exc:  # pragma: no cover - optional dependency of the reference
        pytest.skip(f"reference bench not importable: {exc}")
    ref_recs = [rb.TrialRecord(**r.__dict__) for r in _records()]
    rp.write_trials_csv(_records(), tmp_path / "a.csv")
    rb.write_trials_csv(ref_recs, tmp_path / "b.csv")
    assert (tmp_path / "a.csv").read_bytes() == (tmp_path / "b.csv").read_bytes()
    g = _grid()
    ref_grid = rb.SweepGrid(g.n_values, g.m_values, g.trials, [rb.SweepCell(**c.__dict__) for c in g.cells], g.skipped)
    rp.write_sweep_csv(g, tmp_path / "c.csv")
    rb.write_sweep_csv(ref_grid, tmp_path / "d.csv")
    assert (tmp_path / "c.csv").read_bytes() == (tmp_path / "d.csv").read_bytes()


@pytest.mark.gpu
def test_run_trials_and_sweep_on_gpu(tmp_path):
    from paper_2510_07674_b200.problems import load_scene

    scene = load_scene("tetris5")
    recs, s = rp.run_trials(scene, 3, seed=4, no_trajopt=True)
    assert [r.seed for r in recs] == [4, 5, 6] and s.trials == 3 and s.successes == sum(r.success for r in recs)
    grid = rp.run_sweep(scene, [1024, 4096], [512, 2048], 2, seed=1)
    assert grid.skipped == [(1024, 2048)] and len(grid.cells) == 3
    rp.write_trials_csv(recs, tmp_path / "t.csv")
    assert (tmp_path / "t.csv").read_text().startswith("trial,seed,success,restarts,steps,final_cost,path_length\n")
