"""Trial and batch-size-sweep reporting around ``bench_api.solve_scene``, with the
reference's record types and CSV formats (reference bench.py:275-510), so GPU runs emit
files the reference's readers and plots accept unchanged.

* ``run_trials``: sequential timed solves with per-trial seeds ``seed + i``
  (bench.py:322-365); ``summarize``: success rate, mean and normal-approximation 95 % CI
  of the successful trials' times (bench.py:297-319).
* ``run_sweep``: the placement-stage (n, m) grid, n-major, cells with m > n skipped and
  recorded (bench.py:409-460).
* CSV: ``write_trials_csv`` (bench.py:374-382), ``write_sweep_csv`` / ``read_sweep_csv``
  (bench.py:463-510). Floats are written with ``repr`` and missing values as "".
"""
from __future__ import annotations

import csv
import math
import re
import statistics
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

from .bench_api import solve_scene


@dataclass(frozen=True)
class TrialRecord:
    trial: int
    seed: int
    success: bool
    time_ms: float
    restarts: int
    steps: int
    final_cost: float
    path_length: Optional[float]


@dataclass(frozen=True)
class TrialSummary:
    trials: int
    successes: int
    success_rate: float
    mean_ms: float
    ci95_ms: float


def summarize(records: Sequence[TrialRecord]) -> TrialSummary:
    ok_times = [r.time_ms for r in records if r.success]
    n, k = len(records), len(ok_times)
    if k == 0:
        mean, ci = math.nan, math.nan
    elif k == 1:
        mean, ci = ok_times[0], 0.0
    else:
        mean = statistics.mean(ok_times)
        ci = 1.96 * statistics.stdev(ok_times) / math.sqrt(k)
    return TrialSummary(trials=n, successes=k, success_rate=(k / n) if n else math.nan, mean_ms=mean, ci95_ms=ci)


def run_trials(scene, trials: int, *, seed: int = 0, threads: int = 1, solver_overrides: Optional[dict] = None,
               trajopt_overrides: Optional[dict] = None, quadratic_only: bool = False, no_trajopt: bool = False,
               warm_seeds=None, precision: str = "fp32", model=None) -> Tuple[List[TrialRecord], TrialSummary]:
    if trials < 1:
        raise ValueError("trials must be >= 1")
    out = []
    for i in range(trials):
        s = solve_scene(scene, seed=seed + i, threads=threads, solver_overrides=solver_overrides,
                        trajopt_overrides=trajopt_overrides, quadratic_only=quadratic_only, no_trajopt=no_trajopt,
                        warm_seeds=warm_seeds, precision=precision, model=model)
        out.append(TrialRecord(trial=i, seed=seed + i, success=s.success, time_ms=s.time_ms, restarts=s.restarts,
                               steps=s.steps, final_cost=s.final_cost, path_length=s.path_length))
    return out, summarize(out)


def _num(v) -> str:
    return "" if v is None else repr(float(v))


def write_trials_csv(records: Sequence[TrialRecord], path) -> None:
    rows = [["trial", "seed", "success", "restarts", "steps", "final_cost", "path_length"]]
    rows += [[r.trial, r.seed, int(r.success), r.restarts, r.steps, _num(r.final_cost), _num(r.path_length)]
             for r in records]
    with open(path, "w", newline="") as fh:
        csv.writer(fh, lineterminator="\n").writerows(rows)


@dataclass(frozen=True)
class SweepCell:
    n: int
    m: int
    trials: int
    success_rate: float
    mean_ms: float
    ci95_ms: float


@dataclass
class SweepGrid:
    n_values: List[int]
    m_values: List[int]
    trials: int
    cells: List[SweepCell]
    skipped: List[Tuple[int, int]]


def run_sweep(scene, n_values: Sequence[int], m_values: Sequence[int], trials: int, *, seed: int = 0,
              threads: int = 1, solver_overrides: Optional[dict] = None, quadratic_only: bool = False,
              precision: str = "fp32", model=None) -> SweepGrid:
    cells, skipped = [], []
    for n in (int(v) for v in n_values):
        for m in (int(v) for v in m_values):
            if m > n:
                skipped.append((n, m))
                continue
            _, s = run_trials(scene, trials, seed=seed, threads=threads,
                              solver_overrides={**(solver_overrides or {}), "n": n, "m": m},
                              quadratic_only=quadratic_only, no_trajopt=True, precision=precision, model=model)
            cells.append(SweepCell(n, m, trials, s.success_rate, s.mean_ms, s.ci95_ms))
    return SweepGrid([int(v) for v in n_values], [int(v) for v in m_values], trials, cells, skipped)


def write_sweep_csv(grid: SweepGrid, path) -> None:
    lines = ["n,m,trials,success_rate,mean_ms,ci95_ms"]
    lines += [f"# skipped n={n} m={m}: need m <= n" for n, m in grid.skipped]
    lines += [f"{c.n},{c.m},{c.trials},{_num(c.success_rate)},{_num(c.mean_ms)},{_num(c.ci95_ms)}" for c in grid.cells]
    with open(path, "w", newline="") as fh:
        fh.write("\n".join(lines) + "\n")


_SKIPPED = re.compile(r"# skipped n=(\d+) m=(\d+)")


def read_sweep_csv(path) -> SweepGrid:
    cells, skipped = [], []
    for raw in open(path, newline=""):
        line = raw.strip()
        if not line or line.startswith("n,"):
            continue
        if line.startswith("#"):
            hit = _SKIPPED.match(line)
            if hit:
                skipped.append((int(hit.group(1)), int(hit.group(2))))
            continue
        f = line.split(",")
        cells.append(SweepCell(int(f[0]), int(f[1]), int(f[2]), float(f[3]), float(f[4]), float(f[5])))
    ns = sorted({c.n for c in cells} | {n for n, _ in skipped})
    ms = sorted({c.m for c in cells} | {m for _, m in skipped})
    return SweepGrid(ns, ms, cells[0].trials if cells else 0, cells, skipped)
