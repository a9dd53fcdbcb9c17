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


# ---------------------------------------------------------------------------
# cost traces and selection efficacy (reference bench.py:518-630)
# ---------------------------------------------------------------------------
def trace_solve(scene, *, seed: int = 0, threads: int = 1, solver_overrides: Optional[dict] = None,
                quadratic_only: bool = False, precision: str = "fp64"):
    """Cost evolution of one sampling pass, mixing selected and rejected rows
    (bench.py:518-572): the first sampling batch of restart 0 is ranked once; the traced
    subset is the best half of the selection plus an equal number of rejected particles
    spread evenly over the rejected cost range; all traced rows run the full two-phase
    schedule in ONE fused kernel launch whose device trace buffers record, after every
    step, the cost in the active phase's mode and the QUADRATIC < epsilon flag."""
    import numpy as np
    import torch

    from . import _native as nat
    from .bench_api import _solver_config
    from .particle_opt import (TRACE_PARTICLE_CAP, TraceData, _sort_indices, restart_stream, sample_uniform,
                               torch_dtype)
    from .problems import MotionProblem, as_cost_model

    if isinstance(scene.problem, MotionProblem):
        raise ValueError("tracing applies to placement scenes")
    model = as_cost_model(scene.problem, precision=precision)
    config = _solver_config(scene, seed, solver_overrides, quadratic_only)
    batch = sample_uniform(model, config.n, restart_stream(config.seed, 0))
    costs = model.evaluate(batch.values, "linear")
    order = _sort_indices(costs, config.n)  # the stable ranking; its first m rows are select_topk
    n_traced = min(config.m, TRACE_PARTICLE_CAP)
    n_rej = min(n_traced // 2, config.n - config.m)
    n_sel = n_traced - n_rej
    top = order[:config.m]
    if n_rej:
        pool = order[config.m:]
        pick = torch.as_tensor(np.round(np.linspace(0, len(pool) - 1, n_rej)).astype(np.int64), device=pool.device)
        ids = torch.cat([top[:n_sel], pool[pick]])
    else:
        ids = top[:n_sel].clone()
    selected = np.zeros(len(ids), dtype=bool)
    selected[:n_sel] = True
    steps_total = config.k_lin + config.k_quad
    rows = ids.to(torch.int32).contiguous()
    P = len(rows)
    out_v = torch.empty((P, model.dimension), dtype=batch.values.dtype, device="cuda")
    out_c = torch.empty(P, dtype=batch.values.dtype, device="cuda")
    fl = torch.zeros(P, dtype=torch.uint8, device="cuda")
    tc = torch.zeros((steps_total, P), dtype=torch_dtype(model.precision), device="cuda")
    ts = torch.zeros((steps_total, P), dtype=torch.uint8, device="cuda")
    nat.check(nat.load().spasm_descent_schedule(
        model.handle, model.dtype_id, nat.ptr(batch.values), nat.ptr(rows), P, config.k_lin, config.k_quad,
        config.eta_init, config.alpha, config.epsilon, nat.ptr(out_v), nat.ptr(out_c), nat.ptr(fl), None, nat.ptr(tc),
        nat.ptr(ts), P, nat.stream_handle()), "descent_schedule (traced)")
    return TraceData(steps=np.arange(1, steps_total + 1), particle_ids=ids.cpu().numpy().astype(np.int64),
                     selected=selected, costs=tc.double().cpu().numpy(), satisfied=ts.cpu().numpy().astype(bool))


def export_trace(trace, csv_path, *, svg_path=None) -> None:
    """Write the per-step cost table, step-major (bench.py:575-589): byte-identical to the
    reference's writer for the same TraceData."""
    with open(csv_path, "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(["step", "particle_id", "cost", "selected", "satisfied"])
        for si, step in enumerate(trace.steps):
            for pi, pid in enumerate(trace.particle_ids):
                w.writerow([int(step), int(pid), repr(float(trace.costs[si, pi])), int(trace.selected[pi]),
                            int(trace.satisfied[si, pi])])
    if svg_path is not None:
        # the reference's plots.plot_trace needs matplotlib, which this image does not ship
        import matplotlib  # noqa: F401  (raises ModuleNotFoundError exactly as the reference would)

        raise NotImplementedError("SVG trace plots are out of scope (SURVEY.md section 2: plots)")


def selection_efficacy(scene, *, trials: int = 20, seed: int = 0, threads: int = 1,
                       solver_overrides: Optional[dict] = None, precision: str = "fp64") -> Tuple[float, float]:
    """Satisfaction rate after the schedule: the selected top-m particles versus an
    equal-size random subset of the rejected ones, pooled over trials (bench.py:597-630).

    Sampling, ranking, the fused schedule and the satisfaction test run on the GPU. The
    rejected subset is the reference's ``rng.choice(pool, m, replace=False)`` on the
    restart stream continued past the batch draw: numpy's own Generator on the same
    SeedSequence state advanced by the n*D doubles the uniform draw consumed, so the subset
    is the reference's exactly."""
    import numpy as np
    import torch

    from .bench_api import _solver_config
    from .particle_opt import _sort_indices, restart_stream, run_descent_schedule, sample_uniform
    from .problems import MotionProblem, as_cost_model

    if isinstance(scene.problem, MotionProblem):
        raise ValueError("placement scenes only")
    model = as_cost_model(scene.problem, precision=precision)
    sel_hits = rej_hits = total = 0
    for i in range(trials):
        config = _solver_config(scene, seed + i, solver_overrides, False)
        if config.n - config.m < config.m:
            raise ValueError("need n >= 2*m to draw the rejected subset")
        batch = sample_uniform(model, config.n, restart_stream(config.seed, 0))
        costs = model.evaluate(batch.values, "linear")
        top = _sort_indices(costs, config.m)
        rng = np.random.default_rng(np.random.SeedSequence(entropy=config.seed, spawn_key=(0,)))
        rng.bit_generator.advance(config.n * model.dimension)
        pool = np.setdiff1d(np.arange(config.n), top.cpu().numpy())
        rejected = torch.as_tensor(rng.choice(pool, size=config.m, replace=False), device="cuda")
        values = torch.cat([batch.values[top], batch.values[rejected]])
        run_descent_schedule(model, values, config, threads=threads)
        sat = model.satisfaction(values, config.epsilon)
        sat = sat.cpu().numpy() if hasattr(sat, "cpu") else np.asarray(sat)
        sel_hits += int(np.count_nonzero(sat[:config.m]))
        rej_hits += int(np.count_nonzero(sat[config.m:]))
        total += config.m
    return sel_hits / total, rej_hits / total
