"""Benchmark: SPaSM two-stage particle optimizer on B200 (BASELINE.json metric).

One "step" is one full ``solve_scene`` call (reference bench.py:168-268) through the
public API: host scene + config in, host placement + trajectory out. It runs stage 1
(sample, stable top-M, fused K_lin+K_quad descent, satisfying extraction, restarts) and,
when the workload's scene carries a robot, stage 2 (grasp IK lifting, trajectory init,
and the persistent augmented-Lagrangian solve). The default workload is BASELINE
configs[1] (C2: 3-block stacking with cuboid obstacles, 16k particles, full pipeline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c1|c2|c3|c5]
                    [--precision fp32|fp64] [--impl b200|reference]

Multi-GPU (torchrun, one rank per GPU): weak scaling. Each restart's particle batch is
world x the per-GPU (n, m), sharded contiguously across ranks (sharded.solve_sharded: one
NCCL all-gather of the local elite keys and one of the satisfying candidates per restart,
no collective inside the step loop; result identical to one GPU solving the whole batch).
Rank 0 prints one JSON line with whole-job throughput over the max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "solve time ms (p50) at 100% success; particle-iterations/sec at 1/2/4/8 B200"

# name: (scene, solver overrides, stage-1 only, description)
WORKLOADS = {
    "c1": ("single1", {}, False,
           "C1 7-DOF arm, single-block pick-and-place, 1024 particles, stage 1 + stage 2 (32 waypoints)"),
    "c1f": ("single1f", {}, False,
            "C1 with the Franka-like explicit 7-DOF chain (Panda link offsets / limits, 11 collision spheres), "
            "single-block pick-and-place, 1024 particles, stage 1 + stage 2 (32 waypoints)"),
    "c2": ("tower3c", {}, False,
           "C2 3-block stacking with cuboid obstacles, 16k particles, stage 1 + stage 2; cuboids 0.2x0.2x0.3 m and "
           "0.1x0.1x0.2 m as grids of r=0.05 m spheres at 0.1 m pitch (2x2x3 + 1x1x2 = 14 obstacle spheres)"),
    "c3": ("tetris5", {"n": 65536, "m": 8192}, True, "C3 Tetris packing, 5 objects, 64k particles, stage 1"),
    "c3p": ("tetris5", {"n": 65536, "m": 8192}, False,
            "C3 Tetris packing, 5 objects, 64k particles, stage 1 + stage 2 (motion-constrained placements: lift + "
            "trajectory AL, B=5, T=11)"),
    "c3_4": ("tetris4", {"n": 65536, "m": 8192}, True, "C3 Tetris packing, 4 objects, 64k particles, stage 1"),
    "c3_6": ("tetris6", {"n": 65536, "m": 8192}, True, "C3 Tetris packing, 6 objects, 64k particles, stage 1"),
    "c4": ("tower6r", {"n": 16384, "m": 2048}, True,
           "C4 reactive replanning: 6-block rearrangement, one sphere obstacle moving 3 cm per tick, each tick "
           "warm-started from the previous placement, 16k particles, stage 1"),
    "c5": ("tetris8", {"n": 1 << 20, "m": 1 << 17}, True, "C5 8-object skeleton, 1M particles (M = N/8), stage 1"),
}


# ---------------------------------------------------------------------------
# algorithmic work counts
# ---------------------------------------------------------------------------
def stage1_flops_per_iteration(model, mode="linear", gradient_only=False):
    """FP32 FLOPs of one fused cost-gradient-update step of one particle.
    ``gradient_only``: the reference's step evaluates the gradient only (particle_opt.py:
    214-228), so its count drops the per-pair cost accumulation (2 flops per pair linear,
    3 quadratic) and the height-term cost."""
    from paper_2510_07674_b200.problems import TetrisCostModel

    p = model.problem
    D = model.dimension
    if isinstance(model, TetrisCostModel):
        n = p.n_blocks
        counts = [len(b.sphere_set) for b in p.blocks]
        S = sum(counts)
        E = sum(counts[i] * counts[j] for i in range(n) for j in range(i + 1, n)) + S * len(p.wall_radii)
        f = (22 if mode == "linear" else 24) * E + 3 * S + 4 * n + 2 * D
        if gradient_only:
            f -= (2 if mode == "linear" else 3) * E + 2 * n
        if model.free_yaw:
            f += 10 * E + 8 * S
        return f
    B = p.n_blocks
    O = len(p.obstacle_radii)
    pairs = B * (B - 1) // 2 + B * O
    f = 22 * pairs + 30 * (B - 1) + 4 * B + 2 * D
    if gradient_only:
        f -= (2 if mode == "linear" else 3) * pairs + 2 * B
    return f


def al_flops_per_inner_step(scene, T):
    """FLOPs of one AL inner step (value + exact gradient + clamped update) of one trajectory
    particle, counted from the shapes (trajopt.py:416-653, 993-1002):
      FK per waypoint 124 per joint + 18 per arm sphere + 63 (tool frame);
      path length 4 per dof + 1; sphere-pair penetration + gradient 20 per pair;
      held-block sphere placement 18; Jacobian-transpose products 15 per sphere + 17 per
      joint (arm) and per joint again (held); start/placement chains 40 per joint per
      segment; update 4 per dof."""
    chain = scene.chain
    J = chain.dof
    S = len(chain.sphere_table()[1])
    prob = scene.problem
    n_static = len(scene.obstacle_radii)
    if hasattr(prob, "blocks") or hasattr(prob, "n_blocks"):
        counts = [1] * prob.n_blocks if not hasattr(prob, "blocks") else [len(b.sphere_set) for b in prob.blocks]
    else:
        counts = []
    B = max(1, len(counts))
    f = 0
    for b in range(B):
        later = sum(counts[b + 1:]) if counts else 0
        earlier = sum(counts[:b]) if counts else 0
        obs = n_static + later + earlier
        SB = counts[b] if counts else 0
        for t in range(T):
            f += 124 * J + 18 * S + 63 + 4 * J + 1 + 20 * S * obs + 15 * S + 17 * J + 4 * J
            if counts and 1 <= t <= T - 2:
                f += 18 * SB + 20 * SB * obs + 15 * SB + 17 * J
        f += 40 * J
    return f


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML polled every 2 ms)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, index=0, period=0.002):
        self.index = index
        self.period = period
        self.sm = []
        self.bits = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:  # no NVML: report no samples
            self._ok = False
        return self

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.sm.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.bits |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                pass
            time.sleep(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._ok:
            self._t.join(timeout=1)

    def summary(self):
        reasons = []
        if self._ok:
            for name, attr in self.REASONS.items():
                if self.bits & int(getattr(self._nv, attr, 0)):
                    reasons.append(name)
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.sm), "source": "nvml (2 ms polling during the timed region)"}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK",
                                                                                                          "0"))


def measure_schedule_kernel(model, cfg, repeats=10):
    """Average device time of the fused stage-1 descent kernel on one M-row batch (CUDA
    events on the launching stream, L2 flushed between launches)."""
    import torch

    from paper_2510_07674_b200 import _native as nat
    from paper_2510_07674_b200 import particle_opt as po

    batch = po.sample_uniform(model, cfg.m, po.restart_stream(123, 0))
    src = batch.values.contiguous()
    out_v = torch.empty_like(src)
    out_c = torch.empty(cfg.m, dtype=src.dtype, device="cuda")
    fl = torch.empty(cfg.m, dtype=torch.uint8, device="cuda")
    lib = nat.load()
    stream = torch.cuda.current_stream()

    def launch():
        nat.check(lib.spasm_descent_schedule(model.handle, model.dtype_id, nat.ptr(src), None, cfg.m, cfg.k_lin,
                                             cfg.k_quad, cfg.eta_init, cfg.alpha, cfg.epsilon, nat.ptr(out_v),
                                             nat.ptr(out_c), nat.ptr(fl), None, None, None, 0, stream.cuda_stream))

    for _ in range(3):
        launch()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    times = []
    for _ in range(repeats):
        flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launch()
        e1.record(stream)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = statistics.mean(times)
    flops = cfg.m * (cfg.k_lin * stage1_flops_per_iteration(model, "linear")
                     + cfg.k_quad * stage1_flops_per_iteration(model, "quadratic"))
    flops_g = cfg.m * (cfg.k_lin * stage1_flops_per_iteration(model, "linear", gradient_only=True)
                       + cfg.k_quad * stage1_flops_per_iteration(model, "quadratic", gradient_only=True))
    return ms, flops, flops_g


def _traffic(key):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        return json.load(open(path)).get(key)
    return None


def fp32_peak():
    """Measured FP32 CUDA-core peak at the current clock (spasm_fp32_peak: saturating FFMA /
    FFMA2 kernels on every SM), TFLOP/s."""
    import ctypes

    import torch

    from paper_2510_07674_b200 import _native as nat

    out = (ctypes.c_double * 3)()
    nat.check(nat.load().spasm_fp32_peak(ctypes.addressof(out), ctypes.addressof(out) + 8,
                                         ctypes.addressof(out) + 16, torch.cuda.current_stream().cuda_stream),
              "spasm_fp32_peak")
    return {"tflops": out[0], "ffma_tflops": out[1], "ffma2_tflops": out[2]}


def run_b200(args, workload=None, sub=False):
    import torch

    workload = workload or args.workload
    rank, world, local = dist_env()
    local = local % max(1, torch.cuda.device_count())
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        # nccl on a real multi-GPU node; SPASM_DIST_BACKEND=gloo lets several ranks share one
        # GPU to exercise the sharded path (tests only; the collectives then stage via host)
        dist.init_process_group(os.environ.get("SPASM_DIST_BACKEND", "nccl"))
    else:
        torch.cuda.set_device(0)
    from paper_2510_07674_b200.bench_api import _solver_config, effective_max_restarts, solve_scene
    from paper_2510_07674_b200.problems import as_cost_model, load_scene

    from paper_2510_07674_b200.sharded import TorchComm

    scene_name, over, stage1_only, desc = WORKLOADS[workload]
    scene = load_scene(scene_name)
    model = as_cost_model(scene.problem, precision=args.precision)
    base = _solver_config(scene, 0, over, False)
    # weak scaling: every rank keeps the per-GPU batch (n, m); the restart's global batch is
    # world x (n, m), sharded contiguously (sharded.solve_sharded, NCCL elite exchange)
    over = {**over, "n": base.n * world, "m": base.m * world}
    cfg = _solver_config(scene, 0, over, False)
    cfg.max_restarts = effective_max_restarts(cfg)
    comm = TorchComm() if world > 1 else None

    def step(seed):
        return solve_scene(scene, seed=seed, solver_overrides=over, no_trajopt=stage1_only, precision=args.precision,
                           model=model, comm=comm)

    replan = None
    if workload == "c4":
        # one step = one replan tick: move the obstacle, rebuild the scene/model, re-solve
        # warm-started from the previous tick's placement (replan.py)
        from paper_2510_07674_b200.problems.scenes import tower6r
        from paper_2510_07674_b200.replan import obstacle_center

        replan = {"tick": 0, "warm": None, "tick_ms": []}

        def step(seed):  # noqa: F811
            t0 = time.perf_counter()
            k = replan["tick"]
            replan["tick"] += 1
            sc = load_scene(tower6r(obstacle_center=obstacle_center(k)))
            mdl = as_cost_model(sc.problem, precision=args.precision)
            sol = solve_scene(sc, seed=seed, solver_overrides=over, no_trajopt=True, precision=args.precision,
                              model=mdl, warm_seeds=replan["warm"], comm=comm)
            if sol.success:  # all returned placements seed the next tick (SPASM_C4_WARM=best: only the best)
                keep_all = os.environ.get("SPASM_C4_WARM", "all") == "all" and sol.particles is not None
                replan["warm"] = (sol.particles if keep_all else sol.placement[None, :]).copy()
            replan["tick_ms"].append((time.perf_counter() - t0) * 1e3)
            return sol

    steps = args.sub_steps if sub else args.steps
    warmup = args.warmup
    seed0 = 0
    for i in range(warmup):
        step(seed0 + 100000 + i)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    dev_ms, wall_ms, sols = [], [], []
    with ClockSampler(local) as clocks:
        for i in range(steps):
            flush.fill_(i & 0xFF)  # L2 flush between timed solves (outside the events)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            e0.record(stream)
            sol = step(seed0 + i)
            e1.record(stream)
            e1.synchronize()
            wall_ms.append((time.perf_counter() - t0) * 1e3)
            dev_ms.append(e0.elapsed_time(e1))
            sols.append(sol)
    its = sum(s.stats.get("stage1_iterations", 0) + s.stats.get("stage2_iterations", 0) for s in sols)
    succ = sum(int(s.success) for s in sols)
    launches = sum(s.stats.get("stage1_launches", 0) + s.stats.get("stage2_launches", 0) for s in sols)
    al_ms = [s.stats["al_device_ms"] for s in sols if "al_device_ms" in s.stats]
    al_its = sum(s.stats.get("stage2_iterations", 0) for s in sols)
    total_dev, total_wall = sum(dev_ms), sum(wall_ms)
    if world > 1:
        # every rank holds the same (global) result and work count; time = max over ranks
        red_dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
        t = torch.tensor([total_dev, total_wall], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_dev, total_wall = t.tolist()
        c = torch.tensor([launches], device=red_dev, dtype=torch.float64)
        dist.all_reduce(c)
        launches = int(c.item())
    clk = clocks.summary()
    sm_mhz = clk["sm_mhz"] or 1965.0
    nominal = 2 * 128 * 148 * sm_mhz * 1e6 / 1e12  # FP32 CUDA-core TFLOP/s at the measured SM clock
    pk = fp32_peak()
    peak = pk["tflops"]
    if not stage1_only and al_ms:
        T = load_scene(scene_name).trajopt_overrides.get("k_interp", 5) * (
            load_scene(scene_name).trajopt_overrides.get("k_waypoint", 1) + 1) + 1
        f_step = al_flops_per_inner_step(scene, T)
        kern_ms = statistics.mean(al_ms)
        flops = f_step * al_its / len(al_ms)
        roof = {"bound": "fp32", "achieved": flops / (kern_ms * 1e-3) / 1e12, "peak": peak, "unit": "TFLOP/s",
                "kernel": "k_solve_al (persistent AL solve, CTA per trajectory particle)", "kernel_ms": kern_ms,
                "flops_per_launch": flops, "flops_per_inner_step": f_step,
                "traffic": _traffic(f"{workload}_{args.precision}_k_solve_al"),
                "note": "latency-bound: a few dozen CTAs x serial inner steps; see DESIGN.md section 3"}
    else:
        kern_ms, flops, flops_g = measure_schedule_kernel(model, base)  # one rank's m-row launch
        roof = {"bound": "fp32", "achieved": flops / (kern_ms * 1e-3) / 1e12, "peak": peak, "unit": "TFLOP/s",
                "kernel": "k_schedule (fused K_lin+K_quad descent)", "kernel_ms": kern_ms, "flops_per_launch": flops,
                "flops_per_launch_gradient_only": flops_g,
                "frac_gradient_only": flops_g / (kern_ms * 1e-3) / 1e12 / peak,
                "traffic": _traffic(f"{workload}_{args.precision}_k_schedule")}
    roof["frac"] = roof["achieved"] / peak
    roof["peak_nominal"] = nominal
    roof["peak_note"] = (f"measured FP32 CUDA-core peak (spasm_fp32_peak: saturating FFMA "
                         f"{pk['ffma_tflops']:.1f} / FFMA2 {pk['ffma2_tflops']:.1f} TFLOP/s on 148 SMs, taken after "
                         f"the timed region; MEASURED_PEAKS.json has no FP32 figure); nominal 2*128*148*f_SM at the "
                         f"sampled {sm_mhz:.0f} MHz is peak_nominal")
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return None
    replan_line = None
    if replan is not None:
        from paper_2510_07674_b200.replan import rate_sweep

        replan_line = {**rate_sweep(replan["tick_ms"][warmup:]), "step_m": 0.03,
                       "warm_started_ticks": steps, "note": "tick = obstacle move + scene/model rebuild + solve"}
    cpu = cpu_baseline(args, workload) if (world == 1 and not args.no_cpu and not sub) else None
    D = model.dimension
    p_ret = cfg.p_return
    h2d = 0 if stage1_only else p_ret * D * 8  # stage-1 placements re-enter the device for lifting
    d2h = 64 + p_ret * (D + 3) * 8
    if not stage1_only:
        t_wp = sols[0].trajectory.segments.size if sols and sols[0].trajectory is not None else 0
        d2h += 64 + 8 * t_wp
    ref_out = _reference_outcomes(workload, [seed0 + i for i in range(steps)], sols)
    line = {
        "metric": METRIC,
        "value": its / (total_dev * 1e-3),
        "unit": "particle-iterations/s",
        "n_gpus": world,
        "steps": steps,
        "warmup": warmup,
        "ms_per_step": total_dev / steps,
        # reference bench.solve_scene span: stage 1 (+ lift + AL), excluding scene load and the
        # final independent validate (bench.py:190-247); p50_step_ms is the whole timed step
        "p50_solve_ms": statistics.median(s.time_ms for s in sols),
        # the metric's "at 100 % success": p50 over the successful solves (differs when the
        # workload's scene is not always solvable, e.g. C3p, where the reference fails too)
        "p50_solve_ms_successes": (statistics.median(s.time_ms for s in sols if s.success)
                                   if any(s.success for s in sols) else None),
        "p50_step_ms": statistics.median(wall_ms),
        "success_rate": succ / steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (bundled scene tables; particles drawn on device from numpy-identical PCG64 streams)",
        "config": {"workload": desc, "scene": scene_name, "n": cfg.n, "m": cfg.m, "k_lin": cfg.k_lin,
                   "k_quad": cfg.k_quad, "max_restarts": cfg.max_restarts, "p_return": p_ret,
                   "stage2": not stage1_only, "l2": "flushed (256 MB write) between timed solves",
                   "parallelism": (f"dp{world}: stage-1 particles sharded across ranks, NCCL all-gather of "
                                   "elite keys + candidates once per restart; stage 2 on every rank"
                                   if world > 1 else "single GPU")},
        "e2e": {"value": its / (total_wall * 1e-3), "unit": "particle-iterations/s",
                "p50_solve_ms": statistics.median(wall_ms), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "bench_api.solve_scene (host scene/config in, host placement/trajectory out)"},
        "roofline": roof,
        "cpu_baseline": cpu,
        "clocks": clk,
        "gpu_launches": launches,
        "replan": replan_line,
        "reference_outcomes": ref_out,
        "breakdown": {"stage1_ms_mean": statistics.mean(s.stats.get("stage1_ms", 0.0) for s in sols),
                      "al_device_ms_mean": statistics.mean(al_ms) if al_ms else None,
                      "stage2_outers_mean": statistics.mean(s.stats.get("stage2_outers", 0) for s in sols)},
    }
    if world > 1:
        dist.destroy_process_group()
    return line


# workload -> key prefix of the reference's own per-seed pipeline outcomes
# (tests/golden/pipeline_reference.json, made by tests/golden/make_golden_pipeline.py)
_REF_OUTCOME_KEYS = {"c3p": "tetris5@64k", "c2": "tower3c", "c1": "single1", "c1f": "single1f"}


def _reference_outcomes(workload, seeds, sols):
    """Per-seed success of this run next to the reference's own solve_scene on the same seeds
    (the fixture holds the seeds the reference was run on; others are not compared)."""
    key = _REF_OUTCOME_KEYS.get(workload)
    path = os.path.join(ROOT, "tests", "golden", "pipeline_reference.json")
    if key is None or not os.path.exists(path):
        return None
    gold = json.load(open(path))["pipeline"]
    rows = [(seed, bool(sol.success), gold[f"{key}/{seed}"]["success"]) for seed, sol in zip(seeds, sols)
            if f"{key}/{seed}" in gold]
    if not rows:
        return None
    return {"seeds_compared": len(rows), "success_here": sum(r[1] for r in rows),
            "success_reference": sum(r[2] for r in rows), "same_outcome": sum(r[1] == r[2] for r in rows),
            "per_seed": [[s, int(a), int(b)] for s, a, b in rows],
            "source": f"tests/golden/pipeline_reference.json ({key}/*: the reference's bench.solve_scene, "
                      "variant-B fix, float64)"}


def _oracle_solve(scene, over, stage1_only, seed, threads, max_restarts=None):
    from oracle import pipeline as op

    return op.solve_scene(scene, seed=seed, threads=threads, solver_overrides=over, no_trajopt=stage1_only,
                          max_restarts=max_restarts)


_REF = {}


def _reference_impl():
    """The reference's own CPU implementation when it is staged in baseline/_ref
    (scripts/stage_reference.py: the offline pip install of /root/reference/pkg + the
    variant-B fix), driven through its stock ``seqplace.bench.solve_scene``; otherwise the
    float64 oracle port (oracle/pipeline.py)."""
    if "kind" not in _REF:
        path = os.path.join(ROOT, "baseline", "_ref")
        _REF["kind"] = "port"
        if os.path.isdir(os.path.join(path, "seqplace")) and os.environ.get("SPASM_REFERENCE_ARM", "ref") != "port":
            sys.path.insert(0, path)
            import seqplace.bench as rb

            _REF.update(kind="reference", bench=rb, scenes={},
                        orig={k: getattr(rb, k) for k in ("solve", "solve_al")})
    return _REF["kind"]


class _RefRun:
    """One stock seqplace.bench.solve_scene call with the work it did recorded: the names the
    reference's bench binds at import (bench.py:28-51) are wrapped so the stage-1 config /
    report and the AL batch / outer count are seen on the way through (nothing is changed)."""

    def __init__(self, success, time_ms, stage1_iterations, stage2_iterations):
        self.success, self.time_ms = success, time_ms
        self.stage1_iterations, self.stage2_iterations = stage1_iterations, stage2_iterations


def _reference_solve(scene_name, over, stage1_only, seed, threads, max_restarts=None):
    rb, rec = _REF["bench"], {}
    if scene_name not in _REF["scenes"]:
        from oracle.refscene import ref_scene

        _REF["scenes"][scene_name] = ref_scene(scene_name)
    scene = _REF["scenes"][scene_name]

    def w_solve(model, config, **kw):
        res = _REF["orig"]["solve"](model, config, **kw)
        rec["cfg"], rec["res"] = config, res
        return res

    def w_al(values, *a, **kw):
        rec["P"] = len(values)
        try:
            al = _REF["orig"]["solve_al"](values, *a, **kw)
        except rb.TrajOptFailure as exc:
            rec["outers"], rec["inner"] = len(exc.report.outers), a[2].inner_steps
            raise
        rec["outers"], rec["inner"] = len(al.report.outers), a[2].inner_steps
        return al

    rb.solve, rb.solve_al = w_solve, w_al
    try:
        so = dict(over)
        if max_restarts:
            so["max_restarts"] = max_restarts
        sol = rb.solve_scene(scene, seed=seed, threads=threads, solver_overrides=so, no_trajopt=stage1_only)
    finally:
        rb.solve, rb.solve_al = _REF["orig"]["solve"], _REF["orig"]["solve_al"]
    cfg, res = rec["cfg"], rec["res"]
    runs = res.report.restarts + 1 if res.success else cfg.max_restarts
    it2 = rec.get("outers", 0) * rec.get("P", 0) * rec.get("inner", 0)
    return _RefRun(bool(sol.success), sol.time_ms, runs * cfg.m * (cfg.k_lin + cfg.k_quad), it2)


def _cpu_solve(scene, scene_name, over, stage1_only, seed, threads, max_restarts=None):
    if _reference_impl() == "reference":
        return _reference_solve(scene_name, over, stage1_only, seed, threads, max_restarts)
    return _oracle_solve(scene, over, stage1_only, seed, threads, max_restarts)


def _host_info():
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "")
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "numpy": np.__version__}


def _arm_label(threads):
    if _reference_impl() == "reference":
        return (f"stock seqplace.bench.solve_scene from baseline/_ref (reference pkg, variant-B fix), numpy "
                f"float64, threads={threads}")
    return f"oracle/pipeline.py (float64 numpy port of the reference), threads={threads}"


def cpu_baseline(args, workload=None, budget_s=20.0):
    """The reference's CPU implementation (baseline/_ref when staged, else the oracle port)
    timed on this host's cores on a bounded sample of the same workload, with all host
    threads and with threads=1."""
    from paper_2510_07674_b200.problems import load_scene

    scene_name, over, stage1_only, desc = WORKLOADS[workload or args.workload]
    scene = load_scene(scene_name)
    threads = os.cpu_count() or 1
    # large stage-1-only workloads: one restart per sample solve; pipelines: whole solves
    mr = 1 if stage1_only else None

    def sample(th, budget, max_solves):
        its, t_total, times = 0, 0.0, []
        t_start = time.perf_counter()
        while len(times) < max_solves and (not times or time.perf_counter() - t_start < budget):
            r = _cpu_solve(scene, scene_name, over, stage1_only, len(times), th, max_restarts=mr)
            t_total += r.time_ms * 1e-3
            times.append(r.time_ms)
            its += r.stage1_iterations + r.stage2_iterations
        return its / t_total, times

    value, times = sample(threads, budget_s, 3)
    one = None
    if threads > 1 and statistics.median(times) < 8000:  # threads=1 figure, one bounded solve
        v1, t1 = sample(1, 0.0, 1)
        one = {"value": v1, "p50_solve_ms": statistics.median(t1), "cores": 1}
    return {"value": value, "unit": "particle-iterations/s", "cores": threads, "kind": _reference_impl(),
            "p50_solve_ms": statistics.median(times), "threads_1": one, "host": _host_info(),
            "sample": f"{len(times)} {'single-restart stage-1' if stage1_only else 'full two-stage'} solve(s) of "
                      f"{scene_name} ({_arm_label(threads)})"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2510_07674_b200.problems import load_scene

    from paper_2510_07674_b200.bench_api import _solver_config as _sc

    scene_name, over, stage1_only, desc = WORKLOADS[args.workload]
    scene = load_scene(scene_name)
    if world > 1:  # the b200 arm's weak-scaled workload: world x the per-GPU (n, m) per restart
        b0 = _sc(scene, 0, over, False)
        over = {**over, "n": b0.n * world, "m": b0.m * world}
    threads = os.cpu_count() or 1
    mr = 1 if stage1_only else None
    kind = _reference_impl()
    for i in range(args.warmup):  # warm numpy / thread pools on cheap stage-1 samples
        _cpu_solve(scene, scene_name, over, True, 100000 + i, threads, max_restarts=1)
    times, its, succ = [], 0, 0
    for i in range(args.steps):
        r = _cpu_solve(scene, scene_name, over, stage1_only, i, threads, max_restarts=mr)
        times.append(r.time_ms)
        its += r.stage1_iterations + r.stage2_iterations
        succ += int(r.success)
    value = its / (sum(times) * 1e-3)
    from paper_2510_07674_b200.bench_api import _solver_config, effective_max_restarts

    c = _solver_config(scene, 0, over, False)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "particle-iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sum(times) / args.steps,
        "p50_solve_ms": statistics.median(times), "success_rate": succ / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "scene": scene_name, "n": c.n, "m": c.m, "k_lin": c.k_lin, "k_quad": c.k_quad,
                   "max_restarts": effective_max_restarts(c), "p_return": c.p_return, "stage2": not stage1_only},
        "cpu_baseline": {"value": value, "unit": "particle-iterations/s", "cores": threads, "kind": kind,
                         "host": _host_info(),
                         "sample": f"{args.steps} {'stage-1 (bounded to 1 restart)' if stage1_only else 'full two-stage'} "
                                   f"solves of {scene_name} ({_arm_label(threads)})"},
        "e2e": {"value": value, "unit": "particle-iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--precision", default="fp32", choices=["fp32", "fp64"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-sub", action="store_true", help="skip the C5 / C3 sub-records of the default C2 line")
    ap.add_argument("--sub-steps", type=int, default=10, help="timed steps of each sub-record")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return
    line = run_b200(args)
    if line is None:  # ranks != 0
        return
    if args.gpus == 1 and dist_env()[1] == 1 and args.workload == "c2" and not args.no_sub:
        # same-process sub-records of the other headline configs (C5: the particle-iterations/s
        # clause at 1M particles and k_schedule_tile's FP32 roofline; C3: 64k tetris5; C1 with
        # the builtin arm and with the Franka-like chain), each with its own clocks / roofline,
        # so the driver's default run carries them
        line["sub_records"] = {}
        for w in ("c5", "c3", "c1", "c1f"):
            sub = run_b200(args, workload=w, sub=True)
            keep = ("value", "unit", "ms_per_step", "p50_solve_ms", "p50_solve_ms_successes", "p50_step_ms",
                    "success_rate", "steps", "warmup", "config", "e2e", "roofline", "clocks", "gpu_launches",
                    "breakdown", "reference_outcomes")
            line["sub_records"][w] = {k: sub[k] for k in keep if k in sub}
    if args.gpus == 1 and dist_env()[1] == 1 and args.workload == "c3p" and not args.no_sub:
        # C3's 4- and 6-object variants (stage 1 at 64k) beside the 5-object full pipeline
        line["sub_records"] = {}
        for w in ("c3_4", "c3_6"):
            sub = run_b200(args, workload=w, sub=True)
            keep = ("value", "unit", "ms_per_step", "p50_solve_ms", "p50_solve_ms_successes", "p50_step_ms", "success_rate", "steps", "warmup",
                    "config", "e2e", "roofline", "clocks", "gpu_launches", "breakdown")
            line["sub_records"][w] = {k: sub[k] for k in keep if k in sub}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
