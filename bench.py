"""Benchmark: SPaSM two-stage particle optimizer on B200 (BASELINE.json metric).

One "step" = one full stage-1 solve (sample -> stable top-M -> fused K_lin+K_quad descent
-> satisfying extraction + re-check, restarts included) of the workload's scene on
synthetic, on-device-sampled particles, through the reference-facing API
``particle_opt.solve`` (host config in, host placements out).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c5] [--impl b200|reference]

Multi-GPU (torchrun, one rank per GPU): each rank solves its own seeds (replicas, weak
scaling); rank 0 prints one JSON line with whole-job throughput over max-over-ranks time.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "solve time ms (p50) at 100% success; particle-iterations/sec at 1/2/4/8 B200"

WORKLOADS = {
    # name: (scene, overrides, description)
    "c2": ("tower3c", {"n": 16384, "m": 2048},
           "C2 3-block stacking with cuboid obstacles (sphere-grid cuboids), 16k particles, stage 1"),
    "c3": ("tetris5", {"n": 65536, "m": 8192},
           "C3 Tetris packing, 5 objects, 64k particles, stage 1"),
    "c5": ("tetris8", {"n": 1 << 20, "m": 1 << 17},
           "C5 8-object skeleton, 1M particles (M = N/8), stage 1"),
}


def flops_per_particle_iteration(model, mode="linear"):
    """Algorithmic FP32 FLOPs of one fused cost-gradient-update step."""
    from paper_2510_07674_b200.problems import TetrisCostModel

    p = model.problem
    D = model.dimension
    if isinstance(model, TetrisCostModel):
        n = p.n_blocks
        S = sum(len(b.sphere_set) for b in p.blocks)
        counts = [len(b.sphere_set) for b in p.blocks]
        E = sum(counts[i] * counts[j] for i in range(n) for j in range(i + 1, n)) + S * len(p.wall_radii)
        per_pair = 22 if mode == "linear" else 24
        f = per_pair * E + 3 * S + 4 * n + 2 * D
        if model.free_yaw:
            f += 10 * E + 8 * S
        return f
    B = p.n_blocks
    O = len(p.obstacle_radii)
    pairs = B * (B - 1) // 2
    return 22 * (pairs + B * O) + 30 * (B - 1) + 4 * B + 2 * D


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i - 3] for r in self.rows if len(r) >= 7 for i in range(3, 7)
                          if r[i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def build_workload(name, precision):
    from paper_2510_07674_b200 import particle_opt as po
    from paper_2510_07674_b200.bench_api import effective_max_restarts
    from paper_2510_07674_b200.problems import as_cost_model, load_scene

    scene_name, over, desc = WORKLOADS[name]
    scene = load_scene(scene_name)
    model = as_cost_model(scene.problem, precision=precision)
    base = {**scene.solver_overrides, **over}
    cfg = po.OptimizerConfig(**base)
    cfg.max_restarts = effective_max_restarts(cfg)
    return scene, model, cfg, desc


def measure_schedule_kernel(model, cfg, repeats=10):
    """Average device time of the fused descent kernel (dominant kernel) on one M-row batch,
    timed with CUDA events on the launching stream."""
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
    f_lin = flops_per_particle_iteration(model, "linear")
    f_quad = flops_per_particle_iteration(model, "quadratic")
    flops = cfg.m * (cfg.k_lin * f_lin + cfg.k_quad * f_quad)
    return ms, flops


def run_b200(args):
    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    else:
        torch.cuda.set_device(0)
    from paper_2510_07674_b200 import particle_opt as po

    scene, model, cfg, desc = build_workload(args.workload, args.precision)
    seed0 = 1000 * rank
    # warm-up (also builds workspaces / loads modules)
    for i in range(args.warmup):
        cfg.seed = seed0 + 100000 + i
        po.solve(model, cfg)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    dev_ms, wall_ms, pits, evals, succ, launches = [], [], 0, 0, 0, 0
    with ClockSampler(local) as clocks:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)  # L2 flush between timed iterations (outside the events)
            cfg.seed = seed0 + i
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e0.record(stream)
            res = po.solve(model, cfg)  # host config in, host placements out (e2e path)
            e1.record(stream)
            e1.synchronize()
            wall_ms.append((time.perf_counter() - t0) * 1e3)
            dev_ms.append(e0.elapsed_time(e1))
            restarts_run = min(res.report.restarts + 1, cfg.max_restarts) if res.success else cfg.max_restarts
            pits += restarts_run * cfg.m * (cfg.k_lin + cfg.k_quad)
            evals += restarts_run * cfg.n
            succ += int(res.success)
            launches += res.report.launches
    total_dev = sum(dev_ms)
    total_wall = sum(wall_ms)
    if world > 1:
        t = torch.tensor([total_dev, total_wall], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_dev, total_wall = t.tolist()
        c = torch.tensor([pits, succ, launches], device="cuda", dtype=torch.float64)
        dist.all_reduce(c)
        pits, succ, launches = [int(v) for v in c.tolist()]
    kern_ms, kern_flops = measure_schedule_kernel(model, cfg)
    clk = clocks.summary()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    sm_mhz = clk["sm_mhz"] or 1965.0
    peak = 2 * 128 * 148 * sm_mhz * 1e6 / 1e12  # FP32 CUDA-core TFLOP/s at the measured SM clock
    achieved = kern_flops / (kern_ms * 1e-3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(f"{args.workload}_{args.precision}")
    cpu = cpu_baseline(args) if (rank == 0 and world == 1 and not args.no_cpu) else None
    line = {
        "metric": METRIC,
        "value": pits / (total_dev * 1e-3),
        "unit": "particle-iterations/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_dev / args.steps,
        "p50_solve_ms": statistics.median(dev_ms),
        "success_rate": succ / (args.steps * world),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32" if args.precision == "fp32" else "f64",
        "data": "synthetic (scene tables; particles sampled on device from numpy-identical PCG64 restart streams)",
        "config": {"workload": desc, "scene": WORKLOADS[args.workload][0], "n": cfg.n, "m": cfg.m,
                   "k_lin": cfg.k_lin, "k_quad": cfg.k_quad, "max_restarts": cfg.max_restarts,
                   "l2": "flushed (256 MB write) between timed solves", "parallelism": f"replicas x{world}"},
        "e2e": {"value": pits / (total_wall * 1e-3), "unit": "particle-iterations/s",
                "p50_solve_ms": statistics.median(wall_ms),
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": int(64 + cfg.p_return * (model.dimension + 3) * 8)},
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic, "kernel": "k_schedule (fused descent)",
                     "kernel_ms": kern_ms, "flops_per_launch": kern_flops,
                     "peak_note": "FP32 CUDA-core 2*128*148*f_SM at the median SM clock sampled under load "
                                  "(no FP32 figure in MEASURED_PEAKS.json)"},
        "cpu_baseline": cpu,
        "clocks": clk,
        "gpu_launches": launches,
        "initial_evals_per_s": evals / (total_dev * 1e-3),
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(args, budget_s=15.0):
    """The oracle port timed on this host's cores on a bounded sample of the workload."""
    from oracle import stage1 as orc
    from paper_2510_07674_b200.problems import load_scene

    scene_name, over, desc = WORKLOADS[args.workload]
    scene = load_scene(scene_name)
    o = orc.oracle_model(scene.problem)
    base = {**scene.solver_overrides, **over}
    threads = os.cpu_count() or 1
    cfg = orc.OracleConfig(**base)
    pits, t_total, solves = 0, 0.0, 0
    t_start = time.perf_counter()
    # bounded sample: one restart per solve (max_restarts=1), as many solves as fit the budget
    while time.perf_counter() - t_start < budget_s and solves < 3:
        cfg.seed = solves
        cfg.max_restarts = 1
        t0 = time.perf_counter()
        orc.solve(o, cfg, threads=threads)
        t_total += time.perf_counter() - t0
        pits += cfg.m * (cfg.k_lin + cfg.k_quad)
        solves += 1
    return {"value": pits / t_total, "unit": "particle-iterations/s", "cores": threads, "kind": "port",
            "sample": f"{solves} single-restart solve(s) of {scene_name} at n={cfg.n}, m={cfg.m} "
                      f"(oracle/stage1.py, numpy float64, {threads} threads)"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import stage1 as orc
    from paper_2510_07674_b200.problems import load_scene

    scene_name, over, desc = WORKLOADS[args.workload]
    scene = load_scene(scene_name)
    o = orc.oracle_model(scene.problem)
    threads = os.cpu_count() or 1
    cfg = orc.OracleConfig(**{**scene.solver_overrides, **over})
    cfg.max_restarts = 1  # bounded sample per step: one restart
    for i in range(args.warmup):
        cfg.seed = 100000 + i
        if i == 0:
            orc.solve(o, cfg, threads=threads)
    times, pits = [], 0
    for i in range(args.steps):
        cfg.seed = i
        t0 = time.perf_counter()
        orc.solve(o, cfg, threads=threads)
        times.append((time.perf_counter() - t0) * 1e3)
        pits += cfg.m * (cfg.k_lin + cfg.k_quad)
    value = pits / (sum(times) * 1e-3)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "particle-iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sum(times) / args.steps,
        "p50_solve_ms": statistics.median(times), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": {"workload": desc, "scene": scene_name, "n": cfg.n,
                                                        "m": cfg.m, "max_restarts": 1},
        "cpu_baseline": {"value": value, "unit": "particle-iterations/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} single-restart solves of {scene_name} (oracle/stage1.py)"},
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
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
