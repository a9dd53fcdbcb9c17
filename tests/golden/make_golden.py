"""Generate the golden fixtures that pin the oracle (and, through it, the CUDA path)
to the REFERENCE implementation itself.

Run in the build container, where the reference is importable read-only:

    python tests/golden/make_golden.py

It imports /root/reference/pkg/src/seqplace (never modified, never copied) and freezes
its outputs into tests/golden/stage1_<case>.npz. The GPU box never needs the reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {
    # case: (scene name, yaw override or None)
    "domino2": ("domino2", None),
    "tetris5": ("tetris5", None),
    "tetris8": ("tetris8", None),
    "tower4": ("tower4", None),
    "tetris5_free": ("tetris5", "quantized-free"),
    "tower4_free": ("tower4", "quantized-free"),
}


def build_problem(scene, yaw):
    from seqplace.problems import TetrisProblem, TowerProblem

    p = scene.problem
    if yaw is None:
        return p
    if isinstance(p, TetrisProblem):
        return TetrisProblem(blocks=p.blocks, box=p.box, z_star=p.z_star, yaw_mode=yaw, weights=p.weights,
                             initial_poses=p.initial_poses, tight_packing=p.tight_packing)
    return TowerProblem(n_blocks=p.n_blocks, side=p.side, box=p.box, obstacle_centers=p.obstacle_centers,
                        obstacle_radii=p.obstacle_radii, yaw_mode=yaw, weights=p.weights,
                        footprint_halfwidth=p.footprint_halfwidth, table_height=p.table_height,
                        initial_poses=p.initial_poses)


def main():
    sys.path.insert(0, REF)
    from seqplace import particle_opt as po
    from seqplace.problems import as_cost_model, load_scene

    for case, (name, yaw) in CASES.items():
        scene = load_scene(name)
        problem = build_problem(scene, yaw)
        model = as_cost_model(problem)
        rng = np.random.default_rng(20251007)
        D = model.dimension
        vals = rng.uniform(model.lower, model.upper, size=(40, D))
        # edge rows: both clamp corners, and (placement scenes) a wide spread slightly outside
        extra = [model.lower.copy(), model.upper.copy(), 0.5 * (model.lower + model.upper)]
        vals = np.concatenate([vals, np.array(extra)])
        out = {"values": vals, "lower": model.lower, "upper": model.upper}
        for mode in ("linear", "quadratic"):
            out[f"cost_{mode}"] = model.evaluate(vals, mode)
            out[f"grad_{mode}"] = model.gradient(vals, mode)
        # restart stream draws
        batch = po.sample_uniform(model, 24, po.restart_stream(7, 3))
        out["draw_seed7_restart3"] = batch.values
        # schedule replay from the first 16 rows with the scene's solver settings
        cfg = po.OptimizerConfig(**{**scene.solver_overrides, "n": 64, "m": 16, "seed": 0})
        x = vals[:16].copy()
        x, fl, steps = po.run_descent_schedule(model, x, cfg)
        out["sched_in"] = vals[:16]
        out["sched_out"] = x
        out["sched_flagged"] = fl
        out["sched_cfg"] = np.array([cfg.k_lin, cfg.k_quad, cfg.eta_init, cfg.alpha, cfg.epsilon])
        # full solves (small batches so the CPU reference finishes in seconds)
        for seed in (0, 1):
            scfg = po.OptimizerConfig(**{**scene.solver_overrides, "n": 1024, "m": 128, "seed": seed,
                                         "max_restarts": 3})
            res = po.solve(model, scfg)
            out[f"solve{seed}_cfg"] = np.array([scfg.n, scfg.m, scfg.k_lin, scfg.k_quad, scfg.eta_init, scfg.alpha,
                                               scfg.epsilon, scfg.p_return, scfg.max_restarts, seed], dtype=float)
            out[f"solve{seed}_success"] = np.array(res.success)
            out[f"solve{seed}_indices"] = res.indices
            out[f"solve{seed}_costs"] = res.costs
            out[f"solve{seed}_particles"] = res.particles
            out[f"solve{seed}_report"] = np.array([res.report.restarts, res.report.steps, res.report.n_satisfying,
                                                   res.report.flagged])
        path = os.path.join(HERE, f"stage1_{case}.npz")
        np.savez_compressed(path, **out)
        print("wrote", path, {k: np.shape(v) for k, v in out.items() if k.startswith("solve0")})

    # engine known-answer fixtures (particle_opt.py:195-211)
    sel = {}
    rng = np.random.default_rng(5)
    costs = np.floor(rng.uniform(0, 6, size=300)).astype(float)  # heavy ties
    from seqplace.particle_opt import ParticleBatch

    sel["tie_costs"] = costs
    sel["tie_order"] = po.select_topk(ParticleBatch(values=np.zeros((300, 1)), costs=costs), 300)
    cont = rng.uniform(size=5000)
    sel["cont_costs"] = cont
    sel["cont_top"] = po.select_topk(ParticleBatch(values=np.zeros((5000, 1)), costs=cont), 700)
    np.savez_compressed(os.path.join(HERE, "stage1_engine.npz"), **sel)
    print("wrote engine fixtures")


if __name__ == "__main__":
    main()
