"""Golden fixtures for the stage-2 (trajectory) hot path, from the REFERENCE itself.

As shipped, the reference's trajopt._evaluate lacks its `place_mode` parameter and reads
undefined names. This script copies the reference package to a temp
dir (the original under /root/reference is never modified), applies the test-pinned
"variant B" patch (placement term in the same mode as the collision terms):

    def _evaluate(..., want_grad)  ->  def _evaluate(..., want_grad, place_mode=None)
    + pmode = mode; pquad = pmode == QUADRATIC      (right after `quad = mode == QUADRATIC`)

and freezes its outputs into tests/golden/stage2_*.npz.

    python tests/golden/make_golden_stage2.py
"""
from __future__ import annotations

import os
import shutil
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src/seqplace"
HERE = os.path.dirname(os.path.abspath(__file__))


def patched_reference():
    root = tempfile.mkdtemp(prefix="spasm_refB_")
    dst = os.path.join(root, "seqplace")
    shutil.copytree(REF, dst)
    p = os.path.join(dst, "trajopt.py")
    src = open(p).read()
    old_sig = "def _evaluate(values, geo: _Geometry, config: TrajOptConfig, mode, lam, mu, want_grad):"
    assert src.count(old_sig) == 1
    src = src.replace(old_sig, old_sig[:-2] + ", place_mode=None):")
    anchor = "    quad = mode == QUADRATIC\n"
    assert src.count(anchor) == 1
    src = src.replace(anchor, anchor + "    pmode = mode\n    pquad = pmode == QUADRATIC\n")
    open(p, "w").write(src)
    sys.path.insert(0, root)
    return root


def main():
    root = patched_reference()
    from seqplace import robot, trajopt
    from seqplace.particle_opt import OptimizerConfig, solve
    from seqplace.problems import as_cost_model, load_scene

    rng = np.random.default_rng(77)
    out = {}
    # ---- FK / Jacobians on both bundled arms
    for name, chain in (("spatial7", robot.spatial_arm_7dof(1.3)), ("planar3", robot.planar_arm())):
        Q = rng.uniform(chain.lower, chain.upper, size=(32, chain.dof))
        f = robot.fk_batch(chain, Q)
        out[f"fk_{name}_q"] = Q
        out[f"fk_{name}_ee"] = f.ee_position
        out[f"fk_{name}_rot"] = f.rotation
        out[f"fk_{name}_origins"] = f.joint_origins
        out[f"fk_{name}_axes"] = f.joint_axes
        out[f"fk_{name}_lpos"] = f.link_positions
        out[f"fk_{name}_lrot"] = f.link_rotations
        out[f"fk_{name}_yawjac"] = robot.yaw_jacobian_batch(f)
    # ---- IK + polish on the tower4 / tetris5 staged grasp targets
    for scene_name in ("tower4", "tetris5"):
        sc = load_scene(scene_name)
        targets = [robot.grasp_pose(p, sc.grasp) for p in sc.problem.initial_poses]
        sol, ok, score = robot.ik_solve_batch(sc.chain, targets, seed=3)
        tp = np.array([t.translation for t in targets])
        ty = np.array([t.yaw for t in targets])
        pol, pok = trajopt._polish_tool_down(sc.chain, sol, tp, ty)
        out[f"ik_{scene_name}_tpos"] = tp
        out[f"ik_{scene_name}_tyaw"] = ty
        out[f"ik_{scene_name}_sol"] = sol
        out[f"ik_{scene_name}_ok"] = ok
        out[f"ik_{scene_name}_score"] = score
        out[f"polish_{scene_name}_sol"] = pol
        out[f"polish_{scene_name}_ok"] = pok
    # ---- AL value/gradient and validation on random trajectories (manipulation + motion)
    for scene_name in ("tower4", "tetris5", "corridor3"):
        sc = load_scene(scene_name)
        cfg = trajopt.TrajOptConfig(**sc.trajopt_overrides)
        B = 1 if scene_name == "corridor3" else len(sc.problem.initial_poses)
        T = cfg.waypoints_per_segment
        chain = sc.chain
        vals = rng.uniform(chain.lower, chain.upper, size=(3, B, T, chain.dof))
        lam = rng.uniform(0, 2, size=(3, 3))
        mu = rng.uniform(5, 20, size=3)
        kw = {} if scene_name == "corridor3" else dict(grasp=sc.grasp, static_centers=sc.obstacle_centers,
                                                         static_radii=sc.obstacle_radii)
        out[f"al_{scene_name}_values"] = vals
        out[f"al_{scene_name}_lam"] = lam
        out[f"al_{scene_name}_mu"] = mu
        for mode in ("linear", "quadratic"):
            obj, cons = trajopt.trajectory_cost(vals, sc.problem, chain, cfg, mode=mode, **kw)
            lag, grad = trajopt.al_value_and_gradient(vals, sc.problem, chain, cfg, lam, mu, mode=mode, **kw)
            out[f"al_{scene_name}_{mode}_obj"] = obj
            out[f"al_{scene_name}_{mode}_cons"] = cons
            out[f"al_{scene_name}_{mode}_lag"] = lag
            out[f"al_{scene_name}_{mode}_grad"] = grad
        viol = []
        for p in range(3):
            att = tuple(range(B)) if scene_name != "corridor3" else (None,)
            okv, worst = trajopt.validate(trajopt.Trajectory(vals[p], att), sc.problem, chain,
                                          epsilon=cfg.validation_epsilon, **kw)
            viol.append([okv, worst])
        out[f"val_{scene_name}"] = np.array(viol, dtype=float)
    # ---- full pipeline pieces on tower4: stage-1 -> lift -> init -> AL solve
    sc = load_scene("tower4")
    model = as_cost_model(sc.problem)
    res = solve(model, OptimizerConfig(**{**sc.solver_overrides, "seed": 0}))
    assert res.success
    lift = trajopt.lift_placements(sc.problem, res.particles, sc.chain, sc.grasp, seed=0,
                                   static_centers=sc.obstacle_centers, static_radii=sc.obstacle_radii)
    cfg = trajopt.TrajOptConfig(**sc.trajopt_overrides)
    strm = np.random.default_rng(np.random.SeedSequence(entropy=0, spawn_key=(1 << 20,)))
    vals = trajopt.init_trajectories(lift.endpoints, sc.chain, cfg, strm)
    out["pipe_tower4_placements"] = res.particles
    out["pipe_tower4_endpoints"] = lift.endpoints
    out["pipe_tower4_kept"] = lift.kept
    out["pipe_tower4_init"] = vals
    try:
        al = trajopt.solve_al(vals, sc.problem, sc.chain, cfg, grasp=sc.grasp, static_centers=sc.obstacle_centers,
                              static_radii=sc.obstacle_radii)
        out["pipe_tower4_al_values"] = al.trajectory.segments
        out["pipe_tower4_al_objective"] = np.array(al.objective)
        out["pipe_tower4_al_index"] = np.array(al.particle_index)
        out["pipe_tower4_al_outers"] = np.array(len(al.report.outers))
        r0 = al.report.outers[0]
        out["pipe_tower4_outer0_cons"] = r0.constraints
        out["pipe_tower4_outer0_obj"] = r0.objective
        out["pipe_tower4_outer0_viol"] = r0.violation
    except trajopt.TrajOptFailure as exc:
        out["pipe_tower4_al_failure"] = np.array(exc.best_violation)
    # ---- motion scene AL solve (corridor3)
    sc = load_scene("corridor3")
    cfg = trajopt.TrajOptConfig(**sc.trajopt_overrides)
    ends = trajopt.motion_endpoints(sc.problem)
    strm = np.random.default_rng(np.random.SeedSequence(entropy=0, spawn_key=(1 << 20,)))
    vals = trajopt.init_trajectories(ends, sc.chain, cfg, strm)
    al = trajopt.solve_al(vals, sc.problem, sc.chain, cfg)
    out["motion_corridor3_init"] = vals
    out["motion_corridor3_values"] = al.trajectory.segments
    out["motion_corridor3_objective"] = np.array(al.objective)
    out["motion_corridor3_outers"] = np.array(len(al.report.outers))
    path = os.path.join(HERE, "stage2.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, len(out), "arrays")
    shutil.rmtree(root, ignore_errors=True)


if __name__ == "__main__":
    main()
