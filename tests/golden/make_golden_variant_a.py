"""Golden fixtures for solve_al's "variant A" placement mode, from the REFERENCE itself.

Variant A is the solve_al docstring's intent (reference trajopt.py:958-965): the placement
constraint is evaluated in QUADRATIC mode inside solve_al while the collision terms stay
LINEAR. As shipped the reference cannot run it (trajopt._evaluate lacks `place_mode`,
SURVEY.md 0.4); this script copies the reference to a temp dir and applies

    def _evaluate(..., want_grad)  ->  def _evaluate(..., want_grad, place_mode=None)
    + pmode = mode if place_mode is None else place_mode; pquad = pmode == QUADRATIC

then freezes tests/golden/stage2_variant_a.npz:
  * _evaluate(values, LINEAR, place_mode=QUADRATIC) value / constraints / gradient on the
    stage2.npz random trajectories (tower4, tetris5);
  * solve_al on the tower4 pipeline init (stage2.npz pipe_tower4_init) and on a tower3c
    pipeline init, whose variant-A outcome is a TrajOptFailure in the reference (SURVEY.md
    0.5): best violation and per-outer constraints / violations.

    python tests/golden/make_golden_variant_a.py
"""
from __future__ import annotations

import os
import shutil
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src/seqplace"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))


def patched_reference_a():
    root = tempfile.mkdtemp(prefix="spasm_refA_")
    dst = os.path.join(root, "seqplace")
    shutil.copytree(REF, dst)
    p = os.path.join(dst, "trajopt.py")
    src = open(p).read()
    old_sig = "def _evaluate(values, geo: _Geometry, config: TrajOptConfig, mode, lam, mu, want_grad):"
    assert src.count(old_sig) == 1
    src = src.replace(old_sig, old_sig[:-2] + ", place_mode=None):")
    anchor = "    quad = mode == QUADRATIC\n"
    assert src.count(anchor) == 1
    src = src.replace(anchor, anchor + "    pmode = mode if place_mode is None else place_mode\n"
                                       "    pquad = pmode == QUADRATIC\n")
    open(p, "w").write(src)
    sys.path.insert(0, root)
    return root


def main():
    root = patched_reference_a()
    from seqplace import trajopt
    from seqplace.geometry import LINEAR, QUADRATIC
    from seqplace.particle_opt import OptimizerConfig, solve
    from seqplace.problems import as_cost_model, load_scene

    from oracle.refscene import ref_scene

    g2 = dict(np.load(os.path.join(HERE, "stage2.npz")))
    out = {}
    for name in ("tower4", "tetris5"):
        sc = load_scene(name)
        cfg = trajopt.TrajOptConfig(**sc.trajopt_overrides)
        geo = trajopt._build_geometry(sc.problem, sc.chain, sc.grasp, sc.obstacle_centers, sc.obstacle_radii)
        vals, lam, mu = g2[f"al_{name}_values"], g2[f"al_{name}_lam"], g2[f"al_{name}_mu"]
        obj, cons, lag, grad = trajopt._evaluate(vals, geo, cfg, LINEAR, lam, mu, True, place_mode=QUADRATIC)
        out[f"eval_{name}_obj"], out[f"eval_{name}_cons"] = obj, cons
        out[f"eval_{name}_lag"], out[f"eval_{name}_grad"] = lag, grad
    inits = {"tower4": g2["pipe_tower4_init"]}
    sc = ref_scene("tower3c")
    res = solve(as_cost_model(sc.problem), OptimizerConfig(**{**sc.solver_overrides, "seed": 0}))
    lift = trajopt.lift_placements(sc.problem, res.particles, sc.chain, sc.grasp, seed=0,
                                   static_centers=sc.obstacle_centers, static_radii=sc.obstacle_radii)
    cfg = trajopt.TrajOptConfig(**sc.trajopt_overrides)
    strm = np.random.default_rng(np.random.SeedSequence(entropy=0, spawn_key=(1 << 20,)))
    inits["tower3c"] = trajopt.init_trajectories(lift.endpoints, sc.chain, cfg, strm)
    for name, init in inits.items():
        sc = load_scene(name) if name == "tower4" else ref_scene(name)
        cfg = trajopt.TrajOptConfig(**sc.trajopt_overrides)
        out[f"solve_{name}_init"] = init
        try:
            al = trajopt.solve_al(init, sc.problem, sc.chain, cfg, grasp=sc.grasp,
                                  static_centers=sc.obstacle_centers, static_radii=sc.obstacle_radii)
            outers, out[f"solve_{name}_failure"] = al.report.outers, np.array(np.nan)
            out[f"solve_{name}_objective"] = np.array(al.objective)
            out[f"solve_{name}_index"] = np.array(al.particle_index)
        except trajopt.TrajOptFailure as exc:
            outers, out[f"solve_{name}_failure"] = exc.report.outers, np.array(exc.best_violation)
        out[f"solve_{name}_outers"] = np.array(len(outers))
        out[f"solve_{name}_cons"] = np.stack([r.constraints for r in outers])
        out[f"solve_{name}_viol"] = np.stack([r.violation for r in outers])
        print(name, "variant A:", "failure" if np.isfinite(out[f"solve_{name}_failure"]) else "success",
              float(out[f"solve_{name}_failure"]), len(outers), "outers")
    path = os.path.join(HERE, "stage2_variant_a.npz")
    np.savez_compressed(path, **out)
    print("wrote", path)
    shutil.rmtree(root, ignore_errors=True)


if __name__ == "__main__":
    main()
