import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
from conftest import golden
from oracle import stage2 as o2
from paper_2510_07674_b200 import trajopt as tj
from paper_2510_07674_b200.problems import load_scene
G = golden("stage2.npz")
sc = load_scene("tower4")
cfg = tj.TrajOptConfig(**sc.trajopt_overrides)
ends = G["pipe_tower4_endpoints"]
got = tj.init_trajectories(ends, sc.chain, cfg, tj.trajectory_stream(0))
ref = G["pipe_tower4_init"]
print("init type", type(got), got.shape, ref.shape, "maxdiff", np.abs(got - ref).max(), "neq", np.sum(got != ref))
idx = np.argwhere(got != ref)[:5]
for i in idx:
    print(tuple(i), repr(got[tuple(i)]), repr(ref[tuple(i)]))

def run(o, n):
    c = tj.TrajOptConfig(**{**sc.trajopt_overrides, "outer_iters": o, "inner_steps": n})
    try:
        res = tj.solve_al(G["pipe_tower4_init"], sc.problem, sc.chain, c, grasp=sc.grasp,
                          static_centers=sc.obstacle_centers, static_radii=sc.obstacle_radii)
        return "ok", res.report.outers
    except tj.TrajOptFailure as exc:
        return "fail", exc.report.outers

for trial in range(3):
    st, outers = run(3, 5)
    print("trial", trial, st, len(outers))
    for r in outers:
        plain = r.multipliers + r.mu[:, None] * r.constraints
        for p, i in np.argwhere(plain != r.updated_multipliers):
            print("  outer", r.index, p, i, repr(r.multipliers[p, i]), repr(r.mu[p]), repr(r.constraints[p, i]),
                  "got", repr(r.updated_multipliers[p, i]), "plain", repr(plain[p, i]))
    print("  cons", [r.constraints.tolist() for r in outers][:1])
    st, outers = run(15, 100)
