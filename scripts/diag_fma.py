import sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np
from conftest import golden
from paper_2510_07674_b200 import trajopt as tj
from paper_2510_07674_b200.problems import load_scene
G = golden("stage2.npz")
sc = load_scene("tower4")
cfg = tj.TrajOptConfig(**{**sc.trajopt_overrides, "outer_iters": 3, "inner_steps": 5})
try:
    res = tj.solve_al(G["pipe_tower4_init"], sc.problem, sc.chain, cfg, grasp=sc.grasp,
                      static_centers=sc.obstacle_centers, static_radii=sc.obstacle_radii)
    outers = res.report.outers
except tj.TrajOptFailure as exc:
    outers = exc.report.outers
for r in outers:
    plain = r.multipliers + r.mu[:, None] * r.constraints
    ld = (r.multipliers.astype(np.longdouble) + r.mu[:, None].astype(np.longdouble) * r.constraints.astype(np.longdouble)).astype(np.float64)
    bad = np.argwhere(plain != r.updated_multipliers)
    for p, i in bad:
        print("outer", r.index, p, i, repr(r.multipliers[p, i]), repr(r.mu[p]), repr(r.constraints[p, i]),
              "got", repr(r.updated_multipliers[p, i]), "plain", repr(plain[p, i]), "fma~", repr(ld[p, i]))
