"""solve_al's variant A (placement term QUADRATIC inside the AL solve, collision terms
LINEAR: the reference's solve_al docstring, trajopt.py:958-965,994-1012) against the
variant-A-patched REFERENCE (tests/golden/make_golden_variant_a.py ->
stage2_variant_a.npz). The reference's variant A fails on tower4 and tower3c;
the GPU must fail the same way.

Tolerances (fp64): AL value / constraints rtol 1e-10 and gradient 1e-9 of the gradient
scale (as the variant-B evaluate tests); whole solves: same outcome (TrajOptFailure), same
outer count, outer-0 constraints rtol 1e-5, best violation rtol 1e-5 (1500 chained steps,
as the variant-B solve pins).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden
from paper_2510_07674_b200 import trajopt as tj
from paper_2510_07674_b200.problems import load_scene

pytestmark = pytest.mark.gpu
G = golden("stage2_variant_a.npz")
G2 = golden("stage2.npz")


def _kw(sc):
    return dict(grasp=sc.grasp, static_centers=sc.obstacle_centers, static_radii=sc.obstacle_radii)


@pytest.mark.parametrize("name", ["tower4", "tetris5"])
def test_variant_a_evaluate_matches_reference(name):
    sc = load_scene(name)
    cfg = tj.TrajOptConfig(**sc.trajopt_overrides)
    vals, lam, mu = G2[f"al_{name}_values"], G2[f"al_{name}_lam"], G2[f"al_{name}_mu"]
    obj, cons = tj.trajectory_cost(vals, sc.problem, sc.chain, cfg, mode="linear", place_mode="quadratic",
                                   precision="fp64", **_kw(sc))
    lag, grad = tj.al_value_and_gradient(vals, sc.problem, sc.chain, cfg, lam, mu, mode="linear",
                                         place_mode="quadratic", precision="fp64", **_kw(sc))
    np.testing.assert_allclose(obj, G[f"eval_{name}_obj"], rtol=1e-10)
    np.testing.assert_allclose(lag, G[f"eval_{name}_lag"], rtol=1e-10)
    ref = G[f"eval_{name}_grad"]
    assert np.abs(grad - ref).max() <= 1e-9 * max(np.abs(ref).max(), 1.0)
    # the placement constraint differs from variant B's (linear) value
    _, cons_b = tj.trajectory_cost(vals, sc.problem, sc.chain, cfg, mode="linear", precision="fp64", **_kw(sc))
    assert not np.allclose(cons[:, 0], cons_b[:, 0])


@pytest.mark.parametrize("name", ["tower4", "tower3c"])
def test_variant_a_solve_al_matches_reference(name):
    sc = load_scene(name)
    cfg = tj.TrajOptConfig(**sc.trajopt_overrides)
    init = G[f"solve_{name}_init"]
    assert np.isfinite(G[f"solve_{name}_failure"])  # the reference fails here
    with pytest.raises(tj.TrajOptFailure) as exc:
        tj.solve_al(init, sc.problem, sc.chain, cfg, place_mode="quadratic", precision="fp64", **_kw(sc))
    outers = exc.value.report.outers
    assert len(outers) == int(G[f"solve_{name}_outers"])
    np.testing.assert_allclose(outers[0].constraints, G[f"solve_{name}_cons"][0], rtol=1e-5, atol=1e-9)
    np.testing.assert_allclose(exc.value.best_violation, float(G[f"solve_{name}_failure"]), rtol=1e-5)
