"""Sharded stage 1 on the GPU: the device halves spasm_shard_select /
spasm_shard_descend, driven for G virtual ranks in one process and for 2 real processes
sharing cuda:0 over a gloo group, must reproduce the single-GPU solve exactly (same
kernels, same per-particle arithmetic): success, restarts, indices bit-identical,
particles and costs bit-identical; fp64 also matches the CPU oracle's indices."""
from __future__ import annotations

import os
import tempfile

import numpy as np
import pytest
import torch

from oracle import stage1 as orc
from paper_2510_07674_b200 import particle_opt as po
from paper_2510_07674_b200.problems import as_cost_model, load_scene
from paper_2510_07674_b200.sharded import NativeShardOps, merge_candidates, shard_range, solve_sharded

pytestmark = pytest.mark.gpu


def _virtual_ranks(model, cfg, world, warm=None):
    """solve_sharded's restart loop with `world` ranks simulated in one process."""
    ops = []
    for r in range(world):
        lo, hi = shard_range(cfg.n, world, r)
        plo, phi = shard_range(cfg.m, world, r)
        ops.append((NativeShardOps(model, cfg, po._SAMPLERS["pcg64"], warm, hi - lo, phi - plo), lo, hi, plo, phi))
    for restart in range(cfg.max_restarts):
        elite_all = torch.stack([o.select(restart, lo, hi - lo) for o, lo, hi, _, _ in ops])
        blocks = torch.stack([o.descend(restart, elite_all, plo, phi) for o, _, _, plo, phi in ops]).cpu().numpy()
        n_sat, flagged, chosen = merge_candidates(blocks, model.dimension, cfg.p_return, cfg.epsilon)
        if n_sat:
            return restart, chosen
    return cfg.max_restarts, None


def _virtual_ranks_select(model, cfg, world, warm=None):
    """The same restart loop over the exact top-m select protocol (sharded.topm_exchange),
    its collectives emulated in lock step: sums of the 256-bin digit counts, gathers."""
    from paper_2510_07674_b200.sharded import allot_top_m

    ops = []
    for r in range(world):
        lo, hi = shard_range(cfg.n, world, r)
        plo, phi = shard_range(cfg.m, world, r)
        ops.append((NativeShardOps(model, cfg, po._SAMPLERS["pcg64"], warm, hi - lo, phi - plo), lo, hi, plo, phi))
    for restart in range(cfg.max_restarts):
        for o, lo, hi, _, _ in ops:
            o.select(restart, lo, hi - lo, elite=False)
        sts = [o.topm_init() for o, *_ in ops]
        for _ in range(ops[0][0].key_bits // 8):
            hsum = torch.stack([o.topm_hist(st) for (o, *_), st in zip(ops, sts)]).sum(0)
            for (o, *_), st in zip(ops, sts):
                o.topm_pick(st, hsum)
        take = allot_top_m(torch.stack([o.topm_local(st) for (o, *_), st in zip(ops, sts)]).cpu().numpy())
        assert int(take.sum()) == cfg.m
        cap = max(1, int(take.max()))
        runs = torch.stack([o.topm_contrib(int(take[r]), cap) for r, (o, *_) in enumerate(ops)])
        blocks = torch.stack([o.descend(restart, runs, plo, phi) for o, _, _, plo, phi in ops]).cpu().numpy()
        n_sat, flagged, chosen = merge_candidates(blocks, model.dimension, cfg.p_return, cfg.epsilon)
        if n_sat:
            return restart, chosen
    return cfg.max_restarts, None


CASES = [("tetris5", {"n": 4096, "m": 512, "seed": 3, "max_restarts": 4}),
         ("tower4", {"n": 3000, "m": 700, "seed": 2, "max_restarts": 3}),
         ("tetris8", {"n": 8192, "m": 1024, "seed": 0, "max_restarts": 2}),
         ("tetris5", {"n": 37, "m": 33, "seed": 5, "max_restarts": 3})]


@pytest.mark.parametrize("protocol", ["gather", "select"])
@pytest.mark.parametrize("precision", ["fp32", "fp64"])
@pytest.mark.parametrize("ci", range(len(CASES)))
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_virtual_ranks_match_single_gpu_solve(precision, ci, world, protocol):
    name, over = CASES[ci]
    scene = load_scene(name)
    model = as_cost_model(scene.problem, precision=precision)
    cfg = po.OptimizerConfig(**{**scene.solver_overrides, **over})
    ref = po.solve(model, cfg)
    restart, chosen = (_virtual_ranks if protocol == "gather" else _virtual_ranks_select)(model, cfg, world)
    if chosen is None:
        assert not ref.success and ref.report.restarts == cfg.max_restarts
        return
    assert restart == ref.report.restarts
    assert (len(chosen) > 0) == ref.success
    np.testing.assert_array_equal(chosen[:, 1].astype(np.int64), ref.indices)
    np.testing.assert_array_equal(chosen[:, 4:], ref.particles)
    np.testing.assert_array_equal(chosen[:, 2], ref.costs)


def test_fp64_sharded_matches_cpu_oracle():
    scene = load_scene("tetris5")
    kw = {**scene.solver_overrides, "n": 2048, "m": 256, "seed": 0, "max_restarts": 3}
    model = as_cost_model(scene.problem, precision="fp64")
    ref = orc.solve(orc.oracle_model(scene.problem), orc.OracleConfig(**kw))
    restart, chosen = _virtual_ranks(model, po.OptimizerConfig(**kw), 4)
    assert restart == ref.restarts
    np.testing.assert_array_equal(chosen[:, 1].astype(np.int64), ref.indices)
    np.testing.assert_allclose(chosen[:, 4:], ref.particles, rtol=1e-9, atol=1e-12)


def test_virtual_ranks_warm_start():
    scene = load_scene("tower4")
    model = as_cost_model(scene.problem, precision="fp32")
    cfg = po.OptimizerConfig(**{**scene.solver_overrides, "n": 2000, "m": 300, "seed": 9, "max_restarts": 2})
    seed_res = po.solve(model, po.OptimizerConfig(**{**scene.solver_overrides, "n": 4096, "m": 512, "seed": 1}))
    warm = seed_res.particles[:3]
    ref = po.solve(model, cfg, warm_seeds=warm)
    restart, chosen = _virtual_ranks(model, cfg, 3, warm=warm)
    assert restart == ref.report.restarts
    np.testing.assert_array_equal(chosen[:, 1].astype(np.int64), ref.indices)


def test_select_protocol_with_heavy_key_ties():
    """tower4 from warm seeds at exact zero-cost tilings: many rows share the same key, so
    the threshold key K* carries ties split across ranks (allotted to the lowest rows)."""
    scene = load_scene("tower4")
    model = as_cost_model(scene.problem, precision="fp32")
    cfg = po.OptimizerConfig(**{**scene.solver_overrides, "n": 3000, "m": 700, "seed": 9, "max_restarts": 2})
    seed_res = po.solve(model, po.OptimizerConfig(**{**scene.solver_overrides, "n": 4096, "m": 512, "seed": 1}))
    warm = np.repeat(seed_res.particles[:1], 900, axis=0)  # 900 identical rows spanning ranks 0-2
    ref = po.solve(model, cfg, warm_seeds=warm)
    for world in (2, 5, 8):
        restart, chosen = _virtual_ranks_select(model, cfg, world, warm=warm)
        assert restart == ref.report.restarts
        np.testing.assert_array_equal(chosen[:, 1].astype(np.int64), ref.indices)


def _proc(rank, world, init_file, out, protocol):
    import torch.distributed as dist

    dist.init_process_group("gloo", init_method=f"file://{init_file}", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        scene = load_scene("tetris5")
        model = as_cost_model(scene.problem, precision="fp32")
        cfg = po.OptimizerConfig(**{**scene.solver_overrides, "n": 8192, "m": 1024, "seed": 4, "max_restarts": 4})
        res = solve_sharded(model, cfg, protocol=protocol)
        np.savez(out + f".{rank}.npz", success=res.success, restarts=res.report.restarts, indices=res.indices,
                 particles=res.particles, costs=res.costs)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("protocol", ["gather", "select"])
def test_two_processes_gloo_match_single_gpu(protocol):
    import torch.multiprocessing as mp

    scene = load_scene("tetris5")
    model = as_cost_model(scene.problem, precision="fp32")
    cfg = po.OptimizerConfig(**{**scene.solver_overrides, "n": 8192, "m": 1024, "seed": 4, "max_restarts": 4})
    ref = po.solve(model, cfg)
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "res")
        mp.spawn(_proc, args=(2, os.path.join(d, "store"), out, protocol), nprocs=2, join=True)
        for r in range(2):
            got = dict(np.load(out + f".{r}.npz"))
            assert bool(got["success"]) == ref.success
            assert int(got["restarts"]) == ref.report.restarts
            np.testing.assert_array_equal(got["indices"], ref.indices)
            np.testing.assert_array_equal(got["particles"], ref.particles)
