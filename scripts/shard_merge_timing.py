"""Exchange + merge cost of one sharded C5 restart with G virtual ranks on one GPU: the
all-gather protocol (every rank ranks G x m records against G-1 runs) against the exact
top-m select protocol (m records in total), both bit-identical. Times the descend launch
(merge + re-draw + schedule + candidates) per rank with CUDA events, and the merge kernel
alone from the difference to a world-1 descend of the same slice size.
Usage: python scripts/shard_merge_timing.py [G] [n_per_rank]"""
import statistics
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_sharded_gpu import _virtual_ranks, _virtual_ranks_select  # noqa: E402

from paper_2510_07674_b200 import particle_opt as po  # noqa: E402
from paper_2510_07674_b200.problems import as_cost_model, load_scene  # noqa: E402
from paper_2510_07674_b200.sharded import NativeShardOps, allot_top_m, shard_range  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 8
n_rank = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
scene = load_scene("tetris8")
model = as_cost_model(scene.problem, precision="fp32")
cfg = po.OptimizerConfig(**{**scene.solver_overrides, "n": G * n_rank, "m": G * n_rank // 8, "seed": 0,
                            "max_restarts": 1})
ops = []
for r in range(G):
    lo, hi = shard_range(cfg.n, G, r)
    plo, phi = shard_range(cfg.m, G, r)
    ops.append((NativeShardOps(model, cfg, po._SAMPLERS["pcg64"], None, hi - lo, phi - plo), lo, hi, plo, phi))


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    out = fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1), out


res = {}
for proto in ("gather", "select"):
    t_sel, t_desc, vol = [], [], 0
    for rep in range(3):
        if proto == "gather":
            ms, runs = timed(lambda: torch.stack([o.select(0, lo, hi - lo) for o, lo, hi, _, _ in ops]))
        else:
            def xchg():
                for o, lo, hi, _, _ in ops:
                    o.select(0, lo, hi - lo, elite=False)
                sts = [o.topm_init() for o, *_ in ops]
                for _ in range(4):
                    hs = torch.stack([o.topm_hist(st) for (o, *_), st in zip(ops, sts)]).sum(0)
                    for (o, *_), st in zip(ops, sts):
                        o.topm_pick(st, hs)
                take = allot_top_m(torch.stack([o.topm_local(st) for (o, *_), st in zip(ops, sts)]).cpu().numpy())
                cap = max(1, int(take.max()))
                return torch.stack([o.topm_contrib(int(take[r]), cap) for r, (o, *_) in enumerate(ops)])
            ms, runs = timed(xchg)
        t_sel.append(ms / G)
        vol = runs.numel() * 8
        per = []
        for o, _, _, plo, phi in ops:
            ms, _ = timed(lambda: o.descend(0, runs, plo, phi))
            per.append(ms)
        t_desc.append(statistics.mean(per))
    res[proto] = (statistics.median(t_sel), statistics.median(t_desc), vol)
    print(f"{proto:7s} G={G} n/rank={n_rank}: select/exchange {res[proto][0]:.3f} ms/rank, descend (merge + schedule) "
          f"{res[proto][1]:.3f} ms/rank, gathered {vol / 2**20:.1f} MiB per rank")
print(f"descend saving per rank: {res['gather'][1] - res['select'][1]:.3f} ms; gathered bytes "
      f"{res['gather'][2] / max(1, res['select'][2]):.1f}x less")
