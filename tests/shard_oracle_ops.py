"""Oracle-backed stand-ins for the device halves of a sharded restart (test infrastructure).

They implement the contract of ``spasm_shard_select`` / ``spasm_shard_descend``
(include/spasm.h) in numpy on top of oracle/stage1.py, so the CPU tests can drive
``sharded.solve_sharded``'s host logic (partitioning, the two all-gathers over a gloo
group, the candidate merge, restart control) at world_size > 1 without a GPU.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import stage1 as orc

ALL_ONES = np.uint64(0xFFFFFFFFFFFFFFFF)


def order_key64(c):
    """Order-preserving uint64 image of float64 costs (common.cuh order_key); NaN last."""
    c = np.asarray(c, dtype=np.float64)
    b = c.view(np.uint64)
    sign = (b >> np.uint64(63)).astype(bool)
    k = np.where(sign, ~b, b | np.uint64(1 << 63))
    return np.where(np.isnan(c), ALL_ONES, k)


def merge_runs(runs, m):
    """Global first m rows of the gathered (world, m, 2) records (lexicographic key, row)."""
    r = np.asarray(runs).reshape(-1, 2).view(np.uint64)
    r = r[r[:, 1] != ALL_ONES]
    order = np.lexsort((r[:, 1], r[:, 0]))[:m]
    return r[order, 1].astype(np.int64)


class OracleShardOps:
    def __init__(self, omodel, cfg: orc.OracleConfig, warm=None):
        self.o = omodel
        self.cfg = cfg
        self.warm = None if warm is None or len(warm) == 0 else np.atleast_2d(np.asarray(warm, float))
        self._draws = {}
        self.launches = 0

    def _batch(self, restart):
        if restart not in self._draws:
            v = orc.sample_uniform(self.o, self.cfg.n, orc.restart_stream(self.cfg.seed, restart))
            if self.warm is not None:
                v[: len(self.warm)] = np.clip(self.warm, self.o.lower, self.o.upper)
            self._draws = {restart: v}
        return self._draws[restart]

    def select(self, restart, row_lo, n_local):
        v = self._batch(restart)[row_lo: row_lo + n_local]
        m = self.cfg.m
        rec = np.full((m, 2), ALL_ONES, dtype=np.uint64)
        if n_local:
            c = self.o.evaluate(v, orc.LINEAR)
            order = np.argsort(c, kind="stable")[:m]
            rec[: len(order), 0] = order_key64(c[order])
            rec[: len(order), 1] = (row_lo + order).astype(np.uint64)
        return torch.from_numpy(rec.view(np.int64).copy())

    def descend(self, restart, elite_all, pos_lo, pos_hi):
        cfg = self.cfg
        D = self.o.dimension
        top = merge_runs(elite_all.cpu().numpy(), cfg.m)
        rows = top[pos_lo:pos_hi]
        x = self._batch(restart)[rows].copy()
        x, fl, _ = orc.run_descent_schedule(self.o, x, cfg)
        final = self.o.evaluate(x, orc.QUADRATIC) if len(x) else np.zeros(0)
        sat = final < cfg.epsilon
        idx = np.flatnonzero(sat)
        order = idx[np.argsort(final[idx], kind="stable")][: cfg.p_return]
        cand = np.zeros(3 + cfg.p_return * (4 + D))
        cand[0], cand[1], cand[2] = sat.sum(), fl.sum(), len(order)
        recheck = self.o.evaluate(x[order], orc.QUADRATIC) if len(order) else np.zeros(0)
        for c, q in enumerate(order):
            r = cand[3 + c * (4 + D): 3 + (c + 1) * (4 + D)]
            r[0], r[1], r[2], r[3] = pos_lo + q, rows[q], final[q], recheck[c]
            r[4:] = x[q]
        return torch.from_numpy(cand)
