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
    """Global first m rows of the gathered (world, run_len, 2) records (lexicographic key, row)."""
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

    key_bits = 64

    def select(self, restart, row_lo, n_local, elite=True):
        v = self._batch(restart)[row_lo: row_lo + n_local]
        m = self.cfg.m
        c = self.o.evaluate(v, orc.LINEAR) if n_local else np.zeros(0)
        order = np.argsort(c, kind="stable")
        self._keys = order_key64(c[order])  # the rank's sorted (key, global row) records
        self._rows = (row_lo + order).astype(np.uint64)
        if not elite:
            return None
        rec = np.full((m, 2), ALL_ONES, dtype=np.uint64)
        k = min(m, n_local)
        rec[:k, 0] = self._keys[:k]
        rec[:k, 1] = self._rows[:k]
        return torch.from_numpy(rec.view(np.int64).copy())

    # the top-m select protocol (spasm_shard_topm_*), on the rank's sorted keys
    def topm_init(self):
        return {"prefix": 0, "remaining": self.cfg.m, "pass": 0}

    def topm_hist(self, st):
        shift = self.key_bits - 8 * (st["pass"] + 1)
        k = self._keys.astype(object)
        sel = [int(x) for x in k if (int(x) >> (shift + 8)) == (st["prefix"] >> (shift + 8))]
        h = np.zeros(256, dtype=np.int64)
        for x in sel:
            h[(x >> shift) & 0xFF] += 1
        return torch.from_numpy(h)

    def topm_pick(self, st, hist_sum):
        h = np.asarray(hist_sum.cpu().numpy() if hasattr(hist_sum, "cpu") else hist_sum, dtype=np.int64)
        shift = self.key_bits - 8 * (st["pass"] + 1)
        rem, d = st["remaining"], 0
        while d < 255 and rem > h[d]:
            rem -= h[d]
            d += 1
        st["prefix"] |= d << shift
        st["remaining"] = int(rem)
        st["pass"] += 1

    def topm_local(self, st):
        ks = np.uint64(st["prefix"])
        less = int(np.searchsorted(self._keys, ks, side="left"))
        ties = int(np.searchsorted(self._keys, ks, side="right")) - less
        return torch.tensor([less, ties, st["remaining"]], dtype=torch.int64)

    def topm_contrib(self, take, cap):
        rec = np.full((cap, 2), ALL_ONES, dtype=np.uint64)
        rec[:take, 0] = self._keys[:take]
        rec[:take, 1] = self._rows[:take]
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
