"""CPU ORACLE for the stage-1 hot path -- test infrastructure, not product code.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this module, and only as the checker or the timed CPU baseline. The
product path (paper_2510_07674_b200) never imports it and has no CPU fallback.

A float64 numpy restatement of the reference's stage-1 algorithm
(/root/reference/pkg/src/seqplace, cited as file:line below):

  geometry.py:131-202            sphere penetration, linear/quadratic modes, subgradients
  problems/_interactions.py:23-178  pair-entry tables, batched cost + pose gradient
  problems/tetris.py:54-70,159-245  wall spheres, bounds, height term, row layout
  problems/tower.py:144-322      stability (suffix CoM vs yawed footprint), heights, overlaps
  particle_opt.py:146-400        sampling, stable top-M, LR schedule, clamped NaN-freezing
                                 steps, two-phase schedule, restart loop, extraction

Pinned against the reference itself: tests/golden/make_golden.py imported the
reference in the build container and froze its outputs (costs, gradients, draws,
schedules, full solves) into tests/golden/*.npz; tests/test_oracle_golden.py checks
this restatement against them (CPU, no GPU needed).
"""
from __future__ import annotations

import time
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass
from typing import Optional

import numpy as np

LINEAR = "linear"
QUADRATIC = "quadratic"


# ---------------------------------------------------------------------------
# batched sphere-overlap core (problems/_interactions.py)
# ---------------------------------------------------------------------------
class PairTable:
    """Flat (a, b, weight, rsum) entries: body-body pairs (i<j, spheres in C order)
    followed by body-static pairs (_interactions.py:46-73). Gradient scatter uses
    np.add.at over the entries' owning bodies instead of per-body entry lists."""

    def __init__(self, locals_, radii, static_c, static_r, w_bb, w_bs):
        self.n_bodies = len(locals_)
        self.loc = np.concatenate([np.asarray(c, float) for c in locals_]) if locals_ else np.zeros((0, 3))
        self.rad = np.concatenate([np.asarray(r, float) for r in radii]) if radii else np.zeros(0)
        self.body = np.concatenate([np.full(len(c), b) for b, c in enumerate(locals_)]).astype(int)
        self.sc = np.asarray(static_c, float).reshape(-1, 3)
        self.sr = np.asarray(static_r, float).reshape(-1)
        start = np.concatenate([[0], np.cumsum([len(c) for c in locals_])])
        a, b, w = [], [], []
        for i in range(self.n_bodies):
            for j in range(i + 1, self.n_bodies):
                ii, jj = np.meshgrid(np.arange(start[i], start[i + 1]), np.arange(start[j], start[j + 1]),
                                     indexing="ij")
                a.append(ii.ravel())
                b.append(jj.ravel())
                w.append(np.full(ii.size, float(w_bb)))
        nm = len(self.loc)
        if len(self.sc):
            ii, ss = np.meshgrid(np.arange(nm), np.arange(len(self.sc)), indexing="ij")
            a.append(ii.ravel())
            b.append(nm + ss.ravel())
            w.append(np.full(ii.size, float(w_bs)))
        self.a = np.concatenate(a) if a else np.zeros(0, int)
        self.b = np.concatenate(b) if b else np.zeros(0, int)
        self.w = np.concatenate(w) if w else np.zeros(0)
        all_r = np.concatenate([self.rad, self.sr])
        self.rsum = all_r[self.a] + all_r[self.b] if len(self.a) else np.zeros(0)
        self.nm = nm
        self.a_body = self.body[self.a] if len(self.a) else np.zeros(0, int)
        self.b_mov = self.b < nm
        self.b_body = np.where(self.b_mov, self.body[np.minimum(self.b, max(nm - 1, 0))], -1)

    def _rotated(self, yaw):
        if yaw is None:
            return np.broadcast_to(self.loc, (1,) + self.loc.shape), None
        c = np.cos(yaw)[:, self.body]
        s = np.sin(yaw)[:, self.body]
        lx, ly, lz = self.loc[:, 0], self.loc[:, 1], self.loc[:, 2]
        rot = np.stack([c * lx - s * ly, s * lx + c * ly, np.broadcast_to(lz, c.shape)], axis=-1)
        drot = np.stack([-s * lx - c * ly, c * lx - s * ly, np.zeros_like(c)], axis=-1)
        return rot, drot

    def _diff(self, pos, yaw):
        rot, drot = self._rotated(yaw)
        mov = pos[:, self.body, :] + rot
        world = np.concatenate([mov, np.broadcast_to(self.sc, (pos.shape[0],) + self.sc.shape)], axis=1)
        diff = world[:, self.a, :] - world[:, self.b, :]
        d = np.sqrt(np.sum(diff * diff, axis=-1))
        return diff, d, drot

    def margin(self, pos, yaw, static_band=1e-2):
        """Per row, the smallest |rsum - d| over all entries: distance to a hinge kink
        (where fp32 and fp64 may legitimately disagree on the active set). Static (wall)
        entries are scaled by 1/static_band: the fp32 kernel evaluates them in an exact
        cancellation-free form whose error is ~1e-8, so their kink band is ~100x narrower."""
        if len(self.a) == 0:
            return np.full(pos.shape[0], np.inf)
        _, d, _ = self._diff(pos, yaw)
        gap = np.abs(self.rsum - d)
        gap = np.where(self.b_mov[None, :], gap, gap / static_band)
        return np.min(gap, axis=1)

    def cost(self, pos, yaw, mode):
        if len(self.a) == 0:
            return np.zeros(pos.shape[0])
        _, d, _ = self._diff(pos, yaw)
        pen = np.maximum(0.0, self.rsum - d)
        return (pen * pen if mode == QUADRATIC else pen) @ self.w

    def grad(self, pos, yaw, mode):
        P = pos.shape[0]
        gp = np.zeros((P, self.n_bodies, 3))
        gy = None if yaw is None else np.zeros((P, self.n_bodies))
        if len(self.a) == 0:
            return gp, gy
        diff, d, drot = self._diff(pos, yaw)
        pen = np.maximum(0.0, self.rsum - d)
        live = (pen > 0.0) & (d > 0.0)
        f = self.w if mode == LINEAR else 2.0 * self.w * pen
        s = np.where(live, -f / np.where(d > 0.0, d, 1.0), 0.0)
        g = s[..., None] * diff  # d cost / d centre(a)
        ga = np.zeros((P, self.n_bodies, 3))
        for k in range(3):
            np.add.at(ga[..., k].T, self.a_body, g[..., k].T)
        gbm = np.zeros((P, self.n_bodies, 3))
        mb = np.flatnonzero(self.b_mov)
        for k in range(3):
            np.add.at(gbm[..., k].T, self.b_body[mb], g[:, mb, k].T)
        gp = ga - gbm
        if gy is not None:
            ta = np.sum(g * drot[:, self.a, :], axis=-1)
            ya = np.zeros((P, self.n_bodies))
            np.add.at(ya.T, self.a_body, ta.T)
            tb = np.sum(g[:, mb, :] * drot[:, self.b[mb], :], axis=-1)
            yb = np.zeros((P, self.n_bodies))
            np.add.at(yb.T, self.b_body[mb], tb.T)
            gy = ya - yb
        return gp, gy


# ---------------------------------------------------------------------------
# placement cost models (problems/tetris.py, problems/tower.py)
# ---------------------------------------------------------------------------
class OracleModel:
    dimension: int
    lower: np.ndarray
    upper: np.ndarray

    def satisfaction(self, values, epsilon=1e-3):  # particle_opt.py:57-58
        return self.evaluate(values, QUADRATIC) < epsilon

    def clamp(self, values):
        return np.clip(values, self.lower, self.upper)


class TetrisOracle(OracleModel):
    """tetris.py:159-245 over the pair table. ``problem`` needs blocks (with
    sphere_set, width, height), box, z_star, yaw_mode, weights, wall_centers/radii."""

    def __init__(self, problem):
        self.free = problem.yaw_mode != "fixed"
        self.per = 4 if self.free else 3
        n = len(problem.blocks)
        self.n = n
        lo = np.empty((n, self.per))
        hi = np.empty((n, self.per))
        for b, blk in enumerate(problem.blocks):
            lo[b, :3] = problem.box.min
            hi[b, :3] = [problem.box.max[0] - blk.width, problem.box.max[1] - blk.height, problem.box.max[2]]
            if self.free:
                lo[b, 3], hi[b, 3] = -np.pi, np.pi
        self.lower, self.upper = lo.ravel(), hi.ravel()
        self.dimension = n * self.per
        w = problem.weights
        self.core = PairTable([b.sphere_set.centers for b in problem.blocks], [b.sphere_set.radii for b in problem.blocks],
                              problem.wall_centers, problem.wall_radii, w.block_block, w.block_wall)
        self.w_h = float(w.height)
        self.z_star = float(problem.z_star)

    def _split(self, v):
        v = np.asarray(v, float).reshape(len(v), self.n, self.per)
        return v[..., :3], (v[..., 3] if self.free else None)

    def kink_margin(self, values):
        pos, yaw = self._split(values)
        return np.minimum(self.core.margin(pos, yaw), np.min(np.abs(pos[..., 2] - self.z_star), axis=1))

    def evaluate(self, values, mode):
        pos, yaw = self._split(values)
        dz = pos[..., 2] - self.z_star
        h = np.abs(dz) if mode == LINEAR else dz * dz
        return self.core.cost(pos, yaw, mode) + self.w_h * h.sum(axis=1)

    def gradient(self, values, mode):
        pos, yaw = self._split(values)
        gp, gy = self.core.grad(pos, yaw, mode)
        dz = pos[..., 2] - self.z_star
        gp[..., 2] += self.w_h * (np.sign(dz) if mode == LINEAR else 2.0 * dz)
        out = np.empty((len(pos), self.n, self.per))
        out[..., :3] = gp
        if self.free:
            out[..., 3] = gy
        return out.reshape(len(pos), -1)


class TowerOracle(OracleModel):
    """tower.py:144-322."""

    def __init__(self, problem):
        self.free = problem.yaw_mode != "fixed"
        self.per = 4 if self.free else 3
        n = problem.n_blocks
        self.n = n
        lo = np.empty((n, self.per))
        hi = np.empty((n, self.per))
        lo[:, :3] = problem.box.min
        hi[:, :3] = problem.box.max
        if self.free:
            lo[:, 3], hi[:, 3] = -np.pi, np.pi
        self.lower, self.upper = lo.ravel(), hi.ravel()
        self.dimension = n * self.per
        self.side = float(problem.side)
        self.half = float(problem.footprint_halfwidth)
        self.r = 0.5 * self.side
        self.targets = (np.arange(n) + 1.0) * self.side
        self.oc = np.asarray(problem.obstacle_centers, float).reshape(-1, 3)
        self.orad = np.asarray(problem.obstacle_radii, float).reshape(-1)
        self.w = problem.weights
        self.pi, self.pj = np.triu_indices(n, k=1)

    def _split(self, v):
        v = np.asarray(v, float).reshape(len(v), self.n, self.per)
        return v[..., :3], (v[..., 3] if self.free else None)

    def _stability(self, pos, yaw):
        # suffix mean of the blocks above support i (tower.py:208-212)
        xy = pos[..., :2]
        suffix = np.cumsum(xy[:, ::-1], axis=1)[:, ::-1]
        cnt = np.arange(self.n - 1, 0, -1, dtype=float)
        rel = suffix[:, 1:] / cnt[None, :, None] - xy[:, :-1]
        if yaw is None:
            loc, dloc, c, s = rel, None, None, None
        else:
            c, s = np.cos(yaw[:, :-1]), np.sin(yaw[:, :-1])
            loc = np.stack([c * rel[..., 0] + s * rel[..., 1], -s * rel[..., 0] + c * rel[..., 1]], -1)
            dloc = np.stack([-s * rel[..., 0] + c * rel[..., 1], -c * rel[..., 0] - s * rel[..., 1]], -1)
        delta = loc - np.clip(loc, -self.half, self.half)
        dist = np.sqrt(np.sum(delta * delta, axis=-1))
        unit = np.where(dist[..., None] > 0, delta / np.where(dist > 0, dist, 1.0)[..., None], 0.0)
        return dist, unit, dloc, c, s, cnt

    def _pairs(self, pos):
        diff = pos[:, self.pi] - pos[:, self.pj]
        d = np.sqrt(np.sum(diff * diff, axis=-1))
        pen = np.maximum(0.0, self.side - d)
        odiff = pos[:, :, None, :] - self.oc[None, None]
        od = np.sqrt(np.sum(odiff * odiff, axis=-1))
        open_ = np.maximum(0.0, (self.r + self.orad) - od)
        return diff, d, pen, odiff, od, open_

    def kink_margin(self, values):
        pos, yaw = self._split(values)
        dist, _, _, _, _, _ = self._stability(pos, yaw)
        xy = pos[..., :2]
        suffix = np.cumsum(xy[:, ::-1], axis=1)[:, ::-1]
        cnt = np.arange(self.n - 1, 0, -1, dtype=float)
        rel = suffix[:, 1:] / cnt[None, :, None] - xy[:, :-1]
        edge = np.min(np.abs(np.abs(rel) - self.half), axis=(1, 2)) if yaw is None else np.full(len(pos), np.inf)
        _, d, _, _, od, _ = self._pairs(pos)
        m = np.minimum(np.min(np.abs(self.side - d), axis=1), np.min(np.where(dist > 0, dist, np.inf), axis=1))
        m = np.minimum(m, np.min(np.abs(pos[..., 2] - self.targets), axis=1))
        if len(self.oc):
            m = np.minimum(m, np.min(np.abs((self.r + self.orad) - od), axis=(1, 2)))
        return np.minimum(m, edge)

    def evaluate(self, values, mode):
        sq = mode == QUADRATIC
        pos, yaw = self._split(values)
        dist = self._stability(pos, yaw)[0]
        total = self.w.stability * (dist * dist if sq else dist).sum(1)
        dz = pos[..., 2] - self.targets
        total = total + self.w.height * (dz * dz if sq else np.abs(dz)).sum(1)
        _, _, pen, _, _, open_ = self._pairs(pos)
        total = total + self.w.collision * (pen * pen if sq else pen).sum(1)
        if len(self.oc):
            total = total + self.w.collision * (open_ * open_ if sq else open_).sum((1, 2))
        return total

    def gradient(self, values, mode):
        sq = mode == QUADRATIC
        pos, yaw = self._split(values)
        P, n = pos.shape[0], self.n
        gp = np.zeros((P, n, 3))
        gy = np.zeros((P, n)) if self.free else None
        dist, unit, dloc, c, s, cnt = self._stability(pos, yaw)
        fac = self.w.stability * (2.0 * dist if sq else (dist > 0).astype(float))
        gl = fac[..., None] * unit
        if yaw is None:
            gw = gl
        else:
            gw = np.stack([c * gl[..., 0] - s * gl[..., 1], s * gl[..., 0] + c * gl[..., 1]], -1)
            gy[:, :-1] += np.sum(gl * dloc, axis=-1)
        gp[:, 1:, :2] += np.cumsum(gw / cnt[None, :, None], axis=1)
        gp[:, :-1, :2] -= gw
        dz = pos[..., 2] - self.targets
        gp[..., 2] += self.w.height * (2.0 * dz if sq else np.sign(dz))
        diff, d, pen, odiff, od, open_ = self._pairs(pos)
        live = (pen > 0) & (d > 0)
        sc = np.where(live, -(self.w.collision * (2.0 * pen if sq else 1.0)) / np.where(d > 0, d, 1.0), 0.0)
        g = sc[..., None] * diff
        for k in range(3):
            np.add.at(gp[..., k].T, self.pi, g[..., k].T)
            np.add.at(gp[..., k].T, self.pj, -g[..., k].T)
        if len(self.oc):
            live = (open_ > 0) & (od > 0)
            sc = np.where(live, -(self.w.collision * (2.0 * open_ if sq else 1.0)) / np.where(od > 0, od, 1.0), 0.0)
            gp += np.sum(sc[..., None] * odiff, axis=2)
        out = np.empty((P, n, self.per))
        out[..., :3] = gp
        if self.free:
            out[..., 3] = gy
        return out.reshape(P, -1)


def oracle_model(problem):
    """as_cost_model restated (problems/__init__.py:48-57)."""
    if hasattr(problem, "blocks") and hasattr(problem, "z_star"):
        return TetrisOracle(problem)
    if hasattr(problem, "n_blocks") and hasattr(problem, "side"):
        return TowerOracle(problem)
    raise TypeError(f"no placement cost model for {type(problem).__name__}")


# ---------------------------------------------------------------------------
# engine (particle_opt.py)
# ---------------------------------------------------------------------------
@dataclass
class OracleConfig:
    n: int = 4096
    m: int = 512
    k_lin: int = 25
    k_quad: int = 5
    eta_init: float = 0.1
    alpha: float = 0.05
    epsilon: float = 1e-3
    p_return: int = 32
    max_restarts: int = 64
    seed: int = 0


def restart_stream(seed, restart):  # particle_opt.py:176-178
    return np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(restart,)))


def sample_uniform(model, n, rng):  # particle_opt.py:181-192
    return rng.uniform(model.lower, model.upper, size=(n, model.dimension))


def select_topk(costs, m):  # particle_opt.py:195-200
    return np.argsort(costs, kind="stable")[:m]


def lr_schedule(k, k_lin, eta):  # particle_opt.py:203-211
    return eta * (1.0 - k / k_lin)


class _Chunks:
    """Contiguous row chunks over a thread pool; concatenated in order (particle_opt.py:146-173)."""

    def __init__(self, threads=1):
        self.threads = max(1, int(threads))
        self.pool = ThreadPoolExecutor(self.threads) if self.threads > 1 else None

    def __call__(self, fn, values, mode):
        if self.pool is None or len(values) < 2 * self.threads:
            return fn(values, mode)
        parts = list(self.pool.map(lambda c: fn(c, mode), np.array_split(values, self.threads)))
        return np.concatenate(parts)

    def close(self):
        if self.pool is not None:
            self.pool.shutdown()


def step_values(model, values, flagged, mode, rate, run=None):  # particle_opt.py:214-228
    g = (run or (lambda f, v, m: f(v, m)))(model.gradient, values, mode)
    bad = ~np.all(np.isfinite(g), axis=1)
    if bad.any():
        flagged |= bad
        g = np.where(bad[:, None], 0.0, g)
    values -= rate * g
    np.clip(values, model.lower, model.upper, out=values)


def run_descent_schedule(model, values, cfg, run=None, trace_sink=None, epsilon=None):  # particle_opt.py:266-300
    eps = cfg.epsilon if epsilon is None else epsilon
    ev = run or (lambda f, v, m: f(v, m))
    flagged = np.zeros(len(values), bool)
    step = 0
    for k in range(1, cfg.k_lin + 1):
        step_values(model, values, flagged, LINEAR, lr_schedule(k, cfg.k_lin, cfg.eta_init), run)
        step += 1
        if trace_sink:
            trace_sink(step, LINEAR, ev(model.evaluate, values, LINEAR), ev(model.evaluate, values, QUADRATIC) < eps)
    for _ in range(cfg.k_quad):
        step_values(model, values, flagged, QUADRATIC, cfg.alpha, run)
        step += 1
        if trace_sink:
            cq = ev(model.evaluate, values, QUADRATIC)
            trace_sink(step, QUADRATIC, cq, cq < eps)
    return values, flagged, step


@dataclass
class OracleResult:
    success: bool
    particles: np.ndarray
    costs: np.ndarray
    indices: np.ndarray
    restarts: int
    steps: int
    n_satisfying: int
    flagged: int
    time_ms: float


def solve(model, cfg: OracleConfig, warm_seeds=None, threads=1) -> OracleResult:  # particle_opt.py:303-400
    t0 = time.perf_counter()
    run = _Chunks(threads)
    steps = flagged_total = 0
    try:
        for restart in range(cfg.max_restarts):
            vals = sample_uniform(model, cfg.n, restart_stream(cfg.seed, restart))
            if warm_seeds is not None and len(warm_seeds):
                w = np.atleast_2d(np.asarray(warm_seeds, float))
                vals[: len(w)] = np.clip(w, model.lower, model.upper)
            costs = run(model.evaluate, vals, LINEAR)
            top = select_topk(costs, cfg.m)
            x = vals[top].copy()
            x, fl, k = run_descent_schedule(model, x, cfg, run)
            steps += k
            flagged_total += int(fl.sum())
            final = run(model.evaluate, x, QUADRATIC)
            sat = final < cfg.epsilon
            if sat.any():
                idx = np.flatnonzero(sat)
                order = idx[np.argsort(final[idx], kind="stable")][: cfg.p_return]
                order = order[model.satisfaction(x[order], cfg.epsilon)]
                return OracleResult(len(order) > 0, x[order], final[order], top[order], restart, steps,
                                    int(sat.sum()), flagged_total, (time.perf_counter() - t0) * 1e3)
    finally:
        run.close()
    return OracleResult(False, np.zeros((0, model.dimension)), np.zeros(0), np.zeros(0, int), cfg.max_restarts,
                        steps, 0, flagged_total, (time.perf_counter() - t0) * 1e3)
