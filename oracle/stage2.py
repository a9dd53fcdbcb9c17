"""CPU ORACLE for the stage-2 hot path -- test infrastructure, not product code.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may use it. float64 numpy restatement of the reference's trajectory stage
(/root/reference/pkg/src/seqplace, file:line below):

  robot.py:71-84, 160-180      Rodrigues joint rotation, batched forward kinematics
  robot.py:214-224             exact tool-yaw Jacobian
  robot.py:227-302             batched damped-least-squares IK (4x4), 16 seeded restarts
  robot.py:325-347             grasp / inverse grasp maps
  trajopt.py:305-367           per-problem geometry (arm sphere tables, obstacle families)
  trajopt.py:416-653           AL objective, constraints and exact gradient (variant B)
  trajopt.py:726-787           tool-down polish (5x5 DLS), arm worst penetration
  trajopt.py:795-876           lifting placements into joint space (<= 4 IK draws)
  trajopt.py:892-923           piecewise-linear trajectory initialization
  trajopt.py:936-1063          augmented-Lagrangian outer/inner loop
  trajopt.py:1071-1153         independent validation

Reference defect: as shipped, trajopt._evaluate has no `place_mode`
parameter and reads undefined names. The reference's own tests pin "variant B": the
placement term uses the same mode as the collision terms (`pmode = mode`). This oracle
implements `place_mode` explicitly; None means variant B. Goldens come from a patched
COPY of the reference made by tests/golden/make_golden_stage2.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from types import SimpleNamespace
from typing import List, Optional

import numpy as np

from . import stage1

LINEAR, QUADRATIC = "linear", "quadratic"
FLIP = np.diag([1.0, -1.0, -1.0])
IK_POS_TOL, IK_YAW_TOL, IK_DAMPING = 1e-4, 1e-3, 1e-3
POLISH_ANGLE_TOL = 0.005
POLISH_MAX_ITERS = 1000
INNER_STEP_CLAMP = 0.1
LIFT_DRAW_STRIDE = 1000003
TRAJ_STREAM = 1 << 20


def wrap(a):
    """normalize_yaw: into (-pi, pi] (geometry.py:31-38)."""
    a = np.asarray(a, float)
    w = np.remainder(a + np.pi, 2 * np.pi) - np.pi
    return np.where(w <= -np.pi, w + 2 * np.pi, w)


# ---------------------------------------------------------------------------
# kinematics
# ---------------------------------------------------------------------------
def rodrigues(axis, q):
    q = np.asarray(q, float)
    c = np.cos(q)[..., None, None]
    s = np.sin(q)[..., None, None]
    k = np.array([[0.0, -axis[2], axis[1]], [axis[2], 0.0, -axis[0]], [-axis[1], axis[0], 0.0]])
    return c * np.eye(3) + s * k + (1.0 - c) * np.outer(axis, axis)


def fk(chain, Q):
    """Batched FK over (..., dof): translate by the offset, then rotate about the axis."""
    Q = np.asarray(Q, float)
    lead = Q.shape[:-1]
    J = len(chain.joints)
    p = np.zeros(lead + (3,))
    R = np.broadcast_to(np.eye(3), lead + (3, 3)).copy()
    origins = np.zeros(lead + (J, 3))
    axes = np.zeros(lead + (J, 3))
    lpos = np.zeros(lead + (J, 3))
    lrot = np.zeros(lead + (J, 3, 3))
    for i, jt in enumerate(chain.joints):
        p = p + np.einsum("...ij,j->...i", R, jt.offset)
        axes[..., i, :] = np.einsum("...ij,j->...i", R, jt.axis)
        origins[..., i, :] = p
        R = np.einsum("...ij,...jk->...ik", R, rodrigues(jt.axis, Q[..., i]))
        lpos[..., i, :] = p
        lrot[..., i, :, :] = R
    ee = p + np.einsum("...ij,j->...i", R, chain.tool_translation)
    Ree = np.einsum("...ij,jk->...ik", R, chain.tool_rotation)
    return SimpleNamespace(ee=ee, rot=Ree, origins=origins, axes=axes, lpos=lpos, lrot=lrot)


def yaw_of(rot):
    return np.arctan2(rot[..., 1, 0], rot[..., 0, 0])


def yaw_jac(rot, axes):
    """d yaw / d q from dR/dq_j = [z_j]x R (robot.py:214-224)."""
    r00, r10 = rot[..., 0, 0], rot[..., 1, 0]
    den = r00 * r00 + r10 * r10
    dcol = np.cross(axes, rot[..., :, 0][..., None, :])
    num = r00[..., None] * dcol[..., 1] - r10[..., None] * dcol[..., 0]
    bad = den < 1e-12
    return np.where(bad[..., None], 0.0, num / np.where(bad, 1.0, den)[..., None])


def chain_limits(chain):
    return np.array([j.lower for j in chain.joints]), np.array([j.upper for j in chain.joints])


def arm_table(chain):
    cs, rs, ls = [], [], []
    for i, sp in enumerate(chain.link_spheres):
        if sp is None:
            continue
        cs.append(sp.centers)
        rs.append(sp.radii)
        ls += [i] * len(sp.centers)
    if not cs:
        return np.zeros((0, 3)), np.zeros(0), np.zeros(0, int)
    return np.concatenate(cs), np.concatenate(rs), np.array(ls, int)


def ik_solve_batch(chain, tpos, tyaw, restarts=16, seed=0, max_iters=200, damping=IK_DAMPING):
    """robot.py:227-302. tpos (T,3), tyaw (T,) (already wrapped, as Pose stores them)."""
    lo, hi = chain_limits(chain)
    dof = len(lo)
    nt = len(tpos)
    if nt == 0:
        return np.zeros((0, dof)), np.zeros(0, bool), np.zeros(0)
    seeds = np.empty((nt, restarts, dof))
    for t in range(nt):
        g = np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(t,)))
        seeds[t] = g.uniform(lo, hi, size=(restarts, dof))
    Q = seeds.reshape(-1, dof)
    tp = np.repeat(tpos, restarts, axis=0)
    ty = np.repeat(tyaw, restarts)
    for _ in range(max_iters):
        f = fk(chain, Q)
        pe = tp - f.ee
        ye = wrap(ty - yaw_of(f.rot))
        conv = (np.linalg.norm(pe, axis=1) < IK_POS_TOL) & (np.abs(ye) < IK_YAW_TOL)
        if conv.all():
            break
        jl = np.cross(f.axes, f.ee[:, None, :] - f.origins)
        J4 = np.concatenate([np.swapaxes(jl, 1, 2), f.axes[:, None, :, 2]], axis=1)
        A = J4 @ np.swapaxes(J4, 1, 2) + damping * np.eye(4)
        y = np.linalg.solve(A, np.concatenate([pe, ye[:, None]], 1)[..., None])[..., 0]
        dq = np.einsum("nji,nj->ni", J4, y)
        dq = dq * np.minimum(1.0, 0.5 / np.maximum(np.max(np.abs(dq), axis=1), 1e-12))[:, None]
        dq[conv] = 0.0
        Q = np.clip(Q + dq, lo, hi)
    f = fk(chain, Q)
    pn = np.linalg.norm(tp - f.ee, axis=1)
    ye = np.abs(wrap(ty - yaw_of(f.rot)))
    ok = (pn < IK_POS_TOL) & (ye < IK_YAW_TOL)
    score = (pn + ye).reshape(nt, restarts)
    ok = ok.reshape(nt, restarts)
    best = np.argmin(np.where(ok, 0.0, 1e6) + score, axis=1)
    r = np.arange(nt)
    return Q.reshape(nt, restarts, dof)[r, best], ok[r, best], score[r, best]


def polish_tool_down(chain, Q, tpos, tyaw):
    """trajopt.py:726-776."""
    Q = np.array(Q, float)
    if len(Q) == 0:
        return Q, np.zeros(0, bool)
    lo, hi = chain_limits(chain)
    cos_tol = math.cos(POLISH_ANGLE_TOL)
    fc = (hi - lo) >= 2 * math.pi - 1e-9
    for _ in range(POLISH_MAX_ITERS):
        f = fk(chain, Q)
        pe = tpos - f.ee
        ye = wrap(tyaw - yaw_of(f.rot))
        ax = f.rot[..., :, 2]
        done = (np.linalg.norm(pe, axis=1) < IK_POS_TOL) & (np.abs(ye) < IK_YAW_TOL) & (-ax[..., 2] > cos_tol)
        if done.all():
            break
        jl = np.cross(f.axes, f.ee[:, None, :] - f.origins)
        jy = yaw_jac(f.rot, f.axes)
        jd = np.cross(f.axes, ax[:, None, :])[..., 2]
        J5 = np.concatenate([np.swapaxes(jl, 1, 2), jy[:, None, :], jd[:, None, :]], axis=1)
        e5 = np.concatenate([pe, ye[:, None], (-1.0 - ax[..., 2])[:, None]], axis=1)
        A = J5 @ np.swapaxes(J5, 1, 2) + IK_DAMPING * np.eye(5)
        y = np.linalg.solve(A, e5[..., None])[..., 0]
        dq = np.einsum("nji,nj->ni", J5, y)
        dq = dq * np.minimum(1.0, 0.5 / np.maximum(np.max(np.abs(dq), axis=1), 1e-12))[:, None]
        dq[done] = 0.0
        Q = Q + dq
        Q[:, fc] = lo[fc] + np.mod(Q[:, fc] - lo[fc], 2 * math.pi)
        Q = np.clip(Q, lo, hi)
    f = fk(chain, Q)
    ok = (np.linalg.norm(tpos - f.ee, axis=1) < IK_POS_TOL) & (np.abs(wrap(tyaw - yaw_of(f.rot))) < IK_YAW_TOL) \
        & (-f.rot[..., 2, 2] > cos_tol)
    return Q, ok


def grasp_target(pose_xyzyaw, grasp):
    """grasp_pose restated on (x, y, z, yaw) rows (robot.py:325-334); yaw wrapped like Pose."""
    x, y, z, yaw = pose_xyzyaw
    c, s = math.cos(yaw), math.sin(yaw)
    ox, oy, oz = grasp.offset
    return np.array([x + c * ox - s * oy, y + s * ox + c * oy, z + oz]), float(wrap(yaw + grasp.yaw_offset))


# ---------------------------------------------------------------------------
# geometry (trajopt.py:305-367)
# ---------------------------------------------------------------------------
def _is_tower(problem):
    return hasattr(problem, "n_blocks") and hasattr(problem, "side") and not hasattr(problem, "z_star")


def _is_motion(problem):
    return hasattr(problem, "start") and hasattr(problem, "goal")


def _free_twin_model(problem):
    twin = SimpleNamespace(**{k: getattr(problem, k) for k in dir(problem) if not k.startswith("__")
                              and not callable(getattr(problem, k))})
    twin.yaw_mode = "quantized-free"
    if _is_tower(problem):
        return stage1.TowerOracle(twin)
    return stage1.TetrisOracle(twin)


def _rz(yaw):
    c, s = math.cos(yaw), math.sin(yaw)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def build_geometry(problem, chain, grasp, static_centers=None, static_radii=None):
    if static_centers is None:
        static_centers = getattr(problem, "obstacle_centers", None)
        static_radii = getattr(problem, "obstacle_radii", None)
    sc = np.zeros((0, 3)) if static_centers is None else np.asarray(static_centers, float).reshape(-1, 3)
    sr = np.zeros(0) if static_radii is None else np.asarray(static_radii, float).reshape(-1)
    loc, rad, link = arm_table(chain)
    mask = link[:, None] >= np.arange(len(chain.joints))[None, :]
    g = SimpleNamespace(problem=problem, chain=chain, grasp=grasp, static_c=sc, static_r=sr, arm_local=loc,
                        arm_r=rad, arm_link=link, arm_mask=mask, manip=not _is_motion(problem))
    if not g.manip:
        g.B = 1
        g.fixed_c, g.fixed_r = [sc], [sr]
        return g
    if grasp is None:
        raise ValueError("manipulation problems need a grasp specification")
    if problem.initial_poses is None:
        raise ValueError("manipulation problems need staged initial poses")
    if _is_tower(problem):
        locs = [np.zeros((1, 3)) for _ in range(problem.n_blocks)]
        rads = [np.array([0.5 * problem.side]) for _ in range(problem.n_blocks)]
    else:
        locs = [b.sphere_set.centers.copy() for b in problem.blocks]
        rads = [b.sphere_set.radii.copy() for b in problem.blocks]
    B = len(locs)
    g.B = B
    g.block_u = [l - grasp.offset for l in locs]
    g.block_r = rads
    init_w = [l @ _rz(p.yaw).T + np.array([p.x, p.y, p.z]) for l, p in zip(locs, problem.initial_poses)]
    g.fixed_c = [np.concatenate([sc] + init_w[b + 1:]) for b in range(B)]
    g.fixed_r = [np.concatenate([sr] + rads[b + 1:]) for b in range(B)]
    tg = [grasp_target([p.x, p.y, p.z, p.yaw], grasp) for p in problem.initial_poses]
    g.pick_pos = np.array([t[0] for t in tg])
    g.pick_yaw = np.array([t[1] for t in tg])
    g.place = _free_twin_model(problem)
    g.anchor = problem.yaw_mode == "fixed"
    return g


@dataclass
class TrajConfig:
    k_waypoint: int = 1
    k_interp: int = 5
    w_start: float = 50.0
    w_arm: float = 1.0
    w_block: float = 1.0
    w_place: float = 1.0
    mu0: float = 10.0
    beta: float = 2.0
    outer_iters: int = 20
    inner_steps: int = 50
    lr_init: float = 0.05
    lr_final: float = 0.005
    validation_epsilon: float = 0.02


def _pen(diff, rsum, mode):
    d = np.sqrt(np.sum(diff * diff, axis=-1))
    pen = np.maximum(0.0, rsum - d)
    return d, pen, (pen * pen if mode == QUADRATIC else pen)


def _pen_back(diff, d, pen, mode, factor):
    live = (pen > 0.0) & (d > 0.0)
    slope = np.where(live, 1.0 / np.where(d > 0, d, 1.0), 0.0)
    if mode == QUADRATIC:
        slope = slope * 2.0 * pen
    return (-factor * slope)[..., None] * diff


def evaluate(values, g, cfg, mode, lam, mu, want_grad, place_mode=None):
    """trajopt.py:416-653 with an explicit place_mode (None -> variant B: same as mode)."""
    pmode = mode if place_mode is None else place_mode
    P, B, T, dof = values.shape
    f = fk(g.chain, values)
    ee, rot, axes, org = f.ee, f.rot, f.axes, f.origins
    S = len(g.arm_local)
    arm_w = (np.einsum("...sik,sk->...si", f.lrot[..., g.arm_link, :, :], g.arm_local) + f.lpos[..., g.arm_link, :]
             if S else np.zeros((P, B, T, 0, 3)))
    inner = slice(1, T - 1)
    if g.manip:
        rotF = rot @ FLIP
        held = [np.einsum("ptik,sk->ptsi", rotF[:, b, inner], g.block_u[b]) + ee[:, b, inner, None, :]
                for b in range(B)]
        eef, rotf = ee[:, :, -1], rot[:, :, -1]
        psi = yaw_of(rotf) - g.grasp.yaw_offset
        cp, sp = np.cos(psi), np.sin(psi)
        ox, oy, oz = g.grasp.offset
        pose = np.stack([eef[..., 0] - (cp * ox - sp * oy), eef[..., 1] - (sp * ox + cp * oy), eef[..., 2] - oz], -1)
        placed = []
        for b in range(B):
            u = g.block_u[b]
            placed.append(np.stack([eef[:, b, None, 0] + cp[:, b, None] * u[:, 0] - sp[:, b, None] * u[:, 1],
                                    eef[:, b, None, 1] + sp[:, b, None] * u[:, 0] + cp[:, b, None] * u[:, 1],
                                    eef[:, b, None, 2] + u[:, 2]], -1))
    leg = values[:, :, 1:] - values[:, :, :-1]
    legn = np.linalg.norm(leg, axis=-1)
    obj = legn.sum(axis=(1, 2))
    if g.manip:
        d0 = ee[:, :, 0] - g.pick_pos[None]
        ax0 = rot[:, :, 0, :, 2]
        cosd = np.clip(-ax0[..., 2], -1.0, 1.0)
        th = np.arccos(cosd)
        dy0 = wrap(yaw_of(rot[:, :, 0]) - g.pick_yaw[None])
        obj = obj + cfg.w_start * (np.sum(d0 * d0, axis=(1, 2)) + np.sum(th * th, 1) + np.sum(dy0 * dy0, 1))
    arm_terms, held_terms = [], []
    c_arm = np.zeros(P)
    c_blk = np.zeros(P)
    for b in range(B):
        fc, fr = g.fixed_c[b], g.fixed_r[b]
        if S and len(fc):
            diff = arm_w[:, b, :, :, None, :] - fc[None, None, None]
            d, pen, v = _pen(diff, g.arm_r[:, None] + fr[None], mode)
            c_arm += v.sum(axis=(1, 2, 3))
            arm_terms.append((b, None, diff, d, pen))
        if g.manip:
            for j in range(b):
                if S:
                    diff = arm_w[:, b, :, :, None, :] - placed[j][:, None, None]
                    d, pen, v = _pen(diff, g.arm_r[:, None] + g.block_r[j][None], mode)
                    c_arm += v.sum(axis=(1, 2, 3))
                    arm_terms.append((b, j, diff, d, pen))
            if len(fc):
                diff = held[b][:, :, :, None, :] - fc[None, None, None]
                d, pen, v = _pen(diff, g.block_r[b][:, None] + fr[None], mode)
                c_blk += v.sum(axis=(1, 2, 3))
                held_terms.append((b, None, diff, d, pen))
            for j in range(b):
                diff = held[b][:, :, :, None, :] - placed[j][:, None, None]
                d, pen, v = _pen(diff, g.block_r[b][:, None] + g.block_r[j][None], mode)
                c_blk += v.sum(axis=(1, 2, 3))
                held_terms.append((b, j, diff, d, pen))
    c_place = np.zeros(P)
    if g.manip:
        rows = np.concatenate([pose, psi[..., None]], -1).reshape(P, 4 * B)
        c_place = g.place.evaluate(rows, pmode)
        if g.anchor:
            wpsi = wrap(psi)
            c_place = c_place + np.sum(wpsi * wpsi if pmode == QUADRATIC else np.abs(wpsi), axis=1)
    cons = np.stack([cfg.w_place * c_place, cfg.w_arm * c_arm, cfg.w_block * c_blk], 1)
    lag = obj + np.sum(lam * cons, 1) + 0.5 * mu * np.sum(cons * cons, 1)
    if not want_grad:
        return obj, cons, lag, None
    scale = lam + mu[:, None] * cons
    s_pl, s_arm, s_blk = scale[:, 0] * cfg.w_place, scale[:, 1] * cfg.w_arm, scale[:, 2] * cfg.w_block
    grad = np.zeros_like(values)
    unit = np.where(legn[..., None] > 1e-12, leg / np.maximum(legn, 1e-12)[..., None], 0.0)
    grad[:, :, :-1] -= unit
    grad[:, :, 1:] += unit
    g3_arm = np.zeros_like(arm_w)
    if g.manip:
        g3_held = [np.zeros_like(h) for h in held]
        g3_pl = [np.zeros((P, len(u), 3)) for u in g.block_u]
    for b, j, diff, d, pen in arm_terms:
        ga = _pen_back(diff, d, pen, mode, s_arm[:, None, None, None])
        g3_arm[:, b] += ga.sum(axis=3)
        if j is not None:
            g3_pl[j] -= ga.sum(axis=(1, 2))
    if g.manip:
        for b, j, diff, d, pen in held_terms:
            ga = _pen_back(diff, d, pen, mode, s_blk[:, None, None, None])
            g3_held[b] += ga.sum(axis=3)
            if j is not None:
                g3_pl[j] -= ga.sum(axis=(1, 2))
    if S:
        rel = arm_w[..., :, None, :] - org[..., None, :, :]
        cr = np.cross(axes[..., None, :, :], rel) * g.arm_mask[None, None, None, :, :, None]
        grad += np.einsum("pbtsjd,pbtsd->pbtj", cr, g3_arm)
    if g.manip:
        for b in range(B):
            rel = held[b][:, :, :, None, :] - org[:, b, inner, None, :, :]
            cr = np.cross(axes[:, b, inner, None, :, :], rel)
            grad[:, b, inner] += np.einsum("ptsjd,ptsd->ptj", cr, g3_held[b])
        gpose = s_pl[:, None, None] * g.place.gradient(rows, pmode).reshape(P, B, 4)
        if g.anchor:
            wpsi = wrap(psi)
            gpose[:, :, 3] += s_pl[:, None] * (2.0 * wpsi if pmode == QUADRATIC else np.sign(wpsi))
        jlf = np.cross(axes[:, :, -1], eef[:, :, None, :] - org[:, :, -1])
        yjf = yaw_jac(rotf, axes[:, :, -1])
        for j in range(B):
            g3 = g3_pl[j]
            if not np.any(g3):
                continue
            u = g.block_u[j]
            drx = -sp[:, j, None] * u[:, 0] - cp[:, j, None] * u[:, 1]
            dry = cp[:, j, None] * u[:, 0] - sp[:, j, None] * u[:, 1]
            gy = np.sum(g3[..., 0] * drx + g3[..., 1] * dry, axis=1)
            grad[:, j, -1] += np.einsum("pd,pjd->pj", g3.sum(axis=1), jlf[:, j])
            grad[:, j, -1] += gy[:, None] * yjf[:, j]
        dox = sp * ox + cp * oy
        doy = -cp * ox + sp * oy
        gyp = gpose[..., 0] * dox + gpose[..., 1] * doy + gpose[..., 3]
        grad[:, :, -1] += np.einsum("pbd,pbjd->pbj", gpose[..., :3], jlf)
        grad[:, :, -1] += gyp[..., None] * yjf
        jl0 = np.cross(axes[:, :, 0], ee[:, :, 0, None, :] - org[:, :, 0])
        grad[:, :, 0] += cfg.w_start * 2.0 * np.einsum("pbd,pbjd->pbj", d0, jl0)
        sth = np.sqrt(np.maximum(1.0 - cosd * cosd, 0.0))
        fac = np.where(sth > 1e-8, -2.0 * th / np.maximum(sth, 1e-8), np.where(cosd > 0.0, -2.0, 0.0))
        dcos = -np.cross(axes[:, :, 0], ax0[:, :, None, :])[..., 2]
        grad[:, :, 0] += cfg.w_start * fac[..., None] * dcos
        grad[:, :, 0] += cfg.w_start * 2.0 * dy0[..., None] * yaw_jac(rot[:, :, 0], axes[:, :, 0])
    return obj, cons, lag, grad


# ---------------------------------------------------------------------------
# validation (trajopt.py:1071-1153)
# ---------------------------------------------------------------------------
def validate(segs, g, epsilon=0.02):
    segs = np.asarray(segs, float)
    B, T, _ = segs.shape
    lo, hi = chain_limits(g.chain)
    worst = 0.0
    placed_c, rows = [], []
    if g.manip:
        f = fk(g.chain, segs[:, -1])
        for b in range(B):
            eyaw = float(wrap(yaw_of(f.rot[b])))
            yaw = float(wrap(eyaw - g.grasp.yaw_offset))
            c, s = math.cos(yaw), math.sin(yaw)
            ox, oy, oz = g.grasp.offset
            px, py, pz = f.ee[b, 0] - (c * ox - s * oy), f.ee[b, 1] - (s * ox + c * oy), f.ee[b, 2] - oz
            placed_c.append((g.block_u[b] + g.grasp.offset) @ _rz(yaw).T + np.array([px, py, pz]))
            rows.append([px, py, pz, yaw])
    fa = fk(g.chain, segs)
    S = len(g.arm_local)
    arm = (np.einsum("btsik,sk->btsi", fa.lrot[:, :, g.arm_link], g.arm_local) + fa.lpos[:, :, g.arm_link]
           if S else np.zeros((B, T, 0, 3)))
    for b in range(B):
        oc = [g.fixed_c[b if g.manip else 0]] + [placed_c[j] for j in range(b)]
        orr = [g.fixed_r[b if g.manip else 0]] + [g.block_r[j] for j in range(b)]
        oc, orr = np.concatenate(oc), np.concatenate(orr)
        ex = np.maximum(segs[b] - hi, lo - segs[b])
        worst = max(worst, float(np.max(ex, initial=0.0)))
        if len(oc):
            if S:
                d = np.linalg.norm(arm[b][:, :, None, :] - oc[None, None], axis=-1)
                worst = max(worst, float(np.max((g.arm_r[None, :, None] + orr[None, None]) - d, initial=0.0)))
            if g.manip and T > 2:
                hw = np.einsum("tik,sk->tsi", fa.rot[b, 1:T - 1] @ FLIP, g.block_u[b]) + fa.ee[b, 1:T - 1, None]
                d = np.linalg.norm(hw[:, :, None, :] - oc[None, None], axis=-1)
                worst = max(worst, float(np.max((g.block_r[b][None, :, None] + orr[None, None]) - d, initial=0.0)))
        if g.manip:
            worst = max(worst, float(np.linalg.norm(fa.ee[b, 0] - g.pick_pos[b])))
            worst = max(worst, abs(float(wrap(wrap(yaw_of(fa.rot[b, 0])) - g.pick_yaw[b]))))
            worst = max(worst, math.acos(float(np.clip(-fa.rot[b, 0, 2, 2], -1.0, 1.0))))
    if g.manip:
        r = np.array(rows).reshape(1, 4 * B)
        place = float(g.place.evaluate(r, LINEAR)[0])
        if g.anchor:
            place += float(np.sum(np.abs(wrap(r[0, 3::4]))))
        worst = max(worst, place)
    else:
        worst = max(worst, float(np.max(np.abs(segs[0, 0] - g.problem.start), initial=0.0)))
        worst = max(worst, float(np.max(np.abs(segs[0, -1] - g.problem.goal), initial=0.0)))
    return bool(worst < epsilon), worst


# ---------------------------------------------------------------------------
# lifting, initialization, AL solve
# ---------------------------------------------------------------------------
class LiftFailure(RuntimeError):
    pass


class TrajOptFailure(RuntimeError):
    def __init__(self, best_violation, report):
        super().__init__(f"no feasible trajectory found (best violation {best_violation:.4g})")
        self.best_violation = best_violation
        self.report = report


def arm_worst_pen(chain, Q, g, centers, radii):
    f = fk(chain, Q)
    sph = np.einsum("nsik,sk->nsi", f.lrot[:, g.arm_link], g.arm_local) + f.lpos[:, g.arm_link]
    d = np.linalg.norm(sph[:, :, None, :] - centers[None, None], axis=-1)
    return ((g.arm_r[:, None] + radii[None]) - d).max(axis=(1, 2))


def lift_placements(problem, placements, chain, grasp, seed=0, static_centers=None, static_radii=None,
                    candidates=4):
    g = build_geometry(problem, chain, grasp)
    placements = np.atleast_2d(np.asarray(placements, float))
    P, B = placements.shape[0], g.B
    per = placements.shape[1] // B
    targets = [grasp_target([p.x, p.y, p.z, p.yaw], grasp) for p in problem.initial_poses]
    for row in placements:
        r = row.reshape(B, per)
        for b in range(B):
            yaw = float(wrap(r[b, 3])) if per == 4 else 0.0
            targets.append(grasp_target([r[b, 0], r[b, 1], r[b, 2], yaw], grasp))
    tpos = np.array([t[0] for t in targets])
    tyaw = np.array([t[1] for t in targets])
    sc = np.zeros((0, 3)) if static_centers is None else np.asarray(static_centers, float).reshape(-1, 3)
    sr = np.zeros(0) if static_radii is None else np.asarray(static_radii, float).reshape(-1)
    score = len(sc) > 0
    nt = len(targets)
    dof = len(chain.joints)
    sol_best = np.zeros((nt, dof))
    ok = np.zeros(nt, bool)
    best_pen = np.full(nt, np.inf)
    for a in range(max(1, int(candidates))):
        sol, succ, _ = ik_solve_batch(chain, tpos, tyaw, seed=seed + a * LIFT_DRAW_STRIDE)
        sol, pol = polish_tool_down(chain, sol, tpos, tyaw)
        dok = succ & pol
        pen = arm_worst_pen(chain, sol, g, sc, sr) if score else np.zeros(nt)
        better = dok & (~ok | (pen < best_pen))
        sol_best[better] = sol[better]
        best_pen[better] = pen[better]
        ok |= dok
        if not score and ok.all():
            break
    if not ok[:B].all():
        raise LiftFailure(f"staged pose {int(np.flatnonzero(~ok[:B])[0])} is not reachable tool-down")
    keep = np.flatnonzero(ok[B:].reshape(P, B).all(axis=1))
    if len(keep) == 0:
        raise LiftFailure("every particle contains an unreachable placement")
    ends = np.empty((len(keep), B, 2, dof))
    ends[:, :, 0] = sol_best[:B][None]
    ends[:, :, 1] = sol_best[B:].reshape(P, B, dof)[keep]
    return ends, keep


def trajectory_stream(seed):
    return np.random.default_rng(np.random.SeedSequence(entropy=seed, spawn_key=(TRAJ_STREAM,)))


def init_trajectories(endpoints, chain, cfg, rng):
    lo, hi = chain_limits(chain)
    P, B = endpoints.shape[:2]
    K, n = cfg.k_waypoint, cfg.k_interp
    nodes = np.empty((P, B, K + 2, len(lo)))
    nodes[:, :, 0] = endpoints[:, :, 0]
    nodes[:, :, -1] = endpoints[:, :, 1]
    if K:
        nodes[:, :, 1:-1] = rng.uniform(lo, hi, size=(P, B, K, len(lo)))
    T = n * (K + 1) + 1
    out = np.empty((P, B, T, len(lo)))
    for leg in range(K + 1):
        a = nodes[:, :, leg]
        d = nodes[:, :, leg + 1] - a
        for s in range(n):
            out[:, :, leg * n + s] = a + d * (s / n)
    out[:, :, -1] = nodes[:, :, -1]
    return out


@dataclass
class OuterRecord:
    index: int
    mu: np.ndarray
    multipliers: np.ndarray
    constraints: np.ndarray
    updated_multipliers: np.ndarray
    objective: np.ndarray
    feasible: np.ndarray
    violation: np.ndarray


@dataclass
class AlOutcome:
    values: np.ndarray
    objective: float
    particle_index: int
    outers: List[OuterRecord] = field(default_factory=list)


def solve_al(values, problem, chain, cfg, grasp=None, static_centers=None, static_radii=None, place_mode=None):
    g = build_geometry(problem, chain, grasp, static_centers, static_radii)
    x = np.array(values, float)
    P, B = x.shape[:2]
    lam = np.zeros((P, 3))
    mu = np.full(P, float(cfg.mu0))
    prev = np.full(P, np.inf)
    lo, hi = chain_limits(chain)
    denom = max(cfg.inner_steps - 1, 1)
    best_obj, best_p, best_x, least = math.inf, -1, None, math.inf
    outers = []
    if g.manip:
        pp = np.tile(g.pick_pos, (P, 1))
        py = np.tile(g.pick_yaw, P)
    for outer in range(cfg.outer_iters):
        for k in range(cfg.inner_steps):
            lr = cfg.lr_init + (cfg.lr_final - cfg.lr_init) * (k / denom)
            _, _, _, grad = evaluate(x, g, cfg, LINEAR, lam, mu, True, place_mode)
            x = np.clip(x - np.clip(lr * grad, -INNER_STEP_CLAMP, INNER_STEP_CLAMP), lo, hi)
            if not g.manip:
                x[:, 0, 0] = problem.start
                x[:, 0, -1] = problem.goal
        if g.manip:
            r, _ = polish_tool_down(chain, x[:, :, 0].reshape(P * B, -1), pp, py)
            x[:, :, 0] = r.reshape(P, B, -1)
        obj, cons, _, _ = evaluate(x, g, cfg, LINEAR, lam, mu, False, place_mode)
        upd = lam + mu[:, None] * cons
        feas = np.zeros(P, bool)
        viol = np.empty(P)
        for p in range(P):
            feas[p], viol[p] = validate(x[p], g, cfg.validation_epsilon)
        least = min(least, float(viol.min()))
        outers.append(OuterRecord(outer, mu.copy(), lam.copy(), cons.copy(), upd.copy(), obj.copy(), feas.copy(),
                                  viol.copy()))
        for p in np.flatnonzero(feas):
            if obj[p] < best_obj:
                best_obj, best_p, best_x = float(obj[p]), int(p), x[p].copy()
        if best_x is not None:
            break
        lam = upd
        v = cons.max(axis=1)
        mu = np.where(v > prev / 10.0, mu * cfg.beta, mu)
        prev = v
    if best_x is None:
        raise TrajOptFailure(least, outers)
    return AlOutcome(best_x, best_obj, best_p, outers)
