"""CPU restatement of the reference's trajectory optimisation -- TEST INFRASTRUCTURE ONLY.

Parity oracle for SURVEY.md section 8 rows a19/a20 and config 5, imported
only by tests/ and bench.py's CPU legs.  Restates in NumPy float64:

* capsule vs obstacle distance + endpoint gradients   collision.py:115-152, 207-237
* swept-capsule collision rows and Jacobians          costs.py:554-619
* velocity / smoothness / stencil / limit / rest rows costs.py:174-341
* the plan_trajectory cost set with its anchors       tasks.py:347-403
* solver.solve over it (dense normal equations)       solver.py:289-429
  (the reference switches to SuperLU above 200 tangent dimensions,
  solver.py:327-361 -- the same linear system, solved by LU)
* trajectory_signed_distances                         tasks.py:251-275

Pinned against reference plan_trajectory runs in
tests/golden/reference_golden.npz (traj_*) by tests/test_oracle.py.
"""

from __future__ import annotations

import xml.etree.ElementTree as ET
from dataclasses import dataclass

import numpy as np

from . import collision_oracle as co
from . import ik_oracle as o

ANCHOR_WEIGHT = 1e3  # tasks.py:37
ACCEL = np.array([-1.0, 16.0, -30.0, 16.0, -1.0]) / 12.0  # costs.py:295
JERK = np.array([-1.0, 2.0, 0.0, -2.0, 1.0]) / 2.0  # costs.py:296


def velocity_limits(ch: o.Chain, urdf_text: str) -> np.ndarray:
    """RobotModel.velocity_limits (robot.py:113-126): +inf where absent."""
    root = ET.fromstring(urdf_text)
    vel, mimic = {}, set()
    for je in root.findall("joint"):
        lim = je.find("limit")
        if lim is not None and lim.get("velocity") is not None:
            vel[je.get("name")] = float(lim.get("velocity"))
        if je.find("mimic") is not None:
            mimic.add(je.get("name"))
    out = np.full(ch.n, np.inf)
    for j, name in enumerate(ch.joint_names):
        if ch.qcol[j] >= 0 and name not in mimic and name in vel:
            out[ch.qcol[j]] = vel[name]
    return out


# ---------------------------------------------------------------------------
# capsule distances (collision.py:124-152, 207-237)
# ---------------------------------------------------------------------------

def _seg_seg(p1, q1, p2, q2):
    d1, d2, r = q1 - p1, q2 - p2, p1 - p2
    a, e, f = float(d1 @ d1), float(d2 @ d2), float(d2 @ r)
    if a < 1e-16 and e < 1e-16:
        return 0.0, 0.0
    if a < 1e-16:
        return 0.0, float(np.clip(f / e, 0.0, 1.0))
    c = float(d1 @ r)
    if e < 1e-16:
        return float(np.clip(-c / a, 0.0, 1.0)), 0.0
    b = float(d1 @ d2)
    den = a * e - b * b
    s = float(np.clip((b * f - c * e) / den, 0.0, 1.0)) if den > 1e-16 else 0.0
    t = (b * s + f) / e
    if t < 0.0:
        return float(np.clip(-c / a, 0.0, 1.0)), 0.0
    if t > 1.0:
        return float(np.clip((b - c) / a, 0.0, 1.0)), 1.0
    return s, t


def capsule_obstacle(c0, c1, radius, ob: co.Obstacle):
    """Capsule c0 -> c1 (radius) vs a static obstacle: (d, dd/dc0, dd/dc1), over (..., 3)."""
    c0 = np.asarray(c0, float)
    c1 = np.asarray(c1, float)
    radius = np.broadcast_to(np.asarray(radius, float), c0.shape[:-1])
    if ob.kind == "halfspace":
        da, db = c0 @ ob.a, c1 @ ob.a
        d = np.minimum(da, db) - ob.r - radius
        first = (da <= db)[..., None]
        return d, np.where(first, ob.a, 0.0), np.where(first, 0.0, ob.a)
    if ob.kind == "sphere":
        seg = c1 - c0
        dd = np.sum(seg * seg, axis=-1)
        u = np.where(dd < 1e-16, 0.0,
                     np.clip(np.sum((ob.a - c0) * seg, axis=-1) / np.where(dd < 1e-16, 1.0, dd), 0.0, 1.0))
        p = c0 + u[..., None] * seg
        direction, n = co._unit_or_zero(p - ob.a)
        return n - radius - ob.r, (1.0 - u)[..., None] * direction, u[..., None] * direction
    d = np.empty(c0.shape[:-1])
    ga = np.empty(c0.shape)
    gb = np.empty(c0.shape)
    for idx in np.ndindex(*c0.shape[:-1]):
        s, t = _seg_seg(c0[idx], c1[idx], ob.a, ob.b)
        p = c0[idx] + s * (c1[idx] - c0[idx])
        qp = ob.a + t * (ob.b - ob.a)
        direction, n = co._unit_or_zero(p - qp)
        d[idx] = n - radius[idx] - ob.r
        ga[idx] = (1.0 - s) * direction
        gb[idx] = s * direction
    return d, ga, gb


def swept_rows(ch, sp: co.Spheres, obstacles, q0, q1, eta=0.05, sharpness=co.SOFTMIN_SHARPNESS, hard=False,
               jac=True):
    """swept_collision_cost raw rows (B, P) and Jacobians wrt q0, q1 (B, P, n); costs.py:554-619."""
    lq0, lp0, jp0, ja0 = o.fk(ch, q0)
    lq1, lp1, jp1, ja1 = o.fk(ch, q1)
    b = q0.shape[0]
    pairs = [(l, oi) for l in sp.links for oi in range(len(obstacles))]
    rows = np.zeros((b, len(pairs)))
    J0 = np.zeros((b, len(pairs), ch.n)) if jac else None
    J1 = np.zeros((b, len(pairs), ch.n)) if jac else None
    for p_idx, (link, oi) in enumerate(pairs):
        c0, rad = co._world_spheres(sp, lq0, lp0, link)
        c1, _ = co._world_spheres(sp, lq1, lp1, link)
        ds, ga, gb = capsule_obstacle(c0, c1, np.broadcast_to(rad[None, :], c0.shape[:-1]), obstacles[oi])
        d_agg, w = co.softmin(ds, sharpness, hard)
        rows[:, p_idx] = co.activation(d_agg, eta)
        if not jac:
            continue
        act_d = co.activation_deriv(d_agg, eta)
        r0 = np.zeros((b, ch.n))
        r1 = np.zeros((b, ch.n))
        for k in range(c0.shape[1]):
            pj0 = o.point_jacobian(ch, c0[:, k], jp0, ja0, link, rotational=False)
            pj1 = o.point_jacobian(ch, c1[:, k], jp1, ja1, link, rotational=False)
            r0 += w[:, k, None] * np.einsum("bi,bij->bj", ga[:, k], pj0)
            r1 += w[:, k, None] * np.einsum("bi,bij->bj", gb[:, k], pj1)
        J0[:, p_idx] = act_d[:, None] * r0
        J1[:, p_idx] = act_d[:, None] * r1
    return rows, J0, J1


# ---------------------------------------------------------------------------
# the plan_trajectory problem (tasks.py:347-403)
# ---------------------------------------------------------------------------

@dataclass
class TrajCosts:
    """TrajRequest defaults: CostWeights(rest=0, world_collision=30) (tasks.py:196-198)."""

    timesteps: int = 20
    dt: float = 0.1
    w_anchor: float = ANCHOR_WEIGHT
    w_smooth: float = 10.0
    w_vel: float = 10.0
    w_acc: float = 1.0
    w_jerk: float = 0.1
    w_limit: float = 100.0
    w_rest: float = 0.0
    w_self: float = 5.0
    w_world: float = 30.0
    eta_world: float = 0.05
    eta_self: float = 0.01
    sharpness: float = co.SOFTMIN_SHARPNESS
    hard: bool = False


def traj_stack(ch, sp, obstacles, x, q_start, q_goal, tc: TrajCosts, vlim, rest=None, jac=True):
    """Weighted residual (M,) and dense Jacobian (M, T*n) of the trajectory problem."""
    T, n = tc.timesteps, ch.n
    qs = np.asarray(x, float).reshape(T, n)
    rest = ch.rest if rest is None else np.asarray(rest, float)
    N = T * n
    rows, jrows = [], []

    def add(r, blocks):
        """r (m,), blocks {timestep: (m, n)}"""
        rows.append(r)
        if jac:
            J = np.zeros((r.size, N))
            for t, blk in blocks.items():
                J[:, t * n:(t + 1) * n] += blk
            jrows.append(J)

    eye = np.eye(n)
    add(tc.w_anchor * (qs[0] - q_start), {0: tc.w_anchor * eye})
    add(tc.w_anchor * (qs[-1] - q_goal), {T - 1: tc.w_anchor * eye})
    budget = vlim * tc.dt
    for t in range(1, T):
        step = qs[t] - qs[t - 1]
        add(tc.w_smooth * step, {t - 1: -tc.w_smooth * eye, t: tc.w_smooth * eye})
        if tc.w_vel > 0:
            over = np.where(np.isfinite(budget), np.maximum(0.0, np.abs(step) - budget), 0.0)
            active = np.isfinite(budget) & (np.abs(step) > budget)
            g = np.where(active, np.sign(step), 0.0)
            add(tc.w_vel * over, {t - 1: -tc.w_vel * np.diag(g), t: tc.w_vel * np.diag(g)})
    for t in range(2, T - 2):
        for coeffs, scale, w in ((ACCEL, tc.dt * tc.dt, tc.w_acc), (JERK, tc.dt ** 3, tc.w_jerk)):
            if w <= 0:
                continue
            c = coeffs / scale
            r = sum(ck * qs[t - 2 + k] for k, ck in enumerate(c))
            add(w * r, {t - 2 + k: w * ck * eye for k, ck in enumerate(c)})
    lower, upper = ch.lower, ch.upper
    self_r = world_r = None
    if tc.w_self > 0 and sp.pairs:
        self_r = co.self_rows(ch, sp, qs, tc.eta_self, tc.sharpness, tc.hard, jac)
    if tc.w_world > 0 and obstacles:
        world_r = co.world_rows(ch, sp, obstacles, qs, tc.eta_world, tc.sharpness, tc.hard, jac)
    for t in range(T):
        q = qs[t]
        if tc.w_limit > 0:
            r = np.maximum(0.0, q - upper) + np.maximum(0.0, lower - q)
            g = np.where(q > upper, 1.0, 0.0) + np.where(q < lower, -1.0, 0.0)
            add(tc.w_limit * r, {t: tc.w_limit * np.diag(g)})
        if tc.w_rest > 0:
            add(tc.w_rest * (q - rest), {t: tc.w_rest * eye})
        if self_r is not None:
            add(tc.w_self * self_r[0][t], {t: tc.w_self * self_r[1][t]} if jac else {})
        if world_r is not None:
            add(tc.w_world * world_r[0][t], {t: tc.w_world * world_r[1][t]} if jac else {})
    if tc.w_world > 0 and obstacles:
        sw, j0, j1 = swept_rows(ch, sp, obstacles, qs[:-1], qs[1:], tc.eta_world, tc.sharpness, tc.hard, jac)
        for t in range(1, T):
            add(tc.w_world * sw[t - 1], {t - 1: tc.w_world * j0[t - 1], t: tc.w_world * j1[t - 1]} if jac else {})
    r = np.concatenate(rows)
    return r, (np.concatenate(jrows) if jac else None)


def solve_traj(ch, sp, obstacles, q_init, q_start, q_goal, tc: TrajCosts, vlim, rest=None, max_iterations=150,
               **kw):
    """solver.solve on the plan_trajectory problem (tasks.py:404): (qs, cost, hist, iters, termination)."""
    T, n = tc.timesteps, ch.n

    def stack(x, jac):
        return traj_stack(ch, sp, obstacles, x, q_start, q_goal, tc, vlim, rest, jac)

    x, cost, hist, iters, term = co.lm(stack, np.asarray(q_init, float).reshape(-1),
                                       max_iterations=max_iterations, **kw)
    return x.reshape(T, n), cost, hist, iters, term


def straight_line(q_start, q_goal, T):
    """tasks.py:344-345."""
    alphas = np.linspace(0.0, 1.0, T)
    return q_start[None, :] * (1 - alphas[:, None]) + q_goal[None, :] * alphas[:, None]


def signed_distances(ch, sp, obstacles, qs):
    """trajectory_signed_distances (tasks.py:251-275): (static (T,), swept (T-1,))."""
    qs = np.asarray(qs, float)
    T = qs.shape[0]
    static = np.full(T, np.inf)
    swept = np.full(max(T - 1, 0), np.inf)
    if not obstacles or not sp.links:
        return static, swept
    lq, lp, _, _ = o.fk(ch, qs)
    for link in sp.links:
        c, rad = co._world_spheres(sp, lq, lp, link)
        for ob in obstacles:
            d, _ = co.sphere_obstacle(c, rad[None, :], ob)
            static = np.minimum(static, d.min(axis=1))
            if T > 1:
                ds, _, _ = capsule_obstacle(c[:-1], c[1:], np.broadcast_to(rad[None, :], c[:-1].shape[:-1]), ob)
                swept = np.minimum(swept, ds.min(axis=1))
    return static, swept
