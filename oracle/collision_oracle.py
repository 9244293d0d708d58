"""CPU restatement of the reference's collision costs and generic LM -- TEST INFRASTRUCTURE ONLY.

Parity oracle for SURVEY.md section 8 rows a15-a19 (collision IK, config 4),
imported only by tests/ and bench.py's CPU legs.  Restates, in NumPy float64
vectorised over lanes:

* sphere / capsule / half-space distances + gradients  collision.py:115-237
* Eq. 1 activation and its derivative                   collision.py:245-269
* soft-minimum aggregation                              costs.py:409-420
* world / self collision rows and Jacobians             costs.py:423-551
* sphere tables from URDF + sidecar, default self pairs robot.py:174-190, 209-218, 355-361
* the generic classic-LM ``solve`` (rejection loop, termination criteria,
  dense Cholesky)                                       solver.py:289-429

Pinned against tests/golden/reference_golden.npz (world/self rows and
Jacobians, and reference ``solve`` runs) by tests/test_oracle.py.
"""

from __future__ import annotations

import json
import math
import xml.etree.ElementTree as ET
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

from . import ik_oracle as o

SOFTMIN_SHARPNESS = 100.0  # costs.py:44


# ---------------------------------------------------------------------------
# primitives and sphere tables
# ---------------------------------------------------------------------------

@dataclass
class Obstacle:
    kind: str  # sphere | capsule | halfspace
    a: np.ndarray = field(default_factory=lambda: np.zeros(3))  # center / endpoint a / normal
    b: np.ndarray = field(default_factory=lambda: np.zeros(3))  # endpoint b
    r: float = 0.0  # radius / half-space offset


def sphere(center, radius):
    return Obstacle("sphere", np.asarray(center, float), np.zeros(3), float(radius))


def capsule(a, b, radius):
    return Obstacle("capsule", np.asarray(a, float), np.asarray(b, float), float(radius))


def halfspace(normal, offset):
    n = np.asarray(normal, float)
    return Obstacle("halfspace", n / np.linalg.norm(n), np.zeros(3), float(offset))


@dataclass
class Spheres:
    """Collision spheres per link (links in model order) + default self pairs."""

    links: list            # link indices that carry spheres, model order
    centers: dict          # link -> (S, 3) local centers
    radii: dict            # link -> (S,)
    pairs: list            # self-collision (link_a, link_b) index pairs


def load_spheres(ch: o.Chain, urdf_text: str, sidecar: dict | None) -> Spheres:
    """robot.py:209-218 (URDF <collision><sphere>), :355-361 (sidecar override), :174-190 (pairs)."""
    root = ET.fromstring(urdf_text)
    table = {}
    for le in root.findall("link"):
        entries = []
        for coll in le.findall("collision"):
            sp = coll.find("geometry/sphere")
            if sp is None:
                continue
            org = coll.find("origin")
            c = np.fromstring(org.get("xyz", "0 0 0"), sep=" ") if org is not None else np.zeros(3)
            entries.append((c, float(sp.get("radius"))))
        if entries:
            table[le.get("name")] = entries
    for name, ents in ((sidecar or {}).get("collision_spheres") or {}).items():
        table[name] = [(np.asarray(e["center"], float), float(e["radius"])) for e in ents]
    links = [ch.link(nm) for nm in ch.links if table.get(nm)]
    centers = {ch.link(nm): np.array([c for c, _ in table[nm]]) for nm in table}
    radii = {ch.link(nm): np.array([r for _, r in table[nm]]) for nm in table}
    # default self pairs: all sphere links minus parent/child pairs and ignores (robot.py:174-190)
    adjacent = {frozenset((ch.links[p], ch.links[c])) for p, c in zip(ch.parent, ch.child)}
    ignored = {frozenset(p) for p in ((sidecar or {}).get("self_collision_ignore") or [])}
    named = [ch.links[l] for l in links]
    pairs = []
    for i, a in enumerate(named):
        for b in named[i + 1:]:
            if frozenset((a, b)) in adjacent or frozenset((a, b)) in ignored:
                continue
            pairs.append((ch.link(a), ch.link(b)))
    return Spheres(links, centers, radii, pairs)


def load_spheres_files(ch, urdf_path, sidecar_path=None) -> Spheres:
    with open(urdf_path) as f:
        text = f.read()
    side = None
    if sidecar_path:
        with open(sidecar_path) as f:
            side = json.load(f)
    return load_spheres(ch, text, side)


# ---------------------------------------------------------------------------
# distances (collision.py)
# ---------------------------------------------------------------------------

def _unit_or_zero(v):
    n = np.linalg.norm(v, axis=-1)
    small = n < 1e-12
    d = np.where(small[..., None], 0.0, v / np.where(small, 1.0, n)[..., None])
    return d, np.where(small, 0.0, n)


def _closest_param(a, b, p):
    """collision.py:115-121, vectorised over p (..., 3)."""
    d = b - a
    dd = float(d @ d)
    if dd < 1e-16:
        return np.zeros(p.shape[:-1])
    return np.clip((p - a) @ d / dd, 0.0, 1.0)


def sphere_obstacle(center, radius, ob: Obstacle):
    """collision.py:192-204: (d, d d / d center) for a sphere vs a static obstacle."""
    if ob.kind == "sphere":
        direction, n = _unit_or_zero(center - ob.a)
        return n - radius - ob.r, direction
    if ob.kind == "capsule":
        u = _closest_param(ob.a, ob.b, center)
        p = ob.a + u[..., None] * (ob.b - ob.a)
        direction, n = _unit_or_zero(center - p)
        return n - radius - ob.r, direction
    d = center @ ob.a - ob.r - radius
    return d, np.broadcast_to(ob.a, center.shape).copy()


def activation(d, eta):
    """collision.py:245-257 (Eq. 1)."""
    return np.where(d < 0.0, -d + 0.5 * eta, np.where(d < eta, (0.5 / eta) * (eta - d) ** 2, 0.0))


def activation_deriv(d, eta):
    """collision.py:260-269."""
    return np.where(d < 0.0, -1.0, np.where(d < eta, -(eta - d) / eta, 0.0))


def softmin(ds, sharpness=SOFTMIN_SHARPNESS, hard=False):
    """costs.py:409-420 over the last axis; returns (aggregate, weights)."""
    if hard or ds.shape[-1] == 1:
        k = np.argmin(ds, axis=-1)
        w = np.zeros(ds.shape)
        np.put_along_axis(w, k[..., None], 1.0, axis=-1)
        return np.take_along_axis(ds, k[..., None], axis=-1)[..., 0], w
    dmin = ds.min(axis=-1)
    z = np.exp(-sharpness * (ds - dmin[..., None]))
    s = z.sum(axis=-1)
    return dmin - np.log(s) / sharpness, z / s[..., None]


# ---------------------------------------------------------------------------
# collision rows (costs.py:423-551), vectorised over lanes
# ---------------------------------------------------------------------------

def _world_spheres(sp: Spheres, lq, lp, link):
    c = o.qrot(lq[:, link, None, :], sp.centers[link][None]) + lp[:, link, None, :]
    return c, sp.radii[link]


def world_rows(ch, sp: Spheres, obstacles, q, eta=0.05, sharpness=SOFTMIN_SHARPNESS, hard=False, jac=True):
    """world_collision_cost raw rows (B, P) and Jacobians (B, P, n); P = links x obstacles."""
    lq, lp, jp, ja = o.fk(ch, q)
    b = q.shape[0]
    pairs = [(l, oi) for l in sp.links for oi in range(len(obstacles))]
    rows = np.zeros((b, len(pairs)))
    J = np.zeros((b, len(pairs), ch.n)) if jac else None
    for p_idx, (link, oi) in enumerate(pairs):
        c, rad = _world_spheres(sp, lq, lp, link)
        ds, gs = sphere_obstacle(c, rad[None, :], obstacles[oi])
        d_agg, w = softmin(ds, sharpness, hard)
        rows[:, p_idx] = activation(d_agg, eta)
        if not jac:
            continue
        act_d = activation_deriv(d_agg, eta)
        row = np.zeros((b, ch.n))
        for k in range(c.shape[1]):
            pj = o.point_jacobian(ch, c[:, k], jp, ja, link, rotational=False)
            row += w[:, k, None] * np.einsum("bi,bij->bj", gs[:, k], pj)
        J[:, p_idx] = act_d[:, None] * row
    return rows, J


def self_rows(ch, sp: Spheres, q, eta=0.01, sharpness=SOFTMIN_SHARPNESS, hard=False, jac=True):
    """self_collision_cost raw rows (B, P) and Jacobians (B, P, n); P = default self pairs."""
    lq, lp, jp, ja = o.fk(ch, q)
    b = q.shape[0]
    rows = np.zeros((b, len(sp.pairs)))
    J = np.zeros((b, len(sp.pairs), ch.n)) if jac else None
    for p_idx, (la, lb) in enumerate(sp.pairs):
        ca, ra = _world_spheres(sp, lq, lp, la)
        cb, rb = _world_spheres(sp, lq, lp, lb)
        direction = ca[:, :, None, :] - cb[:, None, :, :]  # (B, Sa, Sb, 3)
        dist = np.linalg.norm(direction, axis=-1)
        ds = (dist - ra[None, :, None] - rb[None, None, :]).reshape(b, -1)
        dirs = np.where((dist > 1e-12)[..., None], direction / np.where(dist > 1e-12, dist, 1.0)[..., None], 0.0)
        dirs = dirs.reshape(b, -1, 3)
        d_agg, w = softmin(ds, sharpness, hard)
        rows[:, p_idx] = activation(d_agg, eta)
        if not jac:
            continue
        act_d = activation_deriv(d_agg, eta)
        row = np.zeros((b, ch.n))
        k = 0
        for i in range(ca.shape[1]):
            pja = o.point_jacobian(ch, ca[:, i], jp, ja, la, rotational=False)
            for j in range(cb.shape[1]):
                pjb = o.point_jacobian(ch, cb[:, j], jp, ja, lb, rotational=False)
                row += w[:, k, None] * np.einsum("bi,bij->bj", dirs[:, k], pja - pjb)
                k += 1
        J[:, p_idx] = act_d[:, None] * row
    return rows, J


# ---------------------------------------------------------------------------
# collision IK cost stack: [pose, limit, rest, world, self] with weights
# ---------------------------------------------------------------------------

@dataclass
class CollisionCosts:
    """CostWeights-driven stack used by the viewer (server.py:60-97) and config 4."""

    w_pos: float = 50.0
    w_ori: float = 10.0
    w_limit: float = 100.0
    w_rest: float = 0.01
    w_world: float = 20.0
    w_self: float = 5.0
    eta_world: float = 0.05
    eta_self: float = 0.01
    sharpness: float = SOFTMIN_SHARPNESS
    hard: bool = False


def stack_residual_jacobian(ch, sp, obstacles, link, tinv_q, tinv_t, q, cc: CollisionCosts, jac=True):
    """Weighted residual (B, M) and Jacobian (B, M, n) of the collision-IK stack."""
    eng = o.LaneEngine(ch, link, tinv_q, tinv_t, (cc.w_pos, cc.w_ori, cc.w_limit, cc.w_rest))
    if jac:
        r0, j0 = eng.residuals_and_jacobian(q)
    else:
        r0, j0 = eng.residuals(q), None
    parts_r, parts_j = [r0], [j0]
    if obstacles and cc.w_world > 0.0:
        wr, wj = world_rows(ch, sp, obstacles, q, cc.eta_world, cc.sharpness, cc.hard, jac)
        parts_r.append(cc.w_world * wr)
        parts_j.append(cc.w_world * wj if jac else None)
    if sp.pairs and cc.w_self > 0.0:
        sr, sj = self_rows(ch, sp, q, cc.eta_self, cc.sharpness, cc.hard, jac)
        parts_r.append(cc.w_self * sr)
        parts_j.append(cc.w_self * sj if jac else None)
    r = np.concatenate(parts_r, axis=1)
    return r, (np.concatenate(parts_j, axis=1) if jac else None)


def solve_lm(ch, sp, obstacles, link, tq, tt, q0, cc: CollisionCosts, **kw):
    """solver.py:364-429 for one collision-IK problem (dense Cholesky path, D <= 200)."""
    iq, it = o.target_inverse(np.atleast_2d(tq), np.atleast_2d(tt))

    def stack(q, jac):
        r, J = stack_residual_jacobian(ch, sp, obstacles, link, iq, it, q[None], cc, jac=jac)
        return r[0], (J[0] if jac else None)

    return lm(stack, q0, **kw)


def lm(stack, q0, max_iterations=100, damping0=1e-4, up=10.0, down=1.0 / 3.0, grad_tol=1e-8, step_tol=1e-10,
       max_rejections=20):
    """The classic LM of solver.py:364-429 over a residual/Jacobian callable
    stack(q, jac) -> (r, J); dense Cholesky (scipy cho_factor / cho_solve)."""
    q = np.asarray(q0, float).copy()
    n = q.size
    r, J = stack(q, True)
    cost = float(r @ r)
    hist = [cost]
    damping = damping0
    termination, iters = "max_iterations", 0
    for _ in range(max_iterations):
        h0 = J.T @ J
        grad = J.T @ r
        diag = np.maximum(np.diag(h0).copy(), o.DIAG_FLOOR)
        if np.max(np.abs(grad), initial=0.0) < grad_tol:
            termination = "gradient_converged"
            break
        accepted, step = False, None
        for _ in range(max_rejections):
            h = h0.copy()
            h[np.arange(n), np.arange(n)] += damping * diag
            try:
                c, low = scipy.linalg.cho_factor(h)
                delta = scipy.linalg.cho_solve((c, low), -grad)
            except scipy.linalg.LinAlgError:
                delta = None
            if delta is not None:
                qn = q + delta
                rn, _ = stack(qn, False)
                cn = float(rn @ rn)
                if cn < cost:
                    q, cost = qn, cn
                    damping = max(damping * down, o.LAMBDA_MIN)
                    accepted, step = True, delta
                    break
            damping *= up
            if damping > o.LAMBDA_MAX:
                break
        if not accepted:
            termination = "numerical_failure" if damping > o.LAMBDA_MAX else "step_converged"
            break
        iters += 1
        hist.append(cost)
        if np.max(np.abs(step), initial=0.0) < step_tol:
            termination = "step_converged"
            break
        r, J = stack(q, True)
    return q, cost, hist, iters, termination


class CollisionLaneEngine(o.LaneEngine):
    """IkLaneProblem (beam.py:71-240) with the collision rows appended (config 4)."""

    def __init__(self, ch, sp, obstacles, link, tinv_q, tinv_t, cc: CollisionCosts, group=None):
        super().__init__(ch, link, tinv_q, tinv_t, (cc.w_pos, cc.w_ori, cc.w_limit, cc.w_rest), group=group)
        self.sp, self.obstacles, self.cc = sp, obstacles, cc

    def residuals(self, q, kin=None, ba=None, bxy=None):
        return stack_residual_jacobian(self.ch, self.sp, self.obstacles, self.link, self.tq, self.tt, q, self.cc,
                                       jac=False)[0]

    def residuals_and_jacobian(self, q, ba=None, bxy=None):
        return stack_residual_jacobian(self.ch, self.sp, self.obstacles, self.link, self.tq, self.tt, q, self.cc)

    def start(self, q0):
        q0 = np.asarray(q0, dtype=float)
        r = self.residuals(q0)
        c = np.einsum("bm,bm->b", r, r)
        return o.Lanes(q0.copy(), np.full(q0.shape[0], o.LAMBDA0), c, [c.copy()])


def ik_beam_collision(ch, sp, obstacles, link, tq, tt, seeds, cc: CollisionCosts, **kw):
    """IK-Beam (tasks.py:119-161) over the collision stack."""
    return o.ik_beam(ch, link, tq, tt, seeds, engine=lambda q_, t_, group: CollisionLaneEngine(
        ch, sp, obstacles, link, q_, t_, cc, group=group), **kw)
