"""CPU restatement of the reference IK-Beam hot path -- TEST INFRASTRUCTURE ONLY.

This module is the parity ORACLE for the B200 build.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it, and only as the checker or the timed CPU
baseline.  The product package (``paper_2505_03728_b200``) never imports it;
there is no CPU fallback.

It restates, in plain NumPy at float64 (or any float dtype, for precision
experiments), the reference ``kinoptik`` code path named by BASELINE.json:

* URDF subset -> joint tables          ``robot.py:52-144``, ``robot.py:198-369``
* batched forward kinematics           ``robot.py:404-448``
* geometric point/link Jacobian        ``robot.py:486-506``
* quaternion / SO(3) / SE(3) kernels   ``liegroups.py:33-85``, ``:130-141``,
                                       ``:176-191``, ``:203-252``
* the lane-batched LM engine           ``beam.py:37-240``
* IK-Beam control flow                 ``tasks.py:88-161``
* reachable benchmark targets          ``benchmark.py:83-93``

Parity is PINNED: ``tests/test_oracle.py`` checks this module against the
golden vectors in ``tests/golden/`` that ``tests/golden/make_golden.py``
produced by importing the reference itself (read-only) in the build
container.
"""

from __future__ import annotations

import json
import math
import xml.etree.ElementTree as ET
from dataclasses import dataclass

import numpy as np

# beam.py:37-42
LAMBDA0, LAMBDA_UP, LAMBDA_DOWN = 1e-4, 10.0, 1.0 / 3.0
LAMBDA_MIN, LAMBDA_MAX, DIAG_FLOOR = 1e-12, 1e10, 1e-8
# liegroups.py:23
SERIES_BELOW = 1e-7
# benchmark.py:36
TARGET_KEY_BASE = 1 << 48

FIXED, REVOLUTE, PRISMATIC = 0, 1, 2


# ---------------------------------------------------------------------------
# quaternion / Lie-group kernels (liegroups.py)
# ---------------------------------------------------------------------------

def qmul(a, b):
    """Hamilton product, (w, x, y, z) -- liegroups.py:48-53."""
    aw, av = a[..., :1], a[..., 1:]
    bw, bv = b[..., :1], b[..., 1:]
    w = aw * bw - np.sum(av * bv, axis=-1, keepdims=True)
    v = aw * bv + bw * av + np.cross(av, bv)
    return np.concatenate([w, v], axis=-1)


def qconj(q):
    out = np.array(q, copy=True)
    out[..., 1:] *= -1.0
    return out


def qrot(q, p):
    """p + 2w(v x p) + v x (2 v x p) -- liegroups.py:62-67."""
    v, w = q[..., 1:], q[..., :1]
    t = 2.0 * np.cross(v, p)
    return p + w * t + np.cross(v, t)


def qmat(q):
    """Rotation matrix of a unit quaternion -- liegroups.py:70-85."""
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    m = np.empty(q.shape[:-1] + (3, 3), dtype=q.dtype)
    m[..., 0, 0] = 1.0 - 2.0 * (y * y + z * z)
    m[..., 0, 1] = 2.0 * (x * y - w * z)
    m[..., 0, 2] = 2.0 * (x * z + w * y)
    m[..., 1, 0] = 2.0 * (x * y + w * z)
    m[..., 1, 1] = 1.0 - 2.0 * (x * x + z * z)
    m[..., 1, 2] = 2.0 * (y * z - w * x)
    m[..., 2, 0] = 2.0 * (x * z - w * y)
    m[..., 2, 1] = 2.0 * (y * z + w * x)
    m[..., 2, 2] = 1.0 - 2.0 * (x * x + y * y)
    return m


def qcanon(q):
    """Unit-normalise, w >= 0 (lead vector component at w == 0) -- liegroups.py:33-45."""
    q = np.asarray(q, dtype=float)
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    sign = np.where(q[..., :1] < 0.0, -1.0, 1.0)
    at_zero = q[..., 0] == 0.0
    if np.any(at_zero):
        v = q[..., 1:]
        lead = np.take_along_axis(v, np.argmax(np.abs(v), axis=-1)[..., None], axis=-1)
        sign = np.where(at_zero[..., None], np.where(lead < 0.0, -1.0, 1.0), sign)
    return q * sign


def qexp(omega):
    """so(3) exp -> canonical quaternion -- liegroups.py:115-127."""
    omega = np.asarray(omega, dtype=float)
    th = np.linalg.norm(omega, axis=-1, keepdims=True)
    k = np.where(th < SERIES_BELOW, 0.5 - th * th / 48.0,
                 np.sin(0.5 * th) / np.where(th == 0.0, 1.0, th))
    return qcanon(np.concatenate([np.cos(0.5 * th), k * omega], axis=-1))


def qlog(q):
    """so(3) log, angle in [0, pi] -- liegroups.py:130-141."""
    q = q * np.where(q[..., :1] < 0.0, -1.0, 1.0).astype(q.dtype)  # dtype-preserving (float32 runs)
    w, v = q[..., :1], q[..., 1:]
    s = np.linalg.norm(v, axis=-1, keepdims=True)
    ang = 2.0 * np.arctan2(s, w)
    scale = np.where(s < SERIES_BELOW, 2.0 / np.maximum(w, 0.5) * (1.0 - s * s / 3.0),
                     ang / np.where(s == 0.0, 1.0, s))
    return scale * v


def hat(v):
    out = np.zeros(v.shape[:-1] + (3, 3), dtype=v.dtype)
    out[..., 0, 1], out[..., 0, 2] = -v[..., 2], v[..., 1]
    out[..., 1, 0], out[..., 1, 2] = v[..., 2], -v[..., 0]
    out[..., 2, 0], out[..., 2, 1] = -v[..., 1], v[..., 0]
    return out


def so3_jl_inv(omega):
    """Inverse SO(3) left Jacobian -- liegroups.py:176-191."""
    th = np.linalg.norm(omega, axis=-1)[..., None, None]
    k = hat(omega)
    half = np.where(th == 0.0, 1.0, 0.5 * th)
    b = np.where(th < SERIES_BELOW, 1.0 / 12.0 + th * th / 720.0,
                 (1.0 - half * np.cos(half) / np.sin(half)) / np.where(th == 0.0, 1.0, th * th))
    return np.eye(3, dtype=omega.dtype) - 0.5 * k + b * (k @ k)


def se3_log(q, t):
    """Translation-first twist of (q, t) -- liegroups.py:203-207."""
    om = qlog(q)
    v = (so3_jl_inv(om) @ t[..., None])[..., 0]
    return np.concatenate([v, om], axis=-1)


def _q_block(rho, phi):
    """Barfoot's Q coupling block -- liegroups.py:210-235.

    The small-angle branch keeps the reference's coefficients verbatim
    (including the sign slip of its c2/c3 series, harmless below 1e-7 rad in
    float64 because those terms scale with theta^2); the oracle must reproduce
    the reference, not the textbook.
    """
    th = np.linalg.norm(phi, axis=-1)[..., None, None]
    p, f = hat(rho), hat(phi)
    fp, pf = f @ p, p @ f
    fpf = fp @ f
    small = th < SERIES_BELOW
    t2 = th * th
    s = np.where(small, 1.0, th)
    s2 = s * s
    s3, s4, s5 = s * s2, s2 * s2, s * s2 * s2
    sn, cs = np.sin(s), np.cos(s)
    c1 = np.where(small, 1.0 / 6.0 - t2 / 120.0, (s - sn) / s3)
    c2 = np.where(small, 1.0 / 24.0 - t2 / 720.0, (1.0 - 0.5 * s2 - cs) / s4)
    c3 = 0.5 * np.where(small, c2 + 3.0 * (1.0 / 120.0 - t2 / 5040.0),
                        c2 - 3.0 * (s - sn - s3 / 6.0) / s5)
    return 0.5 * p + c1 * (fp + pf + fpf) - c2 * (f @ fp + pf @ f - 3.0 * fpf) - c3 * (fpf @ f + f @ fpf)


def se3_jr_inv(xi):
    """Jr^-1(xi) = Jl^-1(-xi) = [[A, -A Q A], [0, A]] -- liegroups.py:238-252."""
    xi = -xi
    rho, phi = xi[..., :3], xi[..., 3:]
    a = so3_jl_inv(phi)
    out = np.zeros(xi.shape[:-1] + (6, 6), dtype=xi.dtype)
    out[..., :3, :3] = a
    out[..., 3:, 3:] = a
    out[..., :3, 3:] = -a @ _q_block(rho, phi) @ a
    return out


def se3_adjoint(q, t):
    """Adjoint on translation-first twists -- liegroups.py:255-262."""
    r = qmat(q)
    out = np.zeros(r.shape[:-2] + (6, 6), dtype=r.dtype)
    out[..., :3, :3] = r
    out[..., 3:, 3:] = r
    out[..., :3, 3:] = hat(t) @ r
    return out


def wrap_angle(a):
    """(-pi, pi] -- liegroups.py:270-273."""
    w = np.mod(np.asarray(a, dtype=float) + math.pi, 2.0 * math.pi) - math.pi
    return np.where(w == -math.pi, math.pi, w)


def se2_exp(delta):
    """se(2) (vx, vy, w) -> (angle, translation) -- liegroups.py:276-287."""
    v, w = delta[..., :2], delta[..., 2]
    small = np.abs(w) < SERIES_BELOW
    safe = np.where(w == 0.0, 1.0, w)
    w2 = w * w
    s = np.where(small, 1.0 - w2 / 6.0, np.sin(safe) / safe)
    c = np.where(small, 0.5 * w - w * w2 / 24.0, (1.0 - np.cos(safe)) / safe)
    return wrap_angle(w), np.stack([s * v[..., 0] - c * v[..., 1], c * v[..., 0] + s * v[..., 1]], axis=-1)


def rot2(a):
    c, s = np.cos(a), np.sin(a)
    out = np.empty(np.shape(a) + (2, 2))
    out[..., 0, 0], out[..., 0, 1], out[..., 1, 0], out[..., 1, 1] = c, -s, s, c
    return out


SE2_EMBED = np.zeros((6, 3))  # costs.py:88-92
SE2_EMBED[0, 0] = SE2_EMBED[1, 1] = SE2_EMBED[5, 2] = 1.0


# ---------------------------------------------------------------------------
# robot tables (robot.py)
# ---------------------------------------------------------------------------

@dataclass
class Chain:
    """Joint tables of a parsed URDF, topological (BFS) order -- robot.py:74-144."""

    links: list
    joint_names: list
    parent: np.ndarray
    child: np.ndarray
    oq: np.ndarray
    op: np.ndarray
    axis: np.ndarray
    kind: np.ndarray
    qcol: np.ndarray
    mult: np.ndarray
    offset: np.ndarray
    ancestors: np.ndarray
    lower: np.ndarray
    upper: np.ndarray
    rest: np.ndarray

    @property
    def n(self):
        return self.lower.size

    def link(self, name):
        return self.links.index(name)


def _rpy_quat(rpy):
    """URDF rpy -> Rz(y) * Ry(p) * Rx(r), each factor canonicalised -- robot.py:198-206."""
    r = qexp(np.array([rpy[0], 0.0, 0.0]))
    p = qexp(np.array([0.0, rpy[1], 0.0]))
    y = qexp(np.array([0.0, 0.0, rpy[2]]))
    return qcanon(qmul(qcanon(qmul(y, p)), r))


def load_chain(urdf_text: str, sidecar: dict | None = None) -> Chain:
    """Subset URDF parse restating robot.py:221-369 (validation errors omitted)."""
    root = ET.fromstring(urdf_text)
    link_names = [e.get("name") for e in root.findall("link")]
    raw = []
    for je in root.findall("joint"):
        kind = je.get("type")
        ax_el = je.find("axis")
        axis = np.fromstring(ax_el.get("xyz"), sep=" ") if ax_el is not None else np.array([1.0, 0, 0])
        if kind != "fixed":
            axis = axis / np.linalg.norm(axis)
        org = je.find("origin")
        xyz = np.fromstring(org.get("xyz", "0 0 0"), sep=" ") if org is not None else np.zeros(3)
        rpy = np.fromstring(org.get("rpy", "0 0 0"), sep=" ") if org is not None else np.zeros(3)
        lim = je.find("limit")
        limits = None
        if lim is not None and lim.get("lower") is not None and lim.get("upper") is not None:
            limits = (float(lim.get("lower")), float(lim.get("upper")))
        if kind == "continuous":
            limits = None
        mim = je.find("mimic")
        mimic = None
        if mim is not None:
            mimic = (mim.get("joint"), float(mim.get("multiplier", "1")), float(mim.get("offset", "0")))
        raw.append(dict(name=je.get("name"), kind=kind, parent=je.find("parent").get("link"),
                        child=je.find("child").get("link"), xyz=xyz, rpy=rpy, axis=axis,
                        limits=limits, mimic=mimic))
    children = {}
    for j in raw:
        children.setdefault(j["parent"], []).append(j)
    has_parent = {j["child"] for j in raw}
    root_link = [l for l in link_names if l not in has_parent][0]
    order, links, queue = [], [root_link], [root_link]
    while queue:
        for j in children.get(queue.pop(0), []):
            order.append(j)
            links.append(j["child"])
            queue.append(j["child"])
    actuated = [j["name"] for j in order if j["kind"] != "fixed" and j["mimic"] is None]
    col = {nm: i for i, nm in enumerate(actuated)}
    nj, nl = len(order), len(links)
    kind_code = {"fixed": FIXED, "revolute": REVOLUTE, "continuous": REVOLUTE, "prismatic": PRISMATIC}
    ch = Chain(links=links, joint_names=[j["name"] for j in order],
               parent=np.array([links.index(j["parent"]) for j in order], dtype=int),
               child=np.array([links.index(j["child"]) for j in order], dtype=int),
               oq=np.stack([_rpy_quat(j["rpy"]) for j in order]) if nj else np.zeros((0, 4)),
               op=np.stack([j["xyz"] for j in order]) if nj else np.zeros((0, 3)),
               axis=np.stack([j["axis"] for j in order]) if nj else np.zeros((0, 3)),
               kind=np.array([kind_code[j["kind"]] for j in order], dtype=int),
               qcol=np.full(nj, -1, dtype=int), mult=np.ones(nj), offset=np.zeros(nj),
               ancestors=np.zeros((nl, nj), dtype=bool),
               lower=np.full(len(actuated), -np.inf), upper=np.full(len(actuated), np.inf),
               rest=np.zeros(len(actuated)))
    for i, j in enumerate(order):
        if j["kind"] == "fixed":
            continue
        if j["mimic"] is not None:
            ch.qcol[i], ch.mult[i], ch.offset[i] = col[j["mimic"][0]], j["mimic"][1], j["mimic"][2]
        else:
            ch.qcol[i] = col[j["name"]]
            if j["limits"] is not None:
                ch.lower[col[j["name"]]], ch.upper[col[j["name"]]] = j["limits"]
    parent_joint = np.full(nl, -1, dtype=int)
    for i in range(nj):
        parent_joint[ch.child[i]] = i
    for l in range(nl):
        i = parent_joint[l]
        while i >= 0:
            ch.ancestors[l, i] = True
            i = parent_joint[ch.parent[i]]
    if sidecar and sidecar.get("rest_pose") is not None:
        ch.rest = np.asarray(sidecar["rest_pose"], dtype=float).reshape(-1)
    else:
        fin = np.isfinite(ch.lower) & np.isfinite(ch.upper)
        ch.rest = np.where(fin, 0.5 * (np.where(fin, ch.lower, 0) + np.where(fin, ch.upper, 0)), 0.0)
    return ch


def load_chain_files(urdf_path, sidecar_path=None) -> Chain:
    with open(urdf_path) as f:
        text = f.read()
    side = None
    if sidecar_path is not None:
        with open(sidecar_path) as f:
            side = json.load(f)
    return load_chain(text, side)


def fk(ch: Chain, q):
    """Batched FK -> (link quat, link pos, joint anchor, joint world axis) -- robot.py:404-448."""
    q = np.asarray(q)
    dt = q.dtype
    lead = q.shape[:-1]
    nl, nj = len(ch.links), len(ch.kind)
    lq = np.empty(lead + (nl, 4), dtype=dt)
    lp = np.empty(lead + (nl, 3), dtype=dt)
    jp = np.empty(lead + (nj, 3), dtype=dt)
    ja = np.empty(lead + (nj, 3), dtype=dt)
    lq[..., 0, :] = np.array([1.0, 0.0, 0.0, 0.0], dtype=dt)
    lp[..., 0, :] = 0.0
    oq, op, ax = ch.oq.astype(dt), ch.op.astype(dt), ch.axis.astype(dt)
    for j in range(nj):
        pq, pp = lq[..., ch.parent[j], :], lp[..., ch.parent[j], :]
        fq = qmul(pq, oq[j])
        fpos = pp + qrot(pq, op[j])
        jp[..., j, :] = fpos
        ja[..., j, :] = qrot(fq, ax[j])
        c = ch.child[j]
        if ch.kind[j] == FIXED:
            lq[..., c, :], lp[..., c, :] = fq, fpos
            continue
        th = q[..., ch.qcol[j]] * dt.type(ch.mult[j]) + dt.type(ch.offset[j])
        if ch.kind[j] == REVOLUTE:
            mot = np.empty(lead + (4,), dtype=dt)
            mot[..., 0] = np.cos(0.5 * th)
            mot[..., 1:] = np.sin(0.5 * th)[..., None] * ax[j]
            lq[..., c, :], lp[..., c, :] = qmul(fq, mot), fpos
        else:
            lq[..., c, :], lp[..., c, :] = fq, fpos + th[..., None] * ja[..., j, :]
    return lq, lp, jp, ja


def point_jacobian(ch: Chain, point, jp, ja, link, rotational=True):
    """Geometric Jacobian over the ancestor joints, mimic folded -- robot.py:486-506."""
    rows = 6 if rotational else 3
    jac = np.zeros(jp.shape[:-2] + (rows, ch.n), dtype=jp.dtype)
    for j in range(len(ch.kind)):
        if not ch.ancestors[link, j] or ch.kind[j] == FIXED:
            continue
        c, m = ch.qcol[j], jp.dtype.type(ch.mult[j])
        if ch.kind[j] == REVOLUTE:
            jac[..., :3, c] += m * np.cross(ja[..., j, :], point - jp[..., j, :])
            if rotational:
                jac[..., 3:, c] += m * ja[..., j, :]
        else:
            jac[..., :3, c] += m * ja[..., j, :]
    return jac


# ---------------------------------------------------------------------------
# lane engine (beam.py) -- per-lane targets so many targets batch together
# ---------------------------------------------------------------------------

@dataclass
class Lanes:
    """beam.py:45-68 LaneState; ``ba``/``bxy`` = base angle / xy (None: fixed base)."""

    q: np.ndarray
    lam: np.ndarray
    cost: np.ndarray
    hist: list
    ba: np.ndarray | None = None
    bxy: np.ndarray | None = None

    def take(self, idx):
        return Lanes(self.q[idx].copy(), self.lam[idx].copy(), self.cost[idx].copy(),
                     [h[idx].copy() for h in self.hist], None if self.ba is None else self.ba[idx].copy(),
                     None if self.bxy is None else self.bxy[idx].copy())


class LaneEngine:
    """IkLaneProblem restated (beam.py:71-240) with one target per lane.

    ``tinv_q``/``tinv_t`` hold target^-1 per lane (beam.py:89-91).  Lanes of
    different targets never interact except through the batched solve's
    all-lanes LinAlgError escalation (beam.py:209-213), which this restatement
    applies per target group (``group`` ids) exactly as the reference would
    when it solves one target at a time.
    """

    def __init__(self, ch: Chain, link: int, tinv_q, tinv_t, weights, group=None, dtype=np.float64,
                 use_base=False, base_weight=0.0):
        self.ch, self.link, self.dt = ch, link, np.dtype(dtype)
        self.tq = np.asarray(tinv_q, dtype=self.dt)
        self.tt = np.asarray(tinv_t, dtype=self.dt)
        wp, wo, wl, wr = weights
        n = ch.n
        rows = [np.full(3, wp), np.full(3, wo), np.full(n, wl), np.full(n, wr)]
        if use_base:
            rows.append(np.full(3, base_weight))
        self.w = np.concatenate(rows).astype(self.dt)
        self.lo, self.hi = ch.lower.astype(self.dt), ch.upper.astype(self.dt)
        self.rest = ch.rest.astype(self.dt)
        self.group = group
        self.use_base = use_base
        self.dim = n + (3 if use_base else 0)

    def _compose(self, fq, fp, ba, bxy):
        """beam.py:104-112."""
        if not self.use_base:
            return fq, fp
        bq = np.zeros(ba.shape + (4,))
        bq[..., 0], bq[..., 3] = np.cos(0.5 * ba), np.sin(0.5 * ba)
        bp = np.concatenate([bxy, np.zeros(ba.shape + (1,))], axis=-1)
        return qmul(bq, fq), qrot(bq, fp) + bp

    def _pose(self, lq, lp, ba=None, bxy=None):
        fq, fpos = lq[..., self.link, :], lp[..., self.link, :]
        cq, cp = self._compose(fq, fpos, ba, bxy)
        eq = qmul(self.tq, cq)
        et = self.tt + qrot(self.tq, cp)
        return se3_log(eq, et), fq, fpos

    def residuals(self, q, kin=None, ba=None, bxy=None):
        """beam.py:114-131."""
        lq, lp, _, _ = kin if kin is not None else fk(self.ch, q)
        pose, _, _ = self._pose(lq, lp, ba, bxy)
        lim = np.maximum(0.0, q - self.hi) + np.maximum(0.0, self.lo - q)
        parts = [pose, lim, q - self.rest]
        if self.use_base:
            parts.append(np.concatenate([bxy, ba[..., None]], axis=-1))
        return np.concatenate(parts, axis=-1) * self.w

    def residuals_and_jacobian(self, q, ba=None, bxy=None):
        """beam.py:133-180."""
        kin = fk(self.ch, q)
        lq, lp, jp, ja = kin
        r = self.residuals(q, kin, ba, bxy)
        n = self.ch.n
        pose, fq, fpos = self._pose(lq, lp, ba, bxy)
        jg = point_jacobian(self.ch, fpos, jp, ja, self.link)
        rt = np.swapaxes(qmat(fq), -1, -2)
        body = np.concatenate([rt @ jg[..., :3, :], rt @ jg[..., 3:, :]], axis=-2)
        jri = se3_jr_inv(pose)
        jac = np.zeros(q.shape[:-1] + (self.w.size, self.dim), dtype=self.dt)
        jac[..., :6, :n] = jri @ body
        i = np.arange(n)
        jac[..., 6 + i, i] = np.where(q > self.hi, 1.0, 0.0) + np.where(q < self.lo, -1.0, 0.0)
        jac[..., 6 + n + i, i] = 1.0
        if self.use_base:
            iq = qconj(fq)
            jac[..., :6, n:] = jri @ se3_adjoint(iq, -qrot(iq, fpos)) @ SE2_EMBED
            rb = 6 + 2 * n
            ca, sa = np.cos(ba), np.sin(ba)
            jac[..., rb, n], jac[..., rb, n + 1] = ca, -sa
            jac[..., rb + 1, n], jac[..., rb + 1, n + 1] = sa, ca
            jac[..., rb + 2, n + 2] = 1.0
        return r, jac * self.w[:, None]

    def start(self, q0) -> Lanes:
        """beam.py:182-196."""
        q0 = np.asarray(q0, dtype=self.dt)
        b = q0.shape[0]
        ba = np.zeros(b) if self.use_base else None
        bxy = np.zeros((b, 2)) if self.use_base else None
        r = self.residuals(q0, None, ba, bxy)
        c = np.einsum("bm,bm->b", r, r)
        return Lanes(q0.copy(), np.full(b, LAMBDA0, dtype=self.dt), c, [c.copy()], ba, bxy)

    def _solve(self, h, g):
        try:
            return -np.linalg.solve(h, g[..., None])[..., 0], np.ones(h.shape[0], dtype=bool)
        except np.linalg.LinAlgError:
            pass
        # the reference solves one target at a time: a singular lane escalates
        # every lane of ITS target only (beam.py:209-213)
        ok = np.ones(h.shape[0], dtype=bool)
        out = np.zeros(g.shape, dtype=g.dtype)
        groups = self.group if self.group is not None else np.zeros(h.shape[0], dtype=int)
        for gid in np.unique(groups):
            sel = groups == gid
            try:
                out[sel] = -np.linalg.solve(h[sel], g[sel][..., None])[..., 0]
            except np.linalg.LinAlgError:
                ok[sel] = False
        return out, ok

    def run(self, st: Lanes, steps: int) -> Lanes:
        """beam.py:198-240: one proposal per step, per-lane accept and damping."""
        n = self.ch.n
        for _ in range(steps):
            r, jac = self.residuals_and_jacobian(st.q, st.ba, st.bxy)
            jtj = np.einsum("bmi,bmj->bij", jac, jac)
            g = np.einsum("bmi,bm->bi", jac, r)
            d = np.maximum(np.einsum("bii->bi", jtj), self.dt.type(DIAG_FLOOR))
            h = jtj + st.lam[:, None, None] * d[:, :, None] * np.eye(self.dim, dtype=self.dt)
            delta, ok = self._solve(h, g)
            qn = st.q + delta[:, :n]
            ban = bxyn = None
            if self.use_base:
                ang, xy = se2_exp(delta[:, n:])
                ban = wrap_angle(st.ba + ang)
                bxyn = st.bxy + (rot2(st.ba) @ xy[..., None])[..., 0]
            rn = self.residuals(qn, None, ban, bxyn)
            cn = np.einsum("bm,bm->b", rn, rn)
            cn = np.where(np.isfinite(cn), cn, np.inf)
            acc = (cn < st.cost) & ok
            st.q = np.where(acc[:, None], qn, st.q)
            if self.use_base:
                st.ba = np.where(acc, ban, st.ba)
                st.bxy = np.where(acc[:, None], bxyn, st.bxy)
            st.cost = np.where(acc, cn, st.cost)
            st.lam = np.where(acc, np.maximum(st.lam * LAMBDA_DOWN, LAMBDA_MIN),
                              np.minimum(st.lam * LAMBDA_UP, LAMBDA_MAX)).astype(self.dt)
            st.hist.append(st.cost.copy())
        return st


class CholeskyLaneEngine(LaneEngine):
    """The lane engine with the damped normal equations solved by a per-lane
    Cholesky factorisation in the ENGINE's dtype (float32 for the FP32 parity
    bar), the way the device solves them.  The reference solves the same SPD
    system with LU (``np.linalg.solve``, beam.py:207-208); for SPD systems the
    two agree to rounding.  A lane whose pivot is not positive is rejected
    (damping x10) -- in FP64 unreachable for finite inputs, since the damping
    term keeps the system SPD."""

    def _solve(self, h, g):
        n = h.shape[-1]
        dt = h.dtype
        lo = np.zeros_like(h)
        ok = np.ones(h.shape[0], dtype=bool)
        for j in range(n):
            s = h[:, j, j] - np.sum(lo[:, j, :j] * lo[:, j, :j], axis=-1)
            ok &= s > 0
            d = np.sqrt(np.where(s > 0, s, dt.type(1))).astype(dt)
            lo[:, j, j] = d
            for i in range(j + 1, n):
                lo[:, i, j] = (h[:, i, j] - np.sum(lo[:, i, :j] * lo[:, j, :j], axis=-1)) / d
        y = np.zeros_like(g)
        for i in range(n):
            y[:, i] = (g[:, i] - np.sum(lo[:, i, :i] * y[:, :i], axis=-1)) / lo[:, i, i]
        x = np.zeros_like(g)
        for i in reversed(range(n)):
            x[:, i] = (y[:, i] - np.sum(lo[:, i + 1:, i] * x[:, i + 1:], axis=-1)) / lo[:, i, i]
        return -x, ok


def cholesky_engine(ch: Chain, link: int, weights=None, dtype=np.float32, **kw):
    """``engine=`` factory for ik_beam: CholeskyLaneEngine lanes in ``dtype``."""
    w = DEFAULT_WEIGHTS if weights is None else weights
    return lambda q_, t_, group: CholeskyLaneEngine(ch, link, q_, t_, w, group=group, dtype=dtype, **kw)


def explain_divergence(h_dev, h_ref, diag, tol=1e-6):
    """For every target whose device winner history leaves ``tol`` (relative) of the
    oracle's, say why: the device's winning seed is identified by its start cost
    (``diag['s1_start']``), then
      * same seed          -> an accept / reject near-tie inside the lane: the relative
                              cost change the oracle made at the first step whose
                              decision differs ("accept_gap");
      * different survivor -> the final argmin (tasks.py:139): the relative gap of the
                              two survivors' final oracle costs ("winner_gap");
      * seed not kept      -> the stable top-keep prune (tasks.py:135): the relative gap
                              between the device seed's stage-1 cost and the oracle's
                              keep-th survivor ("prune_gap").
    Returns a list of (target, kind, first divergent step, gap)."""
    h_dev, h_ref = np.asarray(h_dev, float), np.asarray(h_ref, float)
    rel = np.abs(h_dev - h_ref) / np.maximum(np.abs(h_ref), 1e-300)
    out = []
    for t in np.flatnonzero(rel.max(axis=1) >= tol):
        step = int(np.argmax(rel[t] >= tol))
        starts = diag["s1_start"][t]
        seed = int(np.argmin(np.abs(starts - h_dev[t, 0]) / np.abs(starts)))
        ref_seed = int(diag["order"][t, diag["winner"][t]])
        kept = list(diag["order"][t])
        if seed == ref_seed:
            acc_d = h_dev[t, 1:] < h_dev[t, :-1]
            acc_r = h_ref[t, 1:] < h_ref[t, :-1]
            k = int(np.argmax(acc_d != acc_r)) if np.any(acc_d != acc_r) else max(step - 1, 0)
            gap = abs(h_ref[t, k] - h_ref[t, k + 1]) / abs(h_ref[t, k])
            out.append((int(t), "accept_gap", step, float(gap)))
        elif seed in kept:
            c = diag["s2_cost"][t]
            gap = abs(c[kept.index(seed)] - c[diag["winner"][t]]) / abs(c[diag["winner"][t]])
            out.append((int(t), "winner_gap", step, float(gap)))
        else:
            c1 = diag["s1_cost"][t]
            edge = c1[kept[-1]]
            gap = abs(c1[seed] - edge) / abs(edge)
            out.append((int(t), "prune_gap", step, float(gap)))
    return out


def history_agreement(h_dev, h_ref, rtol=1e-4, atol=1e-6):
    """Per-step cost agreement of two (lanes, steps+1) cost histories up to each
    lane's first accept/reject flip (the first step at which one run accepts its
    proposal and the other rejects).  Returns (fraction of compared (lane, step)
    pairs with |dc| <= rtol*c_ref + atol, flip rate = fraction of lanes that
    flip, number of compared pairs, and the per-lane first flip step (steps+1
    when the lane never flips))."""
    h_dev = np.asarray(h_dev, dtype=float)
    h_ref = np.asarray(h_ref, dtype=float)
    acc_d = h_dev[:, 1:] < h_dev[:, :-1]
    acc_r = h_ref[:, 1:] < h_ref[:, :-1]
    diff = acc_d != acc_r
    steps = h_dev.shape[1] - 1
    first = np.where(diff.any(axis=1), diff.argmax(axis=1) + 1, steps + 1)
    cols = np.arange(h_dev.shape[1])[None, :]
    mask = cols < first[:, None]  # steps before the flip (the flip step itself is not compared)
    ok = np.abs(h_dev - h_ref) <= rtol * np.abs(h_ref) + atol
    n = int(mask.sum())
    return float(ok[mask].mean()) if n else 1.0, float(np.mean(first <= steps)), n, first


# ---------------------------------------------------------------------------
# IK-Beam (tasks.py) and benchmark inputs (benchmark.py)
# ---------------------------------------------------------------------------

def _philox_uniform(lo, hi, key0, key1):
    gen = np.random.Generator(np.random.Philox(key=np.array([key0, key1], dtype=np.uint64)))
    return gen.uniform(lo, hi)


def sample_seeds(ch: Chain, count: int, rng_seed: int):
    """tasks.py:88-106: seed i ~ U(lo, hi) from Philox key (rng_seed, i)."""
    fin_lo, fin_hi = np.isfinite(ch.lower), np.isfinite(ch.upper)
    lo = np.where(fin_lo, ch.lower, -math.pi)
    hi = np.where(fin_hi, ch.upper, math.pi)
    unb = ~(fin_lo & fin_hi)
    out = np.empty((count, ch.n))
    for i in range(count):
        d = _philox_uniform(lo, hi, rng_seed, i)
        out[i] = np.where(unb, -d, d)
    return out


def sample_configuration(ch: Chain, gen):
    """robot.py:164-168."""
    lo = np.where(np.isfinite(ch.lower), ch.lower, -math.pi)
    hi = np.where(np.isfinite(ch.upper), ch.upper, math.pi)
    return gen.uniform(lo, hi)


def reachable_targets(ch: Chain, link: int, count: int, rng_seed: int, start: int = 0):
    """benchmark.py:83-93 -> (wxyz canonical, xyz) arrays of shape (count, 4), (count, 3)."""
    qs = np.empty((count, ch.n))
    for i in range(count):
        gen = np.random.Generator(np.random.Philox(
            key=np.array([rng_seed, TARGET_KEY_BASE + start + i], dtype=np.uint64)))
        qs[i] = sample_configuration(ch, gen)
    lq, lp, _, _ = fk(ch, qs)
    return qcanon(lq[:, link, :]), lp[:, link, :].copy(), qs


def target_inverse(tq, tt):
    """Transform3.inverse with canonical rotation -- liegroups.py:388-390."""
    iq = qcanon(qconj(tq))
    return iq, -qrot(iq, tt)


def pose_errors(ch: Chain, link: int, tq, tt, q, ba=None, bxy=None):
    """tasks.py:109-116: |t(T_t^-1 (B) T)|, |log R(T_t^-1 (B) T)|."""
    lq, lp, _, _ = fk(ch, np.asarray(q, dtype=float))
    cq = qcanon(lq[..., link, :])
    cp = lp[..., link, :]
    if ba is not None:  # Transform2.to_transform3().compose(current), liegroups.py:449-453
        bq = qexp(np.stack([np.zeros_like(ba), np.zeros_like(ba), ba], axis=-1))
        cp = np.concatenate([bxy, np.zeros_like(ba)[..., None]], axis=-1) + qrot(bq, cp)
        cq = qcanon(qmul(bq, cq))
    iq, it = target_inverse(tq, tt)
    rq = qcanon(qmul(iq, cq))
    rt = it + qrot(iq, cp)
    return np.linalg.norm(rt, axis=-1), np.linalg.norm(qlog(rq), axis=-1)


@dataclass
class BeamResult:
    q: np.ndarray
    cost: np.ndarray
    hist: np.ndarray
    pos_err: np.ndarray
    rot_err: np.ndarray
    success: np.ndarray
    base: np.ndarray | None = None  # (B, 3) x, y, angle
    diag: dict | None = None  # stage-1 / stage-2 costs and choices (parity diagnostics)


DEFAULT_WEIGHTS = (50.0, 10.0, 100.0, 0.01)  # costs.py:52-62 (pos, ori, limit, rest)


def ik_beam(ch: Chain, link: int, tq, tt, seeds, weights=DEFAULT_WEIGHTS, total_steps=16,
            prune_after=6, keep=4, pos_tol=0.005, rot_tol=0.05, dtype=np.float64, use_base=False,
            base_weight=0.0, engine=None) -> BeamResult:
    """tasks.py:119-161 over B targets at once (lanes = B x S seeds).

    Each target's lanes are independent, so batching targets reproduces the
    reference's one-target-per-call results (argsort/argmin per target).
    """
    tq, tt = np.atleast_2d(tq), np.atleast_2d(tt)
    b, s = tq.shape[0], seeds.shape[0]
    iq, it = target_inverse(tq, tt)
    lane_t = np.repeat(np.arange(b), s)
    kw = dict(dtype=dtype, use_base=use_base, base_weight=base_weight)
    make = engine or (lambda q_, t_, group: LaneEngine(ch, link, q_, t_, weights, group=group, **kw))
    eng = make(iq[lane_t], it[lane_t], lane_t)
    st = eng.start(np.tile(seeds, (b, 1)))
    st = eng.run(st, prune_after)
    cost = st.cost.reshape(b, s)
    order = np.argsort(cost, axis=1, kind="stable")[:, :keep]
    pick = (order + np.arange(b)[:, None] * s).reshape(-1)
    st2 = st.take(pick)
    eng2 = make(iq[lane_t[pick]], it[lane_t[pick]], lane_t[pick])
    st2 = eng2.run(st2, total_steps - prune_after)
    c2 = st2.cost.reshape(b, keep)
    win = np.argmin(c2, axis=1)
    sel = np.arange(b) * keep + win
    q = st2.q[sel].astype(np.float64)
    hist = np.stack([h[sel] for h in st2.hist], axis=1)
    base = None
    if use_base:
        ba = wrap_angle(st2.ba[sel])  # Transform2 wraps the angle
        base = np.concatenate([st2.bxy[sel], ba[:, None]], axis=1)
        pe, re = pose_errors(ch, link, tq, tt, q, ba, st2.bxy[sel])
    else:
        pe, re = pose_errors(ch, link, tq, tt, q)
    diag = dict(s1_start=st.hist[0].reshape(b, s), s1_cost=cost, order=order, s2_cost=c2, winner=win)
    return BeamResult(q=q, cost=st2.cost[sel], hist=hist, pos_err=pe, rot_err=re,
                      success=(pe < pos_tol) & (re < rot_tol), base=base, diag=diag)
