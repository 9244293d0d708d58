"""CPU restatement of multi-end-effector IK through the generic solver -- TEST INFRASTRUCTURE ONLY.

Config 3 (humanoid multi-EE IK): the reference composes one ``pose_cost`` per
end effector (costs.py:98-166) with ``limit_cost`` (costs.py:174-195) and
``rest_cost`` (costs.py:259-271) and runs ``solver.solve`` (solver.py:364-429).
This module restates that stack for any tree (``ik_oracle.fk`` /
``point_jacobian`` restate robot.py) and reuses the classic LM restatement
``collision_oracle.lm``.  Pinned against reference ``solve`` runs on the
humanoid fixture by tests/test_oracle.py.
"""

from __future__ import annotations

import numpy as np

from . import collision_oracle as co
from . import ik_oracle as o


def multi_pose_stack(ch: o.Chain, poses, w_limit, w_rest, rest, q, jac=True):
    """Weighted residual (M,) and Jacobian (M, n): [pose_e (6 each) | limit n | rest n].
    poses: list of (link, target_wxyz, target_xyz, w_pos, w_ori)."""
    lq, lp, jp, ja = o.fk(ch, q[None])
    rows, jrows = [], []
    for link, tq, tt, wp, wo in poses:
        iq, it = o.target_inverse(np.atleast_2d(tq), np.atleast_2d(tt))
        fq, fpos = lq[0, link], lp[0, link]
        xi = o.se3_log(o.qmul(iq[0], fq), it[0] + o.qrot(iq[0], fpos))
        w = np.array([wp] * 3 + [wo] * 3)
        rows.append(xi * w)
        if jac:
            jg = o.point_jacobian(ch, fpos[None], jp, ja, link)[0]
            rt = o.qmat(fq).T
            body = np.vstack([rt @ jg[:3], rt @ jg[3:]])
            jrows.append((o.se3_jr_inv(xi) @ body) * w[:, None])
    lim = np.maximum(0.0, q - ch.upper) + np.maximum(0.0, ch.lower - q)
    rows += [w_limit * lim, w_rest * (q - rest)]
    r = np.concatenate(rows)
    if not jac:
        return r, None
    g = np.where(q > ch.upper, 1.0, 0.0) + np.where(q < ch.lower, -1.0, 0.0)
    jrows += [w_limit * np.diag(g), w_rest * np.eye(ch.n)]
    return r, np.vstack(jrows)


def solve_multi_pose(ch, poses, q0, w_limit=100.0, w_rest=0.01, rest=None, **kw):
    rest = ch.rest if rest is None else rest
    return co.lm(lambda q, jac: multi_pose_stack(ch, poses, w_limit, w_rest, rest, q, jac), q0, **kw)


# ---------------------------------------------------------------------------
# config 3 as SURVEY.md section 8 (H6) states it: IK-Beam lanes generalised to
# K pose blocks -- the beam.py:133-240 lane LM and the tasks.py:119-161 beam
# control flow over a residual [pose_1 .. pose_K | limit | rest]
# ---------------------------------------------------------------------------

class MultiPoseLaneEngine(o.LaneEngine):
    """IkLaneProblem (beam.py:71-240) with K pose blocks, one target set per lane.
    tinv_q / tinv_t: (lanes, K, 4) / (lanes, K, 3) inverse targets."""

    def __init__(self, ch, links, tinv_q, tinv_t, w_pos, w_ori, w_limit, w_rest, group=None):
        super().__init__(ch, links[0], tinv_q[:, 0], tinv_t[:, 0], (1.0, 1.0, w_limit, w_rest), group=group)
        self.links = list(links)
        self.mq = np.asarray(tinv_q, dtype=float)
        self.mt = np.asarray(tinv_t, dtype=float)
        n = ch.n
        rows = [np.concatenate([np.full(3, wp), np.full(3, wo)]) for wp, wo in zip(w_pos, w_ori)]
        self.w = np.concatenate(rows + [np.full(n, w_limit), np.full(n, w_rest)])

    def _poses(self, lq, lp):
        out = []
        for e, link in enumerate(self.links):
            fq, fp = lq[..., link, :], lp[..., link, :]
            xi = o.se3_log(o.qmul(self.mq[:, e], fq), self.mt[:, e] + o.qrot(self.mq[:, e], fp))
            out.append((xi, fq, fp))
        return out

    def residuals(self, q, kin=None, ba=None, bxy=None):
        lq, lp, _, _ = kin if kin is not None else o.fk(self.ch, q)
        lim = np.maximum(0.0, q - self.hi) + np.maximum(0.0, self.lo - q)
        parts = [xi for xi, _, _ in self._poses(lq, lp)] + [lim, q - self.rest]
        return np.concatenate(parts, axis=-1) * self.w

    def residuals_and_jacobian(self, q, ba=None, bxy=None):
        kin = o.fk(self.ch, q)
        lq, lp, jp, ja = kin
        r = self.residuals(q, kin)
        n, k = self.ch.n, len(self.links)
        jac = np.zeros(q.shape[:-1] + (self.w.size, n))
        for e, (xi, fq, fp) in enumerate(self._poses(lq, lp)):
            jg = o.point_jacobian(self.ch, fp, jp, ja, self.links[e])
            rt = np.swapaxes(o.qmat(fq), -1, -2)
            body = np.concatenate([rt @ jg[..., :3, :], rt @ jg[..., 3:, :]], axis=-2)
            jac[..., 6 * e:6 * e + 6, :] = o.se3_jr_inv(xi) @ body
        i = np.arange(n)
        jac[..., 6 * k + i, i] = np.where(q > self.hi, 1.0, 0.0) + np.where(q < self.lo, -1.0, 0.0)
        jac[..., 6 * k + n + i, i] = 1.0
        return r, jac * self.w[:, None]


def multi_ee_beam(ch, links, tq, tt, seeds, w_pos, w_ori, w_limit=100.0, w_rest=0.01, total_steps=16,
                  prune_after=6, keep=4, pos_tol=0.005, rot_tol=0.05):
    """IK-Beam (tasks.py:119-161) over K end effectors: tq / tt (B, K, 4) / (B, K, 3) targets.
    Returns q, cost, hist, pos_err / rot_err (B, K) and success (every end effector in tolerance)."""
    tq, tt = np.asarray(tq, float), np.asarray(tt, float)
    b, k = tq.shape[:2]
    s = seeds.shape[0]
    iq, it = o.target_inverse(tq.reshape(-1, 4), tt.reshape(-1, 3))
    iq, it = iq.reshape(b, k, 4), it.reshape(b, k, 3)
    lane_t = np.repeat(np.arange(b), s)
    make = lambda idx: MultiPoseLaneEngine(ch, links, iq[idx], it[idx], w_pos, w_ori, w_limit, w_rest, group=idx)
    eng = make(lane_t)
    st = eng.run(eng.start(np.tile(seeds, (b, 1))), prune_after)
    order = np.argsort(st.cost.reshape(b, s), axis=1, kind="stable")[:, :keep]
    pick = (order + np.arange(b)[:, None] * s).reshape(-1)
    st2 = make(lane_t[pick]).run(st.take(pick), total_steps - prune_after)
    win = np.argmin(st2.cost.reshape(b, keep), axis=1)
    sel = np.arange(b) * keep + win
    q = st2.q[sel]
    pe = np.stack([o.pose_errors(ch, links[e], tq[:, e], tt[:, e], q)[0] for e in range(k)], axis=1)
    re = np.stack([o.pose_errors(ch, links[e], tq[:, e], tt[:, e], q)[1] for e in range(k)], axis=1)
    diag = dict(s1_start=st.hist[0].reshape(b, s), s1_cost=st.cost.reshape(b, s), order=order,
                s2_cost=st2.cost.reshape(b, keep), winner=win)
    return dict(q=q, cost=st2.cost[sel], hist=np.stack([h[sel] for h in st2.hist], axis=1), pos_err=pe,
                rot_err=re, success=np.all((pe < pos_tol) & (re < rot_tol), axis=1), diag=diag)
