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
