"""Lane-batched LM engine for IK on the device (the reference's beam.py).

``IkLaneProblem`` keeps the reference's constructor and methods
(beam.py:71-240): ``residuals_and_jacobian``, ``start_state`` and
``run(state, steps)``, but every lane executes in the sm_100a lane kernel
(``kop_lane_*`` in include/kinoptik_b200.h): one CUDA thread per lane, FK,
Jacobian, normal equations, Cholesky and accept/reject in registers.

Semantics per lane are the reference's: one proposal per step, accept iff
the new cost is finite and strictly lower, damping /3 (floor 1e-12) on accept
and x10 (cap 1e10) on reject.  One documented difference: a failed Cholesky
pivot rejects that lane only, where the reference's batched LU raises and
escalates every lane (beam.py:209-213).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as dv
from ._lib import check, lib
from .errors import UnsupportedFeatureError
from .robot import RobotModel, _precision

DAMPING_INIT = 1e-4
DAMPING_UP = 10.0
DAMPING_DOWN = 1.0 / 3.0
DAMPING_MIN = 1e-12
DAMPING_MAX = 1e10
DIAG_CLAMP = 1e-8


@dataclass
class LaneState:
    """State of B lanes (beam.py:45-68); arrays are host float64."""

    q: np.ndarray
    base_angle: np.ndarray | None
    base_xy: np.ndarray | None
    damping: np.ndarray
    cost: np.ndarray
    history: list

    @property
    def lanes(self) -> int:
        return self.q.shape[0]

    def select(self, indices) -> "LaneState":
        return LaneState(q=self.q[indices].copy(),
                         base_angle=None if self.base_angle is None else self.base_angle[indices].copy(),
                         base_xy=None if self.base_xy is None else self.base_xy[indices].copy(),
                         damping=self.damping[indices].copy(), cost=self.cost[indices].copy(),
                         history=[h[indices].copy() for h in self.history])

    def base_state(self):
        """(B, 3) (x, y, angle) array, or None for a fixed base."""
        if self.base_angle is None:
            return None
        return np.concatenate([self.base_xy, self.base_angle[:, None]], axis=1)


class IkLaneProblem:
    """Batched IK objective for one robot, link and target pose (beam.py:71-102)."""

    def __init__(self, model: RobotModel, link: str, target, position_weight: float,
                 orientation_weight: float, limit_weight: float, rest_weight: float, rest_pose=None,
                 use_base: bool = False, base_reg_weight: float = 0.0, precision="fp32"):
        if rest_pose is not None and not np.array_equal(np.asarray(rest_pose, float), model.rest_pose):
            raise UnsupportedFeatureError("a per-problem rest_pose override is not supported; "
                                          "set the model's rest pose instead")
        self.model = model
        self.link_idx = model.link_index(link)
        tinv = target.inverse()
        self.ti_q, self.ti_t = tinv.rotation.wxyz, tinv.translation
        self.use_base = bool(use_base)
        self.rest_pose = model.rest_pose
        n = model.actuated_count
        rows = [np.full(3, position_weight), np.full(3, orientation_weight), np.full(n, limit_weight),
                np.full(n, rest_weight)]
        if self.use_base:
            rows.append(np.full(3, base_reg_weight))
        self.weight = np.concatenate(rows)
        self._w = np.array([position_weight, orientation_weight, limit_weight, rest_weight,
                            base_reg_weight if self.use_base else 0.0], dtype=float)
        self.residual_dim = self.weight.size
        self.tangent_dim = n + (3 if self.use_base else 0)
        self.precision = _precision(precision)
        self._tinv = None

    def _args(self, lanes):
        t = dv.require_cuda()
        if self._tinv is None:
            self._tinv = dv.to_dev(np.concatenate([self.ti_q, self.ti_t])[None])
        lane_t = t.zeros(lanes, dtype=t.int32, device="cuda")
        return self._tinv, lane_t

    def _base_dev(self, lanes, base_angle, base_xy):
        if not self.use_base:
            return None
        if base_angle is None:
            return dv.to_dev(np.zeros((lanes, 3)))
        return dv.to_dev(np.concatenate([np.asarray(base_xy, float).reshape(lanes, 2),
                                         np.asarray(base_angle, float).reshape(lanes, 1)], axis=1))

    def residuals_and_jacobian(self, q, base_angle=None, base_xy=None):
        """Weighted residuals (B, M) and Jacobian (B, M, D) (beam.py:133-180)."""
        q = np.atleast_2d(np.asarray(q, dtype=float))
        b = q.shape[0]
        tinv, lane_t = self._args(b)
        qd, bd = dv.to_dev(q), self._base_dev(b, base_angle, base_xy)
        r, j = dv.empty((b, self.residual_dim)), dv.empty((b, self.residual_dim, self.tangent_dim))
        check(lib().kop_lane_residuals_jacobian(self.model._handle, self.link_idx, self.precision,
                                                self._w.ctypes.data, dv.ptr(tinv), dv.ptr(lane_t), dv.ptr(qd),
                                                dv.ptr(bd), b, dv.ptr(r), dv.ptr(j), dv.stream_handle()),
              "kop_lane_residuals_jacobian")
        return r.cpu().numpy(), j.cpu().numpy()

    def residuals(self, q, base_angle=None, base_xy=None, fk=None):
        return self.residuals_and_jacobian(q, base_angle, base_xy)[0]

    def start_state(self, q0) -> LaneState:
        q0 = np.atleast_2d(np.asarray(q0, dtype=float))
        b = q0.shape[0]
        tinv, lane_t = self._args(b)
        qd, bd = dv.to_dev(q0), self._base_dev(b, None, None)
        lam, cost = dv.empty(b), dv.empty(b)
        check(lib().kop_lane_start(self.model._handle, self.link_idx, self.precision, self._w.ctypes.data,
                                   dv.ptr(tinv), dv.ptr(lane_t), dv.ptr(qd), dv.ptr(bd), b, dv.ptr(lam),
                                   dv.ptr(cost), dv.stream_handle()), "kop_lane_start")
        c = cost.cpu().numpy()
        return LaneState(q=q0.copy(), base_angle=np.zeros(b) if self.use_base else None,
                         base_xy=np.zeros((b, 2)) if self.use_base else None, damping=lam.cpu().numpy(), cost=c,
                         history=[c.copy()])

    def run(self, state: LaneState, steps: int) -> LaneState:
        """Advance every lane by `steps` proposals (beam.py:198-240); mutates and returns state."""
        b = state.lanes
        if steps <= 0 or b == 0:
            return state
        tinv, lane_t = self._args(b)
        q, lam, cost = dv.to_dev(state.q), dv.to_dev(state.damping), dv.to_dev(state.cost)
        bd = self._base_dev(b, state.base_angle, state.base_xy)
        hist = dv.empty((b, steps))
        check(lib().kop_lane_run(self.model._handle, self.link_idx, self.precision, self._w.ctypes.data,
                                 dv.ptr(tinv), dv.ptr(lane_t), b, steps, dv.ptr(q), dv.ptr(bd), dv.ptr(lam),
                                 dv.ptr(cost), dv.ptr(hist), dv.stream_handle()), "kop_lane_run")
        state.q, state.damping, state.cost = q.cpu().numpy(), lam.cpu().numpy(), cost.cpu().numpy()
        if self.use_base:
            bh = bd.cpu().numpy()
            state.base_xy, state.base_angle = bh[:, :2].copy(), bh[:, 2].copy()
        h = hist.cpu().numpy()
        state.history.extend(h[:, i].copy() for i in range(steps))
        return state


def _weights5(weights):
    w = np.zeros(5)
    w[: len(weights)] = np.asarray(weights, dtype=float)
    return np.ascontiguousarray(w)


def lane_run_device(model: RobotModel, link: int, weights, target_inv, lane_target, q, damping, cost,
                    steps: int, history=None, precision="fp32", base_state=None):
    """Device-tensor lane engine: many targets at once (one target index per lane)."""
    w = _weights5(weights)
    check(lib().kop_lane_run(model._handle, int(link), _precision(precision), w.ctypes.data,
                             dv.ptr(target_inv), dv.ptr(lane_target), q.shape[0], int(steps), dv.ptr(q),
                             dv.ptr(base_state), dv.ptr(damping), dv.ptr(cost), dv.ptr(history),
                             dv.stream_handle()), "kop_lane_run")


def lane_start_device(model: RobotModel, link: int, weights, target_inv, lane_target, q, damping, cost,
                      precision="fp32", base_state=None):
    w = _weights5(weights)
    check(lib().kop_lane_start(model._handle, int(link), _precision(precision), w.ctypes.data,
                               dv.ptr(target_inv), dv.ptr(lane_target), dv.ptr(q), dv.ptr(base_state), q.shape[0],
                               dv.ptr(damping), dv.ptr(cost), dv.stream_handle()), "kop_lane_start")
