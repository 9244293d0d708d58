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
        return LaneState(q=self.q[indices].copy(), base_angle=None, base_xy=None,
                         damping=self.damping[indices].copy(), cost=self.cost[indices].copy(),
                         history=[h[indices].copy() for h in self.history])


class IkLaneProblem:
    """Batched IK objective for one robot, link and target pose (beam.py:71-102)."""

    def __init__(self, model: RobotModel, link: str, target, position_weight: float,
                 orientation_weight: float, limit_weight: float, rest_weight: float, rest_pose=None,
                 use_base: bool = False, base_reg_weight: float = 0.0, precision="fp32"):
        if use_base:
            raise UnsupportedFeatureError("mobile-base lanes are not compiled in this build yet")
        if rest_pose is not None and not np.array_equal(np.asarray(rest_pose, float), model.rest_pose):
            raise UnsupportedFeatureError("a per-problem rest_pose override is not supported; "
                                          "set the model's rest pose instead")
        self.model = model
        self.link_idx = model.link_index(link)
        tinv = target.inverse()
        self.ti_q, self.ti_t = tinv.rotation.wxyz, tinv.translation
        self.use_base = False
        self.rest_pose = model.rest_pose
        n = model.actuated_count
        self.weight = np.concatenate([np.full(3, position_weight), np.full(3, orientation_weight),
                                      np.full(n, limit_weight), np.full(n, rest_weight)])
        self._w = np.array([position_weight, orientation_weight, limit_weight, rest_weight], dtype=float)
        self.residual_dim = self.weight.size
        self.tangent_dim = n
        self.precision = _precision(precision)
        self._tinv = None

    def _args(self, lanes):
        t = dv.require_cuda()
        if self._tinv is None:
            self._tinv = dv.to_dev(np.concatenate([self.ti_q, self.ti_t])[None])
        lane_t = t.zeros(lanes, dtype=t.int32, device="cuda")
        return self._tinv, lane_t

    def residuals_and_jacobian(self, q, base_angle=None, base_xy=None):
        """Weighted residuals (B, M) and Jacobian (B, M, n) (beam.py:133-180)."""
        q = np.atleast_2d(np.asarray(q, dtype=float))
        b, n = q.shape[0], self.tangent_dim
        tinv, lane_t = self._args(b)
        qd = dv.to_dev(q)
        r, j = dv.empty((b, self.residual_dim)), dv.empty((b, self.residual_dim, n))
        check(lib().kop_lane_residuals_jacobian(self.model._handle, self.link_idx, self.precision,
                                                self._w.ctypes.data, dv.ptr(tinv), dv.ptr(lane_t),
                                                dv.ptr(qd), b, dv.ptr(r), dv.ptr(j), dv.stream_handle()),
              "kop_lane_residuals_jacobian")
        return r.cpu().numpy(), j.cpu().numpy()

    def residuals(self, q, base_angle=None, base_xy=None, fk=None):
        return self.residuals_and_jacobian(q)[0]

    def start_state(self, q0) -> LaneState:
        q0 = np.atleast_2d(np.asarray(q0, dtype=float))
        b = q0.shape[0]
        tinv, lane_t = self._args(b)
        qd = dv.to_dev(q0)
        lam, cost = dv.empty(b), dv.empty(b)
        check(lib().kop_lane_start(self.model._handle, self.link_idx, self.precision, self._w.ctypes.data,
                                   dv.ptr(tinv), dv.ptr(lane_t), dv.ptr(qd), b, dv.ptr(lam), dv.ptr(cost),
                                   dv.stream_handle()), "kop_lane_start")
        c = cost.cpu().numpy()
        return LaneState(q=q0.copy(), base_angle=None, base_xy=None, damping=lam.cpu().numpy(), cost=c,
                         history=[c.copy()])

    def run(self, state: LaneState, steps: int) -> LaneState:
        """Advance every lane by `steps` proposals (beam.py:198-240); mutates and returns state."""
        b = state.lanes
        if steps <= 0 or b == 0:
            return state
        tinv, lane_t = self._args(b)
        q, lam, cost = dv.to_dev(state.q), dv.to_dev(state.damping), dv.to_dev(state.cost)
        hist = dv.empty((b, steps))
        check(lib().kop_lane_run(self.model._handle, self.link_idx, self.precision, self._w.ctypes.data,
                                 dv.ptr(tinv), dv.ptr(lane_t), b, steps, dv.ptr(q), dv.ptr(lam), dv.ptr(cost),
                                 dv.ptr(hist), dv.stream_handle()), "kop_lane_run")
        state.q, state.damping, state.cost = q.cpu().numpy(), lam.cpu().numpy(), cost.cpu().numpy()
        h = hist.cpu().numpy()
        state.history.extend(h[:, i].copy() for i in range(steps))
        return state


def lane_run_device(model: RobotModel, link: int, weights, target_inv, lane_target, q, damping, cost,
                    steps: int, history=None, precision="fp32"):
    """Device-tensor lane engine: many targets at once (one target index per lane)."""
    w = np.ascontiguousarray(weights, dtype=float)
    check(lib().kop_lane_run(model._handle, int(link), _precision(precision), w.ctypes.data,
                             dv.ptr(target_inv), dv.ptr(lane_target), q.shape[0], int(steps), dv.ptr(q),
                             dv.ptr(damping), dv.ptr(cost), dv.ptr(history), dv.stream_handle()),
          "kop_lane_run")


def lane_start_device(model: RobotModel, link: int, weights, target_inv, lane_target, q, damping, cost,
                      precision="fp32"):
    w = np.ascontiguousarray(weights, dtype=float)
    check(lib().kop_lane_start(model._handle, int(link), _precision(precision), w.ctypes.data,
                               dv.ptr(target_inv), dv.ptr(lane_target), dv.ptr(q), q.shape[0],
                               dv.ptr(damping), dv.ptr(cost), dv.stream_handle()), "kop_lane_start")
