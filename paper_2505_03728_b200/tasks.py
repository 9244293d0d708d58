"""Task drivers: IK-Beam on the device (tasks.py:40-180 of the reference).

``solve_ik_beam(IkRequest) -> IkResult`` keeps the reference signature;
``solve_ik_beam_batch`` / ``IkBeamSolver`` are the batched entry the
reference lacks (it loops targets one by one, benchmark.py:136-151): B
targets x S seeds run as B*S device lanes in one launch sequence.

IK-Beam (tasks.py:119-161): all seeds run ``prune_after`` LM steps, the
``keep`` lowest-cost lanes (stable order) survive, run the remaining steps,
and the lowest-cost survivor wins.  Seeds are Philox-keyed by (rng_seed, i),
shared by every target, and drawn bit-identically to numpy on the device.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _device as dv
from . import costs as ck
from ._lib import KopIkParams, check, lib
from .errors import UnsupportedFeatureError
from .liegroups import Transform2, Transform3
from .robot import RobotModel, _precision
from .solver import SolveReport, VariableSet

BASE_PINNED = 1e12
ANCHOR_WEIGHT = 1e3


@dataclass
class IkRequest:
    model: RobotModel
    target_link: str
    target_pose: Transform3
    weights: ck.CostWeights = field(default_factory=ck.CostWeights)
    seeds: int = 64
    total_steps: int = 16
    prune_after: int = 6
    keep: int = 4
    success_pos_tol: float = 0.005
    success_rot_tol: float = 0.05
    rng_seed: int = 0
    optimize_base: bool = False
    base_reg_weight: float = 0.0
    precision: str = "fp32"

    def __post_init__(self):
        if not 0 < self.prune_after < self.total_steps:
            raise ValueError("need 0 < prune_after < total_steps")
        if not 1 <= self.keep <= self.seeds:
            raise ValueError("need 1 <= keep <= seeds")


@dataclass
class IkResult:
    q: np.ndarray
    base: Transform2 | None
    pos_error: float
    rot_error: float
    success: bool
    report: SolveReport

    def to_json(self, include_timing: bool = False) -> dict:
        out = {"q": self.q.tolist(), "pos_error": self.pos_error, "rot_error": self.rot_error,
               "success": self.success, "report": self.report.to_json(include_timing=include_timing)}
        if self.base is not None:
            out["base"] = {"angle": self.base.angle, "xy": self.base.translation.tolist()}
        return out


def _seed_bounds(model: RobotModel):
    fin_lo, fin_hi = np.isfinite(model.lower_limits), np.isfinite(model.upper_limits)
    lo = np.where(fin_lo, model.lower_limits, -math.pi)
    hi = np.where(fin_hi, model.upper_limits, math.pi)
    return lo, hi, ~(fin_lo & fin_hi)


def philox_uniform_device(key0: int, key1_base: int, count: int, lo, hi, negate=None):
    """Row i = Generator(Philox(key=[key0, key1_base+i])).uniform(lo, hi) (device, bit-exact)."""
    lo = np.ascontiguousarray(lo, dtype=float)
    hi = np.ascontiguousarray(hi, dtype=float)
    n = lo.size
    neg = np.ascontiguousarray(np.zeros(n, np.uint8) if negate is None else np.asarray(negate, np.uint8))
    out = dv.empty((count, n))
    check(lib().kop_sample_uniform(C.c_uint64(int(key0) & (2**64 - 1)), C.c_uint64(int(key1_base) & (2**64 - 1)),
                                   count, n, lo.ctypes.data, hi.ctypes.data, neg.ctypes.data, dv.ptr(out),
                                   dv.stream_handle()), "kop_sample_uniform")
    return out


def sample_seed_configurations_device(model: RobotModel, count: int, rng_seed: int):
    lo, hi, unbounded = _seed_bounds(model)
    return philox_uniform_device(rng_seed, 0, count, lo, hi, unbounded)


def sample_seed_configurations(model: RobotModel, count: int, rng_seed: int) -> np.ndarray:
    """tasks.py:88-106: seed i ~ U(lo, hi) from Philox key (rng_seed, i); (-pi, pi] for continuous."""
    return sample_seed_configurations_device(model, count, rng_seed).cpu().numpy()


def targets_to_array(targets) -> np.ndarray:
    """Transform3 / list of Transform3 / (B,7) array -> (B,7) float64 (w,x,y,z,px,py,pz)."""
    if isinstance(targets, Transform3):
        return targets.as_array()[None]
    if isinstance(targets, (list, tuple)) and targets and isinstance(targets[0], Transform3):
        return np.stack([t.as_array() for t in targets])
    arr = np.asarray(targets, dtype=float)
    if arr.ndim != 2 or arr.shape[1] != 7:
        raise ValueError(f"targets must have shape (B, 7), got {arr.shape}")
    return arr


@dataclass
class BeamBatch:
    """Per-target IK-Beam outputs (device tensors or host arrays).  ``base`` is
    (B, 3) (x, y, angle) with an optimised mobile base, else None."""

    q: object
    cost: object
    history: object
    pos_error: object
    rot_error: object
    success: object
    base: object = None

    FIELDS = ("q", "cost", "history", "pos_error", "rot_error", "success", "base")

    def cpu(self) -> "BeamBatch":
        f = lambda x: x.cpu().numpy() if hasattr(x, "cpu") else x
        return BeamBatch(*(f(getattr(self, k)) for k in self.FIELDS))

    def rows(self, lo: int, hi: int) -> "BeamBatch":
        """Row slice [lo, hi) of every field (views)."""
        return BeamBatch(*((None if getattr(self, k) is None else getattr(self, k)[lo:hi]) for k in self.FIELDS))


class IkBeamSolver:
    """Reusable batched IK-Beam for one (robot, link, request shape).

    Holds the seeds on the device and a grow-only workspace; ``solve_device``
    only enqueues kernels on the current stream (CUDA-graph capturable once
    the workspace has been sized).
    """

    def __init__(self, model: RobotModel, link: str, weights: ck.CostWeights | None = None, seeds: int = 64,
                 total_steps: int = 16, prune_after: int = 6, keep: int = 4, rng_seed: int = 0,
                 success_pos_tol: float = 0.005, success_rot_tol: float = 0.05, precision="fp32",
                 seed_configurations=None, optimize_base: bool = False, base_reg_weight: float = 0.0,
                 world=None, self_collision: bool = False, eta_world: float = 0.05, eta_self: float = 0.01,
                 sharpness: float = ck.SOFTMIN_SHARPNESS, hard_min: bool = False):
        """``world`` (a WorldModel) and/or ``self_collision`` switch the lanes to the
        collision stack (config 4): world rows weighted by ``weights.world_collision``
        and self rows by ``weights.self_collision`` appended to pose / limit / rest."""
        if not 0 < prune_after < total_steps:
            raise ValueError("need 0 < prune_after < total_steps")
        if not 1 <= keep <= seeds:
            raise ValueError("need 1 <= keep <= seeds")
        self.model, self.link = model, link
        self.link_idx = model.link_index(link)
        w = (weights or ck.CostWeights()).ik_row_weights()
        self.total_steps = total_steps
        self.optimize_base = bool(optimize_base)
        self.params = KopIkParams(w[0], w[1], w[2], w[3], seeds, total_steps, prune_after, keep,
                                  success_pos_tol, success_rot_tol, _precision(precision),
                                  1 if self.optimize_base else 0, float(base_reg_weight))
        self.collision = None
        if world is not None or self_collision:
            if optimize_base:
                raise UnsupportedFeatureError("collision lanes with a mobile base are not compiled in")
            from ._lib import KopCollisionCosts
            from .solver import _obstacles

            wts = weights or ck.CostWeights()
            cc = KopCollisionCosts()
            cc.w_position, cc.w_orientation, cc.w_limit, cc.w_rest = w
            self._obs = _obstacles(world) if world is not None and world.obstacles else None
            cc.w_world = wts.world_collision if self._obs is not None else 0.0
            cc.eta_world, cc.num_obstacles = eta_world, len(world.obstacles) if self._obs is not None else 0
            cc.obstacles = self._obs
            cc.w_self, cc.eta_self = (wts.self_collision if self_collision else 0.0), eta_self
            cc.sharpness, cc.hard_min = sharpness, int(hard_min)
            self.collision = cc
        if seed_configurations is not None:
            self.seeds = dv.to_dev(np.asarray(seed_configurations, dtype=float).reshape(seeds, model.actuated_count))
        else:
            self.seeds = sample_seed_configurations_device(model, seeds, rng_seed)
        self._ws = None

    def workspace(self, batch: int):
        need = self._ws_bytes(batch)
        if self._ws is None or self._ws.numel() < need:
            t = dv.require_cuda()
            self._ws = t.empty(need, dtype=t.uint8, device="cuda")
        return self._ws

    def alloc_outputs(self, batch: int) -> BeamBatch:
        t = dv.require_cuda()
        n = self.model.actuated_count
        return BeamBatch(dv.empty((batch, n)), dv.empty(batch), dv.empty((batch, self.total_steps + 1)),
                         dv.empty(batch), dv.empty(batch), t.empty(batch, dtype=t.uint8, device="cuda"),
                         dv.empty((batch, 3)) if self.optimize_base else None)

    def solve_device(self, targets, out: BeamBatch | None = None, history: bool = True,
                     stages: int = 3, workspace=None) -> BeamBatch:
        """targets: device (B,7) float64 tensor.  Enqueues the solve on the current
        stream and returns the device outputs.  ``stages`` 1 / 2 issue only the
        seed+prune or the survivor+winner kernel (for per-kernel timing).
        ``workspace``: a caller-owned uint8 device buffer (for concurrent solves
        on several streams); default the solver's own."""
        targets = dv.to_dev(targets)
        b = targets.shape[0]
        out = out or self.alloc_outputs(b)
        ws = self.workspace(b) if workspace is None else workspace
        if self.collision is not None:
            if stages != 3:
                raise ValueError("collision IK-Beam runs both stages together")
            check(lib().kop_ik_beam_collision(self.model._handle, self.link_idx, C.byref(self.params),
                                              C.byref(self.collision), dv.ptr(targets), b, dv.ptr(self.seeds),
                                              dv.ptr(ws), ws.numel(), dv.ptr(out.q), dv.ptr(out.cost),
                                              dv.ptr(out.history) if history else None, dv.ptr(out.pos_error),
                                              dv.ptr(out.rot_error), dv.ptr(out.success), dv.stream_handle()),
                  "kop_ik_beam_collision")
            return out
        check(lib().kop_ik_beam_stage(self.model._handle, self.link_idx, C.byref(self.params), int(stages),
                                      dv.ptr(targets), b, dv.ptr(self.seeds), dv.ptr(ws), ws.numel(),
                                      dv.ptr(out.q), dv.ptr(out.base), dv.ptr(out.cost),
                                      dv.ptr(out.history) if history else None,
                                      dv.ptr(out.pos_error), dv.ptr(out.rot_error), dv.ptr(out.success),
                                      dv.stream_handle()), "kop_ik_beam")
        return out

    def alloc_host_outputs(self, batch: int) -> BeamBatch:
        """Pinned host tensors shaped like ``alloc_outputs``."""
        dev = self.alloc_outputs(0)
        mk = lambda x, shape: None if x is None else dv.torch().empty(shape, dtype=x.dtype).pin_memory()
        n = self.model.actuated_count
        return BeamBatch(mk(dev.q, (batch, n)), mk(dev.cost, (batch,)), mk(dev.history, (batch, self.total_steps + 1)),
                         mk(dev.pos_error, (batch,)), mk(dev.rot_error, (batch,)), mk(dev.success, (batch,)),
                         mk(dev.base, (batch, 3)))

    def solve_pinned(self, host_targets, host_out: BeamBatch | None = None, chunk: int = 65536,
                     n_streams: int = 4, history: bool = True) -> BeamBatch:
        """Pinned host (B, 7) targets in, pinned host outputs out.  The batch runs
        in chunks round-robin over ``n_streams`` CUDA streams, so the host->device
        copy of one chunk, the kernels of another and the device->host copy of a
        third overlap (copy engines and SMs are separate).  Enqueued behind and
        joined back into the current stream; synchronise before reading."""
        t = dv.require_cuda()
        b = host_targets.shape[0]
        host_out = host_out or self.alloc_host_outputs(b)
        chunk = max(1, min(chunk, b))
        key = (chunk, n_streams)
        if getattr(self, "_pipe_key", None) != key:
            self._pipe = [(t.cuda.Stream(), dv.empty((chunk, 7)), self.alloc_outputs(chunk),
                           t.empty(self._ws_bytes(chunk), dtype=t.uint8, device="cuda")) for _ in range(n_streams)]
            self._pipe_key = key
        cur = t.cuda.current_stream()
        start = t.cuda.Event()
        start.record(cur)
        for i, lo in enumerate(range(0, b, chunk)):
            hi = min(b, lo + chunk)
            st, tg, out, ws = self._pipe[i % n_streams]
            if i < n_streams:
                st.wait_event(start)
            with t.cuda.stream(st):
                tgv = tg[:hi - lo]
                tgv.copy_(host_targets[lo:hi], non_blocking=True)
                ov = out.rows(0, hi - lo)
                self.solve_device(tgv, ov, history=history, workspace=ws)
                hv = host_out.rows(lo, hi)
                for kk in BeamBatch.FIELDS:
                    src = getattr(ov, kk)
                    if src is not None and (history or kk != "history"):
                        getattr(hv, kk).copy_(src, non_blocking=True)
        for st, _, _, _ in self._pipe:
            ev = t.cuda.Event()
            ev.record(st)
            cur.wait_event(ev)
        return host_out

    def _ws_bytes(self, batch: int) -> int:
        if self.collision is not None:
            need = int(lib().kop_ik_beam_collision_workspace_bytes(self.model._handle, self.link_idx,
                                                                   C.byref(self.params), C.byref(self.collision),
                                                                   batch))
        else:
            need = int(lib().kop_ik_beam_workspace_bytes(self.model._handle, self.link_idx, C.byref(self.params),
                                                         batch))
        if need < 0:
            check(need, "kop_ik_beam_workspace_bytes")
        return need

    def solve_host(self, targets, out: BeamBatch | None = None, chunk: int = 0, n_streams: int = 0,
                   history: bool = True) -> BeamBatch:
        """Host arrays in, host arrays out through the C ABI (``kop_ik_beam_host``):
        the library pipelines H2D copies, kernels and D2H copies over its own
        streams.  ``targets``: (B, 7) float64 numpy array or CPU tensor (pinned
        memory overlaps fully); ``out``: host BeamBatch to fill (numpy / CPU
        tensors), default new numpy arrays.  Enqueued behind the current stream
        and joined back into it; returns after synchronising unless ``out`` was
        given (then the caller synchronises)."""
        if self.collision is not None:
            raise UnsupportedFeatureError("the host pipeline runs the plain IK lanes; use solve_device")
        t = dv.require_cuda()
        tg = targets if isinstance(targets, t.Tensor) else t.from_numpy(np.ascontiguousarray(targets_to_array(targets)))
        if tg.dtype != t.float64 or tg.device.type != "cpu" or not tg.is_contiguous() or tg.shape[-1] != 7:
            raise ValueError("targets must be a contiguous host (B, 7) float64 array")
        b = tg.shape[0]
        given = out is not None
        if out is None:
            n = self.model.actuated_count
            out = BeamBatch(np.empty((b, n)), np.empty(b), np.empty((b, self.total_steps + 1)), np.empty(b),
                            np.empty(b), np.empty(b, dtype=np.uint8), np.empty((b, 3)) if self.optimize_base else None)
        if not hasattr(self, "_seeds_host"):
            self._seeds_host = np.ascontiguousarray(self.seeds.cpu().numpy())
        hp = lambda x: None if x is None else (x.data_ptr() if isinstance(x, t.Tensor) else x.ctypes.data)
        check(lib().kop_ik_beam_host(self.model._handle, self.link_idx, C.byref(self.params), hp(tg), b,
                                     self._seeds_host.ctypes.data, hp(out.q), hp(out.base), hp(out.cost),
                                     hp(out.history) if history else None, hp(out.pos_error), hp(out.rot_error),
                                     hp(out.success), chunk, n_streams, dv.stream_handle()), "kop_ik_beam_host")
        if not given:
            t.cuda.current_stream().synchronize()
        return out

    def solve(self, targets) -> BeamBatch:
        """Host in, host out (synchronous), through the host pipeline of the C ABI."""
        arr = targets_to_array(targets)
        if self.collision is not None:
            return self.solve_device(dv.to_dev(arr)).cpu()
        return self.solve_host(arr)


def solve_ik_beam_batch(model: RobotModel, link: str, targets, weights: ck.CostWeights | None = None,
                        seeds: int = 64, total_steps: int = 16, prune_after: int = 6, keep: int = 4,
                        rng_seed: int = 0, precision="fp32", success_pos_tol: float = 0.005,
                        success_rot_tol: float = 0.05, optimize_base: bool = False,
                        base_reg_weight: float = 0.0) -> BeamBatch:
    """IK-Beam over B targets at once (host arrays in and out)."""
    solver = IkBeamSolver(model, link, weights, seeds, total_steps, prune_after, keep, rng_seed,
                          success_pos_tol, success_rot_tol, precision, optimize_base=optimize_base,
                          base_reg_weight=base_reg_weight)
    return solver.solve(targets)


def _result(req: IkRequest, res: BeamBatch, i: int = 0) -> IkResult:
    q = res.q[i].copy()
    hist = [float(h) for h in res.history[i]]
    base = None
    if res.base is not None:
        base = Transform2(float(res.base[i, 2]), res.base[i, :2].copy())
    values = VariableSet.of(q=q) if base is None else VariableSet.of(q=q, base=base)
    report = SolveReport(final_values=values, initial_cost=hist[0], final_cost=float(res.cost[i]),
                         iterations_run=req.total_steps, termination="max_iterations", cost_history=hist)
    return IkResult(q=q, base=base, pos_error=float(res.pos_error[i]), rot_error=float(res.rot_error[i]),
                    success=bool(res.success[i]), report=report)


def _solve(req: IkRequest, use_base: bool) -> IkResult:
    res = solve_ik_beam_batch(req.model, req.target_link, req.target_pose, req.weights, req.seeds,
                              req.total_steps, req.prune_after, req.keep, req.rng_seed, req.precision,
                              req.success_pos_tol, req.success_rot_tol, optimize_base=use_base,
                              base_reg_weight=req.base_reg_weight if use_base else 0.0)
    return _result(req, res)


def solve_ik_beam(req: IkRequest) -> IkResult:
    """Multi-seed IK with mid-optimisation pruning (tasks.py:164-166); never raises
    on unreachable targets.  Like the reference, the base is never optimised here."""
    return _solve(req, use_base=False)


def solve_ik_mobile(req: IkRequest) -> IkResult:
    """IK with the SE(2) base pose as an extra variable (tasks.py:169-180).  Each
    seed starts with the base at identity; base_reg_weight >= BASE_PINNED drops
    the base variable, reproducing solve_ik_beam exactly."""
    if req.base_reg_weight >= BASE_PINNED:
        result = _solve(req, use_base=False)
        result.base = Transform2.identity()
        return result
    return _solve(req, use_base=True)


def solve_ik_collision_batch(model: RobotModel, link: str, targets, world=None, self_collision: bool = True,
                             weights: ck.CostWeights | None = None, seeds: int = 64, total_steps: int = 16,
                             prune_after: int = 6, keep: int = 4, rng_seed: int = 0, precision="fp32",
                             eta_world: float = 0.05, eta_self: float = 0.01, sharpness: float = ck.SOFTMIN_SHARPNESS,
                             hard_min: bool = False, success_pos_tol: float = 0.005,
                             success_rot_tol: float = 0.05) -> BeamBatch:
    """IK-Beam over the collision stack (config 4): pose / limit / rest rows plus
    world-collision (costs.py:499-551) and self-collision (costs.py:435-496) rows."""
    solver = IkBeamSolver(model, link, weights, seeds, total_steps, prune_after, keep, rng_seed, success_pos_tol,
                          success_rot_tol, precision, world=world, self_collision=self_collision,
                          eta_world=eta_world, eta_self=eta_self, sharpness=sharpness, hard_min=hard_min)
    return solver.solve(targets)


@dataclass
class MultiBeamBatch:
    """Multi-end-effector IK-Beam outputs: q (B, n), cost (B,), history (B, total_steps+1),
    pos_error / rot_error (B, E) per end effector, success (B,) (every end effector
    within tolerance)."""

    q: object
    cost: object
    history: object
    pos_error: object
    rot_error: object
    success: object

    def cpu(self) -> "MultiBeamBatch":
        f = lambda x: x.cpu().numpy() if hasattr(x, "cpu") else x
        return MultiBeamBatch(f(self.q), f(self.cost), f(self.history), f(self.pos_error), f(self.rot_error),
                              f(self.success))


def solve_ik_beam_multi(model: RobotModel, links, targets, weights: ck.CostWeights | None = None, seeds: int = 64,
                        total_steps: int = 16, prune_after: int = 6, keep: int = 4, rng_seed: int = 0,
                        precision="fp32", success_pos_tol: float = 0.005, success_rot_tol: float = 0.05,
                        rest=None, device_out: bool = False) -> MultiBeamBatch:
    """IK-Beam over several end effectors of a tree (config 3 as SURVEY.md section 8
    H6 states it): every lane runs the beam.py lane LM over [pose_1..pose_E | limit |
    rest]; the tasks.py:119-161 prune / continue / winner flow picks each target set's
    solution.  ``targets``: (B, E, 7) poses (w, x, y, z, px, py, pz) of ``links``."""
    from ._lib import KopPoseCosts

    if not 0 < prune_after < total_steps:
        raise ValueError("need 0 < prune_after < total_steps")
    if not 1 <= keep <= seeds:
        raise ValueError("need 1 <= keep <= seeds")
    t = dv.require_cuda()
    w = weights or ck.CostWeights()
    links = list(links)
    e = len(links)
    tg = dv.to_dev(targets)
    if tg.dim() != 3 or tg.shape[1] != e or tg.shape[2] != 7:
        raise ValueError(f"targets must have shape (B, {e}, 7), got {tuple(tg.shape)}")
    b, n = tg.shape[0], model.actuated_count
    li = np.ascontiguousarray([model.link_index(l) for l in links], dtype=np.int32)
    wp = np.full(e, float(w.pose_position))
    wo = np.full(e, float(w.pose_orientation))
    rp = np.ascontiguousarray(model.rest_pose if rest is None else rest, dtype=float)
    pc = KopPoseCosts(e, li.ctypes.data, wp.ctypes.data, wo.ctypes.data, float(w.limit), float(w.rest), rp.ctypes.data)
    params = KopIkParams(0.0, 0.0, 0.0, 0.0, seeds, total_steps, prune_after, keep, success_pos_tol, success_rot_tol,
                         _precision(precision), 0, 0.0)
    sd = sample_seed_configurations_device(model, seeds, rng_seed)
    need = int(lib().kop_multi_pose_beam_workspace_bytes(model._handle, C.byref(pc), C.byref(params), b))
    if need < 0:
        check(need, "kop_multi_pose_beam_workspace_bytes")
    ws = t.empty(max(need, 1), dtype=t.uint8, device="cuda")
    out = MultiBeamBatch(dv.empty((b, n)), dv.empty(b), dv.empty((b, total_steps + 1)), dv.empty((b, e)),
                         dv.empty((b, e)), t.empty(b, dtype=t.uint8, device="cuda"))
    check(lib().kop_multi_pose_beam(model._handle, C.byref(pc), C.byref(params), dv.ptr(tg), b, dv.ptr(sd),
                                    dv.ptr(ws), ws.numel(), dv.ptr(out.q), dv.ptr(out.cost), dv.ptr(out.history),
                                    dv.ptr(out.pos_error), dv.ptr(out.rot_error), dv.ptr(out.success),
                                    dv.stream_handle()), "kop_multi_pose_beam")
    return out if device_out else out.cpu()


# trajectory optimisation lives in trajectory.py; re-exported here where the reference keeps it (tasks.py:183-424)
from .trajectory import (TrajectoryPlanner, TrajRequest, TrajResult, plan_trajectory,  # noqa: E402,F401
                         plan_trajectory_batch, trajectory_signed_distances)
