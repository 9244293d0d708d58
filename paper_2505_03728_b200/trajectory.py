"""Trajectory optimisation on the device (config 5; tasks.py:183-424 of the reference).

``plan_trajectory(TrajRequest) -> TrajResult`` keeps the reference signature
and semantics:

1. start / goal poses and the world are expressed in the robot base frame
   (tasks.py:316-323);
2. endpoint IK (tasks.py:278-306): IK-Beam with the rest weight raised to at
   least 0.01, retried with ``rng_seed + 7919 * attempt`` until it succeeds
   and clears the world by ``eta_world`` -- batched over every pending
   endpoint of every trajectory on the device;
3. ``solver.solve`` of the plan_trajectory Problem from the straight-line
   initialisation (tasks.py:344-404) -- one CTA per trajectory, banded
   normal equations (csrc/kop_traj.cu, ``kop_traj_solve``);
4. static / swept signed distances and endpoint pose errors (tasks.py:251-275,
   :406-424) -- ``kop_traj_report``.

``plan_trajectory_batch`` / ``TrajectoryPlanner`` run many requests that share
robot, timestep count, dt, weights and solver options in one launch sequence.
There is no CPU fallback: without the CUDA library every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _device as dv
from . import costs as ck
from ._lib import KopLmOptions, KopTrajCosts, check, lib
from .collision import NULL_OBSTACLE_ROW, WorldModel, obstacle_rows, transform_primitive
from .errors import PlanningError, UnsupportedFeatureError
from .liegroups import Transform3
from .robot import RobotModel, _precision
from .solver import TERMINATIONS, SolveOptions, SolveReport, VariableSet

ANCHOR_WEIGHT = 1e3  # tasks.py:37
MAX_STEPS = 64
MAX_OBSTACLES = 16


@dataclass
class TrajRequest:
    """tasks.py:188-212 (+ ``precision``: "fp64" default, the reference's arithmetic)."""

    model: RobotModel
    start_pose: Transform3
    goal_pose: Transform3
    timesteps: int = 20
    dt: float = 0.1
    world: WorldModel = field(default_factory=WorldModel)
    weights: ck.CostWeights = field(default_factory=lambda: ck.CostWeights(rest=0.0, world_collision=30.0))
    target_link: str | None = None
    eta_world: float = 0.05
    eta_self: float = 0.01
    rng_seed: int = 0
    base_pose: Transform3 = field(default_factory=Transform3.identity)
    max_iterations: int = 150
    anchor_weight: float = ANCHOR_WEIGHT
    ik_retries: int = 5
    precision: str = "fp64"

    def __post_init__(self):
        if self.timesteps < 5:
            raise ValueError("trajectory needs at least 5 timesteps for the stencils")
        if self.dt <= 0.0:
            raise ValueError(f"dt must be positive, got {self.dt}")


@dataclass
class TrajResult:
    qs: np.ndarray  # (T, n)
    report: SolveReport
    collision_free: bool
    min_signed_distance: float
    start_pos_error: float
    start_rot_error: float
    goal_pos_error: float
    goal_rot_error: float
    success: bool

    def to_json(self, include_timing: bool = False) -> dict:
        return {
            "qs": self.qs.tolist(),
            "collision_free": self.collision_free,
            "min_signed_distance": self.min_signed_distance,
            "start_pos_error": self.start_pos_error,
            "start_rot_error": self.start_rot_error,
            "goal_pos_error": self.goal_pos_error,
            "goal_rot_error": self.goal_rot_error,
            "success": self.success,
            "report": self.report.to_json(include_timing=include_timing),
        }


def _obstacle_table(worlds, batch: int) -> tuple[np.ndarray, int]:
    """[B, n_obs, 8] rows; shorter worlds padded with an inert far half-space."""
    n_obs = max((len(w.obstacles) for w in worlds), default=0)
    if n_obs > MAX_OBSTACLES:
        raise UnsupportedFeatureError(f"{n_obs} obstacles: more than {MAX_OBSTACLES} are not compiled in")
    table = np.tile(NULL_OBSTACLE_ROW, (batch, max(n_obs, 1), 1))
    for b, w in enumerate(worlds):
        if w.obstacles:
            table[b, :len(w.obstacles)] = obstacle_rows(w.obstacles)
    return table[:, :n_obs], n_obs


def _chain_link(model: RobotModel, link: str | None) -> int:
    return model.link_index(link or model.link_names[-1])


def trajectory_signed_distances_batch(model: RobotModel, qs, obstacles, n_obs: int, link: str | None = None,
                                      targets=None):
    """Device FP64 report for B trajectories (tasks.py:251-275): static (B, T), swept
    (B, T-1), their minima, and with ``targets`` (B, 2, 7) the endpoint pose errors."""
    qs = dv.to_dev(qs)
    b, steps = qs.shape[0], qs.shape[1]
    obs = dv.to_dev(obstacles) if n_obs else None
    out = {"static": dv.empty((b, steps)), "swept": dv.empty((b, max(steps - 1, 0))),
           "min_static": dv.empty(b), "min_swept": dv.empty(b)}
    tg = dv.to_dev(targets) if targets is not None else None
    if tg is not None:
        out["pos_err"], out["rot_err"] = dv.empty((b, 2)), dv.empty((b, 2))
    check(lib().kop_traj_report(model._handle, _chain_link(model, link), steps, dv.ptr(qs), dv.ptr(obs), n_obs,
                                dv.ptr(tg), b, dv.ptr(out["static"]), dv.ptr(out["swept"]),
                                dv.ptr(out["min_static"]), dv.ptr(out["min_swept"]), dv.ptr(out.get("pos_err")),
                                dv.ptr(out.get("rot_err")), dv.stream_handle()), "kop_traj_report")
    return out


def trajectory_signed_distances(model: RobotModel, qs: np.ndarray, world: WorldModel):
    """Hard-minimum static (T,) and swept (T-1,) signed distances (tasks.py:251-275);
    infinities when the world is empty."""
    qs = np.asarray(qs, dtype=float)
    steps = qs.shape[0]
    if not world.obstacles or not model.collision_spheres:
        return np.full(steps, np.inf), np.full(max(steps - 1, 0), np.inf)
    table, n_obs = _obstacle_table([world], 1)
    out = trajectory_signed_distances_batch(model, qs[None], table, n_obs)
    return out["static"][0].cpu().numpy(), out["swept"][0].cpu().numpy()


def trajectory_problem(model: RobotModel, q_start, q_goal, timesteps: int = 20, dt: float = 0.1,
                       world: WorldModel | None = None, weights: ck.CostWeights | None = None,
                       eta_world: float = 0.05, eta_self: float = 0.01, anchor_weight: float = ANCHOR_WEIGHT,
                       init=None):
    """The Problem plan_trajectory builds (tasks.py:341-403): variables q0..q{T-1}
    from the straight line (or ``init``), anchors, smoothness / velocity /
    stencil / limit / rest / self / world / swept costs.  ``solver.solve`` runs
    it on the device (trajectory path)."""
    from .solver import Problem

    w = weights or ck.CostWeights(rest=0.0, world_collision=30.0)
    world = world or WorldModel()
    q_start, q_goal = np.asarray(q_start, float), np.asarray(q_goal, float)
    alphas = np.linspace(0.0, 1.0, timesteps)
    init = (q_start[None, :] * (1 - alphas[:, None]) + q_goal[None, :] * alphas[:, None]) if init is None \
        else np.asarray(init, float)
    variables = VariableSet()
    names = [f"q{t}" for t in range(timesteps)]
    for t in range(timesteps):
        variables.add(names[t], init[t])
    costs = [ck.rest_cost(names[0], q_start, weight=anchor_weight, name="anchor_start"),
             ck.rest_cost(names[-1], q_goal, weight=anchor_weight, name="anchor_goal")]
    for t in range(1, timesteps):
        costs.append(ck.smoothness_cost(model, names[t - 1], names[t], weight=w.smoothness))
        if w.velocity > 0:
            costs.append(ck.velocity_limit_cost(model, names[t - 1], names[t], dt, weight=w.velocity))
    for t in range(2, timesteps - 2):
        window = names[t - 2:t + 3]
        if w.acceleration > 0:
            costs.append(ck.acceleration_cost(model, window, dt, weight=w.acceleration, name=f"accel{t}"))
        if w.jerk > 0:
            costs.append(ck.jerk_cost(model, window, dt, weight=w.jerk, name=f"jerk{t}"))
    for t in range(timesteps):
        if w.limit > 0:
            costs.append(ck.limit_cost(model, names[t], weight=w.limit, name=f"limit{t}"))
        if w.rest > 0:
            costs.append(ck.rest_cost(names[t], model.rest_pose, weight=w.rest, name=f"rest{t}"))
        if w.self_collision > 0 and model.self_collision_pairs:
            costs.append(ck.self_collision_cost(model, names[t], eta=eta_self, weight=w.self_collision,
                                                name=f"self{t}"))
        if w.world_collision > 0 and world.obstacles:
            costs.append(ck.world_collision_cost(model, names[t], world, eta=eta_world, weight=w.world_collision,
                                                 name=f"world{t}"))
    if w.world_collision > 0 and world.obstacles:
        for t in range(1, timesteps):
            costs.append(ck.swept_collision_cost(model, names[t - 1], names[t], world, eta=eta_world,
                                                 weight=w.world_collision, name=f"swept{t}"))
    return Problem(variables, costs)


class TrajectoryPlanner:
    """Batched plan_trajectory for one (robot, target link, T, dt, weights, options)."""

    def __init__(self, model: RobotModel, target_link: str | None = None, timesteps: int = 20, dt: float = 0.1,
                 weights: ck.CostWeights | None = None, eta_world: float = 0.05, eta_self: float = 0.01,
                 max_iterations: int = 150, anchor_weight: float = ANCHOR_WEIGHT, ik_retries: int = 5,
                 precision="fp64", sharpness: float = ck.SOFTMIN_SHARPNESS, hard_min: bool = False):
        if timesteps < 5:
            raise ValueError("trajectory needs at least 5 timesteps for the stencils")
        if timesteps > MAX_STEPS:
            raise UnsupportedFeatureError(f"{timesteps} timesteps: more than {MAX_STEPS} are not compiled in")
        if dt <= 0.0:
            raise ValueError(f"dt must be positive, got {dt}")
        self.model = model
        self.link = target_link or model.link_names[-1]
        self.link_idx = model.link_index(self.link)
        self.timesteps, self.dt = int(timesteps), float(dt)
        self.weights = weights or ck.CostWeights(rest=0.0, world_collision=30.0)
        self.eta_world, self.eta_self = float(eta_world), float(eta_self)
        self.ik_retries = int(ik_retries)
        self.precision = precision
        self.opts = SolveOptions(max_iterations=max_iterations)
        w = self.weights
        self._vlim = np.ascontiguousarray(model.velocity_limits, dtype=float)
        self._rest = np.ascontiguousarray(model.rest_pose, dtype=float)
        self.costs = KopTrajCosts(
            self.timesteps, self.dt, float(anchor_weight), w.smoothness, w.velocity, w.acceleration, w.jerk,
            w.limit, w.rest, w.self_collision if model.self_collision_pairs else 0.0, self.eta_self,
            w.world_collision, self.eta_world, float(sharpness), int(hard_min),
            self._vlim.ctypes.data_as(C.POINTER(C.c_double)), self._rest.ctypes.data_as(C.POINTER(C.c_double)))
        o = self.opts
        self.lm = KopLmOptions(o.max_iterations, o.initial_damping, o.damping_increase, o.damping_decrease,
                               o.gradient_tolerance, o.step_tolerance, max(0, int(o.max_rejections)), _precision(precision))
        # endpoint IK weights (tasks.py:281-289)
        ikw = ck.CostWeights.from_json({**w.to_json(), "rest": max(w.rest, 0.01)})
        if ikw.pose_position == 0.0:
            ikw.pose_position = ck.CostWeights().pose_position
        if ikw.pose_orientation == 0.0:
            ikw.pose_orientation = ck.CostWeights().pose_orientation
        self.ik_weights = ikw
        self._ik = {}

    # -- step 2: endpoint IK ---------------------------------------------------
    def _ik_solver(self, seed: int):
        from .tasks import IkBeamSolver

        if seed not in self._ik:
            self._ik[seed] = IkBeamSolver(self.model, self.link, self.ik_weights, rng_seed=seed,
                                          precision=self.precision)
        return self._ik[seed]

    def endpoint_ik(self, poses: np.ndarray, rng_seeds: np.ndarray, obstacles: np.ndarray, n_obs: int,
                    ) -> tuple[np.ndarray, np.ndarray]:
        """_endpoint_ik (tasks.py:278-306) for E endpoint poses (E, 7) at once; worlds
        without obstacles carry only inert padding rows.  Returns (q (E, n), found (E,))."""
        e = poses.shape[0]
        n = self.model.actuated_count
        q = np.zeros((e, n))
        found = np.zeros(e, dtype=bool)
        for attempt in range(self.ik_retries):
            pending = np.flatnonzero(~found)
            if pending.size == 0:
                break
            seeds = rng_seeds[pending] + 7919 * attempt
            for seed in np.unique(seeds):
                idx = pending[seeds == seed]
                res = self._ik_solver(int(seed)).solve_device(dv.to_dev(poses[idx]), history=False)
                ok = res.success.bool()
                if n_obs:
                    rep = trajectory_signed_distances_batch(self.model, res.q[:, None, :],
                                                            obstacles[idx], n_obs, self.link)
                    ok &= rep["min_static"] >= self.eta_world
                ok = ok.cpu().numpy()
                qh = res.q.cpu().numpy()
                q[idx[ok]] = qh[ok]
                found[idx[ok]] = True
        return q, found

    # -- step 3 + 4: device solve and report ------------------------------------
    def solve_anchored_device(self, anchors, obstacles=None, n_obs: int = 0, q_init=None, history: bool = True):
        """The plan_trajectory Problem from given anchors (B, 2, n) (device or host):
        enqueues ``kop_traj_solve`` and returns device outputs."""
        t = dv.require_cuda()
        anchors = dv.to_dev(anchors)
        b = anchors.shape[0]
        n = self.model.actuated_count
        out = {"qs": dv.empty((b, self.timesteps, n)), "cost": dv.empty(b), "initial_cost": dv.empty(b),
               "history": dv.empty((b, self.opts.max_iterations + 1)) if history else None,
               "iterations": t.empty(b, dtype=t.int32, device="cuda"),
               "termination": t.empty(b, dtype=t.int32, device="cuda")}
        obs = dv.to_dev(obstacles) if n_obs else None
        qi = dv.to_dev(q_init) if q_init is not None else None
        check(lib().kop_traj_solve(self.model._handle, self.link_idx, C.byref(self.costs), C.byref(self.lm),
                                   dv.ptr(qi), dv.ptr(anchors), dv.ptr(obs), n_obs, b, dv.ptr(out["qs"]),
                                   dv.ptr(out["cost"]), dv.ptr(out["initial_cost"]), dv.ptr(out["history"]),
                                   dv.ptr(out["iterations"]), dv.ptr(out["termination"]), dv.stream_handle()),
              "kop_traj_solve")
        return out

    def normal_equations_device(self, qs, anchors, obstacles=None, n_obs: int = 0):
        """(cost (B,), J^T r (B, T*n), J^T J (B, T*n, T*n)) of the Problem at qs (B, T, n)."""
        qs, anchors = dv.to_dev(qs), dv.to_dev(anchors)
        b = qs.shape[0]
        nr = self.timesteps * self.model.actuated_count
        cost, grad, hess = dv.empty(b), dv.empty((b, nr)), dv.empty((b, nr, nr))
        obs = dv.to_dev(obstacles) if n_obs else None
        check(lib().kop_traj_normal_equations(self.model._handle, self.link_idx, C.byref(self.costs),
                                              self.lm.precision, dv.ptr(qs), dv.ptr(anchors), dv.ptr(obs), n_obs,
                                              b, dv.ptr(cost), dv.ptr(grad), dv.ptr(hess), dv.stream_handle()),
              "kop_traj_normal_equations")
        return cost, grad, hess

    def plan(self, requests, errors: str = "raise") -> list:
        """plan_trajectory for every request (they must share this planner's settings).
        errors="raise": the first request whose endpoint IK fails raises PlanningError (plan_trajectory);
        errors="return": that request's slot holds the PlanningError and the others are still solved."""
        if errors not in ("raise", "return"):
            raise ValueError(f"errors must be 'raise' or 'return', got {errors!r}")
        start = time.perf_counter()
        b = len(requests)
        if b == 0:
            return []
        local_start, local_goal, worlds = [], [], []
        for r in requests:
            base_inv = r.base_pose.inverse()  # tasks.py:316-323
            local_start.append(base_inv.compose(r.start_pose).as_array())
            local_goal.append(base_inv.compose(r.goal_pose).as_array())
            worlds.append(WorldModel([transform_primitive(base_inv, p) for p in r.world.obstacles]))
        obstacles, n_obs = _obstacle_table(worlds, b)
        has_world = np.array([bool(w.obstacles) for w in worlds])
        seeds = np.array([r.rng_seed for r in requests], dtype=np.int64)
        poses = np.concatenate([np.stack(local_start), np.stack(local_goal)])
        q_end, found = self.endpoint_ik(poses, np.concatenate([seeds, seeds]),
                                        np.concatenate([obstacles, obstacles]), n_obs)
        failed = {}
        for i in range(b):
            for j, label in ((i, "start"), (b + i, "goal")):
                if not found[j] and i not in failed:
                    failed[i] = PlanningError(f"could not find a collision-free IK solution for the {label} pose")
                    if errors == "raise":
                        raise failed[i]
        if failed:  # solve the others only; failed requests keep their PlanningError
            keep = [i for i in range(b) if i not in failed]
            sub = self._solve_planned([requests[i] for i in keep], q_end[keep], q_end[[b + i for i in keep]],
                                      obstacles[keep], n_obs, has_world[keep], start) if keep else []
            out = [failed.get(i) for i in range(b)]
            for i, r in zip(keep, sub):
                out[i] = r
            return out
        return self._solve_planned(requests, q_end[:b], q_end[b:], obstacles, n_obs, has_world, start)

    def _solve_planned(self, requests, q_start, q_goal, obstacles, n_obs, has_world, start) -> list:
        b = len(requests)
        local_start, local_goal = [], []
        for r in requests:
            base_inv = r.base_pose.inverse()
            local_start.append(base_inv.compose(r.start_pose).as_array())
            local_goal.append(base_inv.compose(r.goal_pose).as_array())
        anchors = np.stack([q_start, q_goal], axis=1)
        out = self.solve_anchored_device(anchors, obstacles, n_obs)
        targets = np.stack([np.stack(local_start), np.stack(local_goal)], axis=1)
        rep = trajectory_signed_distances_batch(self.model, out["qs"], obstacles, n_obs, self.link, targets)
        host = {k: v.cpu().numpy() for k, v in {**out, **rep}.items() if v is not None}
        elapsed = time.perf_counter() - start
        results = []
        for i in range(b):
            qs = host["qs"][i]
            iters = int(host["iterations"][i])
            term, msg = TERMINATIONS[int(host["termination"][i])]
            hist = [float(h) for h in host["history"][i][:iters + 1]]
            values = VariableSet()
            for tt in range(self.timesteps):
                values.add(f"q{tt}", qs[tt])
            report = SolveReport(final_values=values, initial_cost=float(host["initial_cost"][i]),
                                 final_cost=float(host["cost"][i]), iterations_run=iters, termination=term,
                                 cost_history=hist, solve_time_s=elapsed / b, message=msg)
            min_sd = float(min(host["min_static"][i], host["min_swept"][i]))
            collision_free = (not has_world[i]) or min_sd >= 0.0
            pe, re = host["pos_err"][i], host["rot_err"][i]
            success = collision_free and max(pe) < 0.005 and max(re) < 0.05
            results.append(TrajResult(qs=qs, report=report, collision_free=bool(collision_free),
                                      min_signed_distance=min_sd if has_world[i] else math.inf,
                                      start_pos_error=float(pe[0]), start_rot_error=float(re[0]),
                                      goal_pos_error=float(pe[1]), goal_rot_error=float(re[1]),
                                      success=bool(success)))
        return results


def _planner_for(req: TrajRequest) -> TrajectoryPlanner:
    return TrajectoryPlanner(req.model, req.target_link, req.timesteps, req.dt, req.weights, req.eta_world,
                             req.eta_self, req.max_iterations, req.anchor_weight, req.ik_retries, req.precision)


def plan_trajectory(req: TrajRequest) -> TrajResult:
    """Collision-aware trajectory optimisation from a straight-line initialisation
    (tasks.py:309-424)."""
    return _planner_for(req).plan([req])[0]


def plan_trajectory_batch(requests, errors: str = "return") -> list:
    """plan_trajectory over many requests; requests sharing robot, link, T, dt,
    weights and options run as one batch.  A request whose endpoint IK fails
    does not abort the others: its slot holds the PlanningError (errors="return",
    default) or the first such error is raised (errors="raise")."""
    groups = {}
    for i, r in enumerate(requests):
        key = (id(r.model), r.target_link, r.timesteps, r.dt, tuple(r.weights.to_json().items()), r.eta_world,
               r.eta_self, r.max_iterations, r.anchor_weight, r.ik_retries, r.precision)
        groups.setdefault(key, []).append(i)
    out = [None] * len(requests)
    for idx in groups.values():
        res = _planner_for(requests[idx[0]]).plan([requests[i] for i in idx], errors=errors)
        for i, r in zip(idx, res):
            out[i] = r
    return out
