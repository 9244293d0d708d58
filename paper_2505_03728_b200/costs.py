"""Cost weights and typed cost builders (costs.py of the reference).

The residual rows run on the device: IK-Beam fuses pose / limit / rest rows
into the lane kernel (csrc/kop_lane.cuh), collision rows into the collision
lanes (csrc/kop_collision.cuh).  The builders below keep the reference's
signatures (costs.py:98-551) but return *typed* CostTerms -- a kind plus its
parameters -- that ``solver.solve`` maps onto the device kernels.  Their
``evaluator`` / ``jacobian`` (one term's raw rows and per-variable blocks,
what the reference's closures return) run on the device too
(``terms.py``, csrc/kop_terms.cu).  A CostTerm built from arbitrary Python
callables cannot be SOLVED on the device and is rejected (there is no CPU
fallback).
"""

from __future__ import annotations

from dataclasses import asdict, dataclass, fields

import numpy as np

from .solver import CostTerm


def _typed(name, residual_dim, refs, weight, kind, params, analytic=True) -> CostTerm:
    """A typed CostTerm whose evaluator / jacobian are the device term kernels (terms.py)."""
    from .terms import term_closures

    ct = CostTerm(name=name, residual_dim=residual_dim, variable_refs=refs, weight=weight, kind=kind, params=params)
    ct.evaluator, jac = term_closures(kind, params, len(refs))
    ct.jacobian = jac if analytic else None
    return ct

SOFTMIN_SHARPNESS = 100.0  # 1/m (costs.py:44)
MANIP_EPS = 1e-6


@dataclass
class CostWeights:
    pose_position: float = 50.0
    pose_orientation: float = 10.0
    limit: float = 100.0
    velocity: float = 10.0
    rest: float = 0.01
    smoothness: float = 10.0
    acceleration: float = 1.0
    jerk: float = 0.1
    manipulability: float = 0.0
    self_collision: float = 5.0
    world_collision: float = 20.0

    def __post_init__(self):
        for f in fields(self):
            v = getattr(self, f.name)
            if v < 0.0:
                raise ValueError(f"weight '{f.name}' must be nonnegative, got {v}")
            setattr(self, f.name, float(v))

    def to_json(self) -> dict:
        return asdict(self)

    @staticmethod
    def from_json(data: dict) -> "CostWeights":
        extra = set(data) - {f.name for f in fields(CostWeights)}
        if extra:
            raise ValueError(f"unknown cost weight names: {sorted(extra)}")
        return CostWeights(**data)

    @staticmethod
    def names() -> list:
        return [f.name for f in fields(CostWeights)]

    def ik_row_weights(self):
        """(position, orientation, limit, rest) row weights of the IK lane (beam.py:95-100)."""
        return (self.pose_position, self.pose_orientation, self.limit, self.rest)


# ---------------------------------------------------------------------------
# typed cost builders (device descriptors)
# ---------------------------------------------------------------------------

def pose_cost(model, q_var: str, link: str, target, base_var: str | None = None, position_weight: float = 1.0,
              orientation_weight: float = 1.0, name: str | None = None, analytic: bool = True) -> CostTerm:
    """log(T_target^-1 FK_link(q)) as a translation-first twist (costs.py:98-166)."""
    model.link_index(link)
    w = np.concatenate([np.full(3, float(position_weight)), np.full(3, float(orientation_weight))])
    refs = [q_var] + ([base_var] if base_var else [])
    return _typed(name or f"pose[{link}]", 6, refs, w, "pose",
                  dict(model=model, link=link, target=target, base_var=base_var,
                       position_weight=float(position_weight), orientation_weight=float(orientation_weight)),
                  analytic)


def limit_cost(model, q_var: str, weight: float = 1.0, name: str = "limit", analytic: bool = True) -> CostTerm:
    """max(0, q - upper) + max(0, lower - q) (costs.py:174-195)."""
    n = model.actuated_count
    return _typed(name, n, [q_var], np.full(n, float(weight)), "limit", dict(model=model, weight=float(weight)),
                  analytic)


def rest_cost(q_var: str, q_rest, weight: float = 1.0, name: str = "rest", analytic: bool = True) -> CostTerm:
    """q - q_rest (costs.py:259-271)."""
    q_rest = np.asarray(q_rest, dtype=float).reshape(-1)
    return _typed(name, q_rest.size, [q_var], np.full(q_rest.size, float(weight)), "rest",
                  dict(q_rest=q_rest, weight=float(weight)), analytic)


def world_collision_cost(model, q_var: str, world, eta: float = 0.05, weight: float = 1.0,
                         sharpness: float = SOFTMIN_SHARPNESS, hard_min: bool = False, name: str = "world_collision",
                         analytic: bool = True) -> CostTerm:
    """One activation row per (sphere-bearing link, obstacle) (costs.py:499-551)."""
    links = [nm for nm in model.link_names if model.collision_spheres.get(nm)]
    rows = len(links) * len(world.obstacles)
    if not rows:
        raise ValueError("no (link, obstacle) pairs: empty world or no collision spheres")
    if eta <= 0.0:
        raise ValueError(f"buffer distance must be positive, got {eta}")
    return _typed(name, rows, [q_var], np.full(rows, float(weight)), "world_collision",
                  dict(model=model, world=world, eta=float(eta), weight=float(weight), sharpness=float(sharpness),
                       hard_min=bool(hard_min)), analytic)


def self_collision_cost(model, q_var: str, eta: float = 0.01, weight: float = 1.0,
                        sharpness: float = SOFTMIN_SHARPNESS, hard_min: bool = False, name: str = "self_collision",
                        analytic: bool = True) -> CostTerm:
    """One activation row per self-collision link pair (costs.py:435-496)."""
    pairs = model.self_collision_pairs
    if not pairs:
        raise ValueError("model declares no self-collision pairs")
    if eta <= 0.0:
        raise ValueError(f"buffer distance must be positive, got {eta}")
    return _typed(name, len(pairs), [q_var], np.full(len(pairs), float(weight)), "self_collision",
                  dict(model=model, eta=float(eta), weight=float(weight), sharpness=float(sharpness),
                       hard_min=bool(hard_min)), analytic)


# ---------------------------------------------------------------------------
# trajectory families (costs.py:198-341, 554-619); the device solves them as
# one banded problem when they form a plan_trajectory-shaped Problem
# ---------------------------------------------------------------------------

ACCEL_COEFFS = np.array([-1.0, 16.0, -30.0, 16.0, -1.0]) / 12.0  # costs.py:295
JERK_COEFFS = np.array([-1.0, 2.0, 0.0, -2.0, 1.0]) / 2.0  # costs.py:296


def velocity_limit_cost(model, prev_var: str, curr_var: str, dt: float, weight: float = 1.0,
                        name: str | None = None, analytic: bool = True) -> CostTerm:
    """max(0, |q_t - q_{t-1}| - velocity_limit * dt); unlimited joints 0 (costs.py:198-231)."""
    if dt <= 0.0:
        raise ValueError(f"dt must be positive, got {dt}")
    n = model.actuated_count
    return _typed(name or f"velocity[{prev_var}->{curr_var}]", n, [prev_var, curr_var], np.full(n, float(weight)),
                  "velocity", dict(model=model, dt=float(dt), weight=float(weight)), analytic)


def velocity_limit_cost_direct(model, rate_var: str, weight: float = 1.0, name: str = "velocity_direct") -> CostTerm:
    """max(0, |qdot| - limit) over an explicit rate variable (costs.py:234-256): evaluated by the
    velocity-row kernel with q_prev = 0 and dt = 1; no device solve uses it."""
    n = model.actuated_count
    return _typed(name, n, [rate_var], np.full(n, float(weight)), "velocity_direct",
                  dict(model=model, weight=float(weight)))


def smoothness_cost(model, prev_var: str, curr_var: str, weight: float = 1.0, name: str | None = None,
                    analytic: bool = True) -> CostTerm:
    """q_t - q_{t-1} (costs.py:274-290)."""
    n = model.actuated_count
    return _typed(name or f"smooth[{prev_var}->{curr_var}]", n, [prev_var, curr_var], np.full(n, float(weight)),
                  "smoothness", dict(model=model, weight=float(weight)), analytic)


def _stencil_cost(model, q_vars, dt, coeffs, scale, weight, name, kind, analytic=True):
    if len(q_vars) != 5:
        raise ValueError(f"stencil costs need 5 consecutive timesteps, got {len(q_vars)}")
    if dt <= 0.0:
        raise ValueError(f"dt must be positive, got {dt}")
    n = model.actuated_count
    return _typed(name, n, list(q_vars), np.full(n, float(weight)), kind,
                  dict(model=model, dt=float(dt), coeffs=coeffs / scale, weight=float(weight)), analytic)


def acceleration_cost(model, q_vars, dt: float, weight: float = 1.0, name: str = "acceleration",
                      analytic: bool = True) -> CostTerm:
    """Five-point second difference / dt^2 over q_{t-2..t+2} (costs.py:322-330)."""
    return _stencil_cost(model, q_vars, dt, ACCEL_COEFFS, dt * dt, weight, name, "acceleration", analytic)


def jerk_cost(model, q_vars, dt: float, weight: float = 1.0, name: str = "jerk", analytic: bool = True) -> CostTerm:
    """Five-point third difference / dt^3 over q_{t-2..t+2} (costs.py:333-341)."""
    return _stencil_cost(model, q_vars, dt, JERK_COEFFS, dt ** 3, weight, name, "jerk", analytic)


def swept_collision_cost(model, prev_var: str, curr_var: str, world, eta: float = 0.05, weight: float = 1.0,
                         sharpness: float = SOFTMIN_SHARPNESS, hard_min: bool = False, name: str | None = None,
                         analytic: bool = True) -> CostTerm:
    """Capsules swept by every sphere between consecutive timesteps vs the world,
    one row per (sphere link, obstacle) (costs.py:554-619)."""
    links = [nm for nm in model.link_names if model.collision_spheres.get(nm)]
    rows = len(links) * len(world.obstacles)
    if not rows:
        raise ValueError("no (link, obstacle) pairs: empty world or no collision spheres")
    if eta <= 0.0:
        raise ValueError(f"buffer distance must be positive, got {eta}")
    return _typed(name or f"swept_collision[{prev_var}->{curr_var}]", rows, [prev_var, curr_var],
                  np.full(rows, float(weight)), "swept_collision",
                  dict(model=model, world=world, eta=float(eta), weight=float(weight), sharpness=float(sharpness),
                       hard_min=bool(hard_min)), analytic)


def manipulability_cost(model, q_var: str, link: str, weight: float = 1.0, eps: float = MANIP_EPS,
                        name: str | None = None, analytic: bool = True) -> CostTerm:
    """1 / (Yoshikawa measure + eps) of the translational Jacobian (costs.py:349-401): rows and
    gradient evaluated on the device (kop_term_manipulability); no device solve includes it (no
    configuration uses it)."""
    model.link_index(link)
    return _typed(name or f"manipulability[{link}]", 1, [q_var], np.array([float(weight)]), "manipulability",
                  dict(model=model, link=link, eps=float(eps), weight=float(weight)), analytic)
