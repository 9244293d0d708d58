"""Cost weights and typed cost builders (costs.py of the reference).

The residual rows run on the device: IK-Beam fuses pose / limit / rest rows
into the lane kernel (csrc/kop_lane.cuh), collision rows into the collision
lanes (csrc/kop_collision.cuh).  The builders below keep the reference's
signatures (costs.py:98-551) but return *typed* CostTerms -- a kind plus its
parameters -- that ``solver.solve`` maps onto the device kernels.  A
CostTerm built from arbitrary Python callables cannot run on the device and
is rejected (there is no CPU fallback).
"""

from __future__ import annotations

from dataclasses import asdict, dataclass, fields

import numpy as np

from .solver import CostTerm

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
    return CostTerm(name=name or f"pose[{link}]", residual_dim=6, variable_refs=refs, weight=w,
                    kind="pose", params=dict(model=model, link=link, target=target, base_var=base_var,
                                             position_weight=float(position_weight),
                                             orientation_weight=float(orientation_weight)))


def limit_cost(model, q_var: str, weight: float = 1.0, name: str = "limit", analytic: bool = True) -> CostTerm:
    """max(0, q - upper) + max(0, lower - q) (costs.py:174-195)."""
    n = model.actuated_count
    return CostTerm(name=name, residual_dim=n, variable_refs=[q_var], weight=np.full(n, float(weight)),
                    kind="limit", params=dict(model=model, weight=float(weight)))


def rest_cost(q_var: str, q_rest, weight: float = 1.0, name: str = "rest", analytic: bool = True) -> CostTerm:
    """q - q_rest (costs.py:259-271)."""
    q_rest = np.asarray(q_rest, dtype=float).reshape(-1)
    return CostTerm(name=name, residual_dim=q_rest.size, variable_refs=[q_var],
                    weight=np.full(q_rest.size, float(weight)), kind="rest",
                    params=dict(q_rest=q_rest, weight=float(weight)))


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
    return CostTerm(name=name, residual_dim=rows, variable_refs=[q_var], weight=np.full(rows, float(weight)),
                    kind="world_collision", params=dict(model=model, world=world, eta=float(eta),
                                                        weight=float(weight), sharpness=float(sharpness),
                                                        hard_min=bool(hard_min)))


def self_collision_cost(model, q_var: str, eta: float = 0.01, weight: float = 1.0,
                        sharpness: float = SOFTMIN_SHARPNESS, hard_min: bool = False, name: str = "self_collision",
                        analytic: bool = True) -> CostTerm:
    """One activation row per self-collision link pair (costs.py:435-496)."""
    pairs = model.self_collision_pairs
    if not pairs:
        raise ValueError("model declares no self-collision pairs")
    if eta <= 0.0:
        raise ValueError(f"buffer distance must be positive, got {eta}")
    return CostTerm(name=name, residual_dim=len(pairs), variable_refs=[q_var],
                    weight=np.full(len(pairs), float(weight)), kind="self_collision",
                    params=dict(model=model, eta=float(eta), weight=float(weight), sharpness=float(sharpness),
                                hard_min=bool(hard_min)))
