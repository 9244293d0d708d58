"""Cost weights (costs.py:48-84 of the reference).

The pose / limit / rest residual rows that IK-Beam uses are fused into the
device lane kernel (csrc/kop_lane.cuh); this module carries the weights that
parameterise them.
"""

from __future__ import annotations

from dataclasses import asdict, dataclass, fields

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
