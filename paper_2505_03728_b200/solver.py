"""Solver result types (solver.py:36-224 of the reference).

``SolveReport`` / ``VariableSet`` are the containers IK-Beam returns
(tasks.py:149-158).  The generic block-sparse LM ``solve`` for user-composed
cost sets is the next widening step and is not
provided by this build yet.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .liegroups import Rotation3, Transform2, Transform3


def _tangent_dim(x) -> int:
    if isinstance(x, Transform3):
        return 6
    if isinstance(x, (Transform2, Rotation3)):
        return 3
    return int(np.asarray(x).size)


class VariableSet:
    """Ordered, typed variables (value access only)."""

    def __init__(self):
        self._ids, self._values, self._index = [], [], {}
        self.tangent_offsets = [0]

    @staticmethod
    def of(**variables) -> "VariableSet":
        vs = VariableSet()
        for k, v in variables.items():
            vs.add(k, v)
        return vs

    def add(self, var_id: str, value) -> "VariableSet":
        if var_id in self._index:
            raise ValueError(f"duplicate variable id '{var_id}'")
        if isinstance(value, (list, tuple)) or np.isscalar(value):
            value = np.atleast_1d(np.asarray(value, dtype=float))
        if isinstance(value, np.ndarray):
            value = value.astype(float).reshape(-1)
        elif not isinstance(value, (Transform3, Transform2, Rotation3)):
            raise TypeError(f"unsupported variable type {type(value).__name__}")
        self._index[var_id] = len(self._ids)
        self._ids.append(var_id)
        self._values.append(value)
        self.tangent_offsets.append(self.tangent_offsets[-1] + _tangent_dim(value))
        return self

    @property
    def ids(self):
        return list(self._ids)

    @property
    def tangent_dim(self) -> int:
        return self.tangent_offsets[-1]

    def index(self, var_id: str) -> int:
        try:
            return self._index[var_id]
        except KeyError:
            raise ValueError(f"unknown variable '{var_id}'") from None

    def value(self, var_id: str):
        return self._values[self.index(var_id)]


@dataclass
class SolveReport:
    final_values: VariableSet
    initial_cost: float
    final_cost: float
    iterations_run: int
    termination: str  # max_iterations | gradient_converged | step_converged | numerical_failure
    cost_history: list = field(default_factory=list)
    solve_time_s: float = 0.0
    message: str = ""

    def to_json(self, include_timing: bool = False) -> dict:
        out = {"initial_cost": self.initial_cost, "final_cost": self.final_cost,
               "iterations_run": self.iterations_run, "termination": self.termination,
               "cost_history": list(self.cost_history)}
        if self.message:
            out["message"] = self.message
        if include_timing:
            out["solve_time_s"] = self.solve_time_s
        return out
