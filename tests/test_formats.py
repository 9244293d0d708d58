"""Result / wire formats: IkResult, TrajResult and the
benchmark result dicts validate against the reference's JSON schemas
(schemas/*.schema.json, read in place when /root/reference is present)."""

import json
import os

import numpy as np
import pytest

import paper_2505_03728_b200 as k
from paper_2505_03728_b200.benchmark import _error_stats, _traj_rows, format_table
from paper_2505_03728_b200.solver import SolveReport, VariableSet

SCHEMAS = "/root/reference/pkg/src/kinoptik/schemas"
jsonschema = pytest.importorskip("jsonschema")
pytestmark = pytest.mark.skipif(not os.path.isdir(SCHEMAS), reason="reference schemas not present")


def _validate(obj, name):
    with open(os.path.join(SCHEMAS, name)) as f:
        schema = json.load(f)
    jsonschema.validate(json.loads(json.dumps(obj)), schema)


def _report(hist):
    return SolveReport(final_values=VariableSet.of(q=np.zeros(7)), initial_cost=hist[0], final_cost=hist[-1],
                       iterations_run=len(hist) - 1, termination="max_iterations", cost_history=list(hist),
                       solve_time_s=0.01)


def test_ik_result_schema():
    r = k.IkResult(q=np.linspace(0, 1, 7), base=None, pos_error=1e-5, rot_error=2e-5, success=True,
                   report=_report([1.0, 0.5, 0.1]))
    _validate(r.to_json(), "ik_result.schema.json")
    _validate(r.to_json(include_timing=True), "ik_result.schema.json")
    r.base = k.Transform2(0.3, np.array([0.1, -0.2]))
    _validate(r.to_json(), "ik_result.schema.json")


def test_traj_result_schema():
    r = k.TrajResult(qs=np.zeros((6, 7)), report=_report([3.0, 2.0]), collision_free=True,
                     min_signed_distance=0.02, start_pos_error=1e-6, start_rot_error=1e-6, goal_pos_error=2e-6,
                     goal_rot_error=3e-6, success=True)
    _validate(r.to_json(), "traj_result.schema.json")


def test_benchmark_result_schema_and_table():
    rng = np.random.default_rng(0)
    pos, rot = rng.uniform(0, 1e-4, 50), rng.uniform(0, 1e-4, 50)
    row = {"success_rate": 0.98, **_error_stats(pos, rot)}
    ik = {"task": "ik", "num_targets": 50, "results": {"per_batch_size": {"1": row, "64": row}},
          "timings_ms_informational": {"1": {"total_ms": 5.0, "per_solve_ms": 0.1}}}
    mob = {"task": "ik_mobile", "num_targets": 50, "results": {"static": row, "optimized": row},
           "timings_ms_informational": {"static": {"total_ms": 1.0}}}
    res = [k.TrajResult(qs=np.zeros((6, 7)), report=_report([1.0]), collision_free=True, min_signed_distance=d,
                        start_pos_error=1e-6, start_rot_error=0.0, goal_pos_error=2e-6, goal_rot_error=0.0,
                        success=True) for d in (0.01, 0.03)]
    traj = {"task": "traj", "num_targets": 2, "results": _traj_rows(res), "timings_ms_informational": {}}
    for obj in (ik, mob, traj):
        _validate(obj, "benchmark_result.schema.json")
        assert format_table(obj).startswith(f"task: {obj['task']}")
    assert traj["results"]["min_signed_distance"] == 0.01
