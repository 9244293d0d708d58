"""Host-side planning of device solves (no GPU): which Problem shapes map onto
which kernel, with which parameters, and which are rejected loudly."""

import numpy as np
import pytest

import paper_2505_03728_b200 as k
from conftest import robot_file
from paper_2505_03728_b200.solver import plan


@pytest.fixture(scope="module")
def arm7():
    return k.load_robot(robot_file("arm7.urdf"), robot_file("arm7.sidecar.json"))


def test_trajectory_problem_plans_onto_traj_path(arm7):
    world = k.WorldModel([k.Sphere([0.4, 0.1, 0.5], 0.07)])
    pr = k.trajectory_problem(arm7, arm7.rest_pose, arm7.rest_pose + 0.3, 20, 0.1, world)
    p = plan(pr)
    assert p.path == "traj"
    c = p.costs
    assert (c.timesteps, c.dt, c.w_anchor, c.w_smoothness, c.w_velocity) == (20, 0.1, 1e3, 10.0, 10.0)
    assert (c.w_acceleration, c.w_jerk, c.w_limit, c.w_rest, c.w_self, c.w_world) == (1.0, 0.1, 100.0, 0.0, 5.0, 30.0)
    assert p.traj["n_obs"] == 1 and p.traj["obstacles"].shape == (1, 8)
    np.testing.assert_array_equal(p.traj["anchors"][1], arm7.rest_pose + 0.3)
    # per-timestep rest family next to the anchors
    pr2 = k.trajectory_problem(arm7, arm7.rest_pose, arm7.rest_pose + 0.3, 12, 0.1,
                               weights=k.CostWeights(rest=0.5, world_collision=30.0))
    p2 = plan(pr2)
    assert p2.costs.w_rest == 0.5 and p2.costs.w_anchor == 1e3 and p2.traj["n_obs"] == 0


def test_trajectory_problem_rejects_irregular_structure(arm7):
    pr = k.trajectory_problem(arm7, arm7.rest_pose, arm7.rest_pose + 0.3, 10, 0.1)
    pr.costs = [c for c in pr.costs if c.name != "smooth[q3->q4]"]
    with pytest.raises(k.UnsupportedFeatureError, match="smoothness"):
        plan(pr)
    pr = k.trajectory_problem(arm7, arm7.rest_pose, arm7.rest_pose + 0.3, 10, 0.1)
    pr.costs.append(k.manipulability_cost(arm7, "q3", "flange"))
    with pytest.raises(k.UnsupportedFeatureError):
        plan(pr)
    with pytest.raises(k.UnsupportedFeatureError, match="timesteps"):
        plan(k.trajectory_problem(arm7, arm7.rest_pose, arm7.rest_pose, 65, 0.1))


def test_single_variable_plans(arm7):
    t = k.Transform3.identity()
    p = plan(k.Problem(k.VariableSet.of(q=arm7.rest_pose.copy()),
                       [k.pose_cost(arm7, "q", "flange", t, position_weight=50, orientation_weight=10),
                        k.limit_cost(arm7, "q", weight=100)]))
    assert p.path == "chain" and p.costs.w_position == 50 and p.costs.w_limit == 100
    with pytest.raises(k.UnsupportedFeatureError):
        plan(k.Problem(k.VariableSet.of(q=arm7.rest_pose.copy()), [k.manipulability_cost(arm7, "q", "flange")]))


def test_trajectory_builders_validate(arm7):
    with pytest.raises(ValueError, match="5 consecutive"):
        k.acceleration_cost(arm7, ["a", "b"], 0.1)
    with pytest.raises(ValueError, match="dt"):
        k.velocity_limit_cost(arm7, "a", "b", 0.0)
    with pytest.raises(ValueError, match="no \\(link, obstacle\\)"):
        k.swept_collision_cost(arm7, "a", "b", k.WorldModel())


def test_variable_bookkeeping(arm7):
    vs = k.VariableSet.of(q=np.zeros(3), base=k.Transform2.identity(), pose=k.Transform3.identity())
    assert vs.tangent_slice("base") == slice(3, 6) and vs.tangent_slice("pose") == slice(6, 12)
    up = vs.updated(np.concatenate([[1.0, 2.0, 3.0], [0.1, 0.2, 0.3], np.zeros(6)]))
    np.testing.assert_allclose(up.value("q"), [1, 2, 3])
    np.testing.assert_allclose(up.value("base").log(), [0.1, 0.2, 0.3], atol=1e-12)
    with pytest.raises(ValueError):
        vs.updated(np.zeros(5))
    pr = k.trajectory_problem(arm7, arm7.rest_pose, arm7.rest_pose, 6, 0.1)
    assert pr.sparsity[:3] == [(0, 0), (1, 5), (2, 0)]
