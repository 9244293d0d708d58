"""Config 3: humanoid multi-end-effector IK through the device tree solve
(one warp per problem) vs the reference's own solver.solve runs (goldens) and
the CPU oracle (run on a B200: -m gpu)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2505_03728_b200 as k  # noqa: E402
from oracle import ik_oracle as o  # noqa: E402
from oracle import tree_oracle as to  # noqa: E402

EES = ["left_hand", "right_hand", "left_foot", "right_foot"]


@pytest.fixture(scope="module")
def hum():
    return k.load_robot(k.robot_path("humanoid29.urdf"))


def _problem(model, targets, q0, w=None):
    w = w or k.CostWeights()
    costs = [k.pose_cost(model, "q", e, t, position_weight=w.pose_position, orientation_weight=w.pose_orientation)
             for e, t in zip(EES, targets)]
    costs += [k.limit_cost(model, "q", weight=w.limit), k.rest_cost("q", model.rest_pose, weight=w.rest)]
    return k.Problem(k.VariableSet.of(q=np.asarray(q0, float).copy()), costs)


def test_humanoid_fk_matches_reference(hum, golden):
    quat, pos, _, _ = k.fk_arrays(hum, golden["hum_fk_q"])
    np.testing.assert_allclose(quat, golden["hum_fk_quat"], atol=1e-12)
    np.testing.assert_allclose(pos, golden["hum_fk_pos"], atol=1e-12)


def test_tree_solve_fp64_matches_reference(hum, golden):
    probs = []
    for i in range(5):
        tgs = [k.Transform3.from_parts(golden["hum_tw"][i][e], golden["hum_tp"][i][e]) for e in range(4)]
        probs.append(_problem(hum, tgs, hum.rest_pose))
    reps = k.solve_batch(probs)
    for i, rep in enumerate(reps):
        gh = golden["hum_hist"][i]
        gh = gh[~np.isnan(gh)]
        n = min(len(gh), len(rep.cost_history))
        rel = np.abs(np.array(rep.cost_history[:n]) - gh[:n]) / gh[:n]
        assert rel.max() < 1e-6, (i, rel.max())
        assert rep.iterations_run == golden["hum_iters"][i]
        np.testing.assert_allclose(rep.final_cost, golden["hum_cost"][i], rtol=1e-6)


def test_tree_solve_fp32_reaches_reference_costs(hum, golden):
    probs = []
    for i in range(5):
        tgs = [k.Transform3.from_parts(golden["hum_tw"][i][e], golden["hum_tp"][i][e]) for e in range(4)]
        probs.append(_problem(hum, tgs, hum.rest_pose))
    reps = k.solve_batch(probs, k.SolveOptions(precision="fp32"))
    for i, rep in enumerate(reps):
        assert all(b <= a for a, b in zip(rep.cost_history, rep.cost_history[1:]))
        assert rep.final_cost <= 1.05 * golden["hum_cost"][i] + 1e-5


def test_tree_solve_reachable_batch_converges(hum, chains):
    """Targets = FK of random in-limit configurations; start from the rest pose."""
    ch = o.load_chain_files(k.robot_path("humanoid29.urdf"))
    rng = np.random.default_rng(11)
    qt = np.stack([o.sample_configuration(ch, rng) for _ in range(64)])
    quat, pos, _, _ = k.fk_arrays(hum, qt)
    li = [hum.link_index(e) for e in EES]
    probs = [_problem(hum, [k.Transform3.from_parts(quat[b, l], pos[b, l]) for l in li], hum.rest_pose)
             for b in range(64)]
    reps = k.solve_batch(probs, k.SolveOptions(precision="fp32"))
    init = np.array([r.initial_cost for r in reps])
    final = np.array([r.final_cost for r in reps])
    assert np.all(final <= init) and np.median(final / init) < 1e-2
    # one problem through the oracle as a spot check
    poses = [(ch.link(e), o.qcanon(quat[0, l]), pos[0, l], 50.0, 10.0) for e, l in zip(EES, li)]
    _, c_ref, _, _, _ = to.solve_multi_pose(ch, poses, ch.rest)
    rep64 = k.solve(probs[0])
    np.testing.assert_allclose(rep64.final_cost, c_ref, rtol=1e-5)
