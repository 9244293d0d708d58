"""Per-term evaluation on the device (-m gpu): CostTerm.evaluator / .jacobian /
.raw_residual and solver.assemble of the typed cost builders, backed by
csrc/kop_terms.cu (FP64), pinned to the REFERENCE's own closures evaluated at
the same points (tests/golden/make_golden_terms.py -> reference_golden_terms.npz):
rows within 1e-10, Jacobian blocks within 1e-9.  The reference test suite's
cost gates (test_costs.py) are restated against the package: analytic vs
numeric Jacobians per family (incl. SE(2) / SE(3) bases), zero-at-target,
limit boundary subgradient, stencil exactness, collision behaviour."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2505_03728_b200 as k  # noqa: E402
from paper_2505_03728_b200 import solver as sv  # noqa: E402
from paper_2505_03728_b200.liegroups import Rotation3, Transform2, Transform3  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_golden_terms.npz")
RT, JT = 1e-10, 1e-9


@pytest.fixture(scope="module")
def gt():
    return np.load(GOLD)


@pytest.fixture(scope="module")
def arm7(models):
    return models["arm7"]


def demo_world():
    return k.WorldModel([k.Sphere([0.45, 0.1, 0.55], 0.12), k.Capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
                         k.HalfSpace([0.0, 0.0, 1.0], -0.3)])


def _check(gt, name, cost, points):
    for i, p in enumerate(points):
        np.testing.assert_allclose(cost.evaluator(*p), gt[f"{name}_r"][i], rtol=RT, atol=RT, err_msg=name)
        blocks = cost.jacobian(*p)
        assert len(blocks) == len(p)
        for kk, b in enumerate(blocks):
            np.testing.assert_allclose(b, gt[f"{name}_j{kk}"][i], rtol=JT, atol=JT, err_msg=f"{name} block {kk}")


def _target(gt):
    return Transform3.from_parts(gt["target"][:4], gt["target"][4:])


def test_pose_terms_match_reference(gt, arm7):
    t = _target(gt)
    _check(gt, "pose", k.pose_cost(arm7, "q", "flange", t), [(q,) for q in gt["q"]])
    b2 = [Transform2(a, xy) for a, *xy in gt["base2"]]
    _check(gt, "pose_se2", k.pose_cost(arm7, "q", "flange", t, base_var="b"), list(zip(gt["q"], b2)))
    b3 = [Transform3.from_parts(b[:4], b[4:]) for b in gt["base3"]]
    _check(gt, "pose_se3", k.pose_cost(arm7, "q", "flange", t, base_var="b"), list(zip(gt["q"], b3)))


def test_joint_space_terms_match_reference(gt, arm7):
    _check(gt, "limit", k.limit_cost(arm7, "q"), [(q,) for q in gt["q_wide"]])
    _check(gt, "rest", k.rest_cost("q", arm7.rest_pose), [(q,) for q in gt["q"]])
    _check(gt, "velocity", k.velocity_limit_cost(arm7, "a", "b", dt=0.1), list(zip(gt["q"], gt["q2"])))
    _check(gt, "velocity_direct", k.velocity_limit_cost_direct(arm7, "v"),
           [(2.0 * (q - q0),) for q, q0 in zip(gt["q"], gt["q2"])])
    _check(gt, "smooth", k.smoothness_cost(arm7, "a", "b"), list(zip(gt["q"], gt["q2"])))
    _check(gt, "accel", k.acceleration_cost(arm7, list("abcde"), dt=0.07), [tuple(f) for f in gt["five"]])
    _check(gt, "jerk", k.jerk_cost(arm7, list("abcde"), dt=0.07), [tuple(f) for f in gt["five"]])


def test_collision_terms_match_reference(gt, arm7):
    w = demo_world()
    _check(gt, "world", k.world_collision_cost(arm7, "q", w, eta=0.08), [(q,) for q in gt["q"]])
    _check(gt, "world_hard", k.world_collision_cost(arm7, "q", w, eta=0.3, hard_min=True), [(q,) for q in gt["q"]])
    _check(gt, "self", k.self_collision_cost(arm7, "q", eta=0.05), [(q,) for q in gt["q"]])
    _check(gt, "self_wide", k.self_collision_cost(arm7, "q", eta=0.3), [(q,) for q in gt["q"]])
    _check(gt, "self_hard", k.self_collision_cost(arm7, "q", eta=0.3, hard_min=True), [(q,) for q in gt["q"]])
    _check(gt, "swept", k.swept_collision_cost(arm7, "a", "b", w, eta=0.08), list(zip(gt["q"], gt["q2"])))
    assert np.any(gt["world_r"] != 0) and np.any(gt["self_wide_r"] != 0) and np.any(gt["swept_r"] != 0)


def test_assemble_matches_reference(gt, arm7):
    b2 = Transform2(gt["base2"][0][0], gt["base2"][0][1:])
    vs = k.VariableSet.of(q=gt["q"][0].copy(), b=b2)
    prob = k.Problem(vs, [k.pose_cost(arm7, "q", "flange", _target(gt), base_var="b", position_weight=50,
                                      orientation_weight=10),
                          k.limit_cost(arm7, "q", weight=100), k.rest_cost("q", arm7.rest_pose, weight=0.01)])
    r, jac = sv.assemble(prob, vs)
    np.testing.assert_allclose(r, gt["assemble_r"], rtol=RT, atol=RT)
    dense = jac.to_dense()
    np.testing.assert_allclose(dense, gt["assemble_j"], rtol=JT, atol=JT)
    assert np.max(np.abs(jac.to_csr().toarray() - dense)) == 0.0
    assert prob.sparsity == [(0, 0), (0, 1), (1, 0), (2, 0)]


# ---- the reference suite's cost gates, restated (test_costs.py) ---------------------------
def check_jacobian(cost, values, tol=1e-5):
    analytic = cost.jacobian(*values)
    numeric = sv.numeric_jacobian(cost, values)
    for a, n in zip(analytic, numeric):
        assert np.max(np.abs(np.asarray(a) - n)) < tol


def test_jacobian_cross_checks(arm7):
    """test_costs.py:276-349: analytic vs central differences per family."""
    rng = np.random.default_rng(50)
    target = k.link_transform(arm7, arm7.sample_configuration(rng), "flange")
    pose = k.pose_cost(arm7, "q", "flange", target)
    based = k.pose_cost(arm7, "q", "flange", target, base_var="base")
    for _ in range(5):
        check_jacobian(pose, [arm7.sample_configuration(rng)])
        check_jacobian(based, [arm7.sample_configuration(rng), Transform2(rng.uniform(-2, 2), rng.normal(size=2))])
        check_jacobian(based, [arm7.sample_configuration(rng),
                               Transform3(Rotation3.exp(rng.normal(size=3) * 0.5), rng.normal(size=3))])
    span = arm7.upper_limits - arm7.lower_limits
    for _ in range(5):
        q = rng.uniform(arm7.lower_limits - 0.5 * span, arm7.upper_limits + 0.5 * span)
        q2 = arm7.sample_configuration(rng)
        check_jacobian(k.limit_cost(arm7, "q"), [q])
        check_jacobian(k.velocity_limit_cost(arm7, "a", "b", dt=0.1), [q, q2])
        check_jacobian(k.rest_cost("q", arm7.rest_pose), [q])
        check_jacobian(k.smoothness_cost(arm7, "a", "b"), [q, q2])
    qs = [arm7.sample_configuration(rng) for _ in range(5)]
    check_jacobian(k.acceleration_cost(arm7, list("abcde"), dt=0.07), qs)
    check_jacobian(k.jerk_cost(arm7, list("abcde"), dt=0.07), qs)
    w = demo_world()
    for _ in range(4):
        q, q2 = arm7.sample_configuration(rng), arm7.sample_configuration(rng)
        check_jacobian(k.world_collision_cost(arm7, "q", w, eta=0.08), [q])
        check_jacobian(k.self_collision_cost(arm7, "q", eta=0.05), [q])
        check_jacobian(k.swept_collision_cost(arm7, "a", "b", w, eta=0.08), [q, q2])


def test_pose_and_joint_values(arm7):
    """test_costs.py:40-190 value checks."""
    q = arm7.rest_pose
    target = k.link_transform(arm7, q, "flange")
    assert np.max(np.abs(k.pose_cost(arm7, "q", "flange", target).evaluator(q))) < 1e-12
    moved = Transform3(target.rotation, target.translation - np.array([0.001, 0, 0]))
    r = k.pose_cost(arm7, "q", "flange", moved).evaluator(q)
    assert abs(np.linalg.norm(r[:3]) - 0.001) < 1e-6 and np.linalg.norm(r[3:]) < 1e-9
    base = Transform2(0.4, np.array([2.0, -1.0]))
    tgt = base.to_transform3().compose(k.link_transform(arm7, q, "flange"))
    c = k.pose_cost(arm7, "q", "flange", tgt, base_var="base")
    assert np.max(np.abs(c.evaluator(q, base))) < 1e-12
    assert np.linalg.norm(c.evaluator(q, Transform2.identity())) > 1.0
    lim = k.limit_cost(arm7, "q")
    assert np.allclose(lim.evaluator(arm7.rest_pose), 0.0)
    qa = arm7.rest_pose.copy()
    qa[0] = arm7.upper_limits[0] + 0.2
    ra = lim.evaluator(qa)
    assert ra[0] == pytest.approx(0.2) and np.allclose(ra[1:], 0.0)
    qb = arm7.rest_pose.copy()
    qb[2] = arm7.upper_limits[2]
    assert lim.jacobian(qb)[0][2, 2] == 0.0  # one-sided subgradient 0 at the boundary
    vel = k.velocity_limit_cost(arm7, "a", "b", 0.1)
    budget = arm7.velocity_limits * 0.1
    assert np.allclose(vel.evaluator(q, q), 0.0) and np.allclose(vel.evaluator(q, q + budget), 0.0)
    assert np.allclose(vel.evaluator(q, q + 2 * budget), budget)
    rest = k.rest_cost("q", arm7.rest_pose)
    assert np.allclose(rest.evaluator(arm7.rest_pose + 0.1), 0.1)
    sm = k.smoothness_cost(arm7, "a", "b")
    assert np.allclose(sm.evaluator(q, q + 0.3), 0.3)
    # stencils: zero on constant / linear, exact on quadratics (accel) and cubics (jerk)
    dt = 0.05
    ts = np.arange(5) * dt
    acc = k.acceleration_cost(arm7, list("abcde"), dt)
    jrk = k.jerk_cost(arm7, list("abcde"), dt)
    const = [q.copy() for _ in ts]
    lin = [q + 0.3 * t for t in ts]
    quad = [q + 0.7 * t * t for t in ts]
    cub = [q + 0.5 * t ** 3 for t in ts]
    assert np.allclose(acc.evaluator(*const), 0.0, atol=1e-9) and np.allclose(acc.evaluator(*lin), 0.0, atol=1e-8)
    assert np.allclose(acc.evaluator(*quad), 1.4, atol=1e-6)
    assert np.allclose(jrk.evaluator(*cub), 3.0, atol=1e-5)


def test_collision_behaviour(arm7, models):
    """test_costs.py:209-275 restated."""
    far = k.WorldModel([k.Sphere([5.0, 5.0, 5.0], 0.2)])
    assert np.allclose(k.world_collision_cost(arm7, "q", far).evaluator(arm7.rest_pose), 0.0)
    # one sphere r = 0.1 on a prismatic stick, obstacle 0.15 away: activation 0.05 + 0.5 * 0.1
    stick = k.parse_urdf("""
        <robot name="stick"><link name="base"/><link name="tip"/>
          <joint name="j" type="prismatic">
            <parent link="base"/><child link="tip"/><axis xyz="1 0 0"/>
            <limit lower="-1" upper="1" velocity="1"/>
          </joint>
        </robot>""", collision_spheres={"tip": [{"center": [0, 0, 0], "radius": 0.1}]})
    one = k.world_collision_cost(stick, "q", k.WorldModel([k.Sphere([0.35, 0.0, 0.0], 0.1)]), eta=0.1)
    assert one.evaluator(np.array([0.2]))[0] == pytest.approx(0.1, abs=1e-9)
    # penetrating flange sphere: a step along -gradient reduces the rows
    q = arm7.rest_pose
    flange = k.link_transform(arm7, q, "flange")
    wc = k.world_collision_cost(arm7, "q", k.WorldModel([k.Sphere(flange.apply([0.0, 0.0, 0.035]), 0.06)]),
                                eta=0.05, hard_min=True)
    rows = wc.evaluator(q)
    assert rows.max() > 0.0
    grad = wc.jacobian(q)[0].sum(axis=0)
    assert wc.evaluator(q - 1e-3 * grad / np.linalg.norm(grad)).sum() < rows.sum()
    rng = np.random.default_rng(41)
    for _ in range(20):
        qq = arm7.sample_configuration(rng)
        assert np.all(k.world_collision_cost(arm7, "q", demo_world()).evaluator(qq) >= 0.0)
        assert np.all(k.self_collision_cost(arm7, "q").evaluator(qq) >= 0.0)
    p2r = models["planar_2r"]
    for m in (arm7, p2r):
        assert np.allclose(k.self_collision_cost(m, "q", eta=0.01).evaluator(m.rest_pose), 0.0)
    # swept rows see an obstacle both endpoint configurations miss
    q0, q1 = np.array([0.6, 0.0]), np.array([-0.6, 0.0])
    ee = p2r.link_index("ee")
    mid = 0.5 * (k.forward_kinematics(p2r, q0)[ee].translation + k.forward_kinematics(p2r, q1)[ee].translation)
    world = k.WorldModel([k.Sphere(mid, 0.1)])
    static = k.world_collision_cost(p2r, "q", world, eta=0.01)
    swept = k.swept_collision_cost(p2r, "a", "b", world, eta=0.01)
    assert np.allclose(static.evaluator(q0), 0.0) and np.allclose(static.evaluator(q1), 0.0)
    assert swept.evaluator(q0, q1).max() > 0.0


def test_raw_residual_contract(arm7):
    c = k.pose_cost(arm7, "q", "flange", Transform3.identity())
    assert c.raw_residual([arm7.rest_pose]).shape == (6,)
    with pytest.raises(ValueError):
        c.raw_residual([np.zeros(3)])



def test_manipulability_matches_reference(gt, arm7, models):
    """manipulability_cost (costs.py:349-401) and translational_jacobian_with_derivative
    (robot.py:509-566) on the device vs the reference's own closures."""
    _check(gt, "manip", k.manipulability_cost(arm7, "q", "flange"), [(q,) for q in gt["q"]])
    _check(gt, "manip_p2r", k.manipulability_cost(models["planar_2r"], "q", "ee"), [(q,) for q in gt["q_p2r"]])
    for i, q in enumerate(gt["q"][:4]):
        jac, djac = k.robot.translational_jacobian_with_derivative(arm7, q, "flange")
        np.testing.assert_allclose(jac, gt["tjac"][i], atol=1e-12)
        np.testing.assert_allclose(djac, gt["tdjac"][i], atol=1e-10)


@pytest.mark.parametrize("kind", ["se2", "se3"])
def test_solve_with_base_variable_matches_reference(gt, arm7, kind):
    """solver.solve with pose_cost(base_var=...) (costs.py:98-166) on the device tree LM
    (kop_multi_pose_solve_base): the reference's own solve histories (60 iterations, targets
    up to 1.5 m out of the fixed base's reach) within 1e-6, final q / base within 1e-6."""
    probs = []
    for i in range(4):
        t = gt[f"solve_{kind}_targets"][i]
        tgt = Transform3.from_parts(t[:4], t[4:])
        base0 = Transform2.identity() if kind == "se2" else Transform3.identity()
        vs = k.VariableSet.of(q=arm7.rest_pose.copy(), b=base0)
        probs.append(k.Problem(vs, [k.pose_cost(arm7, "q", "flange", tgt, base_var="b", position_weight=50,
                                                orientation_weight=10),
                                    k.limit_cost(arm7, "q", weight=100), k.rest_cost("q", arm7.rest_pose, weight=0.01)]))
    reps = k.solve_batch(probs, k.SolveOptions(max_iterations=60))
    for i, rep in enumerate(reps):
        gh = gt[f"solve_{kind}_hist"][i]
        gh = gh[~np.isnan(gh)]
        assert rep.iterations_run == gt[f"solve_{kind}_iters"][i]
        h = np.array(rep.cost_history)
        assert h.shape == gh.shape
        assert np.max(np.abs(h - gh) / gh) < 1e-6, (i, np.max(np.abs(h - gh) / gh))
        np.testing.assert_allclose(rep.final_values.value("q"), gt[f"solve_{kind}_q"][i], atol=1e-6)
        b = rep.final_values.value("b")
        got = np.array([b.angle, *b.translation]) if kind == "se2" else b.as_array()
        np.testing.assert_allclose(got, gt[f"solve_{kind}_b"][i], atol=1e-6)
    # FP32 reaches comparable costs: these problems are still descending slowly at iteration 60 in
    # FP64, and the FP32 stopping rule may end them a little earlier
    r32 = k.solve_batch(probs, k.SolveOptions(max_iterations=60, precision="fp32"))
    for i, rep in enumerate(r32):
        assert all(bb <= aa for aa, bb in zip(rep.cost_history, rep.cost_history[1:]))
        assert rep.final_cost <= 1.1 * np.nanmin(gt[f"solve_{kind}_hist"][i]) + 1e-5


def test_terms_on_mimic_chain_and_tree(gt, models):
    """The term kernels on the gripper (a mimic finger and prismatic joints, robot.py:486-506
    folds the mimic multiplier into the column) and on the humanoid tree with an SE(3) base."""
    grip = models["arm7_gripper"]
    tg = Transform3.from_parts(gt["target_grip"][:4], gt["target_grip"][4:])
    _check(gt, "pose_grip", k.pose_cost(grip, "q", "finger_right", tg), [(q,) for q in gt["q_grip"]])
    _check(gt, "manip_grip", k.manipulability_cost(grip, "q", "finger_right"), [(q,) for q in gt["q_grip"]])
    hum = k.load_robot(k.robot_path("humanoid29.urdf"))
    th = Transform3.from_parts(gt["target_hum"][:4], gt["target_hum"][4:])
    bases = [Transform3.from_parts(b[:4], b[4:]) for b in gt["base_hum"]]
    _check(gt, "pose_hum_se3", k.pose_cost(hum, "q", "left_hand", th, base_var="b"), list(zip(gt["q_hum"], bases)))


def test_floating_base_humanoid_solve_matches_reference(gt):
    """Humanoid IK with a planar floating base -- four end-effector poses, an SE(2) base variable,
    limit and rest (the reference's solve, 40 iterations) -- on the device tree LM: 29 + 3 = 32
    tangent columns, every warp lane a column; histories within 1e-6.  (An SE(3) base on the
    29-joint humanoid needs 35 columns: the tree kernel holds <= 32, KOP_EUNSUPPORTED.)"""
    hum = k.load_robot(k.robot_path("humanoid29.urdf"))
    ees = ["left_hand", "right_hand", "left_foot", "right_foot"]
    probs = []
    for i in range(len(gt["hum_base_iters"])):
        tg = gt["hum_base_targets"][i]
        vs = k.VariableSet.of(q=hum.rest_pose.copy(), b=Transform2.identity())
        probs.append(k.Problem(vs, [k.pose_cost(hum, "q", e, Transform3.from_parts(t[:4], t[4:]), base_var="b",
                                                position_weight=50, orientation_weight=10) for e, t in zip(ees, tg)]
                               + [k.limit_cost(hum, "q", weight=100), k.rest_cost("q", hum.rest_pose, weight=0.01)]))
    for i, rep in enumerate(k.solve_batch(probs, k.SolveOptions(max_iterations=40))):
        gh = gt["hum_base_hist"][i]
        gh = gh[~np.isnan(gh)]
        assert rep.iterations_run == gt["hum_base_iters"][i]
        h = np.array(rep.cost_history)
        assert np.max(np.abs(h - gh) / gh) < 1e-6, (i, np.max(np.abs(h - gh) / gh))
        bb = rep.final_values.value("b")
        np.testing.assert_allclose([bb.angle, *bb.translation], gt["hum_base_b"][i], atol=1e-6)
    with pytest.raises(k.UnsupportedFeatureError):
        vs = k.VariableSet.of(q=hum.rest_pose.copy(), b=Transform3.identity())
        k.solve(k.Problem(vs, [k.pose_cost(hum, "q", "left_hand", Transform3.identity(), base_var="b")]))
