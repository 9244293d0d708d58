"""Golden per-term rows: the REFERENCE's cost builders evaluated (read-only).

    python tests/golden/make_golden_terms.py      (build container only)

For every typed cost family the reference's own ``evaluator`` and
``jacobian`` closures (costs.py:98-619) are called at seeded random points
of the arm7 fixture -- pose (no base, SE(2) base, SE(3) base), limit (box
enlarged so rows activate), rest, velocity, velocity_direct, smoothness,
acceleration / jerk stencils, world / self / swept collision against the
reference test suite's demo world (test_costs.py:199-206) -- plus
``solver.assemble`` on a mixed problem and the reference ``solve`` of pose
problems with an SE(2) and an SE(3) base variable.  The device term kernels
(tests/test_gpu_terms.py) and the base-variable solve are pinned to these.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from kinoptik import collision as col  # noqa: E402
from kinoptik import costs as ck  # noqa: E402
from kinoptik import robot, solver  # noqa: E402
from kinoptik.liegroups import Rotation3, Transform2, Transform3  # noqa: E402

ROBOTS = os.path.join(REF, "kinoptik", "robots")
# the humanoid fixture is this repository's own (config 3); the reference parses it
HUMANOID = os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))),
                        "paper_2505_03728_b200", "robots", "humanoid29.urdf")
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden_terms.npz")


def demo_world():
    return col.WorldModel([col.Sphere([0.45, 0.1, 0.55], 0.12), col.Capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
                           col.HalfSpace([0.0, 0.0, 1.0], -0.3)])


def main():
    arm7 = robot.load_robot(os.path.join(ROBOTS, "arm7.urdf"), os.path.join(ROBOTS, "arm7.sidecar.json"))
    rng = np.random.default_rng(77)
    g = {}
    N = 16
    qs = np.stack([arm7.sample_configuration(rng) for _ in range(N)])
    q2 = np.stack([arm7.sample_configuration(rng) for _ in range(N)])
    span = arm7.upper_limits - arm7.lower_limits
    wide = rng.uniform(arm7.lower_limits - 0.5 * span, arm7.upper_limits + 0.5 * span, (N, 7))
    g["q"], g["q2"], g["q_wide"] = qs, q2, wide
    target = robot.link_transform(arm7, arm7.sample_configuration(rng), "flange")
    g["target"] = np.concatenate([target.rotation.wxyz, target.translation])

    def record(name, cost, points):
        r = np.stack([cost.evaluator(*p) for p in points])
        jac = [np.stack([np.asarray(cost.jacobian(*p)[k]) for p in points]) for k in range(len(points[0]))]
        g[f"{name}_r"] = r
        for k, j in enumerate(jac):
            g[f"{name}_j{k}"] = j

    # pose, without / with SE(2) / with SE(3) base
    record("pose", ck.pose_cost(arm7, "q", "flange", target), [(q,) for q in qs])
    b2 = [Transform2(rng.uniform(-2, 2), rng.normal(size=2)) for _ in range(N)]
    g["base2"] = np.array([[b.angle, *b.translation] for b in b2])
    record("pose_se2", ck.pose_cost(arm7, "q", "flange", target, base_var="b"), list(zip(qs, b2)))
    b3 = [Transform3(Rotation3.exp(rng.normal(size=3) * 0.5), rng.normal(size=3)) for _ in range(N)]
    g["base3"] = np.array([np.concatenate([b.rotation.wxyz, b.translation]) for b in b3])
    record("pose_se3", ck.pose_cost(arm7, "q", "flange", target, base_var="b"), list(zip(qs, b3)))
    # joint-space families
    record("limit", ck.limit_cost(arm7, "q"), [(q,) for q in wide])
    record("rest", ck.rest_cost("q", arm7.rest_pose), [(q,) for q in qs])
    record("velocity", ck.velocity_limit_cost(arm7, "a", "b", dt=0.1), list(zip(qs, q2)))
    record("velocity_direct", ck.velocity_limit_cost_direct(arm7, "v"), [(2.0 * (q - q0),) for q, q0 in zip(qs, q2)])
    record("smooth", ck.smoothness_cost(arm7, "a", "b"), list(zip(qs, q2)))
    five = [tuple(arm7.sample_configuration(rng) for _ in range(5)) for _ in range(N)]
    g["five"] = np.array([np.stack(f) for f in five])
    record("accel", ck.acceleration_cost(arm7, list("abcde"), dt=0.07), five)
    record("jerk", ck.jerk_cost(arm7, list("abcde"), dt=0.07), five)
    # collision families (demo world, eta as in test_costs.py:338-349)
    world = demo_world()
    record("world", ck.world_collision_cost(arm7, "q", world, eta=0.08), [(q,) for q in qs])
    record("self", ck.self_collision_cost(arm7, "q", eta=0.05), [(q,) for q in qs])
    record("swept", ck.swept_collision_cost(arm7, "a", "b", world, eta=0.08), list(zip(qs, q2)))
    record("world_hard", ck.world_collision_cost(arm7, "q", world, eta=0.3, hard_min=True), [(q,) for q in qs])
    record("manip", ck.manipulability_cost(arm7, "q", "flange"), [(q,) for q in qs])
    p2r = robot.load_robot(os.path.join(ROBOTS, "planar_2r.urdf"), os.path.join(ROBOTS, "planar_2r.sidecar.json"))
    q2r = np.stack([p2r.sample_configuration(rng) for _ in range(N)])
    g["q_p2r"] = q2r
    record("manip_p2r", ck.manipulability_cost(p2r, "q", "ee"), [(q,) for q in q2r])
    jd = [robot.translational_jacobian_with_derivative(arm7, q, "flange") for q in qs]
    g["tjac"], g["tdjac"] = np.stack([a for a, _ in jd]), np.stack([b for _, b in jd])
    record("self_wide", ck.self_collision_cost(arm7, "q", eta=0.3), [(q,) for q in qs])
    record("self_hard", ck.self_collision_cost(arm7, "q", eta=0.3, hard_min=True), [(q,) for q in qs])

    # mimic + prismatic chain (arm7_gripper) and a tree (the humanoid fixture of this repo)
    grip = robot.load_robot(os.path.join(ROBOTS, "arm7_gripper.urdf"))
    qg = np.stack([grip.sample_configuration(rng) for _ in range(N)])
    g["q_grip"] = qg
    tg_grip = robot.link_transform(grip, grip.sample_configuration(rng), "finger_right")
    g["target_grip"] = np.concatenate([tg_grip.rotation.wxyz, tg_grip.translation])
    record("pose_grip", ck.pose_cost(grip, "q", "finger_right", tg_grip), [(q,) for q in qg])
    record("manip_grip", ck.manipulability_cost(grip, "q", "finger_right"), [(q,) for q in qg])
    hum = robot.load_robot(HUMANOID)
    qh = np.stack([hum.sample_configuration(rng) for _ in range(N)])
    g["q_hum"] = qh
    tg_hum = robot.link_transform(hum, hum.sample_configuration(rng), "left_hand")
    g["target_hum"] = np.concatenate([tg_hum.rotation.wxyz, tg_hum.translation])
    bh = [Transform3(Rotation3.exp(rng.normal(size=3) * 0.3), rng.normal(size=3)) for _ in range(N)]
    g["base_hum"] = np.array([np.concatenate([b.rotation.wxyz, b.translation]) for b in bh])
    record("pose_hum_se3", ck.pose_cost(hum, "q", "left_hand", tg_hum, base_var="b"), list(zip(qh, bh)))
    # humanoid IK with a planar floating base: 4 end-effector poses, SE(2) base, limit + rest (reference solve)
    hh, hq, hb, hit, htg = [], [], [], [], []
    ees = ["left_hand", "right_hand", "left_foot", "right_foot"]
    for i in range(3):
        qt = hum.sample_configuration(rng)
        bt = Transform2(rng.uniform(-0.5, 0.5), rng.normal(size=2) * 0.3).to_transform3()
        tgts = [bt.compose(robot.link_transform(hum, qt, e)) for e in ees]
        vs = solver.VariableSet.of(q=hum.rest_pose.copy(), b=Transform2.identity())
        prob = solver.Problem(vs, [ck.pose_cost(hum, "q", e, t, base_var="b", position_weight=50,
                                                orientation_weight=10) for e, t in zip(ees, tgts)]
                              + [ck.limit_cost(hum, "q", weight=100), ck.rest_cost("q", hum.rest_pose, weight=0.01)])
        rep = solver.solve(prob, solver.SolveOptions(max_iterations=40))
        h = np.full(41, np.nan)
        h[:len(rep.cost_history)] = rep.cost_history
        hh.append(h)
        hq.append(rep.final_values.value("q"))
        b = rep.final_values.value("b")
        hb.append([b.angle, *b.translation])
        hit.append(rep.iterations_run)
        htg.append(np.stack([np.concatenate([t.rotation.wxyz, t.translation]) for t in tgts]))
    g["hum_base_targets"], g["hum_base_hist"], g["hum_base_q"] = np.array(htg), np.array(hh), np.array(hq)
    g["hum_base_b"], g["hum_base_iters"] = np.array(hb), np.array(hit)

    # solver.assemble on a mixed two-variable problem (pose with SE(2) base + limit + rest)
    vs = solver.VariableSet.of(q=qs[0].copy(), b=b2[0])
    prob = solver.Problem(vs, [ck.pose_cost(arm7, "q", "flange", target, base_var="b", position_weight=50,
                                            orientation_weight=10),
                               ck.limit_cost(arm7, "q", weight=100), ck.rest_cost("q", arm7.rest_pose, weight=0.01)])
    r, jac = solver.assemble(prob, vs)
    g["assemble_r"], g["assemble_j"] = r, jac.to_dense()

    # solve with a base variable: targets out of reach of the fixed base (test_tasks.py:110-121 spirit)
    for kind in ("se2", "se3"):
        hist, fq, fb, iters, costs = [], [], [], [], []
        for i in range(4):
            tq = arm7.sample_configuration(rng)
            shift = np.array([rng.uniform(-1.5, 1.5), rng.uniform(-1.5, 1.5), 0.0])
            tgt = robot.link_transform(arm7, tq, "flange")
            tgt = Transform3(tgt.rotation, tgt.translation + shift)
            base0 = Transform2.identity() if kind == "se2" else Transform3.identity()
            vs = solver.VariableSet.of(q=arm7.rest_pose.copy(), b=base0)
            prob = solver.Problem(vs, [ck.pose_cost(arm7, "q", "flange", tgt, base_var="b", position_weight=50,
                                                    orientation_weight=10),
                                       ck.limit_cost(arm7, "q", weight=100),
                                       ck.rest_cost("q", arm7.rest_pose, weight=0.01)])
            rep = solver.solve(prob, solver.SolveOptions(max_iterations=60))
            h = np.full(61, np.nan)
            h[:len(rep.cost_history)] = rep.cost_history
            hist.append(h)
            fq.append(rep.final_values.value("q"))
            b = rep.final_values.value("b")
            fb.append([b.angle, *b.translation] if kind == "se2" else np.concatenate([b.rotation.wxyz, b.translation]))
            iters.append(rep.iterations_run)
            costs.append(np.concatenate([tgt.rotation.wxyz, tgt.translation]))
        g[f"solve_{kind}_targets"] = np.array(costs)
        g[f"solve_{kind}_hist"], g[f"solve_{kind}_q"] = np.array(hist), np.array(fq)
        g[f"solve_{kind}_b"], g[f"solve_{kind}_iters"] = np.array(fb), np.array(iters)
    np.savez_compressed(OUT, **g)
    print(OUT, len(g), "arrays")


if __name__ == "__main__":
    main()
