"""Generate golden vectors by running the REFERENCE implementation (read-only).

Run in the build container only (``/root/reference`` does not exist on the GPU
box); the resulting ``reference_golden.npz`` is committed and is what the
oracle and the CUDA parity tests are pinned against.

    python tests/golden/make_golden.py

Every array below comes from calling the reference's own public functions:
``robot.fk_arrays`` (robot.py:404), ``liegroups.se3_log_arrays`` /
``se3_right_jacobian_inv`` (liegroups.py:203-252), ``beam.IkLaneProblem``
(beam.py:71-240), ``tasks.sample_seed_configurations`` (tasks.py:88),
``tasks.solve_ik_beam`` (tasks.py:164) and
``benchmark.generate_reachable_targets`` (benchmark.py:83).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from kinoptik import beam, liegroups, robot, tasks  # noqa: E402
from kinoptik.benchmark import generate_reachable_targets  # noqa: E402
from kinoptik.liegroups import Transform3  # noqa: E402

ROBOTS = os.path.join(REF, "kinoptik", "robots")
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.npz")


def main():
    arm7 = robot.load_robot(os.path.join(ROBOTS, "arm7.urdf"), os.path.join(ROBOTS, "arm7.sidecar.json"))
    p2r = robot.load_robot(os.path.join(ROBOTS, "planar_2r.urdf"), os.path.join(ROBOTS, "planar_2r.sidecar.json"))
    grip = robot.load_robot(os.path.join(ROBOTS, "arm7_gripper.urdf"))
    g = {}
    rng = np.random.default_rng(1234)

    # --- FK on random in-limit configurations (three fixtures) -------------
    for name, m in (("arm7", arm7), ("planar_2r", p2r), ("arm7_gripper", grip)):
        qs = np.stack([m.sample_configuration(rng) for _ in range(32)])
        quat, pos, jp, ja = robot.fk_arrays(m, qs)
        g[f"fk_{name}_q"], g[f"fk_{name}_quat"], g[f"fk_{name}_pos"] = qs, quat, pos
        g[f"fk_{name}_jpos"], g[f"fk_{name}_jaxis"] = jp, ja
        g[f"tables_{name}_lower"], g[f"tables_{name}_upper"] = m.lower_limits, m.upper_limits
        g[f"tables_{name}_rest"] = m.rest_pose
        g[f"tables_{name}_origin_quat"] = m._origin_quat

    # --- SE(3) log and Jr^-1 on twists spanning small to large angles -------
    xi = rng.normal(size=(64, 6))
    xi[:, 3:] *= np.geomspace(1e-9, 3.0, 64)[:, None] / np.linalg.norm(xi[:, 3:], axis=1, keepdims=True)
    quats, trans = [], []
    for x in xi:
        t = Transform3.exp(x)
        quats.append(t.rotation.wxyz)
        trans.append(t.translation)
    quats, trans = np.array(quats), np.array(trans)
    g["lie_q"], g["lie_t"] = quats, trans
    g["lie_log"] = liegroups.se3_log_arrays(quats, trans)
    g["lie_xi"] = xi
    g["lie_jrinv"] = liegroups.se3_right_jacobian_inv(xi)

    # --- seeds and targets ---------------------------------------------------
    g["seeds_arm7_77"] = tasks.sample_seed_configurations(arm7, 64, 77)
    g["seeds_arm7_3"] = tasks.sample_seed_configurations(arm7, 16, 3)
    g["seeds_p2r_5"] = tasks.sample_seed_configurations(p2r, 64, 5)
    targets = generate_reachable_targets(arm7, "flange", 40, 77)
    g["targets_arm7_77_wxyz"] = np.array([t.rotation.wxyz for t in targets])
    g["targets_arm7_77_pos"] = np.array([t.translation for t in targets])

    # --- lane engine: per-step cost of all 64 seeds on target 0 ------------
    t0 = targets[0]
    w = tasks.IkRequest(model=arm7, target_link="flange", target_pose=t0).weights
    prob = beam.IkLaneProblem(arm7, "flange", t0, w.pose_position, w.pose_orientation, w.limit, w.rest)
    st = prob.start_state(g["seeds_arm7_77"])
    st = prob.run(st, 16)
    g["lane_t0_hist"] = np.stack(st.history, axis=1)
    g["lane_t0_q"], g["lane_t0_damping"] = st.q, st.damping
    r, jac = prob.residuals_and_jacobian(g["seeds_arm7_77"][:8])
    g["lane_t0_r"], g["lane_t0_jac"] = r, jac

    # --- full IK-Beam on the first 40 benchmark targets (rng 77) ----------
    rows = {k: [] for k in ("q", "cost", "hist", "pos", "rot", "succ")}
    for t in targets:
        res = tasks.solve_ik_beam(tasks.IkRequest(model=arm7, target_link="flange", target_pose=t, rng_seed=77))
        rows["q"].append(res.q)
        rows["cost"].append(res.report.final_cost)
        rows["hist"].append(res.report.cost_history)
        rows["pos"].append(res.pos_error)
        rows["rot"].append(res.rot_error)
        rows["succ"].append(res.success)
    for k, v in rows.items():
        g[f"beam_arm7_77_{k}"] = np.array(v)

    # --- unreachable target and planar 2R beam ----------------------------
    far = Transform3.from_parts([1, 0, 0, 0], [10.0, 0.0, 0.5])
    res = tasks.solve_ik_beam(tasks.IkRequest(model=arm7, target_link="flange", target_pose=far, rng_seed=0))
    g["beam_far_q"], g["beam_far_pos"], g["beam_far_hist"] = res.q, res.pos_error, np.array(res.report.cost_history)
    p_targets = generate_reachable_targets(p2r, "ee", 8, 5)
    g["targets_p2r_5_wxyz"] = np.array([t.rotation.wxyz for t in p_targets])
    g["targets_p2r_5_pos"] = np.array([t.translation for t in p_targets])
    ph, pp = [], []
    for t in p_targets:
        res = tasks.solve_ik_beam(tasks.IkRequest(model=p2r, target_link="ee", target_pose=t, rng_seed=5))
        ph.append(res.report.cost_history)
        pp.append(res.q)
    g["beam_p2r_5_hist"], g["beam_p2r_5_q"] = np.array(ph), np.array(pp)

    # --- mobile base (beam.py:98-112, 167-179, 216-221; tasks.py:169-180) ----
    from kinoptik.benchmark import disk_translations

    shifts = disk_translations(12, 2.0, 2024)
    g["mobile_shifts_2024"] = disk_translations(50, 2.0, 2024)
    mtargets = generate_reachable_targets(arm7, "flange", 12, 2024)
    g["mobile_targets_wxyz"] = np.array([t.rotation.wxyz for t in mtargets])
    g["mobile_targets_pos"] = np.array([t.translation for t in mtargets]) + shifts
    mq, mh, mp, mr, mb, ms = [], [], [], [], [], []
    for i, t in enumerate(mtargets):
        sh = Transform3(t.rotation, t.translation + shifts[i])
        res = tasks.solve_ik_mobile(tasks.IkRequest(model=arm7, target_link="flange", target_pose=sh,
                                                    rng_seed=2024, optimize_base=True))
        mq.append(res.q)
        mh.append(res.report.cost_history)
        mp.append(res.pos_error)
        mr.append(res.rot_error)
        mb.append([res.base.translation[0], res.base.translation[1], res.base.angle])
        ms.append(res.success)
    for k, v in (("q", mq), ("hist", mh), ("pos", mp), ("rot", mr), ("base", mb), ("succ", ms)):
        g[f"mobile_{k}"] = np.array(v)
    sh0 = Transform3(mtargets[0].rotation, mtargets[0].translation + shifts[0])
    mprob = beam.IkLaneProblem(arm7, "flange", sh0, w.pose_position, w.pose_orientation, w.limit, w.rest,
                               use_base=True, base_reg_weight=0.3)
    seeds24 = tasks.sample_seed_configurations(arm7, 64, 2024)
    ba = np.linspace(-3.0, 3.0, 8)
    bxy = np.stack([np.linspace(-1, 1, 8), np.linspace(0.5, -0.5, 8)], axis=1)
    r, jac = mprob.residuals_and_jacobian(seeds24[:8], ba, bxy)
    g["mobile_lane_ba"], g["mobile_lane_bxy"], g["mobile_lane_r"], g["mobile_lane_jac"] = ba, bxy, r, jac
    st = mprob.run(mprob.start_state(seeds24), 16)
    g["mobile_lane_hist"] = np.stack(st.history, axis=1)
    g["mobile_lane_q"], g["mobile_lane_base_angle"], g["mobile_lane_base_xy"] = st.q, st.base_angle, st.base_xy

    # --- collision rows (costs.py:423-551) and collision-IK solves (solver.py:364) ---
    from kinoptik import collision as col
    from kinoptik import costs as ck
    from kinoptik import solver as sv

    world = col.WorldModel([col.Sphere([0.45, 0.1, 0.55], 0.12), col.Capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
                            col.HalfSpace([0.0, 0.0, 1.0], -0.3)])  # test_costs.py:199-206 demo_world
    crng = np.random.default_rng(4321)
    cq = np.stack([arm7.sample_configuration(crng) for _ in range(24)])
    wc = ck.world_collision_cost(arm7, "q", world, eta=0.05)
    sc = ck.self_collision_cost(arm7, "q", eta=0.01)
    wch = ck.world_collision_cost(arm7, "q", world, eta=0.08, hard_min=True)
    g["col_q"] = cq
    g["col_world_r"] = np.stack([wc.raw_residual([x]) for x in cq])
    g["col_world_j"] = np.stack([wc.jacobian(x)[0] for x in cq])
    g["col_world_hard_r"] = np.stack([wch.raw_residual([x]) for x in cq])
    g["col_world_hard_j"] = np.stack([wch.jacobian(x)[0] for x in cq])
    g["col_self_r"] = np.stack([sc.raw_residual([x]) for x in cq])
    g["col_self_j"] = np.stack([sc.jacobian(x)[0] for x in cq])
    W = ck.CostWeights()
    rows = {k: [] for k in ("q", "cost", "hist", "iters", "term")}
    for t in targets[:6]:
        costs = [ck.pose_cost(arm7, "q", "flange", t, position_weight=W.pose_position,
                              orientation_weight=W.pose_orientation),
                 ck.limit_cost(arm7, "q", weight=W.limit), ck.rest_cost("q", arm7.rest_pose, weight=W.rest),
                 ck.world_collision_cost(arm7, "q", world, weight=W.world_collision),
                 ck.self_collision_cost(arm7, "q", weight=W.self_collision)]
        rep = sv.solve(sv.Problem(sv.VariableSet.of(q=arm7.rest_pose.copy()), costs))
        rows["q"].append(rep.final_values.value("q"))
        rows["cost"].append(rep.final_cost)
        rows["hist"].append(np.pad(rep.cost_history, (0, 101 - len(rep.cost_history)), constant_values=np.nan))
        rows["iters"].append(rep.iterations_run)
        rows["term"].append(["max_iterations", "gradient_converged", "step_converged",
                             "numerical_failure"].index(rep.termination))
    for k, v in rows.items():
        g[f"colik_{k}"] = np.array(v)

    # --- config 3: humanoid multi-EE IK through solver.solve -------------------
    hum = robot.load_robot(os.path.join(os.path.dirname(OUT), "..", "..", "paper_2505_03728_b200", "robots",
                                        "humanoid29.urdf"))
    ees = ["left_hand", "right_hand", "left_foot", "right_foot"]
    hrng = np.random.default_rng(2929)
    hq = np.stack([hum.sample_configuration(hrng) for _ in range(5)])
    g["hum_q_true"] = hq
    g["hum_fk_q"], g["hum_fk_quat"], g["hum_fk_pos"] = hq, *robot.fk_arrays(hum, hq)[:2]
    hrows = {k: [] for k in ("q", "cost", "hist", "iters", "term", "tw", "tp")}
    for qi in hq:
        tgs = [robot.link_transform(hum, qi, e) for e in ees]
        costs = [ck.pose_cost(hum, "q", e, t, position_weight=W.pose_position, orientation_weight=W.pose_orientation)
                 for e, t in zip(ees, tgs)]
        costs += [ck.limit_cost(hum, "q", weight=W.limit), ck.rest_cost("q", hum.rest_pose, weight=W.rest)]
        rep = sv.solve(sv.Problem(sv.VariableSet.of(q=hum.rest_pose.copy()), costs))
        hrows["q"].append(rep.final_values.value("q"))
        hrows["cost"].append(rep.final_cost)
        hrows["hist"].append(np.pad(rep.cost_history, (0, 101 - len(rep.cost_history)), constant_values=np.nan))
        hrows["iters"].append(rep.iterations_run)
        hrows["term"].append(["max_iterations", "gradient_converged", "step_converged",
                              "numerical_failure"].index(rep.termination))
        hrows["tw"].append([t.rotation.wxyz for t in tgs])
        hrows["tp"].append([t.translation for t in tgs])
    for k, v in hrows.items():
        g[f"hum_{k}"] = np.array(v)

    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays")


if __name__ == "__main__":
    main()
