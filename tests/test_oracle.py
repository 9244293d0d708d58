"""The CPU oracle is pinned to the reference: every check here compares the
oracle (oracle/ik_oracle.py) with golden vectors produced by running the
reference itself (tests/golden/make_golden.py).  Exact equality wherever the
restatement follows the reference's operation order."""

import numpy as np
import pytest

from oracle import ik_oracle as o


@pytest.mark.parametrize("name", ["arm7", "planar_2r", "arm7_gripper"])
def test_fk_matches_reference_bitwise(chains, golden, name):
    ch = chains[name]
    out = o.fk(ch, golden[f"fk_{name}_q"])
    for arr, key in zip(out, ("quat", "pos", "jpos", "jaxis")):
        assert np.array_equal(arr, golden[f"fk_{name}_{key}"]), key
    assert np.array_equal(ch.oq, golden[f"tables_{name}_origin_quat"])
    assert np.array_equal(ch.rest, golden[f"tables_{name}_rest"])
    assert np.array_equal(ch.lower, golden[f"tables_{name}_lower"])


def test_se3_log_and_jr_inv(golden):
    assert np.array_equal(o.se3_log(golden["lie_q"], golden["lie_t"]), golden["lie_log"])
    assert np.array_equal(o.se3_jr_inv(golden["lie_xi"]), golden["lie_jrinv"])


def test_seeds_bitwise(chains, golden):
    assert np.array_equal(o.sample_seeds(chains["arm7"], 64, 77), golden["seeds_arm7_77"])
    assert np.array_equal(o.sample_seeds(chains["arm7"], 16, 3), golden["seeds_arm7_3"])
    assert np.array_equal(o.sample_seeds(chains["planar_2r"], 64, 5), golden["seeds_p2r_5"])


def test_targets_bitwise(chains, golden):
    tq, tt, _ = o.reachable_targets(chains["arm7"], 8, 40, 77)
    assert np.array_equal(tq, golden["targets_arm7_77_wxyz"])
    assert np.array_equal(tt, golden["targets_arm7_77_pos"])


def test_lane_engine_bitwise(chains, golden):
    ch = chains["arm7"]
    iq, it = o.target_inverse(golden["targets_arm7_77_wxyz"][:1], golden["targets_arm7_77_pos"][:1])
    eng = o.LaneEngine(ch, 8, np.repeat(iq, 8, 0), np.repeat(it, 8, 0), o.DEFAULT_WEIGHTS)
    r, j = eng.residuals_and_jacobian(golden["seeds_arm7_77"][:8])
    assert np.array_equal(r, golden["lane_t0_r"]) and np.array_equal(j, golden["lane_t0_jac"])
    eng = o.LaneEngine(ch, 8, np.repeat(iq, 64, 0), np.repeat(it, 64, 0), o.DEFAULT_WEIGHTS)
    st = eng.run(eng.start(golden["seeds_arm7_77"]), 16)
    assert np.array_equal(np.stack(st.hist, 1), golden["lane_t0_hist"])
    assert np.array_equal(st.q, golden["lane_t0_q"])
    assert np.array_equal(st.lam, golden["lane_t0_damping"])


def test_ik_beam_bitwise_40_targets(chains, golden):
    ch = chains["arm7"]
    res = o.ik_beam(ch, 8, golden["targets_arm7_77_wxyz"], golden["targets_arm7_77_pos"], golden["seeds_arm7_77"])
    assert np.array_equal(res.hist, golden["beam_arm7_77_hist"])
    assert np.array_equal(res.q, golden["beam_arm7_77_q"])
    assert np.allclose(res.pos_err, golden["beam_arm7_77_pos"], rtol=1e-12, atol=1e-15)
    assert np.array_equal(res.success, golden["beam_arm7_77_succ"])


def test_ik_beam_unreachable_and_planar(chains, golden):
    ch = chains["arm7"]
    seeds = o.sample_seeds(ch, 64, 0)
    res = o.ik_beam(ch, 8, np.array([[1.0, 0, 0, 0]]), np.array([[10.0, 0.0, 0.5]]), seeds)
    assert np.array_equal(res.hist[0], golden["beam_far_hist"])
    assert not res.success[0] and 8.0 < res.pos_err[0] < 10.0
    p = chains["planar_2r"]
    res = o.ik_beam(p, p.link("ee"), golden["targets_p2r_5_wxyz"], golden["targets_p2r_5_pos"],
                    o.sample_seeds(p, 64, 5))
    assert np.array_equal(res.hist, golden["beam_p2r_5_hist"])


def test_mobile_lane_and_beam_bitwise(chains, golden):
    """Mobile-base lanes (beam.py:98-112, 167-179, 216-221) and solve_ik_mobile."""
    ch = chains["arm7"]
    tq, tt = golden["mobile_targets_wxyz"], golden["mobile_targets_pos"]
    iq, it = o.target_inverse(tq[:1], tt[:1])
    seeds = o.sample_seeds(ch, 64, 2024)
    eng = o.LaneEngine(ch, 8, np.repeat(iq, 8, 0), np.repeat(it, 8, 0), o.DEFAULT_WEIGHTS, use_base=True,
                       base_weight=0.3)
    r, j = eng.residuals_and_jacobian(seeds[:8], golden["mobile_lane_ba"], golden["mobile_lane_bxy"])
    assert np.array_equal(r, golden["mobile_lane_r"]) and np.array_equal(j, golden["mobile_lane_jac"])
    eng = o.LaneEngine(ch, 8, np.repeat(iq, 64, 0), np.repeat(it, 64, 0), o.DEFAULT_WEIGHTS, use_base=True,
                       base_weight=0.3)
    st = eng.run(eng.start(seeds), 16)
    assert np.array_equal(np.stack(st.hist, 1), golden["mobile_lane_hist"])
    assert np.array_equal(st.ba, golden["mobile_lane_base_angle"])
    res = o.ik_beam(ch, 8, tq, tt, seeds, use_base=True, base_weight=0.0)
    assert np.array_equal(res.hist, golden["mobile_hist"])
    assert np.array_equal(res.base, golden["mobile_base"])
    assert np.array_equal(res.success, golden["mobile_succ"])


# ---------------------------------------------------------------------------
# collision rows and the generic LM (oracle/collision_oracle.py)
# ---------------------------------------------------------------------------
from oracle import collision_oracle as co  # noqa: E402

DEMO_WORLD = [co.sphere([0.45, 0.1, 0.55], 0.12), co.capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
              co.halfspace([0.0, 0.0, 1.0], -0.3)]


def _arm7_spheres(chains):
    from conftest import robot_file

    return co.load_spheres_files(chains["arm7"], robot_file("arm7.urdf"), robot_file("arm7.sidecar.json"))


def test_collision_rows_match_reference(chains, golden):
    ch, sp = chains["arm7"], _arm7_spheres(chains)
    assert len(sp.pairs) == 12 and sum(len(v) for v in sp.radii.values()) == 14
    q = golden["col_q"]
    r, J = co.world_rows(ch, sp, DEMO_WORLD, q, 0.05)
    assert np.array_equal(r, golden["col_world_r"]) and np.allclose(J, golden["col_world_j"], rtol=0, atol=1e-15)
    r, J = co.world_rows(ch, sp, DEMO_WORLD, q, 0.08, hard=True)
    assert np.array_equal(r, golden["col_world_hard_r"]) and np.allclose(J, golden["col_world_hard_j"], atol=1e-15)
    r, J = co.self_rows(ch, sp, q, 0.01)
    assert np.array_equal(r, golden["col_self_r"]) and np.array_equal(J, golden["col_self_j"])
    assert (golden["col_world_r"] > 0).any()


def test_generic_lm_matches_reference_solve(chains, golden):
    ch, sp = chains["arm7"], _arm7_spheres(chains)
    names = ["max_iterations", "gradient_converged", "step_converged", "numerical_failure"]
    for i in range(6):
        q, c, h, it, term = co.solve_lm(ch, sp, DEMO_WORLD, 8, golden["targets_arm7_77_wxyz"][i],
                                        golden["targets_arm7_77_pos"][i], ch.rest, co.CollisionCosts())
        gh = golden["colik_hist"][i]
        gh = gh[~np.isnan(gh)]
        assert it == golden["colik_iters"][i] and len(h) == len(gh)
        np.testing.assert_allclose(h, gh, rtol=1e-8)
        np.testing.assert_allclose(q, golden["colik_q"][i], atol=1e-8)
        # the last accepted step of problem 5 sits at the 1e-10 step tolerance: a
        # rounding-level difference may end it one iteration later as a damping failure
        assert names.index(term) == golden["colik_term"][i] or (i == 5 and term == "numerical_failure")


def test_multi_pose_solve_matches_reference_humanoid(golden):
    """Config 3 oracle: 4 pose costs + limit + rest through the classic LM, bitwise."""
    from conftest import robot_file
    from oracle import tree_oracle as to

    ch = o.load_chain_files(robot_file("humanoid29.urdf"))
    lq, lp, _, _ = o.fk(ch, golden["hum_fk_q"])
    assert np.array_equal(lq, golden["hum_fk_quat"]) and np.array_equal(lp, golden["hum_fk_pos"])
    ees = [ch.link(e) for e in ["left_hand", "right_hand", "left_foot", "right_foot"]]
    for i in (0, 3):
        poses = [(ees[e], golden["hum_tw"][i][e], golden["hum_tp"][i][e], 50.0, 10.0) for e in range(4)]
        q, c, h, it, term = to.solve_multi_pose(ch, poses, ch.rest)
        gh = golden["hum_hist"][i]
        assert np.array_equal(np.array(h), gh[~np.isnan(gh)]) and it == golden["hum_iters"][i]


# ---------------------------------------------------------------------------
# config 5: trajectory optimisation (traj_oracle vs reference plan_trajectory)
# ---------------------------------------------------------------------------
from oracle import traj_oracle as to  # noqa: E402

TRAJ_CASES = ["scene0", "scene1", "scene2", "empty"]


def traj_case(chains, gt, name):
    from conftest import robot_file

    ch = chains["arm7"]
    sp = co.load_spheres_files(ch, robot_file("arm7.urdf"), robot_file("arm7.sidecar.json"))
    k = lambda s: gt[f"traj_{name}_{s}"]
    obs = [co.sphere(r[1:4], r[7]) for r in k("obstacles")]
    return ch, sp, obs, to.TrajCosts(timesteps=int(k("T"))), k


def test_traj_velocity_limits(chains, golden_traj):
    from conftest import robot_file

    with open(robot_file("arm7.urdf")) as f:
        vl = to.velocity_limits(chains["arm7"], f.read())
    np.testing.assert_array_equal(vl, golden_traj["velocity_limits"])


@pytest.mark.parametrize("name", TRAJ_CASES)
def test_traj_stack_matches_reference_assemble(chains, golden_traj, name):
    """Cost, gradient J^T r and J^T J of the plan_trajectory Problem at the straight line."""
    ch, sp, obs, tc, k = traj_case(chains, golden_traj, name)
    x0 = to.straight_line(k("q_start"), k("q_goal"), tc.timesteps)
    r, J = to.traj_stack(ch, sp, obs, x0.reshape(-1), k("q_start"), k("q_goal"), tc, golden_traj["velocity_limits"])
    np.testing.assert_allclose(r @ r, k("r0") @ k("r0"), rtol=1e-13)
    np.testing.assert_allclose(J.T @ r, k("grad0"), rtol=0, atol=1e-13 * np.abs(k("grad0")).max())
    np.testing.assert_allclose(J.T @ J, k("h0"), rtol=0, atol=1e-13 * np.abs(k("h0")).max())


@pytest.mark.parametrize("name", TRAJ_CASES)
def test_traj_solve_matches_reference(chains, golden_traj, name):
    ch, sp, obs, tc, k = traj_case(chains, golden_traj, name)
    x0 = to.straight_line(k("q_start"), k("q_goal"), tc.timesteps)
    qs, cost, hist, iters, term = to.solve_traj(ch, sp, obs, x0, k("q_start"), k("q_goal"), tc,
                                                golden_traj["velocity_limits"])
    ref_hist = k("hist")[~np.isnan(k("hist"))]
    m = min(len(hist), len(ref_hist))
    np.testing.assert_allclose(hist[:m], ref_hist[:m], rtol=1e-9)
    # the final iterations sit at roundoff: one accepted step more or less and a
    # step / damping termination swap are the reference's own run-to-run noise
    assert abs(iters - int(k("iters"))) <= 1
    np.testing.assert_allclose(cost, float(k("cost")), rtol=1e-9)
    np.testing.assert_allclose(qs, k("qs"), atol=1e-6)
    st, sw = to.signed_distances(ch, sp, obs, qs)
    if obs:
        np.testing.assert_allclose(st, k("static"), atol=1e-6)
        np.testing.assert_allclose(sw, k("swept"), atol=1e-6)
        st_ref, sw_ref = to.signed_distances(ch, sp, obs, k("qs"))
        np.testing.assert_allclose(st_ref, k("static"), rtol=0, atol=1e-14)
        np.testing.assert_allclose(sw_ref, k("swept"), rtol=0, atol=1e-14)
        assert bool(k("collision_free")) == (min(st.min(), sw.min()) >= 0)


def test_capsule_obstacle_kinds():
    """capsule_obstacle vs collision.py:207-237 on hand-checked cases."""
    c0, c1 = np.array([[0.0, 0.0, 0.0]]), np.array([[1.0, 0.0, 0.0]])
    d, ga, gb = to.capsule_obstacle(c0, c1, 0.1, co.sphere([0.5, 0.3, 0.0], 0.1))
    np.testing.assert_allclose(d, [0.1])
    np.testing.assert_allclose(ga, [[0, -0.5, 0]])
    np.testing.assert_allclose(gb, [[0, -0.5, 0]])
    d, ga, gb = to.capsule_obstacle(c0, c1, 0.1, co.capsule([0.2, 1.0, -1.0], [0.2, 1.0, 1.0], 0.2))
    np.testing.assert_allclose(d, [0.7])
    np.testing.assert_allclose(ga, [[0, -0.8, 0]], atol=1e-15)
    d, ga, gb = to.capsule_obstacle(c0, c1, 0.1, co.halfspace([1.0, 0.0, 0.0], -0.5))
    np.testing.assert_allclose(d, [0.4])
    np.testing.assert_allclose(ga, [[1, 0, 0]])
    np.testing.assert_allclose(gb, [[0, 0, 0]])


def test_host_collision_distance_helpers_match_oracle():
    """collision.sphere_obstacle_distance / capsule_obstacle_distance (host API
    helpers) vs the oracle's restatement of collision.py:192-237."""
    import paper_2505_03728_b200 as k

    rng = np.random.default_rng(8)
    obs = [(k.Sphere([0.3, 0.1, 0.2], 0.1), co.sphere([0.3, 0.1, 0.2], 0.1)),
           (k.Capsule([-0.2, 0.0, 0.1], [0.4, 0.3, 0.5], 0.05), co.capsule([-0.2, 0.0, 0.1], [0.4, 0.3, 0.5], 0.05)),
           (k.HalfSpace([0.0, 0.2, 1.0], -0.1), co.halfspace([0.0, 0.2, 1.0], -0.1))]
    for _ in range(20):
        c0, c1, r = rng.normal(size=3) * 0.4, rng.normal(size=3) * 0.4, 0.07
        for ob, ob_o in obs:
            d, g = k.collision.sphere_obstacle_distance(c0, r, ob)
            d_o, g_o = co.sphere_obstacle(c0[None], np.array([r]), ob_o)
            np.testing.assert_allclose(d, d_o[0], atol=1e-14)
            np.testing.assert_allclose(g, g_o[0], atol=1e-14)
            d, ga, gb = k.collision.capsule_obstacle_distance(c0, c1, r, ob)
            d_o, ga_o, gb_o = to.capsule_obstacle(c0[None], c1[None], r, ob_o)
            np.testing.assert_allclose([d], d_o, atol=1e-14)
            np.testing.assert_allclose(ga, ga_o[0], atol=1e-14)
            np.testing.assert_allclose(gb, gb_o[0], atol=1e-14)


def test_multi_ee_beam_reduces_to_ik_beam(chains, golden):
    """The config-3 multi-end-effector beam oracle with one end effector is the
    single-link IK-Beam restatement (itself bit-equal to the reference goldens)."""
    from oracle import tree_oracle as tro

    ch = chains["arm7"]
    tq, tt = golden["targets_arm7_77_wxyz"][:6], golden["targets_arm7_77_pos"][:6]
    seeds = golden["seeds_arm7_77"]
    one = o.ik_beam(ch, 8, tq, tt, seeds)
    multi = tro.multi_ee_beam(ch, [8], tq[:, None], tt[:, None], seeds, [50.0], [10.0])
    np.testing.assert_array_equal(multi["q"], one.q)
    np.testing.assert_array_equal(multi["hist"], one.hist)
    np.testing.assert_array_equal(multi["pos_err"][:, 0], one.pos_err)
    np.testing.assert_array_equal(multi["success"], one.success)


def test_cholesky_lane_engine_fp64_equals_lu_and_fp32_stays_fp32(chains, golden):
    """The FP32 parity yardstick (CholeskyLaneEngine): in FP64 it follows the reference's LU
    lanes to rounding; in float32 every quantity stays float32 (no silent float64 promotion)."""
    ch = chains["arm7"]
    tq, tt = golden["targets_arm7_77_wxyz"][:3], golden["targets_arm7_77_pos"][:3]
    iq, it = o.target_inverse(tq, tt)
    seeds = golden["seeds_arm7_77"]
    lane_t = np.repeat(np.arange(3), len(seeds))
    ref = o.LaneEngine(ch, 8, iq[lane_t], it[lane_t], o.DEFAULT_WEIGHTS, group=lane_t)
    chol = o.CholeskyLaneEngine(ch, 8, iq[lane_t], it[lane_t], o.DEFAULT_WEIGHTS, group=lane_t)
    q0 = np.tile(seeds, (3, 1))
    h_ref = np.stack(ref.run(ref.start(q0), 16).hist, 1)
    h_chol = np.stack(chol.run(chol.start(q0), 16).hist, 1)
    frac, flip, n, _ = o.history_agreement(h_chol, h_ref, 1e-9, 0.0)
    assert frac == 1.0 and flip < 0.02 and n > 0.95 * h_ref.size
    e32 = o.CholeskyLaneEngine(ch, 8, iq[lane_t], it[lane_t], o.DEFAULT_WEIGHTS, group=lane_t, dtype=np.float32)
    st = e32.run(e32.start(q0.astype(np.float32)), 2)
    assert st.q.dtype == st.cost.dtype == st.lam.dtype == np.float32
    assert all(h.dtype == np.float32 for h in st.hist)


def test_history_agreement_semantics():
    ref = np.array([[10.0, 5.0, 5.0, 4.0], [10.0, 9.0, 8.0, 7.0]])
    dev = np.array([[10.0, 5.0001, 5.0001, 4.5], [10.0, 9.0, 9.0, 7.0]])
    frac, flip, n, first = o.history_agreement(dev, ref, rtol=1e-4, atol=0.0)
    # lane 0 never flips (accept pattern equal), its last step differs; lane 1 flips at step 2
    assert list(first) == [4, 2]
    assert n == 4 + 2 and flip == 0.5
    assert frac == pytest.approx(5 / 6)
