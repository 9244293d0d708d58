"""Trajectory optimisation (config 5) on the device vs the oracle and the
reference plan_trajectory goldens (run on a B200: -m gpu).

Bars: the FP64 device solve from the reference's anchors follows the
reference cost history within 1e-8 relative (iteration count within one: the
last steps sit at roundoff, where the reference's own termination flips
between step / damping), final trajectories within 1e-6 rad; the FP64 report
kernel reproduces trajectory_signed_distances within 1e-12 m; FP32 reaches a
final cost within 1% of FP64 and the same collision verdict; the end-to-end
plan_trajectory reproduces the reference's success / collision-free verdicts
on the golden scenes.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2505_03728_b200 as k  # noqa: E402
from conftest import robot_file  # noqa: E402
from oracle import collision_oracle as co  # noqa: E402
from oracle import traj_oracle as to  # noqa: E402
from paper_2505_03728_b200.liegroups import Transform3  # noqa: E402

CASES = ["scene0", "scene1", "scene2", "empty"]


@pytest.fixture(scope="module")
def arm7():
    return k.load_robot(robot_file("arm7.urdf"), robot_file("arm7.sidecar.json"))


def _case(gt, name):
    g = lambda s: gt[f"traj_{name}_{s}"]
    obs = g("obstacles")
    return g, int(g("T")), obs, obs.shape[0]


def _solve(arm7, gt, names, precision="fp64", q_init=None):
    g0, T, _, _ = _case(gt, names[0])
    planner = k.TrajectoryPlanner(arm7, "flange", timesteps=T, precision=precision)
    n_obs = max(_case(gt, nm)[3] for nm in names)
    table = np.tile(k.collision.NULL_OBSTACLE_ROW, (len(names), max(n_obs, 1), 1))[:, :n_obs]
    anchors = []
    for i, nm in enumerate(names):
        g, _, obs, m = _case(gt, nm)
        table[i, :m] = obs
        anchors.append([g("q_start"), g("q_goal")])
    out = planner.solve_anchored_device(np.array(anchors), table, n_obs, q_init=q_init)
    torch.cuda.synchronize()
    return {kk: v.cpu().numpy() for kk, v in out.items() if v is not None}, table, n_obs


@pytest.mark.parametrize("precision,tol,gtol", [("fp64", 1e-12, 1e-9), ("fp32", 2e-4, 0.05)])
@pytest.mark.parametrize("name", CASES)
def test_traj_normal_equations_match_reference(arm7, golden_traj, name, precision, tol, gtol):
    """Cost, J^T r and J^T J at the straight line vs the reference's assemble.
    Interior gradient entries are sums of stencil / smoothness terms of size
    ~1e4 that cancel to ~0 on a straight line, so they get an absolute bar
    (gtol) at the arithmetic's epsilon times that term size."""
    g, T, obs, n_obs = _case(golden_traj, name)
    planner = k.TrajectoryPlanner(arm7, "flange", timesteps=T, precision=precision)
    line = to.straight_line(g("q_start"), g("q_goal"), T)
    cost, grad, hess = planner.normal_equations_device(line[None], np.array([[g("q_start"), g("q_goal")]]),
                                                       obs[None], n_obs)
    r0 = g("r0")
    np.testing.assert_allclose(cost[0].item(), r0 @ r0, rtol=tol)
    np.testing.assert_allclose(grad[0].cpu().numpy(), g("grad0"), rtol=tol, atol=gtol)
    np.testing.assert_allclose(hess[0].cpu().numpy(), g("h0"), rtol=0, atol=tol * np.abs(g("h0")).max())


@pytest.mark.parametrize("name", CASES)
def test_traj_solve_fp64_matches_reference(arm7, golden_traj, name):
    g, T, obs, _ = _case(golden_traj, name)
    out, _, _ = _solve(arm7, golden_traj, [name])
    ref = g("hist")[~np.isnan(g("hist"))]
    iters = int(out["iterations"][0])
    hist = out["history"][0][:iters + 1]
    assert np.isnan(out["history"][0][iters + 1:]).all()
    m = min(len(hist), len(ref))
    np.testing.assert_allclose(hist[:m], ref[:m], rtol=1e-8)
    # extra / missing accepted steps are allowed only once the cost has stalled at roundoff
    if abs(iters - int(g("iters"))) > 1:
        tail = np.concatenate([hist[m - 1:], ref[m - 1:]])
        assert np.ptp(tail) <= 1e-10 * ref[-1]
    np.testing.assert_allclose(out["cost"][0], float(g("cost")), rtol=1e-8)
    np.testing.assert_allclose(out["qs"][0], g("qs"), atol=1e-6)
    np.testing.assert_allclose(out["initial_cost"][0], ref[0], rtol=1e-12)


def test_traj_solve_batch_independent(arm7, golden_traj):
    """Two T=20 scenes solved together == solved alone (CTA per trajectory)."""
    both, _, _ = _solve(arm7, golden_traj, ["scene0", "scene1", "scene0"])
    for i, nm in enumerate(["scene0", "scene1", "scene0"]):
        alone, _, _ = _solve(arm7, golden_traj, [nm])
        np.testing.assert_array_equal(both["qs"][i], alone["qs"][0])
        np.testing.assert_array_equal(both["iterations"][i], alone["iterations"][0])


def test_traj_explicit_init_equals_straight_line(arm7, golden_traj):
    g, T, _, _ = _case(golden_traj, "scene1")
    line = to.straight_line(g("q_start"), g("q_goal"), T)[None]
    a, _, _ = _solve(arm7, golden_traj, ["scene1"])
    b, _, _ = _solve(arm7, golden_traj, ["scene1"], q_init=line)
    np.testing.assert_array_equal(a["qs"], b["qs"])


@pytest.mark.parametrize("name", ["scene0", "scene1", "scene2"])
def test_traj_fp32_close_to_fp64(arm7, golden_traj, name):
    g, T, obs, n_obs = _case(golden_traj, name)
    f32, table, _ = _solve(arm7, golden_traj, [name], precision="fp32")
    f64, _, _ = _solve(arm7, golden_traj, [name])
    assert f32["cost"][0] <= f64["cost"][0] * 1.01
    h = f32["history"][0][:int(f32["iterations"][0]) + 1]
    assert np.all(np.diff(h) < 0)
    rep = k.trajectory.trajectory_signed_distances_batch(arm7, f32["qs"], table, n_obs, "flange")
    assert (min(rep["min_static"][0].item(), rep["min_swept"][0].item()) >= 0) == bool(g("collision_free"))


@pytest.mark.parametrize("name", ["scene0", "scene1", "scene2"])
def test_traj_report_matches_reference(arm7, golden_traj, name):
    g, T, obs, n_obs = _case(golden_traj, name)
    targets = np.stack([g("pa"), g("pb")])[None]
    rep = k.trajectory.trajectory_signed_distances_batch(arm7, g("qs")[None], obs[None], n_obs, "flange", targets)
    np.testing.assert_allclose(rep["static"][0].cpu().numpy(), g("static"), rtol=0, atol=1e-12)
    np.testing.assert_allclose(rep["swept"][0].cpu().numpy(), g("swept"), rtol=0, atol=1e-12)
    np.testing.assert_allclose(rep["pos_err"][0].cpu().numpy(), g("pos_err"), rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(rep["rot_err"][0].cpu().numpy(), g("rot_err"), rtol=1e-6, atol=1e-12)
    st, sw = k.trajectory_signed_distances(arm7, g("qs"), k.WorldModel([k.Sphere(r[1:4], r[7]) for r in obs]))
    np.testing.assert_allclose(st, g("static"), rtol=0, atol=1e-12)
    np.testing.assert_allclose(sw, g("swept"), rtol=0, atol=1e-12)


def test_traj_report_all_obstacle_kinds(arm7, chains):
    """Capsule / half-space / sphere distances of the report kernel vs the oracle."""
    ch = chains["arm7"]
    sp = co.load_spheres_files(ch, robot_file("arm7.urdf"), robot_file("arm7.sidecar.json"))
    obs_o = [co.sphere([0.45, 0.1, 0.55], 0.12), co.capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
             co.halfspace([0.0, 0.0, 1.0], -0.3)]
    world = k.WorldModel([k.Sphere([0.45, 0.1, 0.55], 0.12), k.Capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
                          k.HalfSpace([0.0, 0.0, 1.0], -0.3)])
    rng = np.random.default_rng(5)
    qs = np.stack([to.straight_line(*(rng.uniform(ch.lower, ch.upper, (2, ch.n))), 12) for _ in range(3)])
    for q in qs:
        st, sw = k.trajectory_signed_distances(arm7, q, world)
        st_o, sw_o = to.signed_distances(ch, sp, obs_o, q)
        np.testing.assert_allclose(st, st_o, rtol=0, atol=1e-12)
        np.testing.assert_allclose(sw, sw_o, rtol=0, atol=1e-12)


def test_traj_device_vs_oracle_capsule_world(arm7, chains, golden_traj):
    """World with a capsule and a half-space (the reference goldens only hold
    spheres): FP64 device solve vs the oracle's solve from the same anchors."""
    ch = chains["arm7"]
    sp = co.load_spheres_files(ch, robot_file("arm7.urdf"), robot_file("arm7.sidecar.json"))
    g, _, _, _ = _case(golden_traj, "scene1")
    qa, qb = g("q_start"), g("q_goal")
    T = 12
    mid = k.link_transform(arm7, 0.5 * (qa + qb), "flange").translation
    world = k.WorldModel([k.Capsule(mid - [0, 0, 0.1], mid + [0, 0, 0.1], 0.05), k.HalfSpace([0, 0, 1.0], -0.2)])
    obs_o = [co.capsule(mid - [0, 0, 0.1], mid + [0, 0, 0.1], 0.05), co.halfspace([0, 0, 1.0], -0.2)]
    tc = to.TrajCosts(timesteps=T)
    qs_o, cost_o, hist_o, iters_o, _ = to.solve_traj(ch, sp, obs_o, to.straight_line(qa, qb, T), qa, qb, tc,
                                                     golden_traj["velocity_limits"])
    planner = k.TrajectoryPlanner(arm7, "flange", timesteps=T)
    table = k.collision.obstacle_rows(world.obstacles)[None]
    out = planner.solve_anchored_device(np.array([[qa, qb]]), table, 2)
    hist = out["history"][0].cpu().numpy()[:int(out["iterations"][0]) + 1]
    m = min(len(hist), len(hist_o))
    np.testing.assert_allclose(hist[:m], hist_o[:m], rtol=1e-8)
    np.testing.assert_allclose(out["cost"][0].item(), cost_o, rtol=1e-8)


@pytest.mark.parametrize("T", [5, 6, 7, 9, 64])
def test_traj_device_vs_oracle_lengths(arm7, chains, golden_traj, T):
    """Trajectory lengths at the edges of the FP64 two-sided factorisation:
    T = 5 (separator only below one top block, no bottom half), 6 / 7 / 9
    (bottom half of 1 / 1 / 2 blocks, odd and even splits) and the maximum
    T = 64.  FP64 device solve vs the oracle's from the same anchors."""
    ch = chains["arm7"]
    sp = co.load_spheres_files(ch, robot_file("arm7.urdf"), robot_file("arm7.sidecar.json"))
    g, _, _, _ = _case(golden_traj, "scene1")
    qa, qb = g("q_start"), g("q_goal")
    mid = k.link_transform(arm7, 0.5 * (qa + qb), "flange").translation
    world = k.WorldModel([k.Sphere(mid + [0.02, 0.0, 0.0], 0.07)])
    obs_o = [co.sphere(mid + [0.02, 0.0, 0.0], 0.07)]
    tc = to.TrajCosts(timesteps=T)
    qs_o, cost_o, hist_o, _, _ = to.solve_traj(ch, sp, obs_o, to.straight_line(qa, qb, T), qa, qb, tc,
                                               golden_traj["velocity_limits"])
    planner = k.TrajectoryPlanner(arm7, "flange", timesteps=T, precision="fp64")
    out = planner.solve_anchored_device(np.array([[qa, qb]]), k.collision.obstacle_rows(world.obstacles)[None], 1)
    hist = out["history"][0].cpu().numpy()[:int(out["iterations"][0]) + 1]
    m = min(len(hist), len(hist_o))
    np.testing.assert_allclose(hist[:m], hist_o[:m], rtol=1e-8)
    np.testing.assert_allclose(out["cost"][0].item(), cost_o, rtol=1e-8)
    np.testing.assert_allclose(out["qs"][0].cpu().numpy(), qs_o, atol=1e-6)


def test_plan_trajectory_end_to_end(arm7, golden_traj):
    """plan_trajectory (endpoint IK + solve + report) on the reference's scenes."""
    reqs = []
    for name in ["scene0", "scene1"]:
        g, T, obs, _ = _case(golden_traj, name)
        world = k.WorldModel([k.Sphere(r[1:4], r[7]) for r in obs])
        pa = Transform3.from_parts(g("pa")[:4], g("pa")[4:])
        pb = Transform3.from_parts(g("pb")[:4], g("pb")[4:])
        reqs.append(k.TrajRequest(model=arm7, start_pose=pa, goal_pose=pb, timesteps=T, dt=0.1, world=world,
                                  rng_seed=3000 + int(name[-1]), target_link="flange"))
    res = k.plan_trajectory_batch(reqs)
    for name, r in zip(["scene0", "scene1"], res):
        g = lambda s: golden_traj[f"traj_{name}_{s}"]
        assert r.collision_free == bool(g("collision_free"))
        assert r.success == bool(g("success"))
        assert r.min_signed_distance >= 0.0
        hist = r.report.cost_history
        assert all(b <= a + 1e-15 for a, b in zip(hist, hist[1:]))
        np.testing.assert_allclose(r.qs, g("qs"), atol=1e-4)
    single = k.plan_trajectory(reqs[1])
    np.testing.assert_array_equal(single.qs, res[1].qs)


def test_plan_trajectory_translation_equivariance(arm7, golden_traj):
    """tests/test_tasks.py:228-254 of the reference: moving base + scene moves nothing in joint space."""
    g, _, obs, _ = _case(golden_traj, "scene1")
    pa = Transform3.from_parts(g("pa")[:4], g("pa")[4:])
    pb = Transform3.from_parts(g("pb")[:4], g("pb")[4:])
    world = k.WorldModel([k.Sphere(r[1:4], r[7]) for r in obs])
    shift = np.array([3.0, -2.0, 0.5])
    r0 = k.plan_trajectory(k.TrajRequest(model=arm7, start_pose=pa, goal_pose=pb, timesteps=15, world=world,
                                         rng_seed=5))
    r1 = k.plan_trajectory(k.TrajRequest(
        model=arm7, start_pose=Transform3(pa.rotation, pa.translation + shift),
        goal_pose=Transform3(pb.rotation, pb.translation + shift), timesteps=15,
        world=k.WorldModel([k.Sphere(s.center + shift, s.radius) for s in world.obstacles]), rng_seed=5,
        base_pose=Transform3.from_parts([1, 0, 0, 0], shift)))
    assert np.max(np.abs(r0.qs - r1.qs)) < 1e-9


def test_plan_trajectory_empty_world_near_linear(arm7, golden_traj):
    g, T, _, _ = _case(golden_traj, "empty")
    pa = Transform3.from_parts(g("pa")[:4], g("pa")[4:])
    pb = Transform3.from_parts(g("pb")[:4], g("pb")[4:])
    r = k.plan_trajectory(k.TrajRequest(model=arm7, start_pose=pa, goal_pose=pb, timesteps=10, dt=0.1))
    assert r.success and r.collision_free and r.min_signed_distance == np.inf
    interp = np.linspace(0, 1, 10)[:, None]
    linear = r.qs[0][None, :] * (1 - interp) + r.qs[-1][None, :] * interp
    assert np.max(np.abs(r.qs - linear)) < 1e-3


def test_plan_trajectory_errors(arm7):
    with pytest.raises(ValueError, match="5 timesteps"):
        k.TrajRequest(model=arm7, start_pose=Transform3.identity(), goal_pose=Transform3.identity(), timesteps=3)
    with pytest.raises(k.UnsupportedFeatureError):
        k.TrajectoryPlanner(arm7, "flange", timesteps=65)
    far = Transform3.from_parts([1, 0, 0, 0], [10.0, 0.0, 0.0])
    near = k.link_transform(arm7, arm7.rest_pose, "flange")
    with pytest.raises(k.PlanningError, match="start"):
        k.plan_trajectory(k.TrajRequest(model=arm7, start_pose=far, goal_pose=near, ik_retries=1))


def test_generic_solve_runs_trajectory_problems(arm7, golden_traj):
    """solver.solve / solve_batch on the Problem plan_trajectory builds (the
    trajectory path of the generic solve) == the planner's launch."""
    g, T, obs, n_obs = _case(golden_traj, "scene1")
    world = k.WorldModel([k.Sphere(r[1:4], r[7]) for r in obs])
    pr = k.trajectory_problem(arm7, g("q_start"), g("q_goal"), T, 0.1, world)
    rep = k.solve(pr, k.SolveOptions(max_iterations=150))
    ref, _, _ = _solve(arm7, golden_traj, ["scene1"])
    qs = np.stack([rep.final_values.value(f"q{t}") for t in range(T)])
    np.testing.assert_array_equal(qs, ref["qs"][0])
    assert rep.iterations_run == int(ref["iterations"][0])
    hist = np.array(rep.cost_history)
    h_ref = g("hist")[~np.isnan(g("hist"))]
    m = min(len(hist), len(h_ref))
    np.testing.assert_allclose(hist[:m], h_ref[:m], rtol=1e-8)
    g0, T0, obs0, _ = _case(golden_traj, "scene0")
    pr0 = k.trajectory_problem(arm7, g0("q_start"), g0("q_goal"), T0, 0.1,
                               k.WorldModel([k.Sphere(r[1:4], r[7]) for r in obs0]))
    reps = k.solve_batch([pr0, pr], k.SolveOptions(max_iterations=150))
    np.testing.assert_array_equal(np.stack([reps[1].final_values.value(f"q{t}") for t in range(T)]), qs)
    np.testing.assert_allclose(reps[0].final_cost, float(g0("cost")), rtol=1e-8)


def test_traj_generic_shape_planar_2r_vs_oracle(models, chains):
    """Padded generic kernel shape (n = 2 < 8 -> NQ = 8, 36-entry diagonal
    blocks) with spheres, a capsule obstacle and self pairs: FP64 device solve
    vs the oracle's from the same anchors."""
    m = models["planar_2r"]
    ch = chains["planar_2r"]
    sp = co.load_spheres_files(ch, robot_file("planar_2r.urdf"), robot_file("planar_2r.sidecar.json"))
    qa, qb = np.array([0.2, 0.4]), np.array([1.4, -0.6])
    T = 14
    mid = k.link_transform(m, 0.5 * (qa + qb), m.link_names[-1]).translation
    world = k.WorldModel([k.Capsule(mid - [0.05, 0.0, 0.2], mid + [0.05, 0.0, 0.2], 0.08)])
    obs_o = [co.capsule(mid - [0.05, 0.0, 0.2], mid + [0.05, 0.0, 0.2], 0.08)]
    tc = to.TrajCosts(timesteps=T)
    with open(robot_file("planar_2r.urdf")) as f:
        vl = to.velocity_limits(ch, f.read())
    qs_o, cost_o, hist_o, _, _ = to.solve_traj(ch, sp, obs_o, to.straight_line(qa, qb, T), qa, qb, tc, vl)
    planner = k.TrajectoryPlanner(m, m.link_names[-1], timesteps=T)
    out = planner.solve_anchored_device(np.array([[qa, qb]]), k.collision.obstacle_rows(world.obstacles)[None], 1)
    hist = out["history"][0].cpu().numpy()[:int(out["iterations"][0]) + 1]
    mlen = min(len(hist), len(hist_o))
    np.testing.assert_allclose(hist[:mlen], hist_o[:mlen], rtol=1e-8)
    np.testing.assert_allclose(out["cost"][0].item(), cost_o, rtol=1e-8)
    np.testing.assert_allclose(out["qs"][0].cpu().numpy(), qs_o, atol=1e-6)
