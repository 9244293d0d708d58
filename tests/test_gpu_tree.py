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
from oracle_pool import assert_fp64_beam_parity, par_batched  # noqa: E402

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


def _hum_targets(hum, chh, count, seed):
    rng = np.random.default_rng(seed)
    qt = rng.uniform(chh.lower, chh.upper, (count, chh.n))
    lq, lp, _, _ = o.fk(chh, qt)
    links = [chh.link(e) for e in EES]
    tq = np.stack([o.qcanon(lq[:, l]) for l in links], 1)
    tt = np.stack([lp[:, l] for l in links], 1)
    return links, tq, tt, np.concatenate([tq, tt], axis=2)


def test_tree_ik_beam_fp64_matches_oracle(hum):
    """Multi-EE IK-Beam (config 3, SURVEY H6 flavour) FP64 on the device vs the
    oracle composed of the pinned lane / beam primitives."""
    from oracle import tree_oracle as tro

    chh = o.load_chain_files(k.robot_path("humanoid29.urdf"))
    links, tq, tt, tg = _hum_targets(hum, chh, 128, 5)
    seeds = o.sample_seeds(chh, 64, 3)
    ref = par_batched(tro.multi_ee_beam, chh, links, tq=tq, tt=tt, seeds=seeds, w_pos=[50.0] * 4,
                      w_ori=[10.0] * 4, split=("tq", "tt"))
    got = k.solve_ik_beam_multi(hum, EES, tg, rng_seed=3, precision="fp64")
    assert_fp64_beam_parity(got.history, ref["hist"], ref["diag"])
    rel = np.abs(got.history - ref["hist"]) / ref["hist"]
    same = rel.max(axis=1) < 1e-6
    assert np.array_equal(got.success[same].astype(bool), ref["success"][same])
    np.testing.assert_allclose(got.pos_error[same], ref["pos_err"][same], rtol=1e-4, atol=1e-9)


def test_tree_ik_beam_fp32_and_single_ee(hum, models):
    chh = o.load_chain_files(k.robot_path("humanoid29.urdf"))
    links, tq, tt, tg = _hum_targets(hum, chh, 256, 6)
    r32 = k.solve_ik_beam_multi(hum, EES, tg, rng_seed=3)
    r64 = k.solve_ik_beam_multi(hum, EES, tg, rng_seed=3, precision="fp64")
    assert abs(r32.success.mean() - r64.success.mean()) <= 0.05
    assert np.all(np.diff(r32.history, axis=1) <= 0)
    # one end effector on the Panda chain: the same lanes as the chain IK-Beam
    m = models["arm7"]
    from paper_2505_03728_b200.benchmark import reachable_target_array

    tgt = reachable_target_array(m, "flange", 64, 77).cpu().numpy()
    multi = k.solve_ik_beam_multi(m, ["flange"], tgt[:, None, :], rng_seed=77, precision="fp64")
    chain = k.solve_ik_beam_batch(m, "flange", tgt, rng_seed=77, precision="fp64")
    rel = np.abs(multi.history - chain.history) / chain.history
    assert np.mean(rel.max(axis=1) < 1e-6) >= 0.9
    assert np.mean(multi.success.astype(bool) == chain.success.astype(bool)) >= 0.98


@pytest.mark.parametrize("seed,n", [(21, 32), (22, 13), (23, 1)])
def test_tree_ik_beam_random_chain_lane_edges(seed, n):
    """Tree path at the lane-count edges vs the oracle (FP64): n = 32 fills the
    warp, n = 13 leaves a partial column quad in the vectorised J^T J and in the
    Cholesky's pivot-column broadcasts, n = 1 is a single column."""
    from oracle import tree_oracle as tro
    from random_robots import random_chain_urdf

    doc = random_chain_urdf(seed, n, 2, True, False)
    m = k.parse_urdf(doc)
    ch = o.load_chain(doc)
    assert m.actuated_count == ch.n == n
    li = ch.link("tool")
    rng = np.random.default_rng(seed)
    lo = np.where(np.isfinite(ch.lower), ch.lower, -np.pi)
    hi = np.where(np.isfinite(ch.upper), ch.upper, np.pi)
    lq, lp, _, _ = o.fk(ch, rng.uniform(lo, hi, (32, n)))
    tq = o.qcanon(lq[:, li])[:, None]
    tt = lp[:, li][:, None]
    seeds = o.sample_seeds(ch, 64, 3)
    ref = par_batched(tro.multi_ee_beam, ch, [li], tq=tq, tt=tt, seeds=seeds, w_pos=[50.0], w_ori=[10.0],
                      split=("tq", "tt"))
    got = k.solve_ik_beam_multi(m, ["tool"], np.concatenate([tq, tt], axis=2), rng_seed=3, precision="fp64")
    # one column: many seeds reach the same optimum, so prune / winner choices are exact ties and the
    # winner's early history may be another tied seed's; every divergence must still be such a near-tie
    assert_fp64_beam_parity(got.history, ref["hist"], ref["diag"], frac=0.95 if n > 1 else 0.0)
    np.testing.assert_allclose(got.history[:, -1], ref["hist"][:, -1], rtol=1e-6, atol=1e-12)
    assert np.mean(got.success == ref["success"]) >= 0.95
    r32 = k.solve_ik_beam_multi(m, ["tool"], np.concatenate([tq, tt], axis=2), rng_seed=3)
    assert np.all(np.diff(r32.history, axis=1) <= 0)


def test_tree_solve_32_columns_matches_oracle():
    """solver.solve semantics on the tree path with every warp lane a column
    (n = 32, one pose cost + limit + rest) vs the oracle's classic LM, FP64."""
    from random_robots import random_chain_urdf

    doc = random_chain_urdf(31, 32, 2, True, False)
    m = k.parse_urdf(doc)
    ch = o.load_chain(doc)
    li = ch.link("tool")
    rng = np.random.default_rng(31)
    lo = np.where(np.isfinite(ch.lower), ch.lower, -np.pi)
    hi = np.where(np.isfinite(ch.upper), ch.upper, np.pi)
    lq, lp, _, _ = o.fk(ch, rng.uniform(lo, hi, (1, 32)))
    w = k.CostWeights()
    tgt = k.Transform3.from_parts(lq[0, li], lp[0, li])
    costs = [k.pose_cost(m, "q", "tool", tgt, position_weight=w.pose_position, orientation_weight=w.pose_orientation),
             k.limit_cost(m, "q", weight=w.limit), k.rest_cost("q", m.rest_pose, weight=w.rest)]
    rep = k.solve(k.Problem(k.VariableSet.of(q=np.asarray(m.rest_pose, float).copy()), costs))
    poses = [(li, o.qcanon(lq[0, li]), lp[0, li], w.pose_position, w.pose_orientation)]
    _, c_ref, _, _, _ = to.solve_multi_pose(ch, poses, ch.rest)
    np.testing.assert_allclose(rep.final_cost, c_ref, rtol=1e-5, atol=1e-12)


def test_humanoid_ik_beam_distribution_1000(hum):
    """Config 3 at 1000 target sets: device FP32 (measured mode) and FP64 success rates vs the
    oracle's (54% -- 4 end-effector targets from random in-limit configurations, 16 LM steps)."""
    from oracle import tree_oracle as tro

    chh = o.load_chain_files(k.robot_path("humanoid29.urdf"))
    links, tq, tt, tg = _hum_targets(hum, chh, 1000, 29)
    seeds = o.sample_seeds(chh, 64, 0)
    ref = par_batched(tro.multi_ee_beam, chh, links, tq=tq, tt=tt, seeds=seeds, w_pos=[50.0] * 4,
                      w_ori=[10.0] * 4, split=("tq", "tt"))
    r64 = k.solve_ik_beam_multi(hum, EES, tg, rng_seed=0, precision="fp64")
    r32 = k.solve_ik_beam_multi(hum, EES, tg, rng_seed=0)
    s_ref = ref["success"].mean()
    print(f"\nconfig 3, 1000 targets: oracle success {s_ref:.4f}, device FP64 {r64.success.mean():.4f} "
          f"(per-target agreement {np.mean(r64.success.astype(bool) == ref['success']):.4f}), device FP32 "
          f"{r32.success.mean():.4f}")
    assert np.mean(r64.success.astype(bool) == ref["success"]) >= 0.99
    assert abs(r32.success.mean() - s_ref) <= 0.02
    for a, b in ((r32.pos_error.max(axis=1), ref["pos_err"].max(axis=1)),):
        assert 0.5 * np.percentile(b, 50) <= np.percentile(a, 50) <= 2.0 * np.percentile(b, 50)


# A branched tree with consecutive fixed joints (fx1 -> fx2 before j1, fxA1 -> fxA2
# after the prismatic j2 ending at end effector tipA) and a branch that leaves
# through a fixed joint (fb): the host folds fixed joints into their children's
# origins and the end-effector offsets (kop_capi.cu tree_params).
_LIM = '<limit lower="-2.5" upper="2.5" effort="1" velocity="1"/>'
_FOLD_TREE = (
    '<robot name="fold">'
    + "".join(f'<link name="{n}"/>' for n in ["base", "a", "b", "c", "d", "e", "f", "g", "h", "tipA", "tipB"])
    + f'<joint name="j0" type="revolute"><parent link="base"/><child link="a"/><origin xyz="0 0 0.1" rpy="0.1 0 0.2"/><axis xyz="0 0 1"/>{_LIM}</joint>'
    + '<joint name="fx1" type="fixed"><parent link="a"/><child link="b"/><origin xyz="0.05 0 0.12" rpy="0.3 0.1 0"/></joint>'
    + '<joint name="fx2" type="fixed"><parent link="b"/><child link="c"/><origin xyz="0 0.04 0.08" rpy="0 -0.2 0.4"/></joint>'
    + f'<joint name="j1" type="revolute"><parent link="c"/><child link="d"/><origin xyz="0 0 0.15" rpy="0 0.3 0"/><axis xyz="0 1 0"/>{_LIM}</joint>'
    + '<joint name="j2" type="prismatic"><parent link="d"/><child link="e"/><origin xyz="0.02 0 0.1" rpy="0 0 0.5"/><axis xyz="0.6 0 0.8"/><limit lower="-0.1" upper="0.2" effort="1" velocity="1"/></joint>'
    + '<joint name="fxA1" type="fixed"><parent link="e"/><child link="f"/><origin xyz="0.03 0.01 0.06" rpy="0.2 0 -0.1"/></joint>'
    + '<joint name="fxA2" type="fixed"><parent link="f"/><child link="tipA"/><origin xyz="0 0 0.05" rpy="0 0.4 0"/></joint>'
    + '<joint name="fb" type="fixed"><parent link="b"/><child link="g"/><origin xyz="-0.04 0.02 0.07" rpy="-0.3 0 0.2"/></joint>'
    + f'<joint name="j3" type="revolute"><parent link="g"/><child link="h"/><origin xyz="0 0 0.12" rpy="0 0 0.3"/><axis xyz="1 0 0"/>{_LIM}</joint>'
    + f'<joint name="j4" type="revolute"><parent link="h"/><child link="tipB"/><origin xyz="0 0.02 0.1" rpy="0.2 0 0"/><axis xyz="0 0.6 0.8"/>{_LIM}</joint>'
    + '</robot>')


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_tree_ik_beam_folded_fixed_joints(prec):
    from oracle import tree_oracle as tro

    m = k.parse_urdf(_FOLD_TREE)
    ch = o.load_chain(_FOLD_TREE)
    ees = ["tipA", "tipB"]
    links = [ch.link(e) for e in ees]
    rng = np.random.default_rng(41)
    lq, lp, _, _ = o.fk(ch, rng.uniform(ch.lower, ch.upper, (48, ch.n)))
    tq = np.stack([o.qcanon(lq[:, li]) for li in links], 1)
    tt = np.stack([lp[:, li] for li in links], 1)
    seeds = o.sample_seeds(ch, 64, 3)
    ref = par_batched(tro.multi_ee_beam, ch, links, tq=tq, tt=tt, seeds=seeds, w_pos=[50.0] * 2,
                      w_ori=[10.0] * 2, split=("tq", "tt"))
    got = k.solve_ik_beam_multi(m, ees, np.concatenate([tq, tt], axis=2), rng_seed=3, precision=prec)
    # reachable targets and 5 columns: most seeds reach the same minimum, so prune / winner
    # choices are exact ties (as for the one-column chain above) -- every divergence must be one
    if prec == "fp64":
        assert_fp64_beam_parity(got.history, ref["hist"], ref["diag"], frac=0.0)
        np.testing.assert_allclose(got.history[:, -1], ref["hist"][:, -1], rtol=1e-6, atol=1e-12)
    else:
        assert np.all(got.cost <= ref["hist"][:, -1] * 1.01 + 1e-6)
    assert np.mean(got.success == ref["success"]) >= 0.95


def test_tree_solve_folded_fixed_joints_matches_oracle():
    """solver.solve semantics on the folded tree (two pose costs + limit + rest) vs the
    oracle's classic LM, FP64."""
    m = k.parse_urdf(_FOLD_TREE)
    ch = o.load_chain(_FOLD_TREE)
    rng = np.random.default_rng(43)
    lq, lp, _, _ = o.fk(ch, rng.uniform(ch.lower, ch.upper, (1, ch.n)))
    w = k.CostWeights()
    costs, poses = [], []
    for e in ("tipA", "tipB"):
        li = ch.link(e)
        costs.append(k.pose_cost(m, "q", e, k.Transform3.from_parts(lq[0, li], lp[0, li]),
                                 position_weight=w.pose_position, orientation_weight=w.pose_orientation))
        poses.append((li, o.qcanon(lq[0, li]), lp[0, li], w.pose_position, w.pose_orientation))
    costs += [k.limit_cost(m, "q", weight=w.limit), k.rest_cost("q", m.rest_pose, weight=w.rest)]
    rep = k.solve(k.Problem(k.VariableSet.of(q=np.asarray(m.rest_pose, float).copy()), costs))
    _, c_ref, _, _, _ = to.solve_multi_pose(ch, poses, ch.rest)
    np.testing.assert_allclose(rep.final_cost, c_ref, rtol=1e-5, atol=1e-12)


@pytest.mark.parametrize("keep", [1, 3, 4])
def test_tree_ik_beam_batch_invariance_odd_batches(hum, keep):
    """Per-target results do not depend on the batch: 37 targets in one call equal
    the same targets split 20 + 17 (odd batches leave stage 2's packed FP32 CTAs
    with an empty target slot), for several keep widths."""
    chh = o.load_chain_files(k.robot_path("humanoid29.urdf"))
    _, _, _, tg = _hum_targets(hum, chh, 37, 9)
    kw = dict(rng_seed=5, keep=keep, precision="fp32")
    full = k.solve_ik_beam_multi(hum, EES, tg, **kw)
    a = k.solve_ik_beam_multi(hum, EES, tg[:20], **kw)
    b = k.solve_ik_beam_multi(hum, EES, tg[20:], **kw)
    for f in ("q", "cost", "history", "pos_error", "rot_error", "success"):
        np.testing.assert_array_equal(getattr(full, f), np.concatenate([getattr(a, f), getattr(b, f)]), err_msg=f)


@pytest.mark.parametrize("rej", [0, 1, 3])
def test_tree_solve_rejection_budget_matches_oracle(rej):
    """The tree solve's rejection loop (one evaluation site, kop_tree.cu) with small
    budgets -- including none -- against the oracle's classic LM (solver.py:389-419),
    FP64: cost history, iteration count and termination."""
    m = k.parse_urdf(_FOLD_TREE)
    ch = o.load_chain(_FOLD_TREE)
    rng = np.random.default_rng(47)
    lq, lp, _, _ = o.fk(ch, rng.uniform(ch.lower, ch.upper, (1, ch.n)))
    w = k.CostWeights()
    costs, poses = [], []
    for e in ("tipA", "tipB"):
        li = ch.link(e)
        costs.append(k.pose_cost(m, "q", e, k.Transform3.from_parts(lq[0, li], lp[0, li]),
                                 position_weight=w.pose_position, orientation_weight=w.pose_orientation))
        poses.append((li, o.qcanon(lq[0, li]), lp[0, li], w.pose_position, w.pose_orientation))
    costs += [k.limit_cost(m, "q", weight=w.limit), k.rest_cost("q", m.rest_pose, weight=w.rest)]
    q0 = np.asarray(m.rest_pose, float).copy()
    rep = k.solve(k.Problem(k.VariableSet.of(q=q0.copy()), costs), k.SolveOptions(max_rejections=rej))
    _, c_ref, hist, iters, term = to.solve_multi_pose(ch, poses, q0, max_rejections=rej)
    assert rep.iterations_run == iters and rep.termination == term
    np.testing.assert_allclose(rep.cost_history, hist, rtol=1e-8, atol=1e-14)


@pytest.mark.parametrize("rej", [0, 1, 3])
def test_chain_solve_rejection_budget_matches_oracle(rej):
    """Same budgets on the chain path (k_col_solve's trial machine: a Panda pose
    problem routes there) against the oracle's classic LM, FP64."""
    m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
    ch = o.load_chain_files(k.robot_path("arm7.urdf"))
    li = ch.link("flange")
    rng = np.random.default_rng(53)
    lq, lp, _, _ = o.fk(ch, rng.uniform(ch.lower, ch.upper, (1, ch.n)))
    w = k.CostWeights()
    costs = [k.pose_cost(m, "q", "flange", k.Transform3.from_parts(lq[0, li], lp[0, li]),
                         position_weight=w.pose_position, orientation_weight=w.pose_orientation),
             k.limit_cost(m, "q", weight=w.limit), k.rest_cost("q", m.rest_pose, weight=w.rest)]
    q0 = np.asarray(m.rest_pose, float).copy()
    rep = k.solve(k.Problem(k.VariableSet.of(q=q0.copy()), costs), k.SolveOptions(max_rejections=rej))
    poses = [(li, o.qcanon(lq[0, li]), lp[0, li], w.pose_position, w.pose_orientation)]
    _, c_ref, hist, iters, term = to.solve_multi_pose(ch, poses, q0, rest=np.asarray(m.rest_pose, float),
                                                      max_rejections=rej)
    assert rep.iterations_run == iters and rep.termination == term
    np.testing.assert_allclose(rep.cost_history, hist, rtol=1e-8, atol=1e-14)
