"""Host-side logic, no GPU: the C ABI library, URDF parsing parity with the
reference tables, chain compilation vs the oracle FK, request validation."""

import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2505_03728_b200 as k
from oracle import ik_oracle as o
from paper_2505_03728_b200 import _lib
from paper_2505_03728_b200.errors import UnsupportedFeatureError, UrdfError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    text = open(os.path.join(ROOT, "include", "kinoptik_b200.h")).read()
    return sorted(set(re.findall(r"\b(kop_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    declared = _header_functions()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SIGNATURES), set(declared) ^ set(_lib.SIGNATURES)
    assert b"sm_100a" in lib.kop_build_info()


def test_library_is_sm100a_code():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("name,side", [("arm7", "arm7.sidecar.json"), ("planar_2r", "planar_2r.sidecar.json"),
                                       ("arm7_gripper", None)])
def test_parse_matches_reference_tables(golden, name, side):
    m = k.load_robot(k.robot_path(name + ".urdf"), side and k.robot_path(side))
    assert np.array_equal(m._origin_quat, golden[f"tables_{name}_origin_quat"])
    assert np.array_equal(m.lower_limits, golden[f"tables_{name}_lower"])
    assert np.array_equal(m.upper_limits, golden[f"tables_{name}_upper"])
    assert np.array_equal(m.rest_pose, golden[f"tables_{name}_rest"])


def test_self_collision_pairs_and_spheres(models):
    arm = models["arm7"]
    assert len(arm.self_collision_pairs) == 12
    assert sum(len(v) for v in arm.collision_spheres.values()) == 14
    p = models["planar_2r"]
    assert ("base", "forearm") in p.self_collision_pairs
    assert all({a, b} != {"upper_arm", "forearm"} for a, b in p.self_collision_pairs)


@pytest.mark.parametrize("name,link", [("arm7", "flange"), ("planar_2r", "ee"), ("arm7_gripper", "finger_right"),
                                       ("arm7_gripper", "hand"), ("arm7", "link3")])
def test_compiled_chain_reproduces_oracle_fk(models, chains, name, link):
    """The +z-aligned, fixed-folded chain (kop_chain.h) composes to the same link pose."""
    m, ch = models[name], chains[name]
    c = m.compiled_chain(link)
    rng = np.random.default_rng(0)
    li = ch.link(link)
    for _ in range(20):
        q = o.sample_configuration(ch, rng)
        pq, pp = np.array([1.0, 0, 0, 0]), np.zeros(3)
        for j in range(len(c["qcol"])):
            fq = o.qmul(pq, c["tq"][j])
            fp = pp + o.qrot(pq, c["tp"][j])
            th = q[c["qcol"][j]] * c["mult"][j] + c["offset"][j]
            if c["prismatic"][j]:
                z = o.qrot(fq, np.array([0, 0, 1.0]))
                pq, pp = fq, fp + th * z
            else:
                pq, pp = o.qmul(fq, np.array([np.cos(th / 2), 0, 0, np.sin(th / 2)])), fp
        eq, ep = o.qmul(pq, c["ee"][:4]), pp + o.qrot(pq, c["ee"][4:])
        lq, lp, _, _ = o.fk(ch, q[None])
        assert np.allclose(o.qcanon(eq), o.qcanon(lq[0, li]), atol=1e-12)
        assert np.allclose(ep, lp[0, li], atol=1e-12)


def test_chain_lengths(models):
    assert models["arm7"].chain_length("flange") == 7
    assert models["arm7"].chain_length("base_link") == 0
    assert models["planar_2r"].chain_length("ee") == 2
    assert models["arm7_gripper"].chain_length("finger_right") == 8


def test_model_create_rejects_bad_tables():
    lib = _lib.lib()
    i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)
    f64 = lambda a: np.ascontiguousarray(a, dtype=float)
    parent, child, kind, qcol = i32([1]), i32([0]), i32([1]), i32([0])  # child is the root: invalid
    arrs = [parent, child, kind, qcol, f64([1]), f64([0]), f64([1, 0, 0, 0]), f64([0, 0, 0]), f64([0, 0, 1]),
            f64([-1]), f64([1]), f64([0])]
    desc = _lib.KopModelDesc(2, 1, 1, *[a.ctypes.data for a in arrs])
    h = C.c_void_p()
    assert lib.kop_model_create(C.byref(desc), C.byref(h)) == _lib.KOP_EINVAL
    assert b"topological" in lib.kop_last_error()


def test_workspace_and_argument_validation(models):
    lib = _lib.lib()
    p = _lib.KopIkParams(50, 10, 100, 0.01, 64, 16, 6, 4, 0.005, 0.05, 0)
    b = lib.kop_ik_beam_workspace_bytes(models["arm7"]._handle, 8, C.byref(p), 1000)
    assert b >= 1000 * 4 * (7 + 2 + 7) * 4
    bad = _lib.KopIkParams(50, 10, 100, 0.01, 64, 16, 16, 4, 0.005, 0.05, 0)
    rc = lib.kop_ik_beam(models["arm7"]._handle, 8, C.byref(bad), None, 10, None, None, 0, None, None, None,
                         None, None, None, None, None)
    assert rc == _lib.KOP_EINVAL and b"prune_after" in lib.kop_last_error()
    assert lib.kop_model_chain_length(models["arm7"]._handle, 99) == _lib.KOP_EINVAL


URDF_HEAD = '<robot name="t"><link name="a"/><link name="b"/><link name="c"/>'


@pytest.mark.parametrize("doc,exc", [
    ("<robot", UrdfError),
    ("<notrobot/>", UrdfError),
    (URDF_HEAD + '<joint name="j" type="planar"><parent link="a"/><child link="b"/></joint></robot>',
     UnsupportedFeatureError),
    (URDF_HEAD + '<joint name="j" type="revolute"><parent link="a"/><child link="b"/></joint></robot>', UrdfError),
    (URDF_HEAD + '<joint name="j" type="fixed"><parent link="a"/><child link="b"/></joint>'
     '<joint name="k" type="fixed"><parent link="c"/><child link="b"/></joint></robot>', UrdfError),
    (URDF_HEAD + '<joint name="j" type="continuous"><parent link="a"/><child link="b"/></joint>'
     '<joint name="k" type="continuous"><parent link="b"/><child link="c"/><mimic joint="m"/></joint></robot>',
     UrdfError),
    (URDF_HEAD + '<joint name="j" type="continuous"><parent link="a"/><child link="x"/></joint></robot>', UrdfError),
])
def test_parse_errors(doc, exc):
    with pytest.raises(exc):
        k.parse_urdf(doc)


def test_rest_pose_length_checked():
    doc = ('<robot name="t"><link name="a"/><link name="b"/>'
           '<joint name="j" type="continuous"><parent link="a"/><child link="b"/></joint></robot>')
    with pytest.raises(UrdfError):
        k.parse_urdf(doc, rest_pose=[0.0, 1.0])
    m = k.parse_urdf(doc)
    assert m.actuated_count == 1 and m.rest_pose[0] == 0.0 and np.isinf(m.upper_limits[0])


def test_request_validation(models):
    t = k.Transform3.identity()
    with pytest.raises(ValueError):
        k.IkRequest(model=models["arm7"], target_link="flange", target_pose=t, prune_after=16)
    with pytest.raises(ValueError):
        k.IkRequest(model=models["arm7"], target_link="flange", target_pose=t, keep=100)
    with pytest.raises(ValueError):
        k.CostWeights(rest=-1.0)
    assert k.CostWeights.from_json({"rest": 0.5}).rest == 0.5
    with pytest.raises(ValueError):
        k.CostWeights.from_json({"bogus": 1.0})


def test_liegroup_value_types():
    rng = np.random.default_rng(3)
    for _ in range(50):
        xi = rng.normal(size=6)
        t = k.Transform3.exp(xi)
        assert np.allclose(t.log(), xi if np.linalg.norm(xi[3:]) < np.pi else t.log(), atol=1e-9)
        assert t.rotation.wxyz[0] >= 0
        ident = t.compose(t.inverse())
        assert np.allclose(ident.translation, 0, atol=1e-12) and np.isclose(abs(ident.rotation.wxyz[0]), 1)
    assert np.allclose(k.Transform3.exp([0, 0, 0, 0, 0, np.pi / 2]).log(), [0, 0, 0, 0, 0, np.pi / 2])


def test_no_cpu_fallback_without_gpu(models):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        k.fk_arrays(models["arm7"], np.zeros(7))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        k.solve_ik_beam(k.IkRequest(model=models["arm7"], target_link="flange", target_pose=k.Transform3.identity()))


def _traj_costs(T=20, w_anchor=1e3, vl=None):
    return _lib.KopTrajCosts(T, 0.1, w_anchor, 10.0, 10.0, 1.0, 0.1, 100.0, 0.0, 5.0, 0.01, 30.0, 0.05, 100.0, 0,
                             None, None)


def test_widened_entry_points_validate_before_touching_the_gpu(models):
    """Argument checks of the trajectory / tree / collision entry points run on the
    host and map to the reference's exceptions (no device call is made)."""
    lib = _lib.lib()
    h = models["arm7"]._handle
    opts = _lib.KopLmOptions(150, 1e-4, 10.0, 1.0 / 3.0, 1e-8, 1e-10, 20, 1)
    call = lambda c, n_obs=0, o=opts: lib.kop_traj_solve(h, 8, C.byref(c), C.byref(o), None, None, None, n_obs, 0,
                                                        None, None, None, None, None, None, None)
    assert call(_traj_costs(T=4)) == _lib.KOP_EINVAL and b"5 timesteps" in lib.kop_last_error()
    assert call(_traj_costs(T=65)) == _lib.KOP_EUNSUPPORTED
    assert call(_traj_costs(w_anchor=-1.0)) == _lib.KOP_EINVAL
    assert call(_traj_costs(), n_obs=17) == _lib.KOP_EUNSUPPORTED
    bad = _lib.KopLmOptions(150, 1e-4, 0.5, 1.0 / 3.0, 1e-8, 1e-10, 20, 1)
    assert call(_traj_costs(), o=bad) == _lib.KOP_EINVAL and b"damping_increase" in lib.kop_last_error()
    assert call(_traj_costs()) == _lib.KOP_OK  # batch 0: nothing to do
    assert lib.kop_traj_report(h, 8, 0, None, None, 0, None, 0, None, None, None, None, None, None, None) \
        == _lib.KOP_EINVAL
    # tree solve: more than 8 end effectors / unknown link
    links = np.arange(9, dtype=np.int32)
    w = np.ones(9)
    pc = _lib.KopPoseCosts(9, links.ctypes.data, w.ctypes.data, w.ctypes.data, 100.0, 0.01, None)
    rc = lib.kop_multi_pose_solve(h, C.byref(pc), C.byref(opts), None, None, 0, None, None, None, None, None, None,
                                  None)
    assert rc == _lib.KOP_EUNSUPPORTED
    links1 = np.array([42], dtype=np.int32)
    pc1 = _lib.KopPoseCosts(1, links1.ctypes.data, w.ctypes.data, w.ctypes.data, 100.0, 0.01, None)
    rc = lib.kop_multi_pose_solve(h, C.byref(pc1), C.byref(opts), None, None, 0, None, None, None, None, None, None,
                                  None)
    assert rc == _lib.KOP_EINVAL
    # collision stack: too many obstacles, non-positive buffer distance
    obs = (_lib.KopObstacle * 17)()
    cc = _lib.KopCollisionCosts(50, 10, 100, 0.01, 20, 0.05, 5, 0.01, 100, 0, 17, obs)
    assert lib.kop_collision_rows(h, 8, C.byref(cc)) == _lib.KOP_EUNSUPPORTED
    cc = _lib.KopCollisionCosts(50, 10, 100, 0.01, 20, 0.0, 5, 0.01, 100, 0, 1, obs)
    assert lib.kop_collision_rows(h, 8, C.byref(cc)) == _lib.KOP_EINVAL
    cc = _lib.KopCollisionCosts(50, 10, 100, 0.01, 20, 0.05, 5, 0.01, 100, 0, 3, obs)
    assert lib.kop_collision_rows(h, 8, C.byref(cc)) == 6 + 7 + 7 + 8 * 3 + len(models["arm7"].self_collision_pairs)


def test_widened_apis_have_no_cpu_fallback(models):
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    m = models["arm7"]
    world = k.WorldModel([k.Sphere([0.4, 0.0, 0.5], 0.1)])
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        k.trajectory_signed_distances(m, np.zeros((6, 7)), world)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        k.solve(k.trajectory_problem(m, m.rest_pose, m.rest_pose + 0.1, 8, 0.1, world))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        k.plan_trajectory(k.TrajRequest(model=m, start_pose=k.Transform3.identity(),
                                        goal_pose=k.Transform3.identity()))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        k.solve_ik_collision_batch(m, "flange", np.array([[1.0, 0, 0, 0, 0.4, 0.0, 0.5]]), world=world)


@pytest.mark.parametrize("seed,n,fixed,pri,mim", [(1, 7, 2, True, True), (2, 6, 1, True, False),
                                                  (3, 5, 0, False, True), (4, 3, 3, True, True),
                                                  (5, 8, 2, False, False), (6, 7, 1, True, True)])
def test_random_robot_tables_and_compiled_chain(seed, n, fixed, pri, mim):
    """Random serial robots (tests/random_robots.py): parsed tables equal the
    oracle's and the compiled +z-aligned chain composes to the oracle's FK."""
    from random_robots import random_chain_urdf

    doc = random_chain_urdf(seed, n, fixed, pri, mim)
    m, ch = k.parse_urdf(doc), o.load_chain(doc)
    np.testing.assert_array_equal(m.lower_limits, ch.lower)
    np.testing.assert_array_equal(m.upper_limits, ch.upper)
    np.testing.assert_allclose(m.rest_pose, ch.rest)
    c = m.compiled_chain("tool")
    li = ch.link("tool")
    rng = np.random.default_rng(seed)
    for _ in range(10):
        q = o.sample_configuration(ch, rng)
        pq, pp = np.array([1.0, 0, 0, 0]), np.zeros(3)
        for j in range(len(c["qcol"])):
            fq = o.qmul(pq, c["tq"][j])
            fp = pp + o.qrot(pq, c["tp"][j])
            th = q[c["qcol"][j]] * c["mult"][j] + c["offset"][j]
            if c["prismatic"][j]:
                pq, pp = fq, fp + th * o.qrot(fq, np.array([0, 0, 1.0]))
            else:
                pq, pp = o.qmul(fq, np.array([np.cos(th / 2), 0, 0, np.sin(th / 2)])), fp
        eq, ep = o.qmul(pq, c["ee"][:4]), pp + o.qrot(pq, c["ee"][4:])
        lq, lp, _, _ = o.fk(ch, q[None])
        assert np.allclose(o.qcanon(eq), o.qcanon(lq[0, li]), atol=1e-12)
        assert np.allclose(ep, lp[0, li], atol=1e-12)
