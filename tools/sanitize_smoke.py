"""Smoke-sized launches of every kernel family, for compute-sanitizer.

    compute-sanitizer --tool racecheck python tools/sanitize_smoke.py [fp32|fp64|both]

Each family runs a handful of problems so that a sanitizer pass (which
serialises and instruments every access) finishes in minutes: IK-Beam
(stage 1 / 2 / errors), lanes, FK, Philox, collision IK-Beam, generic LM
(k_col_solve), tree solve + multi-EE beam, trajectories (+ report), mobile
base, host pipeline.  Prints one line per family; exits non-zero on any
Python-side failure (the sanitizer's own report is on stderr).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2505_03728_b200 as k
from paper_2505_03728_b200 import _device as dv, beam as kbeam, trajectory as ktraj
from paper_2505_03728_b200.benchmark import reachable_target_array
from paper_2505_03728_b200.robot import fk_arrays_device, link_poses_device
from paper_2505_03728_b200.tasks import IkBeamSolver

PRECS = {"fp32": ["fp32"], "fp64": ["fp64"], "both": ["fp32", "fp64"]}[sys.argv[1] if len(sys.argv) > 1 else "both"]
ONLY = set(sys.argv[2].split(",")) if len(sys.argv) > 2 else None

DEMO = k.WorldModel([k.Sphere([0.45, 0.1, 0.55], 0.12), k.Capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
                     k.HalfSpace([0.0, 0.0, 1.0], -0.3)])
m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
hum = k.load_robot(k.robot_path("humanoid29.urdf"))
EES = ["left_hand", "right_hand", "left_foot", "right_foot"]


def pose(a):
    a = a.cpu().numpy() if hasattr(a, "cpu") else a
    return k.Transform3.from_parts(a[:4], a[4:])


def fam(name):
    return ONLY is None or name in ONLY


def done(name, prec):
    torch.cuda.synchronize()
    print(f"ok {name} {prec}", flush=True)


tg = reachable_target_array(m, "flange", 8, 77)
for prec in PRECS:
    if fam("fk"):
        q = dv.to_dev(np.random.default_rng(0).uniform(m.lower_limits, m.upper_limits, (33, 7)))
        fk_arrays_device(m, q, precision=prec)
        done("fk", prec)
    if fam("beam"):
        s = IkBeamSolver(m, "flange", rng_seed=77, precision=prec)
        s.solve_device(tg)
        done("beam", prec)
        # seeds not a multiple of a warp, keep 7
        s = IkBeamSolver(m, "flange", seeds=37, keep=7, rng_seed=3, precision=prec)
        s.solve_device(tg[:5])
        done("beam-ragged", prec)
    if fam("host"):
        s = IkBeamSolver(m, "flange", rng_seed=77, precision=prec)
        s.solve_host(tg.cpu().numpy(), chunk=3, n_streams=2)
        done("host-pipeline", prec)
    if fam("mobile"):
        s = IkBeamSolver(m, "flange", rng_seed=77, precision=prec, optimize_base=True)
        s.solve_device(tg[:4])
        done("mobile", prec)
    if fam("lanes"):
        lp = kbeam.IkLaneProblem(m, "flange", pose(tg[0]), 50, 10, 100, 0.01, precision=prec)
        st = lp.start_state(k.sample_seed_configurations(m, 8, 1))
        lp.run(st, 3)
        done("lanes", prec)
    if fam("collision"):
        s = IkBeamSolver(m, "flange", rng_seed=77, precision=prec, world=DEMO, self_collision=True)
        s.solve_device(tg[:3])
        done("collision-beam", prec)
    if fam("lm"):
        probs = []
        for i in range(5):
            T = pose(tg[i])
            probs.append(k.Problem(k.VariableSet.of(q=m.rest_pose.copy()), [
                k.pose_cost(m, "q", "flange", T, position_weight=50, orientation_weight=10),
                k.limit_cost(m, "q", weight=100), k.rest_cost("q", m.rest_pose, weight=0.01),
                k.world_collision_cost(m, "q", DEMO, weight=20), k.self_collision_cost(m, "q", weight=5)]))
        k.solve_batch(probs, k.SolveOptions(precision=prec, max_iterations=12))
        done("generic-lm", prec)
    if fam("tree"):
        qt = dv.to_dev(np.random.default_rng(29).uniform(hum.lower_limits, hum.upper_limits, (3, hum.actuated_count)))
        tgh = torch.stack([link_poses_device(hum, qt, e) for e in EES], dim=1).contiguous()
        k.solve_ik_beam_multi(hum, EES, tgh, seeds=8, keep=2, precision=prec)
        done("tree-beam", prec)
        probs = []
        th = tgh.cpu().numpy()
        for i in range(3):
            probs.append(k.Problem(k.VariableSet.of(q=hum.rest_pose.copy()),
                                   [k.pose_cost(hum, "q", e, pose(th[i, j]), position_weight=50,
                                                orientation_weight=10) for j, e in enumerate(EES)]
                                   + [k.limit_cost(hum, "q", weight=100), k.rest_cost("q", hum.rest_pose, weight=0.01)]))
        k.solve_batch(probs, k.SolveOptions(precision=prec, max_iterations=8))
        done("tree-solve", prec)
    if fam("traj"):
        rng = np.random.default_rng(5)
        for TT in (20, 64):
            qa = rng.uniform(m.lower_limits, m.upper_limits, (2, 7))
            qb = rng.uniform(m.lower_limits, m.upper_limits, (2, 7))
            mid = link_poses_device(m, dv.to_dev(0.5 * (qa + qb)), "flange").cpu().numpy()[:, 4:7]
            obs = np.zeros((2, 1, 8))
            obs[:, 0, 1:4] = mid
            obs[:, 0, 7] = 0.07
            pl = k.TrajectoryPlanner(m, "flange", timesteps=TT, precision=prec, max_iterations=4)
            res = pl.solve_anchored_device(dv.to_dev(np.stack([qa, qb], axis=1)), dv.to_dev(obs), 1)
            ktraj.trajectory_signed_distances_batch(m, res["qs"], dv.to_dev(obs), 1, "flange")
            done(f"traj-T{TT}", prec)
print("sanitize smoke complete", flush=True)
