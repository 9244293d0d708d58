"""One pass of a widened workload, for ncu (launch lists / full captures).

    python tools/prof_workloads.py WORKLOAD [PREC] [N]

WORKLOAD: col_lm (config 4 generic LM), col_beam (config 4 IK-Beam),
tree_lm (config 3 generic LM), tree_beam (config 3 multi-EE IK-Beam),
traj (config 5 trajectories, T = 64), beam (the headline Panda IK-Beam).
Each runs one warm-up call and one profiled call with the bench's inputs.
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2505_03728_b200 as k
from paper_2505_03728_b200 import _device as dv
from paper_2505_03728_b200._lib import check, lib
from paper_2505_03728_b200.benchmark import reachable_target_array
from paper_2505_03728_b200.robot import link_poses_device
from paper_2505_03728_b200.solver import _options, plan
from paper_2505_03728_b200.tasks import IkBeamSolver

W = sys.argv[1]
PREC = sys.argv[2] if len(sys.argv) > 2 else "fp32"
N = int(sys.argv[3]) if len(sys.argv) > 3 else 20000
m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
DEMO = k.WorldModel([k.Sphere([0.45, 0.1, 0.55], 0.12), k.Capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
                     k.HalfSpace([0.0, 0.0, 1.0], -0.3)])
hum = k.load_robot(k.robot_path("humanoid29.urdf"))
EES = ["left_hand", "right_hand", "left_foot", "right_foot"]


def col_lm():
    tg = reachable_target_array(m, "flange", N, 77)
    p = plan(k.Problem(k.VariableSet.of(q=m.rest_pose.copy()), [
        k.pose_cost(m, "q", "flange", k.Transform3.identity(), position_weight=50, orientation_weight=10),
        k.limit_cost(m, "q", weight=100), k.rest_cost("q", m.rest_pose, weight=0.01),
        k.world_collision_cost(m, "q", DEMO, weight=20), k.self_collision_cost(m, "q", weight=5)]))
    opts = _options(k.SolveOptions(precision=PREC))
    q0 = dv.to_dev(np.tile(m.rest_pose, (N, 1)))
    outs = [dv.empty((N, 7)), dv.empty(N), dv.empty(N), None, torch.empty(N, dtype=torch.int32, device="cuda"),
            torch.empty(N, dtype=torch.int32, device="cuda")]
    return lambda: check(lib().kop_lm_solve(m._handle, 8, C.byref(p.costs), C.byref(opts), dv.ptr(tg), dv.ptr(q0), N,
                                            *(dv.ptr(x) for x in outs), dv.stream_handle()), "lm")


def col_beam():
    tg = reachable_target_array(m, "flange", N, 77)
    s = IkBeamSolver(m, "flange", rng_seed=77, precision=PREC, world=DEMO, self_collision=True)
    out = s.alloc_outputs(N)
    return lambda: s.solve_device(tg, out)


def _hum_targets():
    qt = dv.to_dev(np.random.default_rng(29).uniform(hum.lower_limits, hum.upper_limits, (N, hum.actuated_count)))
    return torch.stack([link_poses_device(hum, qt, e) for e in EES], dim=1).contiguous()


def tree_lm():
    tgh = _hum_targets()
    hp = plan(k.Problem(k.VariableSet.of(q=hum.rest_pose.copy()),
                        [k.pose_cost(hum, "q", e, k.Transform3.identity(), position_weight=50, orientation_weight=10)
                         for e in EES] + [k.limit_cost(hum, "q", weight=100),
                                          k.rest_cost("q", hum.rest_pose, weight=0.01)]))
    opts = _options(k.SolveOptions(precision=PREC))
    q0 = dv.to_dev(np.tile(hum.rest_pose, (N, 1)))
    outs = [dv.empty((N, hum.actuated_count)), dv.empty(N), dv.empty(N), None,
            torch.empty(N, dtype=torch.int32, device="cuda"), torch.empty(N, dtype=torch.int32, device="cuda")]
    return lambda: check(lib().kop_multi_pose_solve(hum._handle, C.byref(hp.costs), C.byref(opts), dv.ptr(tgh),
                                                    dv.ptr(q0), N, *(dv.ptr(x) for x in outs), dv.stream_handle()),
                         "tree")


def tree_beam():
    tgh = _hum_targets()
    return lambda: k.solve_ik_beam_multi(hum, EES, tgh, precision=PREC, device_out=True)


def traj():
    rng = np.random.default_rng(5)
    qa = rng.uniform(m.lower_limits, m.upper_limits, (N, 7))
    qb = rng.uniform(m.lower_limits, m.upper_limits, (N, 7))
    mid = link_poses_device(m, dv.to_dev(0.5 * (qa + qb)), "flange").cpu().numpy()[:, 4:7]
    obs = np.zeros((N, 1, 8))
    obs[:, 0, 1:4] = mid
    obs[:, 0, 7] = 0.07
    anchors, obsd = dv.to_dev(np.stack([qa, qb], axis=1)), dv.to_dev(obs)
    pl = k.TrajectoryPlanner(m, "flange", timesteps=64, precision=PREC)
    return lambda: pl.solve_anchored_device(anchors, obsd, 1, history=False)


def beam():
    tg = reachable_target_array(m, "flange", N, 77)
    s = IkBeamSolver(m, "flange", rng_seed=77, precision=PREC)
    out = s.alloc_outputs(N)
    return lambda: s.solve_device(tg, out)


run = {"col_lm": col_lm, "col_beam": col_beam, "tree_lm": tree_lm, "tree_beam": tree_beam, "traj": traj,
       "beam": beam}[W]()
run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
run()
e1.record()
torch.cuda.synchronize()
print(f"{W} {PREC} N={N}: {e0.elapsed_time(e1):.3f} ms", flush=True)
