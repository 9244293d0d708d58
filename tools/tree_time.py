"""Config-3 humanoid multi-EE tree solve timing / profiling driver."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np, torch
import paper_2505_03728_b200 as k
from paper_2505_03728_b200 import _device as dv
from paper_2505_03728_b200._lib import check, lib
from paper_2505_03728_b200.robot import link_poses_device
from paper_2505_03728_b200.solver import _options, plan

NH = int(os.environ.get("NHUM", "100000"))
PREC = os.environ.get("PREC", "fp32")
REPS = int(os.environ.get("REPS", "2"))
hum = k.load_robot(k.robot_path("humanoid29.urdf"))
EES = ["left_hand", "right_hand", "left_foot", "right_foot"]
qt = dv.to_dev(np.random.default_rng(29).uniform(hum.lower_limits, hum.upper_limits, (NH, hum.actuated_count)))
tgh = torch.stack([link_poses_device(hum, qt, e) for e in EES], dim=1).contiguous()
W0 = k.CostWeights()
hp = plan(k.Problem(k.VariableSet.of(q=hum.rest_pose.copy()),
                    [k.pose_cost(hum, "q", e, k.Transform3.identity(), position_weight=W0.pose_position,
                                 orientation_weight=W0.pose_orientation) for e in EES]
                    + [k.limit_cost(hum, "q", weight=W0.limit), k.rest_cost("q", hum.rest_pose, weight=W0.rest)]))
opts = _options(k.SolveOptions(precision=PREC))
q0 = dv.to_dev(np.tile(hum.rest_pose, (NH, 1)))
outs = [dv.empty((NH, hum.actuated_count)), dv.empty(NH), dv.empty(NH), None,
        torch.empty(NH, dtype=torch.int32, device="cuda"), torch.empty(NH, dtype=torch.int32, device="cuda")]
run = lambda: check(lib().kop_multi_pose_solve(hum._handle, C.byref(hp.costs), C.byref(opts), dv.ptr(tgh), dv.ptr(q0),
                                               NH, *(dv.ptr(x) for x in outs), dv.stream_handle()), "tree")
run(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(REPS):
    run()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / REPS
print(json.dumps({"precision": PREC, "problems": NH, "ms": ms, "solves_per_s": NH / ms * 1e3,
                  "mean_iterations": outs[4].float().mean().item(), "cost_p50": outs[1].median().item(),
                  "terminations": torch.bincount(outs[5].long(), minlength=6).tolist()}))
# multi-EE IK-Beam on the same targets (SURVEY H6 flavour of config 3)
if os.environ.get("BEAM", "1") == "1":
    NB = int(os.environ.get("NBEAM", str(NH)))
    k.solve_ik_beam_multi(hum, EES, tgh[:NB], precision=PREC, device_out=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(REPS):
        r = k.solve_ik_beam_multi(hum, EES, tgh[:NB], precision=PREC, device_out=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / REPS
    print(json.dumps({"workload": "multi-EE IK-Beam", "precision": PREC, "targets": NB, "ms": ms,
                      "solves_per_s": NB / ms * 1e3, "success": r.success.float().mean().item(),
                      "pos_err_p50": r.pos_error.median().item()}))
