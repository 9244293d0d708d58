"""Fingerprint of the tree kernels' outputs (A/B bit-identity of kernel
rewrites): SHA-256 of the humanoid multi-EE IK-Beam results and of the
generic tree solve (kop_multi_pose_solve), FP32 and FP64.  Prints one JSON
line; compare the lines of two libraries:

  LIBS="default variants/libkinoptik_b200_X.so" bash tools/gpu_ab.sh python tools/tree_bits.py
"""
import ctypes as C, hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_03728_b200 as k
from paper_2505_03728_b200 import _device as dv
from paper_2505_03728_b200._lib import check, lib
from paper_2505_03728_b200.robot import link_poses_device
from paper_2505_03728_b200.solver import _options, plan

NH = int(os.environ.get("NHUM", "2000"))
hum = k.load_robot(k.robot_path("humanoid29.urdf"))
EES = ["left_hand", "right_hand", "left_foot", "right_foot"]
qt = dv.to_dev(np.random.default_rng(31).uniform(hum.lower_limits, hum.upper_limits, (NH, hum.actuated_count)))
tgh = torch.stack([link_poses_device(hum, qt, e) for e in EES], dim=1).contiguous()
W0 = k.CostWeights()
hp = plan(k.Problem(k.VariableSet.of(q=hum.rest_pose.copy()),
                    [k.pose_cost(hum, "q", e, k.Transform3.identity(), position_weight=W0.pose_position,
                                 orientation_weight=W0.pose_orientation) for e in EES]
                    + [k.limit_cost(hum, "q", weight=W0.limit), k.rest_cost("q", hum.rest_pose, weight=W0.rest)]))
q0 = dv.to_dev(np.tile(hum.rest_pose, (NH, 1)))


def digest(ts):
    h = hashlib.sha256()
    for t in ts:
        h.update(t.detach().cpu().contiguous().numpy().tobytes())
    return h.hexdigest()[:16]


out = {}
for prec in ("fp32", "fp64"):
    r = k.solve_ik_beam_multi(hum, EES, tgh, precision=prec, device_out=True)
    torch.cuda.synchronize()
    out[f"beam_{prec}"] = digest([r.q, r.cost, r.success.int()])
    out[f"beam_{prec}_success"] = float(r.success.float().mean())
    opts = _options(k.SolveOptions(precision=prec))
    outs = [dv.empty((NH, hum.actuated_count)), dv.empty(NH), dv.empty(NH), dv.empty((NH, opts.max_iterations + 1)),
            torch.empty(NH, dtype=torch.int32, device="cuda"), torch.empty(NH, dtype=torch.int32, device="cuda")]
    check(lib().kop_multi_pose_solve(hum._handle, C.byref(hp.costs), C.byref(opts), dv.ptr(tgh), dv.ptr(q0), NH,
                                     *(dv.ptr(x) for x in outs), dv.stream_handle()), "tree")
    torch.cuda.synchronize()
    out[f"solve_{prec}"] = digest(outs)
    out[f"solve_{prec}_iters"] = float(outs[4].float().mean())
print(json.dumps(out))
