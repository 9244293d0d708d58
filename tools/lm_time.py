"""Generic-LM (solver.solve semantics) timing on config 4's collision stack:
FP32 and FP64 time, iterations, termination profiles and FP32-vs-FP64 final
costs per problem.  Usage: [B=100000] [REPS=3] python tools/lm_time.py"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2505_03728_b200 as k
from paper_2505_03728_b200 import _device as dv
from paper_2505_03728_b200._lib import check, lib
from paper_2505_03728_b200.benchmark import reachable_target_array
from paper_2505_03728_b200.solver import _options, plan

B = int(os.environ.get("B", "100000"))
REPS = int(os.environ.get("REPS", "3"))
m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
DEMO = k.WorldModel([k.Sphere([0.45, 0.1, 0.55], 0.12), k.Capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
                     k.HalfSpace([0.0, 0.0, 1.0], -0.3)])
tg = reachable_target_array(m, "flange", B, 77)
prob = k.Problem(k.VariableSet.of(q=m.rest_pose.copy()), [
    k.pose_cost(m, "q", "flange", k.Transform3.identity(), position_weight=50, orientation_weight=10),
    k.limit_cost(m, "q", weight=100), k.rest_cost("q", m.rest_pose, weight=0.01),
    k.world_collision_cost(m, "q", DEMO, weight=20), k.self_collision_cost(m, "q", weight=5)])
p = plan(prob)
res = {}
for prec in ("fp32", "fp64"):
    opts = _options(k.SolveOptions(precision=prec))
    q0 = dv.to_dev(np.tile(m.rest_pose, (B, 1)))
    outs = [dv.empty((B, 7)), dv.empty(B), dv.empty(B), None, torch.empty(B, dtype=torch.int32, device="cuda"),
            torch.empty(B, dtype=torch.int32, device="cuda")]

    def run():
        check(lib().kop_lm_solve(m._handle, 8, C.byref(p.costs), C.byref(opts), dv.ptr(tg), dv.ptr(q0), B,
                                 *(dv.ptr(x) for x in outs), dv.stream_handle()), "kop_lm_solve")
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(REPS):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    res[prec] = {"cost": outs[1].cpu().numpy(), "q": outs[0].cpu().numpy()}
    print(json.dumps({"precision": prec, "problems": B, "ms": ms, "rep_ms": [round(t, 2) for t in ts], "solves_per_s": B / ms * 1e3,
                      "mean_iterations": float(outs[4].float().mean()),
                      "terminations": torch.bincount(outs[5].long(), minlength=7).tolist()}), flush=True)
c32, c64 = res["fp32"]["cost"], res["fp64"]["cost"]
rel = (c32 - c64) / c64
print(json.dumps({"fp32_vs_fp64_final_cost_rel": {"p10": float(np.percentile(rel, 10)),
                                                  "p50": float(np.percentile(rel, 50)),
                                                  "p90": float(np.percentile(rel, 90)),
                                                  "p99": float(np.percentile(rel, 99))},
                  "fp64_cost_p50": float(np.median(c64))}))
