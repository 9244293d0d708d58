"""Config-3 multi-EE IK-Beam timing driver (humanoid, 4 end effectors, 64 seeds,
6+10 steps, keep 4).  NHUM targets, PREC fp32/fp64.  Prints one JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_03728_b200 as k
from paper_2505_03728_b200 import _device as dv
from paper_2505_03728_b200.robot import link_poses_device

NH = int(os.environ.get("NHUM", "100000"))
PREC = os.environ.get("PREC", "fp32")
REPS = int(os.environ.get("REPS", "2"))
hum = k.load_robot(k.robot_path("humanoid29.urdf"))
EES = ["left_hand", "right_hand", "left_foot", "right_foot"]
qt = dv.to_dev(np.random.default_rng(29).uniform(hum.lower_limits, hum.upper_limits, (NH, hum.actuated_count)))
tgh = torch.stack([link_poses_device(hum, qt, e) for e in EES], dim=1).contiguous()
run = lambda: k.solve_ik_beam_multi(hum, EES, tgh, precision=PREC, device_out=True)
res = run()
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(REPS + 1)]
ev[0].record()
for i in range(REPS):
    res = run()
    ev[i + 1].record()
torch.cuda.synchronize()
per = [ev[i].elapsed_time(ev[i + 1]) for i in range(REPS)]
ms = sorted(per)[REPS // 2]  # median rep
print(json.dumps({"precision": PREC, "targets": NH, "ms": ms, "rep_ms": [round(x, 1) for x in per], "solves_per_s": NH / ms * 1e3,
                  "success": res.success.float().mean().item(), "cost_mean": res.cost.double().mean().item()}))
