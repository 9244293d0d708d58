"""Config-5 timing / profiling driver: T-step trajectories from random in-limit
anchor pairs with one r=0.07 sphere at the FK of the joint-space midpoint
(benchmark.py:250-277 without the endpoint IK).  Prints one JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_03728_b200 as k
from paper_2505_03728_b200 import _device as dv
from paper_2505_03728_b200.robot import link_poses_device

NT = int(os.environ.get("NTRAJ", "2000"))
TT = int(os.environ.get("TSTEPS", "64"))
PREC = os.environ.get("PREC", "fp64")
REPS = int(os.environ.get("REPS", "2"))
m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
rng = np.random.default_rng(5)
qa = rng.uniform(m.lower_limits, m.upper_limits, (NT, 7))
qb = rng.uniform(m.lower_limits, m.upper_limits, (NT, 7))
mid = link_poses_device(m, dv.to_dev(0.5 * (qa + qb)), "flange").cpu().numpy()[:, 4:7]
obs = np.zeros((NT, 1, 8)); obs[:, 0, 1:4] = mid; obs[:, 0, 7] = 0.07
anchors = dv.to_dev(np.stack([qa, qb], axis=1)); obsd = dv.to_dev(obs)
pl = k.TrajectoryPlanner(m, "flange", timesteps=TT, precision=PREC)
res = pl.solve_anchored_device(anchors, obsd, 1, history=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(REPS):
    res = pl.solve_anchored_device(anchors, obsd, 1, history=False)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / REPS
it = res["iterations"].float()
print(json.dumps({"precision": PREC, "T": TT, "trajectories": NT, "ms": ms, "trajectories_per_s": NT / ms * 1e3,
                  "mean_iterations": it.mean().item(), "cost_mean": res["cost"].mean().item(),
                  "terminations": torch.bincount(res["termination"].long(), minlength=6).tolist()}))
