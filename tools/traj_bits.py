"""Fingerprint of the trajectory solve's outputs (A/B bit-identity of kernel
rewrites): SHA-256 of final trajectories, costs, iterations and terminations
for FP64 / FP32 at several lengths (T = 64 and odd / short T: the two-sided
factorisation's separator and empty-half cases).  Prints one JSON line;
compare the lines of two libraries:

  LIBS="default variants/libkinoptik_b200_X.so" bash tools/gpu_ab.sh python tools/traj_bits.py
"""
import hashlib, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_03728_b200 as k
from paper_2505_03728_b200 import _device as dv
from paper_2505_03728_b200.robot import link_poses_device

NT = int(os.environ.get("NTRAJ", "300"))
m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
rng = np.random.default_rng(11)
qa = rng.uniform(m.lower_limits, m.upper_limits, (NT, 7))
qb = rng.uniform(m.lower_limits, m.upper_limits, (NT, 7))
mid = link_poses_device(m, dv.to_dev(0.5 * (qa + qb)), "flange").cpu().numpy()[:, 4:7]
obs = np.zeros((NT, 1, 8)); obs[:, 0, 1:4] = mid; obs[:, 0, 7] = 0.07
anchors = dv.to_dev(np.stack([qa, qb], axis=1)); obsd = dv.to_dev(obs)
out = {}
for prec in ("fp64", "fp32"):
    for T in (64, 37, 9, 5):
        pl = k.TrajectoryPlanner(m, "flange", timesteps=T, precision=prec)
        res = pl.solve_anchored_device(anchors, obsd, 1, history=True)
        torch.cuda.synchronize()
        h = hashlib.sha256()
        for key in sorted(res):
            v = res[key]
            if torch.is_tensor(v):
                h.update(key.encode()); h.update(v.detach().cpu().contiguous().numpy().tobytes())
        out[f"{prec}_T{T}"] = h.hexdigest()[:16]
        out[f"{prec}_T{T}_iters"] = float(res["iterations"].float().mean())
print(json.dumps(out))
