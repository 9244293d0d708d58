"""Timeline of the first damped solve of CTA 0 (build with -DKOP_TRAJ_TIMELINE)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_2505_03728_b200 as k
from paper_2505_03728_b200 import _device as dv
from paper_2505_03728_b200._lib import lib
prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
rng = np.random.default_rng(5)
NT = 148
qa = rng.uniform(m.lower_limits, m.upper_limits, (NT, 7)); qb = rng.uniform(m.lower_limits, m.upper_limits, (NT, 7))
obs = np.zeros((NT, 1, 8)); obs[:, 0, 1:4] = [0.4, 0.0, 0.5]; obs[:, 0, 7] = 0.07
pl = k.TrajectoryPlanner(m, "flange", timesteps=64, precision=prec)
pl.solve_anchored_device(dv.to_dev(np.stack([qa, qb], 1)), dv.to_dev(obs), 1, history=False)
torch.cuda.synchronize()
buf = (C.c_longlong * (4 * 72 * 6))()
lib().kop_debug_traj_timeline(buf)
a = np.array(buf, dtype=np.int64).reshape(4, 72, 6)
t0 = a[a > 0].min()
names = ["top main", "bottom main", "top trail", "bottom trail"]
for blk in list(range(0, 6)) + list(range(28, 34)):
    print(blk, " | ".join(f"{names[r]}: " + ",".join(str(int(v - t0)) if v else "-" for v in a[r, blk, :5]) for r in range(4)))
for r in range(4):
    v = a[r, :, :5]; ok = v[:, 0] > 0
    d = np.diff(v[ok], axis=1).mean(axis=0) if ok.any() else []
    print(names[r], "mean per block: rows/work->bar1 arrive", *(round(x) for x in d))
