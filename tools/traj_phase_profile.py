"""Per-phase clock64 cycles of the trajectory kernel (thread 0 of each CTA),
from a -DKOP_TRAJ_PROFILE build:

  python -c "from paper_2505_03728_b200 import _build; _build.build(variant='trajprof', defines=['-DKOP_TRAJ_PROFILE'])"
  KOP_LIB=variants/libkinoptik_b200_trajprof.so python tools/traj_phase_profile.py
"""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_03728_b200 as k
from paper_2505_03728_b200 import _device as dv
from paper_2505_03728_b200._lib import lib
from paper_2505_03728_b200.robot import link_poses_device

NT = int(os.environ.get("NTRAJ", "296"))
m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
rng = np.random.default_rng(5)
qa = rng.uniform(m.lower_limits, m.upper_limits, (NT, 7))
qb = rng.uniform(m.lower_limits, m.upper_limits, (NT, 7))
mid = link_poses_device(m, dv.to_dev(0.5 * (qa + qb)), "flange").cpu().numpy()[:, 4:7]
obs = np.zeros((NT, 1, 8)); obs[:, 0, 1:4] = mid; obs[:, 0, 7] = 0.07
anchors = dv.to_dev(np.stack([qa, qb], axis=1)); obsd = dv.to_dev(obs)
buf = (C.c_ulonglong * 20)()
names = ["eval+J", "eval", "solve setup", "factor", "back subst"]
for prec in ("fp64", "fp32"):
    pl = k.TrajectoryPlanner(m, "flange", timesteps=64, precision=prec)
    pl.solve_anchored_device(anchors, obsd, 1, history=False)
    torch.cuda.synchronize()
    lib().kop_debug_traj_profile(buf, 1)
    res = pl.solve_anchored_device(anchors, obsd, 1, history=False)
    torch.cuda.synchronize()
    lib().kop_debug_traj_profile(buf, 1)
    v = list(buf)
    ns, nj, ne = v[5], v[6], v[7]
    per = {"eval+J": v[0] / max(nj, 1), "eval": v[1] / max(ne, 1), "solve setup": v[2] / max(ns, 1),
           "factor": v[3] / max(ns, 1), "back subst": v[4] / max(ns, 1)}
    tot = sum(v[:5])
    print(json.dumps({"precision": prec, "trajectories": NT, "solves_per_traj": ns / NT, "evalJ_per_traj": nj / NT,
                      "eval_per_traj": ne / NT, "cycles_per_call": {a: round(b) for a, b in per.items()},
                      "share": {a: round(v[i] / tot, 3) for i, a in enumerate(names)},
                      "cycles_per_traj": round(tot / NT),
                      "sweep_cycles_per_solve": {side: {a: round(v[base + i] / max(ns, 1)) for i, a in
                                                        enumerate(["rows", "barrier 1", "diag pairs + factor",
                                                                   "barrier 2"])}
                                                 for side, base in (("top", 8), ("bottom", 12), ("separator", 16))}}))
