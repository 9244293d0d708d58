"""fk_arrays device timing (A/B of k_fk_tree variants via KOP_LIB): python tools/fk_time.py [B]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_03728_b200 as k
from paper_2505_03728_b200 import _device as dv
from paper_2505_03728_b200.robot import fk_arrays_device

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
for name in ("arm7", "humanoid29"):
    m = k.load_robot(k.robot_path(name + ".urdf"), k.robot_path("arm7.sidecar.json") if name == "arm7" else None)
    q = dv.to_dev(np.random.default_rng(3).uniform(np.where(np.isfinite(m.lower_limits), m.lower_limits, -3),
                                                   np.where(np.isfinite(m.upper_limits), m.upper_limits, 3),
                                                   (B, m.actuated_count)))
    byts = B * 8 * (m.actuated_count + 7 * len(m.link_names) + 6 * len(m.joints))
    for prec in ("fp64", "fp32"):
        fk_arrays_device(m, q, prec)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fk_arrays_device(m, q, prec); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        print(json.dumps({"lib": os.environ.get("KOP_LIB", "default"), "robot": name, "prec": prec, "ms": ms,
                          "GBps": byts / ms / 1e6}))
