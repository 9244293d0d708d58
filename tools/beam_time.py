"""Headline IK-Beam stage timing (A/B of library variants via KOP_LIB).
Usage: [KOP_LIB=variants/....so] python tools/beam_time.py PREC [B] [REPS]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_03728_b200 as k
from paper_2505_03728_b200.benchmark import reachable_target_array
from paper_2505_03728_b200.tasks import IkBeamSolver

prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
s = IkBeamSolver(m, "flange", rng_seed=77, precision=prec)
tg = reachable_target_array(m, "flange", B, 77)
out = s.alloc_outputs(B)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for _ in range(2):
    s.solve_device(tg, out)
torch.cuda.synchronize()
t1, t2 = [], []
for _ in range(reps):
    flush.zero_()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); s.solve_device(tg, out, stages=1); e[1].record(); s.solve_device(tg, out, stages=2); e[2].record()
    torch.cuda.synchronize()
    t1.append(e[0].elapsed_time(e[1])); t2.append(e[1].elapsed_time(e[2]))
ms1, ms2 = float(np.median(t1)), float(np.median(t2))
print(json.dumps({"lib": os.environ.get("KOP_LIB", "default"), "prec": prec, "B": B, "stage1_ms": ms1, "stage2_ms": ms2,
                  "solves_per_s": B / (ms1 + ms2) * 1e3, "success": float(out.success.float().mean()),
                  "cost_sum": float(out.cost.sum())}))
