"""Config-4 collision IK-Beam timing / profiling driver (demo world, self pairs)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_03728_b200 as k
from paper_2505_03728_b200.benchmark import reachable_target_array
from paper_2505_03728_b200.tasks import IkBeamSolver

B = int(os.environ.get("B", "100000"))
PREC = os.environ.get("PREC", "fp32")
REPS = int(os.environ.get("REPS", "3"))
m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
DEMO = k.WorldModel([k.Sphere([0.45, 0.1, 0.55], 0.12), k.Capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
                     k.HalfSpace([0.0, 0.0, 1.0], -0.3)])
tg = reachable_target_array(m, "flange", B, 77)
s = IkBeamSolver(m, "flange", rng_seed=77, precision=PREC, world=DEMO, self_collision=True)
out = s.alloc_outputs(B)
s.solve_device(tg, out); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(REPS):
    s.solve_device(tg, out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / REPS
print(json.dumps({"precision": PREC, "targets": B, "ms": ms, "solves_per_s": B / ms * 1e3,
                  "success": out.success.float().mean().item(), "cost_mean": out.cost.mean().item()}))
