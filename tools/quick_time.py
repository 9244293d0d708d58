"""Quick device timing of IK-Beam at several batch sizes (dev tool, not the bench)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_03728_b200 as k
from paper_2505_03728_b200.benchmark import reachable_target_array
from paper_2505_03728_b200.tasks import IkBeamSolver
m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
for prec in sys.argv[1:] or ["fp32"]:
    for twopass in ("0", "1"):
        os.environ["KOP_TWOPASS"] = twopass
        solver = IkBeamSolver(m, "flange", rng_seed=77, precision=prec)
        for B in (1, 1000, 10000, 100000, 1000000):
            if prec == "fp64" and B > 100000: continue
            t = reachable_target_array(m, "flange", B, 77)
            out = solver.alloc_outputs(B)
            for _ in range(3): solver.solve_device(t, out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 5 if B >= 100000 else 20
            e0.record()
            for _ in range(reps): solver.solve_device(t, out)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            print(f"{prec} twopass={twopass} B={B:8d} {ms:9.3f} ms  {B/ms*1e3:12.0f} solves/s  succ {out.success.float().mean().item():.4f}", flush=True)
