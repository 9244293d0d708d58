"""IK-Beam throughput and latency from batch 1 to 1M (BASELINE.json: "Panda
batched-IK solves/sec at batch 1 to 1M").  Device time: CUDA events around
the two/three kernels of one solve, median of the repetitions, L2 not
flushed (small batches are latency-bound).  End-to-end: host targets in,
host results out through the public API (IkBeamSolver.solve for <= 128K,
solve_pinned above)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_03728_b200 as k
from paper_2505_03728_b200.benchmark import reachable_target_array
from paper_2505_03728_b200.tasks import IkBeamSolver

m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
s = IkBeamSolver(m, "flange", rng_seed=77)
full = reachable_target_array(m, "flange", 1_000_000, 77)
for B in (1, 10, 100, 1000, 10_000, 100_000, 1_000_000):
    tg = full[:B].contiguous()
    out = s.alloc_outputs(B)
    s.solve_device(tg, out); torch.cuda.synchronize()
    reps = 20 if B <= 100_000 else 5
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); s.solve_device(tg, out); e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    dev_ms = float(np.median(times))
    host = tg.cpu().numpy()
    if B <= 131072:
        s.solve(host)
        t0 = time.perf_counter()
        for _ in range(reps):
            s.solve(host)
        e2e_ms = (time.perf_counter() - t0) * 1e3 / reps
    else:
        hp = tg.cpu().pin_memory(); ho = s.alloc_host_outputs(B)
        s.solve_pinned(hp, ho); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            s.solve_pinned(hp, ho)
        torch.cuda.synchronize()
        e2e_ms = (time.perf_counter() - t0) * 1e3 / reps
    print(json.dumps({"batch": B, "device_ms": dev_ms, "device_solves_per_s": B / dev_ms * 1e3,
                      "e2e_ms": e2e_ms, "e2e_solves_per_s": B / e2e_ms * 1e3,
                      "success": float(out.success.float().mean())}), flush=True)
