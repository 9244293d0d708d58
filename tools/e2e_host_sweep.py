"""Sweep chunk size / stream count of the C-ABI host pipeline (kop_ik_beam_host via
IkBeamSolver.solve_host): end-to-end rate with pinned host buffers, 1M targets."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_03728_b200 as k
from paper_2505_03728_b200.benchmark import reachable_target_array
from paper_2505_03728_b200.tasks import IkBeamSolver

B = 1_000_000
m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
s = IkBeamSolver(m, "flange", rng_seed=77)
host = reachable_target_array(m, "flange", B, 77).cpu().pin_memory()
out = s.alloc_host_outputs(B)
for chunk in [int(c) for c in os.environ.get("CHUNKS", "32768,65536,131072,262144").split(",")]:
    for ns in [int(c) for c in os.environ.get("STREAMS", "2,4,8").split(",")]:
        s.solve_host(host, out, chunk=chunk, n_streams=ns); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); s.solve_host(host, out, chunk=chunk, n_streams=ns); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        print(json.dumps({"chunk": chunk, "streams": ns, "ms": ms, "solves_per_s": B / ms * 1e3}), flush=True)
