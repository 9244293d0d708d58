"""solve_pinned replayed as one CUDA graph vs eager (end-to-end rate)."""
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
for chunk, ns in ((65536, 4), (131072, 3)):
    s.solve_pinned(host, out, chunk=chunk, n_streams=ns); torch.cuda.synchronize()
    ref = out.q.clone()
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    with torch.cuda.stream(cap):
        g.capture_begin()
        s.solve_pinned(host, out, chunk=chunk, n_streams=ns)
        g.capture_end()
    torch.cuda.synchronize()
    out.q.zero_()
    g.replay(); torch.cuda.synchronize()
    same = bool(torch.equal(out.q, ref))
    for mode in ("eager", "graph"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            if mode == "graph":
                g.replay()
            else:
                s.solve_pinned(host, out, chunk=chunk, n_streams=ns)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(json.dumps({"chunk": chunk, "streams": ns, "mode": mode, "ms": ms, "solves_per_s": B / ms * 1e3,
                          "graph_matches_eager": same}), flush=True)
