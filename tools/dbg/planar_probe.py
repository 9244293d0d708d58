"""Debug probe: padded planar_2r trajectory solves over several T / precisions, each in a fresh process."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
if len(sys.argv) == 1:
    for prec in ("fp64", "fp32"):
        for T in (8, 14, 16, 64):
            for obs in (0, 1):
                r = subprocess.run([sys.executable, __file__, prec, str(T), str(obs)], capture_output=True, text=True)
                print(prec, T, obs, (r.stdout.strip() or r.stderr.strip().splitlines()[-1])[:150], flush=True)
    sys.exit(0)
import numpy as np, torch
import paper_2505_03728_b200 as k
prec, T, nobs = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
m = k.load_robot(k.robot_path("planar_2r.urdf"), k.robot_path("planar_2r.sidecar.json"))
qa, qb = np.array([0.2, 0.4]), np.array([1.4, -0.6])
mid = k.link_transform(m, 0.5 * (qa + qb), m.link_names[-1]).translation
world = k.WorldModel([k.Capsule(mid - [0.05, 0.0, 0.2], mid + [0.05, 0.0, 0.2], 0.08)][:nobs])
rows = k.collision.obstacle_rows(world.obstacles) if nobs else np.zeros((0, 8))
planner = k.TrajectoryPlanner(m, m.link_names[-1], timesteps=T, precision=prec)
out = planner.solve_anchored_device(np.array([[qa, qb]]), rows[None], nobs)
torch.cuda.synchronize()
print("ok cost", out["cost"][0].item(), "iters", int(out["iterations"][0]))
