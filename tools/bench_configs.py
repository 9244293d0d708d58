"""Device timing of the widened configurations (not the driver's bench line):
config 4 collision IK-Beam and the generic collision LM solve, config 2 mobile
IK-Beam.  Prints one JSON line per workload."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_03728_b200 as k
from paper_2505_03728_b200.benchmark import reachable_target_array, disk_translations
from paper_2505_03728_b200.tasks import IkBeamSolver

DEMO = k.WorldModel([k.Sphere([0.45, 0.1, 0.55], 0.12), k.Capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
                     k.HalfSpace([0.0, 0.0, 1.0], -0.3)])
m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))


def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


B = int(os.environ.get("B", "100000"))
tg = reachable_target_array(m, "flange", B, 77)
for prec in ("fp32", "fp64"):
    s = IkBeamSolver(m, "flange", rng_seed=77, precision=prec, world=DEMO, self_collision=True)
    out = s.alloc_outputs(B)
    ms = timeit(lambda: s.solve_device(tg, out))
    print(json.dumps({"workload": "config4 collision IK-Beam (Panda, demo world: sphere+capsule+half-space, self pairs)",
                      "precision": prec, "targets": B, "ms": ms, "solves_per_s": B / ms * 1e3,
                      "success": float(out.success.float().mean())}), flush=True)
# generic solve (solver.solve semantics), q0 = rest pose, 100 iterations max
nb = min(B, 20000)
probs_t = tg[:nb].cpu().numpy()
from paper_2505_03728_b200.solver import plan, _options
import ctypes as C
from paper_2505_03728_b200 import _device as dv
from paper_2505_03728_b200._lib import lib, check
prob = k.Problem(k.VariableSet.of(q=m.rest_pose.copy()), [
    k.pose_cost(m, "q", "flange", k.Transform3.identity(), position_weight=50, orientation_weight=10),
    k.limit_cost(m, "q", weight=100), k.rest_cost("q", m.rest_pose, weight=0.01),
    k.world_collision_cost(m, "q", DEMO, weight=20), k.self_collision_cost(m, "q", weight=5)])
p = plan(prob)
for prec in ("fp32", "fp64"):
    opts = _options(k.SolveOptions(precision=prec))
    q0 = dv.to_dev(np.tile(m.rest_pose, (nb, 1)))
    tdev = dv.to_dev(probs_t)
    outs = [dv.empty((nb, 7)), dv.empty(nb), dv.empty(nb), None, torch.empty(nb, dtype=torch.int32, device="cuda"),
            torch.empty(nb, dtype=torch.int32, device="cuda")]
    def run():
        check(lib().kop_lm_solve(m._handle, 8, C.byref(p.costs), C.byref(opts), dv.ptr(tdev), dv.ptr(q0), nb,
                                 *(dv.ptr(x) for x in outs), dv.stream_handle()), "solve")
    ms = timeit(run, 3)
    it = outs[4].float().mean().item()
    print(json.dumps({"workload": "generic LM solve (solver.solve semantics) on the collision stack, q0 = rest pose",
                      "precision": prec, "problems": nb, "ms": ms, "solves_per_s": nb / ms * 1e3,
                      "mean_iterations": it}), flush=True)
# mobile
sh = tg.cpu().numpy().copy()
sh[:, 4:] += disk_translations(B, 2.0, 2024) if B <= 20000 else np.tile(disk_translations(20000, 2.0, 2024), (B // 20000 + 1, 1))[:B]
shd = dv.to_dev(sh)
s = IkBeamSolver(m, "flange", rng_seed=77, optimize_base=True)
out = s.alloc_outputs(B)
ms = timeit(lambda: s.solve_device(shd, out))
print(json.dumps({"workload": "mobile-base IK-Beam (Panda + SE(2) base, disk-shifted targets)", "precision": "fp32",
                  "targets": B, "ms": ms, "solves_per_s": B / ms * 1e3,
                  "success": float(out.success.float().mean())}), flush=True)
