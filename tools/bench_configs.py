"""Device timing of the widened configurations (not the driver's bench line):
config 4 collision IK-Beam and the generic collision LM solve, config 2 mobile
IK-Beam, config 5 trajectories, config 3 humanoid.  Prints one JSON line per
workload; with CPU=1 (default) each FP64 line carries a ``cpu_baseline``: the
oracle port of the reference (test infrastructure, float64 NumPy) timed on one
host core over a bounded sample of the same workload."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_03728_b200 as k
from paper_2505_03728_b200.benchmark import reachable_target_array, disk_translations
from paper_2505_03728_b200.tasks import IkBeamSolver

DEMO = k.WorldModel([k.Sphere([0.45, 0.1, 0.55], 0.12), k.Capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
                     k.HalfSpace([0.0, 0.0, 1.0], -0.3)])
m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))


CPU = os.environ.get("CPU", "1") == "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cpu_time(fn, count, unit, sample):
    """Single-core wall time of the oracle port over `count` units -> cpu_baseline dict."""
    if not CPU:
        return None
    t0 = time.perf_counter()
    fn()
    dt = time.perf_counter() - t0
    return {"value": count / dt, "unit": unit, "cores": 1, "kind": "port", "sample": sample}


if CPU:
    from oracle import collision_oracle as co, ik_oracle as o, traj_oracle as to, tree_oracle as tro
    ch7 = o.load_chain_files(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
    sp7 = co.load_spheres_files(ch7, k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
    FL = ch7.link("flange")
    DEMO_O = [co.sphere([0.45, 0.1, 0.55], 0.12), co.capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
              co.halfspace([0.0, 0.0, 1.0], -0.3)]


def _peak(fn, dtype, chains):
    import ctypes as C
    from paper_2505_03728_b200._lib import lib as _lib
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    sink = torch.zeros(4096, device="cuda", dtype=dtype)
    fl = C.c_double()
    st = torch.cuda.current_stream().cuda_stream
    getattr(_lib(), fn)(sms * 8, 256, 2000, sink.data_ptr(), C.byref(fl), st)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        getattr(_lib(), fn)(sms * 8, 256, 20000, sink.data_ptr(), C.byref(fl), st)
        e1.record(); torch.cuda.synchronize()
        best = max(best, fl.value / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


PEAK = {"fp32": _peak("kop_fma_peak_kernel", torch.float32, 16), "fp64": _peak("kop_dfma_peak_kernel", torch.float64, 8)}
try:
    with open(os.path.join(ROOT, "profiles", "r01_widened_flops.json")) as _f:
        FLOPS = {(w["workload"], w["precision"]): w for w in json.load(_f)["workloads"]}
except OSError:
    FLOPS = {}


def roofline(key, prec, units_per_s):
    """Executed-flop roofline of a widened workload against the measured FMA-pipe peak."""
    w = FLOPS.get((key, prec))
    if w is None:
        return None
    fpu = w["fp32_flops_per_unit"] if prec == "fp32" else w["fp64_flops_per_unit"]
    ach = fpu * units_per_s / 1e12
    return {"bound": "latency (serial LM chain per problem); compared with the " + prec.upper() + " FMA pipe",
            "achieved": ach, "peak": PEAK[prec], "unit": "TFLOP/s", "frac": ach / PEAK[prec],
            "flops_per_unit": fpu, "basis": "executed flops, ncu SASS counters (profiles/r01_widened_flops.json)",
            "peak_source": "live " + ("FFMA" if prec == "fp32" else "DFMA") + " microbenchmark"}


def timeit(fn, reps=5):
    """Median per-call device time (ms) over `reps` back-to-back calls after one warm-up call."""
    fn(); torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record()
    for i in range(reps):
        fn()
        ev[i + 1].record()
    torch.cuda.synchronize()
    return sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))[reps // 2]


B = int(os.environ.get("B", "100000"))
tg = reachable_target_array(m, "flange", B, 77)
for prec in ("fp32", "fp64"):
    s = IkBeamSolver(m, "flange", rng_seed=77, precision=prec, world=DEMO, self_collision=True)
    out = s.alloc_outputs(B)
    ms = timeit(lambda: s.solve_device(tg, out))
    cpu = None
    if prec == "fp64" and CPU:
        tgh = tg[:2].cpu().numpy()
        seeds = o.sample_seeds(ch7, 64, 77)
        cpu = cpu_time(lambda: co.ik_beam_collision(ch7, sp7, DEMO_O, FL, tgh[:, :4], tgh[:, 4:], seeds,
                                                    co.CollisionCosts()), 2, "solves/s",
                       "2 targets of this workload, oracle port (float64 NumPy), 1 core")
    print(json.dumps({"workload": "config4 collision IK-Beam (Panda, demo world: sphere+capsule+half-space, self pairs)",
                      "precision": prec, "targets": B, "ms": ms, "solves_per_s": B / ms * 1e3,
                      "success": float(out.success.float().mean()), "cpu_baseline": cpu,
                      "roofline": roofline("config4 collision IK-Beam", prec, B / ms * 1e3)}), flush=True)
# generic solve (solver.solve semantics), q0 = rest pose, 100 iterations max
nb = min(B, 100000)
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
    cpu = None
    if prec == "fp64" and CPU:
        def cpu_run():
            for i in range(5):
                co.solve_lm(ch7, sp7, DEMO_O, FL, probs_t[i, :4], probs_t[i, 4:], m.rest_pose.copy(),
                            co.CollisionCosts())
        cpu = cpu_time(cpu_run, 5, "solves/s", "5 problems of this workload, oracle port (float64 NumPy), 1 core")
    print(json.dumps({"workload": "generic LM solve (solver.solve semantics) on the collision stack, q0 = rest pose",
                      "precision": prec, "problems": nb, "ms": ms, "solves_per_s": nb / ms * 1e3,
                      "mean_iterations": it, "cpu_baseline": cpu,
                      "roofline": roofline("generic LM solve (collision stack)", prec, nb / ms * 1e3)}), flush=True)
# mobile
sh = tg.cpu().numpy().copy()
sh[:, 4:] += disk_translations(B, 2.0, 2024) if B <= 20000 else np.tile(disk_translations(20000, 2.0, 2024), (B // 20000 + 1, 1))[:B]
shd = dv.to_dev(sh)
s = IkBeamSolver(m, "flange", rng_seed=77, optimize_base=True)
out = s.alloc_outputs(B)
ms = timeit(lambda: s.solve_device(shd, out))
cpu = None
if CPU:
    seeds = o.sample_seeds(ch7, 64, 77)
    cpu = cpu_time(lambda: o.ik_beam(ch7, FL, sh[:4, :4], sh[:4, 4:], seeds, use_base=True), 4, "solves/s",
                   "4 targets of this workload, oracle port (float64 NumPy), 1 core")
print(json.dumps({"workload": "mobile-base IK-Beam (Panda + SE(2) base, disk-shifted targets)", "precision": "fp32",
                  "targets": B, "ms": ms, "solves_per_s": B / ms * 1e3,
                  "success": float(out.success.float().mean()), "cpu_baseline": cpu,
                  "roofline": roofline("mobile-base IK-Beam", "fp32", B / ms * 1e3)}), flush=True)
# config 5: trajectory optimisation, T=64, random in-limit anchor pairs, one
# r=0.07 sphere at the FK of the joint-space midpoint (benchmark.py:250-277
# without the endpoint IK), plan_trajectory cost set, solver.solve options
from paper_2505_03728_b200.robot import link_poses_device
NT = int(os.environ.get("NTRAJ", "10000"))
TT = int(os.environ.get("TSTEPS", "64"))
rng = np.random.default_rng(5)
qa = rng.uniform(m.lower_limits, m.upper_limits, (NT, 7))
qb = rng.uniform(m.lower_limits, m.upper_limits, (NT, 7))
mid = link_poses_device(m, dv.to_dev(0.5 * (qa + qb)), "flange").cpu().numpy()[:, 4:7]
obs = np.zeros((NT, 1, 8)); obs[:, 0, 1:4] = mid; obs[:, 0, 7] = 0.07
anchors = dv.to_dev(np.stack([qa, qb], axis=1)); obsd = dv.to_dev(obs)
for prec in ("fp32", "fp64"):
    pl = k.TrajectoryPlanner(m, "flange", timesteps=TT, precision=prec)
    res = {}
    def run():
        res.update(pl.solve_anchored_device(anchors, obsd, 1, history=False))
    ms = timeit(run, 2)
    rep = k.trajectory.trajectory_signed_distances_batch(m, res["qs"], obsd, 1, "flange")
    free = (torch.minimum(rep["min_static"], rep["min_swept"]) >= 0).float().mean().item()
    it = res["iterations"].float()
    cpu = None
    if prec == "fp64" and CPU:
        tc = to.TrajCosts(timesteps=TT)
        cpu = cpu_time(lambda: to.solve_traj(ch7, sp7, [co.sphere(mid[0], 0.07)], to.straight_line(qa[0], qb[0], TT),
                                             qa[0], qb[0], tc, m.velocity_limits), 1, "trajectories/s",
                       "trajectory 0 of this workload, oracle port (float64 NumPy, dense normal equations), 1 core")
    print(json.dumps({"cpu_baseline": cpu, "workload": f"config5 trajectory optimisation (Panda, T={TT}, 1 sphere at the midpoint)",
                      "precision": prec, "trajectories": NT, "ms": ms, "trajectories_per_s": NT / ms * 1e3,
                      "mean_iterations": it.mean().item(), "lm_iterations_per_s": it.sum().item() / ms * 1e3,
                      "collision_free": free,
                      "roofline": roofline("config5 trajectory optimisation T=64", prec, NT / ms * 1e3) if TT == 64 else None,
                      "terminations": torch.bincount(res["termination"].long(), minlength=6).tolist()}), flush=True)
# config 3: humanoid (synthetic G1-class, n=29) multi-EE IK through solver.solve
# semantics, 4 pose costs (hands, feet) + limit + rest, q0 = rest pose
hum = k.load_robot(k.robot_path("humanoid29.urdf"))
EES = ["left_hand", "right_hand", "left_foot", "right_foot"]
NH = int(os.environ.get("NHUM", "100000"))
qt = dv.to_dev(np.random.default_rng(29).uniform(hum.lower_limits, hum.upper_limits, (NH, hum.actuated_count)))
tgh = torch.stack([link_poses_device(hum, qt, e) for e in EES], dim=1).contiguous()
W0 = k.CostWeights()
hprob = k.Problem(k.VariableSet.of(q=hum.rest_pose.copy()),
                  [k.pose_cost(hum, "q", e, k.Transform3.identity(), position_weight=W0.pose_position,
                               orientation_weight=W0.pose_orientation) for e in EES]
                  + [k.limit_cost(hum, "q", weight=W0.limit), k.rest_cost("q", hum.rest_pose, weight=W0.rest)])
hp = plan(hprob)
for prec in ("fp32", "fp64"):
    opts = _options(k.SolveOptions(precision=prec))
    q0 = dv.to_dev(np.tile(hum.rest_pose, (NH, 1)))
    outs = [dv.empty((NH, hum.actuated_count)), dv.empty(NH), dv.empty(NH), None,
            torch.empty(NH, dtype=torch.int32, device="cuda"), torch.empty(NH, dtype=torch.int32, device="cuda")]
    def run():
        check(lib().kop_multi_pose_solve(hum._handle, C.byref(hp.costs), C.byref(opts), dv.ptr(tgh), dv.ptr(q0), NH,
                                         *(dv.ptr(x) for x in outs), dv.stream_handle()), "tree")
    ms = timeit(run, 2)
    cpu = None
    if prec == "fp64" and CPU:
        chh = o.load_chain_files(k.robot_path("humanoid29.urdf"))
        tgc = tgh[:3].cpu().numpy()
        links = [chh.link(e) for e in EES]
        def cpu_run():
            for i in range(3):
                poses = [(l, tgc[i, j, :4], tgc[i, j, 4:], W0.pose_position, W0.pose_orientation)
                         for j, l in enumerate(links)]
                tro.solve_multi_pose(chh, poses, hum.rest_pose.copy())
        cpu = cpu_time(cpu_run, 3, "solves/s", "3 problems of this workload, oracle port (float64 NumPy), 1 core")
    print(json.dumps({"cpu_baseline": cpu, "workload": "config3 humanoid multi-EE IK (n=29, 4 pose costs + limit + rest; solver.solve semantics)",
                      "precision": prec, "problems": NH, "ms": ms, "solves_per_s": NH / ms * 1e3,
                      "mean_iterations": outs[4].float().mean().item(),
                      "final_cost_p50": outs[1].median().item(),
                      "roofline": roofline("config3 humanoid multi-EE IK", prec, NH / ms * 1e3)}), flush=True)
# config 3 in the SURVEY H6 flavour: multi-end-effector IK-Beam (64 seeds, 6 + 10 lane-LM steps, keep 4)
for prec in ("fp32", "fp64"):
    nb = NH if prec == "fp32" else min(NH, 20000)
    box = {}
    def run_beam():
        box["r"] = k.solve_ik_beam_multi(hum, EES, tgh[:nb], precision=prec, device_out=True)
    ms = timeit(run_beam, 3)
    res = box["r"]
    cpu = None
    if prec == "fp64" and CPU:
        chh = o.load_chain_files(k.robot_path("humanoid29.urdf"))
        tgc = tgh[:2].cpu().numpy()
        links = [chh.link(e) for e in EES]
        seeds = o.sample_seeds(chh, 64, 0)
        cpu = cpu_time(lambda: tro.multi_ee_beam(chh, links, tgc[:, :, :4], tgc[:, :, 4:], seeds, [50.0] * 4,
                                                 [10.0] * 4), 2, "solves/s",
                       "2 target sets of this workload, oracle port (float64 NumPy), 1 core")
    print(json.dumps({"cpu_baseline": cpu, "workload": "config3 humanoid multi-EE IK-Beam (n=29, 4 end effectors, "
                      "64 seeds, 6+10 lane-LM steps, keep 4; SURVEY 8 H6)", "precision": prec, "targets": nb,
                      "ms": ms, "solves_per_s": nb / ms * 1e3, "success": res.success.float().mean().item(),
                      "roofline": roofline("config3 humanoid multi-EE IK-Beam", prec, nb / ms * 1e3)}), flush=True)
