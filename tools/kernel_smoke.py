"""Small launches of every kernel family, with their outputs saved.

    [KOP_LIB=variants/poison.so] python tools/kernel_smoke.py [fp32|fp64|both] [families] [--out FILE.npz]

Each family runs a handful of problems: IK-Beam (stage 1 / 2 / errors, ragged
request shapes), lanes, FK, Philox, host pipeline, mobile base, collision
IK-Beam, generic LM (k_col_solve), tree solve + multi-EE beam, trajectories
(+ report).  tests/test_gpu_checks.py runs it against the normal library and
the checking builds (kop_check.cuh: shared-memory poison, barrier jitter) and
compares the saved outputs bit for bit -- the substitute for compute-sanitizer,
which is closed on this GPU pool.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2505_03728_b200 as k
from paper_2505_03728_b200 import _device as dv, beam as kbeam, trajectory as ktraj
from paper_2505_03728_b200.benchmark import reachable_target_array
from paper_2505_03728_b200.robot import fk_arrays_device, link_poses_device
from paper_2505_03728_b200.tasks import IkBeamSolver

ARGS = [a for a in sys.argv[1:] if not a.startswith("--")]
OUT = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
if OUT in ARGS:
    ARGS.remove(OUT)
PRECS = {"fp32": ["fp32"], "fp64": ["fp64"], "both": ["fp32", "fp64"]}[ARGS[0] if ARGS else "both"]
ONLY = set(ARGS[1].split(",")) if len(ARGS) > 1 else None
SAVED = {}


def keep(name, prec, obj):
    """Record every array field of obj (tensor / numpy / dict / BeamBatch-like) under name/prec."""
    def arr(x):
        return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)
    if isinstance(obj, dict):
        items = obj.items()
    elif isinstance(obj, (list, tuple)):
        items = enumerate(obj)
    elif hasattr(obj, "__dataclass_fields__"):
        items = ((f, getattr(obj, f)) for f in obj.__dataclass_fields__)
    else:
        items = [("value", obj)]
    for key, v in items:
        if v is None:
            continue
        if hasattr(v, "__dataclass_fields__") or isinstance(v, (dict, list, tuple)):
            keep(f"{name}.{key}", prec, v)
        else:
            SAVED[f"{name}.{key}/{prec}"] = arr(v)

DEMO = k.WorldModel([k.Sphere([0.45, 0.1, 0.55], 0.12), k.Capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
                     k.HalfSpace([0.0, 0.0, 1.0], -0.3)])
m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
hum = k.load_robot(k.robot_path("humanoid29.urdf"))
EES = ["left_hand", "right_hand", "left_foot", "right_foot"]


def pose(a):
    a = a.cpu().numpy() if hasattr(a, "cpu") else a
    return k.Transform3.from_parts(a[:4], a[4:])


def fam(name):
    return ONLY is None or name in ONLY


def done(name, prec):
    torch.cuda.synchronize()
    print(f"ok {name} {prec}", flush=True)


from paper_2505_03728_b200._lib import lib  # noqa: E402

print("build:", lib().kop_build_info().decode(), flush=True)
probe = torch.zeros(4096, dtype=torch.int32, device="cuda")
assert lib().kop_check_probe(probe.data_ptr(), 4096, torch.cuda.current_stream().cuda_stream) == 0
torch.cuda.synchronize()
print("smem probe all-poison:", bool((probe == -1).all()), flush=True)
tg = reachable_target_array(m, "flange", 8, 77)
for prec in PRECS:
    if fam("fk"):
        q = dv.to_dev(np.random.default_rng(0).uniform(m.lower_limits, m.upper_limits, (33, 7)))
        keep("fk", prec, fk_arrays_device(m, q, precision=prec))
        done("fk", prec)
    if fam("beam"):
        s = IkBeamSolver(m, "flange", rng_seed=77, precision=prec)
        keep("beam", prec, s.solve_device(tg))
        done("beam", prec)
        # seeds not a multiple of a warp, keep 7
        s = IkBeamSolver(m, "flange", seeds=37, keep=7, rng_seed=3, precision=prec)
        keep("beam-ragged", prec, s.solve_device(tg[:5]))
        done("beam-ragged", prec)
    if fam("host"):
        s = IkBeamSolver(m, "flange", rng_seed=77, precision=prec)
        keep("host", prec, s.solve_host(tg.cpu().numpy(), chunk=3, n_streams=2))
        done("host-pipeline", prec)
    if fam("mobile"):
        s = IkBeamSolver(m, "flange", rng_seed=77, precision=prec, optimize_base=True)
        keep("mobile", prec, s.solve_device(tg[:4]))
        done("mobile", prec)
    if fam("lanes"):
        lp = kbeam.IkLaneProblem(m, "flange", pose(tg[0]), 50, 10, 100, 0.01, precision=prec)
        st = lp.start_state(k.sample_seed_configurations(m, 8, 1))
        lp.run(st, 3)
        keep("lanes", prec, {"q": st.q, "cost": st.cost, "lam": st.damping, "hist": np.stack(st.history, 1)})
        done("lanes", prec)
    if fam("collision"):
        s = IkBeamSolver(m, "flange", rng_seed=77, precision=prec, world=DEMO, self_collision=True)
        keep("collision-beam", prec, s.solve_device(tg[:3]))
        done("collision-beam", prec)
    if fam("lm"):
        probs = []
        for i in range(5):
            T = pose(tg[i])
            probs.append(k.Problem(k.VariableSet.of(q=m.rest_pose.copy()), [
                k.pose_cost(m, "q", "flange", T, position_weight=50, orientation_weight=10),
                k.limit_cost(m, "q", weight=100), k.rest_cost("q", m.rest_pose, weight=0.01),
                k.world_collision_cost(m, "q", DEMO, weight=20), k.self_collision_cost(m, "q", weight=5)]))
        reps = k.solve_batch(probs, k.SolveOptions(precision=prec, max_iterations=12))
        keep("generic-lm", prec, {"q": np.stack([r.final_values.value("q") for r in reps]),
                                  "hist": np.array([r.cost_history + [np.nan] * (13 - len(r.cost_history))
                                                    for r in reps])})
        done("generic-lm", prec)
    if fam("tree"):
        qt = dv.to_dev(np.random.default_rng(29).uniform(hum.lower_limits, hum.upper_limits, (3, hum.actuated_count)))
        tgh = torch.stack([link_poses_device(hum, qt, e) for e in EES], dim=1).contiguous()
        keep("tree-beam", prec, k.solve_ik_beam_multi(hum, EES, tgh, seeds=8, keep=2, precision=prec))
        done("tree-beam", prec)
        probs = []
        th = tgh.cpu().numpy()
        for i in range(3):
            probs.append(k.Problem(k.VariableSet.of(q=hum.rest_pose.copy()),
                                   [k.pose_cost(hum, "q", e, pose(th[i, j]), position_weight=50,
                                                orientation_weight=10) for j, e in enumerate(EES)]
                                   + [k.limit_cost(hum, "q", weight=100), k.rest_cost("q", hum.rest_pose, weight=0.01)]))
        reps = k.solve_batch(probs, k.SolveOptions(precision=prec, max_iterations=8))
        keep("tree-solve", prec, {"q": np.stack([r.final_values.value("q") for r in reps]),
                                  "hist": np.array([r.cost_history + [np.nan] * (9 - len(r.cost_history))
                                                    for r in reps])})
        done("tree-solve", prec)
    if fam("traj"):
        rng = np.random.default_rng(5)
        for TT in (20, 64):
            qa = rng.uniform(m.lower_limits, m.upper_limits, (2, 7))
            qb = rng.uniform(m.lower_limits, m.upper_limits, (2, 7))
            mid = link_poses_device(m, dv.to_dev(0.5 * (qa + qb)), "flange").cpu().numpy()[:, 4:7]
            obs = np.zeros((2, 1, 8))
            obs[:, 0, 1:4] = mid
            obs[:, 0, 7] = 0.07
            pl = k.TrajectoryPlanner(m, "flange", timesteps=TT, precision=prec, max_iterations=4)
            res = pl.solve_anchored_device(dv.to_dev(np.stack([qa, qb], axis=1)), dv.to_dev(obs), 1)
            keep(f"traj{TT}", prec, res)
            keep(f"traj{TT}-report", prec,
                 ktraj.trajectory_signed_distances_batch(m, res["qs"], dv.to_dev(obs), 1, "flange"))
            done(f"traj-T{TT}", prec)
if OUT:
    np.savez_compressed(OUT, **SAVED)
print(f"kernel smoke complete: {len(SAVED)} arrays", flush=True)
