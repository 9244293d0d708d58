"""Executed-flop counts of the widened-config kernels (for their rooflines).

  python tools/widened_flops.py run            # launches each workload once (small batches)
  ncu --metrics <FLOP_METRICS> --csv --log-file f.csv python tools/widened_flops.py run
  python tools/widened_flops.py parse f.csv    # -> profiles/r01_widened_flops.json

Flops = 2*FFMA + FADD + FMUL (FP32) and 2*DFMA + DADD + DMUL (FP64), from the
per-thread SASS counters, summed over every launch of a kernel and divided by
the units (targets / problems / trajectories) that kernel processed.  These
are EXECUTED flops (the §8(d) algorithmic convention exists only for config 1).
"""
import csv, json, os, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
FLOP_METRICS = ",".join(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum"
                        for op in ("ffma", "fadd", "fmul", "dfma", "dadd", "dmul"))
# (workload, kernel-name substring, precision tag in the template args, units)
WORK = [
    ("config4 collision IK-Beam", ("k_col_beam_stage", "k_beam_errors"), "float", 2000),
    ("generic LM solve (collision stack)", "k_col_solve", "float", 2000),
    ("generic LM solve (collision stack)", "k_col_solve", "double", 2000),
    ("mobile-base IK-Beam", "k_beam_stage", "float", 2000),
    ("config5 trajectory optimisation T=64", "k_traj_solve", "float", 148),
    ("config5 trajectory optimisation T=64", "k_traj_solve", "double", 148),
    ("config3 humanoid multi-EE IK", "k_tree_solve", "float", 2000),
    ("config3 humanoid multi-EE IK", "k_tree_solve", "double", 2000),
    ("config3 humanoid multi-EE IK-Beam", ("k_tree_beam_stage", "k_tree_beam_prune"), "float", 2000),
    ("config3 humanoid multi-EE IK-Beam", ("k_tree_beam_stage", "k_tree_beam_prune"), "double", 2000),
]


def run():
    import numpy as np, torch, ctypes as C
    import paper_2505_03728_b200 as k
    from paper_2505_03728_b200 import _device as dv
    from paper_2505_03728_b200._lib import check, lib
    from paper_2505_03728_b200.benchmark import reachable_target_array, disk_translations
    from paper_2505_03728_b200.robot import link_poses_device
    from paper_2505_03728_b200.solver import _options, plan
    from paper_2505_03728_b200.tasks import IkBeamSolver

    m = k.load_robot(k.robot_path("arm7.urdf"), k.robot_path("arm7.sidecar.json"))
    demo = k.WorldModel([k.Sphere([0.45, 0.1, 0.55], 0.12), k.Capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
                         k.HalfSpace([0.0, 0.0, 1.0], -0.3)])
    n = 2000
    tg = reachable_target_array(m, "flange", n, 77)
    IkBeamSolver(m, "flange", rng_seed=77, world=demo, self_collision=True).solve_device(tg)
    prob = k.Problem(k.VariableSet.of(q=m.rest_pose.copy()), [
        k.pose_cost(m, "q", "flange", k.Transform3.identity(), position_weight=50, orientation_weight=10),
        k.limit_cost(m, "q", weight=100), k.rest_cost("q", m.rest_pose, weight=0.01),
        k.world_collision_cost(m, "q", demo, weight=20), k.self_collision_cost(m, "q", weight=5)])
    p = plan(prob)
    for prec in ("fp32", "fp64"):
        opts = _options(k.SolveOptions(precision=prec))
        q0 = dv.to_dev(np.tile(m.rest_pose, (n, 1)))
        outs = [dv.empty((n, 7)), dv.empty(n), dv.empty(n), None, torch.empty(n, dtype=torch.int32, device="cuda"),
                torch.empty(n, dtype=torch.int32, device="cuda")]
        check(lib().kop_lm_solve(m._handle, 8, C.byref(p.costs), C.byref(opts), dv.ptr(tg), dv.ptr(q0), n,
                                 *(dv.ptr(x) for x in outs), dv.stream_handle()), "solve")
    sh = tg.cpu().numpy().copy()
    sh[:, 4:] += disk_translations(n, 2.0, 2024)
    IkBeamSolver(m, "flange", rng_seed=77, optimize_base=True).solve_device(dv.to_dev(sh))
    nt = 148
    rng = np.random.default_rng(5)
    qa = rng.uniform(m.lower_limits, m.upper_limits, (nt, 7))
    qb = rng.uniform(m.lower_limits, m.upper_limits, (nt, 7))
    mid = link_poses_device(m, dv.to_dev(0.5 * (qa + qb)), "flange").cpu().numpy()[:, 4:7]
    obs = np.zeros((nt, 1, 8)); obs[:, 0, 1:4] = mid; obs[:, 0, 7] = 0.07
    for prec in ("fp32", "fp64"):
        k.TrajectoryPlanner(m, "flange", timesteps=64, precision=prec).solve_anchored_device(
            np.stack([qa, qb], axis=1), obs, 1, history=False)
    hum = k.load_robot(k.robot_path("humanoid29.urdf"))
    ees = ["left_hand", "right_hand", "left_foot", "right_foot"]
    qt = dv.to_dev(np.random.default_rng(29).uniform(hum.lower_limits, hum.upper_limits, (n, hum.actuated_count)))
    tgh = torch.stack([link_poses_device(hum, qt, e) for e in ees], dim=1).contiguous()
    w0 = k.CostWeights()
    hp = plan(k.Problem(k.VariableSet.of(q=hum.rest_pose.copy()),
                        [k.pose_cost(hum, "q", e, k.Transform3.identity(), position_weight=w0.pose_position,
                                     orientation_weight=w0.pose_orientation) for e in ees]
                        + [k.limit_cost(hum, "q", weight=w0.limit), k.rest_cost("q", hum.rest_pose, weight=w0.rest)]))
    for prec in ("fp32", "fp64"):
        opts = _options(k.SolveOptions(precision=prec))
        q0 = dv.to_dev(np.tile(hum.rest_pose, (n, 1)))
        outs = [dv.empty((n, hum.actuated_count)), dv.empty(n), dv.empty(n), None,
                torch.empty(n, dtype=torch.int32, device="cuda"), torch.empty(n, dtype=torch.int32, device="cuda")]
        check(lib().kop_multi_pose_solve(hum._handle, C.byref(hp.costs), C.byref(opts), dv.ptr(tgh), dv.ptr(q0), n,
                                         *(dv.ptr(x) for x in outs), dv.stream_handle()), "tree")
    torch.cuda.synchronize()
    for prec in ("fp32", "fp64"):  # multi-EE IK-Beam; the prune kernel is attributed to both (no FP work)
        k.solve_ik_beam_multi(hum, ees, tgh, precision=prec, device_out=True)
    torch.cuda.synchronize()


def parse(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hi]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    launches = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        key = (r[0], r[ki])
        launches.setdefault(key, {})[r[mi]] = float(r[vi].replace(",", ""))
    out = []
    for name, sub, prec, units in WORK:
        f32 = f64 = 0.0
        kernels = set()
        for (lid, kname), mets in launches.items():
            subs = sub if isinstance(sub, tuple) else (sub,)
            if not any(x in kname for x in subs):
                continue
            if ("k_beam_errors" not in kname and "k_tree_beam_prune" not in kname
                    and not any(t in kname.split("(")[0] for t in (f"Cfg<{prec}", f"<{prec}>", f"<{prec},"))):
                continue
            if sub == "k_beam_stage" and "1, 1>" not in kname.replace("true", "1"):
                continue  # mobile: BASE shapes only
            kernels.add(kname.split("(")[0])
            g = lambda op: mets.get(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum", 0.0)
            f32 += 2 * g("ffma") + g("fadd") + g("fmul")
            f64 += 2 * g("dfma") + g("dadd") + g("dmul")
        out.append({"workload": name, "precision": "fp32" if prec == "float" else "fp64", "units": units,
                    "kernels": sorted(kernels), "fp32_flops_per_unit": f32 / units,
                    "fp64_flops_per_unit": f64 / units})
    dst = os.path.join(ROOT, "profiles", "r01_widened_flops.json")
    with open(dst, "w") as fh:
        json.dump({"source": "ncu --metrics " + FLOP_METRICS + " of tools/widened_flops.py run",
                   "workloads": out}, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run()
    else:
        parse(sys.argv[2])
