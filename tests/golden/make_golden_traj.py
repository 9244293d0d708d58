"""Golden vectors for trajectory optimisation (config 5) from the REFERENCE.

Build container only (``/root/reference`` is absent on the GPU box); writes
``reference_golden_traj.npz`` next to this file.

    python tests/golden/make_golden_traj.py

Scenes are ``benchmark._blocked_scene(arm7, "flange", 3000, i)``
(benchmark.py:250-277, the acceptance set of test_acceptance.py:96-124) plus
an empty-world case.  Each runs the reference ``tasks.plan_trajectory``
(tasks.py:309-424) with its ``_endpoint_ik`` results (the anchors) and the
``solve`` Problem intercepted, so the oracle and the device solve can be fed
the same anchors; the weighted residual, gradient and Gauss-Newton matrix of
that Problem at the straight-line initialisation come from ``solver.assemble``
(solver.py:287-324).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from kinoptik import benchmark, robot, solver, tasks  # noqa: E402
from kinoptik.benchmark import generate_reachable_targets  # noqa: E402

ROBOTS = os.path.join(REF, "kinoptik", "robots")
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden_traj.npz")
TERMS = ["max_iterations", "gradient_converged", "step_converged", "numerical_failure"]


def run(arm7, pa, pb, world, T, seed):
    anchors, problems = [], []
    orig_ik, orig_solve = tasks._endpoint_ik, tasks.solve

    def ik(req, pose, label):
        q = orig_ik(req, pose, label)
        anchors.append(q)
        return q

    def solve(problem, options=None):
        problems.append(problem)
        return orig_solve(problem, options)

    tasks._endpoint_ik, tasks.solve = ik, solve
    try:
        res = tasks.plan_trajectory(tasks.TrajRequest(model=arm7, start_pose=pa, goal_pose=pb, timesteps=T, dt=0.1,
                                                      world=world, rng_seed=seed, target_link="flange"))
    finally:
        tasks._endpoint_ik, tasks.solve = orig_ik, orig_solve
    r, jac = solver.assemble(problems[0], problems[0].variables)
    J = jac.to_dense()
    static, swept = tasks.trajectory_signed_distances(arm7, res.qs, world)
    rep = res.report
    return {
        "T": T,
        "q_start": anchors[0],
        "q_goal": anchors[1],
        "obstacles": np.array([[0.0, *s.center, 0.0, 0.0, 0.0, s.radius] for s in world.obstacles]).reshape(-1, 8),
        "r0": r,
        "grad0": J.T @ r,
        "h0": J.T @ J,
        "qs": res.qs,
        "cost": rep.final_cost,
        "hist": np.pad(rep.cost_history, (0, 151 - len(rep.cost_history)), constant_values=np.nan),
        "iters": rep.iterations_run,
        "term": TERMS.index(rep.termination),
        "static": static,
        "swept": swept,
        "min_sd": res.min_signed_distance,
        "collision_free": res.collision_free,
        "success": res.success,
        "pos_err": [res.start_pos_error, res.goal_pos_error],
        "rot_err": [res.start_rot_error, res.goal_rot_error],
        "pa": np.concatenate([pa.rotation.wxyz, pa.translation]),
        "pb": np.concatenate([pb.rotation.wxyz, pb.translation]),
    }


def main():
    arm7 = robot.load_robot(os.path.join(ROBOTS, "arm7.urdf"), os.path.join(ROBOTS, "arm7.sidecar.json"))
    g = {"velocity_limits": arm7.velocity_limits}
    cases = []
    for i, T in ((0, 20), (1, 20), (2, 32)):  # T=32: 224 tangent dims, the reference's sparse-LU path
        pa, pb, world = benchmark._blocked_scene(arm7, "flange", 3000, i)
        cases.append((f"scene{i}", pa, pb, world, T, 3000 + i))
    tg = generate_reachable_targets(arm7, "flange", 2, 16)
    from kinoptik.collision import WorldModel

    cases.append(("empty", tg[0], tg[1], WorldModel(), 10, 0))
    for name, pa, pb, world, T, seed in cases:
        out = run(arm7, pa, pb, world, T, seed)
        for k, v in out.items():
            g[f"traj_{name}_{k}"] = np.asarray(v)
        print(name, T, out["iters"], TERMS[out["term"]], out["min_sd"], out["success"], flush=True)
    g["traj_cases"] = np.array([c[0] for c in cases])
    np.savez_compressed(OUT, **g)
    print(f"wrote {OUT}: {len(g)} arrays")


if __name__ == "__main__":
    main()
