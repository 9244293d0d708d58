"""FP64 device vs oracle on the widened rows, >= 100 targets each: the share of
targets whose winner history stays within 1e-6 of the oracle's, and for every
other target the first divergent step and the near-tie that explains it
(oracle.ik_oracle.explain_divergence).  Writes one JSON object per workload.
Usage: python tools/fp64_divergence.py [N]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import paper_2505_03728_b200 as k
from oracle import collision_oracle as co, ik_oracle as o, tree_oracle as tro
from oracle_pool import par_batched
from paper_2505_03728_b200.benchmark import disk_translations, reachable_target_array

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
R = k.robot_path
m = k.load_robot(R("arm7.urdf"), R("arm7.sidecar.json"))
ch = o.load_chain_files(R("arm7.urdf"), R("arm7.sidecar.json"))


def report(name, h_dev, ref_hist, diag):
    rel = np.abs(h_dev - ref_hist) / ref_hist
    ok = rel.max(axis=1) < 1e-6
    ex = o.explain_divergence(h_dev, ref_hist, diag)
    print(json.dumps({"workload": name, "targets": len(ok), "within_1e-6": float(ok.mean()),
                      "divergent": [{"target": t, "kind": kd, "first_step": s, "oracle_gap": g} for t, kd, s, g in ex],
                      "max_gap": max([g for _, _, _, g in ex], default=0.0)}), flush=True)


# plain Panda IK-Beam (rng 77) -- the headline path in FP64
tg = reachable_target_array(m, "flange", N, 77).cpu().numpy()
seeds = o.sample_seeds(ch, 64, 77)
ref = par_batched(o.ik_beam, ch, 8, tq=tg[:, :4], tt=tg[:, 4:], seeds=seeds, split=("tq", "tt"))
got = k.solve_ik_beam_batch(m, "flange", tg, rng_seed=77, precision="fp64")
report("panda ik-beam", got.history, ref.hist, ref.diag)

# request shapes
tgs = reachable_target_array(m, "flange", N, 5).cpu().numpy()
for seeds_n, keep, prune, total in [(10, 3, 1, 2), (64, 1, 6, 16), (100, 7, 3, 9)]:
    s = o.sample_seeds(ch, seeds_n, 9)
    ref = par_batched(o.ik_beam, ch, 8, tq=tgs[:, :4], tt=tgs[:, 4:], seeds=s, total_steps=total, prune_after=prune,
                      keep=keep, split=("tq", "tt"))
    got = k.solve_ik_beam_batch(m, "flange", tgs, seeds=seeds_n, keep=keep, prune_after=prune, total_steps=total,
                                rng_seed=9, precision="fp64")
    report(f"panda ik-beam shape {seeds_n}/{keep}/{prune}/{total}", got.history, ref.hist, ref.diag)

# mobile base (disk-shifted targets)
tgm = reachable_target_array(m, "flange", N, 2024).cpu().numpy()
tgm[:, 4:] += disk_translations(N, 2.0, 2024)
s = o.sample_seeds(ch, 64, 2024)
ref = par_batched(o.ik_beam, ch, 8, tq=tgm[:, :4], tt=tgm[:, 4:], seeds=s, use_base=True, split=("tq", "tt"))
got = k.solve_ik_beam_batch(m, "flange", tgm, rng_seed=2024, precision="fp64", optimize_base=True)
report("mobile ik-beam", got.history, ref.hist, ref.diag)

# collision IK-Beam (config 4)
DEMO = k.WorldModel([k.Sphere([0.45, 0.1, 0.55], 0.12), k.Capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
                     k.HalfSpace([0.0, 0.0, 1.0], -0.3)])
DEMO_O = [co.sphere([0.45, 0.1, 0.55], 0.12), co.capsule([-0.5, -0.4, 0.2], [-0.5, 0.4, 0.6], 0.1),
          co.halfspace([0.0, 0.0, 1.0], -0.3)]
sp = co.load_spheres_files(ch, R("arm7.urdf"), R("arm7.sidecar.json"))
tgc = reachable_target_array(m, "flange", N, 31).cpu().numpy()
s = o.sample_seeds(ch, 64, 31)
ref = par_batched(co.ik_beam_collision, ch, sp, DEMO_O, 8, tq=tgc[:, :4], tt=tgc[:, 4:], seeds=s,
                  cc=co.CollisionCosts(), split=("tq", "tt"))
got = k.solve_ik_collision_batch(m, "flange", tgc, world=DEMO, rng_seed=31, precision="fp64")
report("collision ik-beam", got.history, ref.hist, ref.diag)

# humanoid multi-EE IK-Beam (config 3)
hum = k.load_robot(R("humanoid29.urdf"))
chh = o.load_chain_files(R("humanoid29.urdf"))
EES = ["left_hand", "right_hand", "left_foot", "right_foot"]
qt = np.random.default_rng(5).uniform(hum.lower_limits, hum.upper_limits, (N, hum.actuated_count))
lq, lp, _, _ = o.fk(chh, qt)
links = [chh.link(e) for e in EES]
tq = np.stack([o.qcanon(lq[:, l]) for l in links], 1)
tt = np.stack([lp[:, l] for l in links], 1)
s = o.sample_seeds(chh, 64, 3)
ref = par_batched(tro.multi_ee_beam, chh, links, tq=tq, tt=tt, seeds=s, w_pos=[50.0] * 4, w_ori=[10.0] * 4,
                  split=("tq", "tt"))
got = k.solve_ik_beam_multi(hum, EES, np.concatenate([tq, tt], axis=2), rng_seed=3, precision="fp64")
report("humanoid multi-EE ik-beam", got.history, ref["hist"], ref["diag"])
