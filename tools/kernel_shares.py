"""Dominant-kernel shares of the widened IK-Beams from ncu launch lists
(`ncu --metrics gpu__time_duration.sum --csv`, tools/gpu_prof_r02.sh LAUNCHES=1):
the second of the two profiled solves (after warm-up) of each workload.

  python tools/kernel_shares.py profiles/r02_ncu   -> profiles/r02_kernel_shares.json
"""
import csv
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "profiles/r02_ncu"
out_path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "r02_kernel_shares.json")
STAGE1 = {"col_beam": "k_col_beam_stage1", "tree_beam": "k_tree_beam_stage1"}
out = {"source": "ncu --metrics gpu__time_duration.sum launch lists of tools/prof_workloads.py "
                 "(profiles/r02_ncu/launches_*.csv), second (profiled) call", "all": {}}
for w, s1 in STAGE1.items():
    for prec in ("fp32", "fp64"):
        path = os.path.join(d, f"launches_{w}_{prec}.csv")
        if not os.path.exists(path):
            continue
        with open(path) as f:
            rows = [r for r in csv.reader(line for line in f if line.startswith('"'))]
        hdr, rows = rows[0], rows[1:]
        ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
        launches = [(r[ik], float(r[iv])) for r in rows]
        starts = [i for i, (k, _) in enumerate(launches) if s1 in k]
        first = starts[-1] - (1 if starts[-1] > 0 and "k_philox" in launches[starts[-1] - 1][0] else 0)
        call = [(k, t) for k, t in launches[first:] if "at::" not in k]  # the solve's own kernels
        tot = sum(t for _, t in call)
        shares = {}
        for k, t in call:
            name = k.split("(")[0].split("<")[0].replace("void ", "").strip()
            shares[name] = shares.get(name, 0.0) + t / tot
        cfg = {"col_beam": "config4", "tree_beam": "config3"}[w]
        out[f"{cfg}_{prec}"] = round(next(v for k, v in shares.items() if s1 in k), 4)
        out["all"][f"{w}_{prec}"] = {k: round(v, 4) for k, v in shares.items()}
with open(out_path, "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
