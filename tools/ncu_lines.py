"""Aggregate ncu per-SASS-instruction stall samples onto CUDA source lines.

usage: python tools/ncu_lines.py <report.ncu-rep> <kernel-regex> <mangled-name> [cubin]
Needs the kernel compiled with -lineinfo (nvdisasm -g gives offset -> file:line).
"""
import csv, io, re, subprocess, sys
from collections import defaultdict

rep, kre, mangled = sys.argv[1:4]
cubin = sys.argv[4] if len(sys.argv) > 4 else "/tmp/cub/kop_kernels.sm_100a.cubin"
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
start = dis.index(".text." + mangled + ":")
end = dis.find("//---------------------", start)
dis = dis[start:end if end > 0 else None]
line_of, cur = {}, None
for ln in dis.splitlines():
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
heads = [i for i, r in enumerate(rows) if "Address" in r]
hi = heads[0]
rows = rows[: heads[1] - 1] if len(heads) > 1 else rows  # one section per profiled launch
h = rows[hi]
ia, iss, ie = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
base = int(rows[hi + 1][ia], 16)
agg = defaultdict(lambda: [0, 0])
tot = [0, 0]
for r in rows[hi + 1:]:
    if len(r) <= ie or not r[ia].startswith("0x"):
        continue
    off = int(r[ia], 16) - base
    key = line_of.get(off, ("?", 0))
    s, e = int(r[iss] or 0), int(r[ie] or 0)
    agg[key][0] += s
    agg[key][1] += e
    tot[0] += s
    tot[1] += e
print(f"total samples {tot[0]}, warp-instructions {tot[1]}")
for (f, l), (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[5]) if len(sys.argv) > 5 else 40]:
    print(f"{f}:{l:<5d} samples {s:8d} ({100*s/tot[0]:5.1f}%)  instr {e:11d} ({100*e/tot[1]:5.1f}%)")
