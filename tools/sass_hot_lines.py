"""Dynamic instruction counts of a kernel per CUDA source line, offline: an ncu
source page (--page source --csv --print-source sass, gzip) of one launch plus
the cubin of the SAME build (nvdisasm -g maps SASS offsets to file:line).

usage: python tools/sass_hot_lines.py SASS.csv.gz CUBIN MANGLED_NAME [TOP]"""
import collections
import csv
import gzip
import io
import re
import subprocess
import sys

path, cubin, mang = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(io.TextIOWrapper(gzip.open(path))))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) > 5]
ia, isrc, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
ist = hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][ia], 16)
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
i = dis.find(".text." + mang + ":")
seg = dis[i:dis.find("//---------------------", i + 10)]
line_of, cur = {}, None
for ln in seg.splitlines():
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
agg, fp, st = collections.Counter(), collections.Counter(), collections.Counter()
tot = 0
for r in data:
    off, n = int(r[ia], 16) - base, int(r[iex] or 0)
    tot += n
    key = line_of.get(off, ("?", 0))
    agg[key] += n
    st[key] += int(r[ist] or 0)
    op = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip()).split()[0].split(".")[0]
    if op in ("FFMA", "FMUL", "FADD"):
        fp[key] += n
stot = sum(st.values())
print(f"{'line':28s} {'inst%':>7s} {'fp%':>6s} {'stall%':>7s}")
for k, v in agg.most_common(top):
    print(f"{k[0] + ':' + str(k[1]):28s} {v / tot * 100:7.2f} {fp[k] / max(v, 1) * 100:6.1f} {st[k] / stot * 100:7.2f}")
