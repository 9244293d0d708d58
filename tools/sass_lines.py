"""Attribute ncu warp-stall samples to CUDA source lines without the GUI.

  python tools/sass_lines.py <report.ncu-rep> <kernel-substring> [top]

Reads the report's SASS page (per-instruction samples, addresses from the
kernel entry), disassembles the matching function from the in-tree .so with
nvdisasm -g (innermost file:line per instruction), and prints the sampled
stall share per source line and per function-sized line range.
"""
import csv, glob, io, os, re, subprocess, sys, tempfile
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.environ.get("KOP_LIB") or os.path.join(ROOT, "paper_2505_03728_b200", "libkinoptik_b200.so")


def sass_samples(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    name = rows[0][1]
    h = rows[1]
    ai, si = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
    reasons = [(i, c[6:]) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    base = int(rows[2][ai], 16)
    return name, [(int(r[ai], 16) - base, int(r[si] or 0),
                   {n: int(r[i] or 0) for i, n in reasons if r[i] not in ("", "0")})
                  for r in rows[2:] if len(r) > si]


def line_map(kernel_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", SO], cwd=tmp, capture_output=True)
    for cub in sorted(glob.glob(os.path.join(tmp, "*.cubin"))):
        txt = subprocess.run(["nvdisasm", "-gi", cub], capture_output=True, text=True).stdout
        for sec in re.split(r"\n\.text\.", txt)[1:]:
            fname = sec.split(":", 1)[0]
            if not all(s in fname for s in kernel_sub.split(",")):
                continue
            chain, m = [], {}
            for ln in sec.splitlines():
                f = re.search(r'//## File "([^"]+)", line (\d+)', ln)
                if f:
                    chain.append(f"{os.path.basename(f.group(1))}:{f.group(2)}")
                    continue
                a = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
                if a:
                    if chain:
                        cur, chain = (chain[0], chain[-1]), []  # (innermost, kernel-body line)
                    m[int(a.group(1), 16)] = cur
            return fname, m
    raise SystemExit(f"no function matching {kernel_sub}")


def main():
    rep, sub = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    kname, samples = sass_samples(rep)
    fname, m = line_map(sub)
    inner, outer, why = Counter(), Counter(), {}
    for addr, s, r in samples:
        lo = m.get(addr, ("?", "?"))
        inner[lo[0]] += s
        outer[lo[1]] += s
        why.setdefault(lo[0], Counter()).update(r)
    tot = sum(inner.values()) or 1
    print(f"{kname[:100]}\nsamples={tot}\n-- by kernel-body line (call sites inlined into it)")
    for k, v in outer.most_common(top):
        print(f"{v / tot:7.2%}  {k}")
    print("-- by innermost line (top stall reasons)")
    for k, v in inner.most_common(top):
        rs = ", ".join(f"{n} {c / max(v, 1):.0%}" for n, c in why[k].most_common(3))
        print(f"{v / tot:7.2%}  {k:28s} {rs}")


if __name__ == "__main__":
    main()
