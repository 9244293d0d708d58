"""Per-kernel registers / spills from `nvcc -Xptxas -v` output on stdin."""
import re, sys
cur = None
rows = []
for ln in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", ln)
    if m:
        cur = {"name": m.group(1)}
        rows.append(cur)
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m and cur is not None and "stack" not in cur:
        cur["stack"], cur["spill_st"], cur["spill_ld"] = map(int, m.groups())
    m = re.search(r"Used (\d+) registers", ln)
    if m and cur is not None:
        cur["regs"] = int(m.group(1))
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for r in rows:
    if pat in r["name"]:
        n = re.sub(r"_ZN3kop\d+", "", r["name"])[:70]
        print(f"{n:70s} regs {r.get('regs','?'):>4} stack {r.get('stack','?'):>5} spill {r.get('spill_st','?')}/{r.get('spill_ld','?')}")
