"""Per-function totals (stall samples, warp instructions, lane utilisation) of one
kernel from `ncu -i REP --page source --csv --print-source cuda,sass` output.
A source line belongs to the enclosing top-level definition of its file (the
last line before it that starts a definition at column 0)."""
import collections
import csv
import os
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
root = sys.argv[2] if len(sys.argv) > 2 else "."
defs = {}


def owner(path, line):
    fn = os.path.basename(path)
    if fn not in defs:
        starts = []
        p = os.path.join(root, "paper_1009_2768_b200", "csrc", fn)
        if os.path.exists(p):
            for i, s in enumerate(open(p), 1):
                if re.match(r"^[A-Za-z_].*\b([A-Za-z_][A-Za-z0-9_]*)\s*\(", s) and not s.startswith(
                        ("template", "#", "namespace", "struct", "constexpr", "enum", "}")):
                    m = re.findall(r"\b([A-Za-z_][A-Za-z0-9_]*)\s*\(", s)
                    name = [x for x in m if x not in ("__launch_bounds__", "__align__")]
                    starts.append((i, name[0] if name else "?"))
        defs[fn] = starts
    best = "?"
    for i, nm in defs[fn]:
        if i <= line:
            best = nm
    return f"{fn}:{best}"


fname = None
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1]
        continue
    if r[0] in ("Line No", "Function Name") or fname is None:
        continue
    try:
        ln = int(r[0])
        smp, ins, thr = float(r[4]), float(r[7]), float(r[8])
    except (ValueError, IndexError):
        continue
    a = agg[owner(fname, ln)]
    a[0] += smp; a[1] += ins; a[2] += thr
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total samples {ts:.0f}  warp instructions {ti:.0f}")
for k, (smp, ins, thr) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"{smp / ts * 100:5.1f}% smp {ins / ti * 100:5.1f}% ins  lanes {thr / max(ins, 1):5.1f}  {k}")
