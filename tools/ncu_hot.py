"""Hot CUDA source lines (stall samples, instructions) of one kernel from
`ncu -i REP --page source --csv --print-source cuda,sass` output."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None
hdr = None
recs = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] == "Function Name" or hdr is None or r[0] == "":
        continue
    try:
        smp = float(r[4])
        ins = float(r[7])
    except (ValueError, IndexError):
        continue
    recs.append((smp, ins, fname, int(r[0]), r[1].strip()[:90]))
ts = sum(x[0] for x in recs) or 1
ti = sum(x[1] for x in recs) or 1
print(f"total samples {ts:.0f}  warp instructions {ti:.0f}")
for smp, ins, f, ln, src in sorted(recs, reverse=True)[:top]:
    print(f"{smp / ts * 100:5.1f}% smp {ins / ti * 100:5.1f}% ins  {f}:{ln}  {src}")
