"""Per-CUDA-source-line instruction counts and stall samples from
`ncu --page source --csv --print-source cuda,sass` output."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
fname = None
recs = []
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    try:
        ins = float(r[7]) if r[7] not in ("-", "") else 0.0
        smp = float(r[4]) if r[4] not in ("-", "") else 0.0
    except (ValueError, IndexError):
        continue
    recs.append((ins, smp, fname, r[0], r[1].strip()[:80]))
ti = sum(x[0] for x in recs) or 1
ts = sum(x[1] for x in recs) or 1
print("by instructions:")
for ins, smp, f, ln, src in sorted(recs, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{ins / ti * 100:5.1f}% inst {smp / ts * 100:5.1f}% stall  {f}:{ln}  {src}")
print("by stall samples:")
for ins, smp, f, ln, src in sorted(recs, key=lambda x: -x[1])[:15]:
    print(f"{ins / ti * 100:5.1f}% inst {smp / ts * 100:5.1f}% stall  {f}:{ln}  {src}")
