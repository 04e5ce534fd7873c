"""Summarise an ncu --page source --print-source sass CSV: opcode mix and stall samples."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
cnt, smp, lsb = Counter(), Counter(), Counter()
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ci["Source"]].strip()
    toks = src.split()
    if not toks:
        continue
    opc = toks[1] if toks[0].startswith("@") else toks[0]
    opc = opc.split(".")[0]
    cnt[opc] += float(r[ci["Instructions Executed"]] or 0)
    smp[opc] += float(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    lsb[opc] += float(r[ci["stall_long_sb"]] or 0)
tot = sum(cnt.values()); ts = sum(smp.values()) or 1
print("total warp instructions", tot)
for k, v in cnt.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{k:10s} {v/tot*100:6.2f}%  stall-samples {smp[k]/ts*100:6.2f}%  long_sb {lsb[k]/ts*100:5.2f}%")
