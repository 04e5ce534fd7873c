"""The pooled-batch shock collision kernel against the lock-step kernel on the
same workload: particles and statistics must be bitwise identical (same keyed
draws, same reduction orders).  usage: batch_vs_lock.py wl steps [f64]"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_1009_2768_b200 import api

wl = sys.argv[1] if len(sys.argv) > 1 else "c4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
f64 = len(sys.argv) > 3 and sys.argv[3] == "f64"
W = bench.workload(wl)
td = torch.float64 if f64 else torch.float32
T = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=td)
sims = []
for flag in ("0", "1"):
    os.environ["TRMCR_SHOCK_BATCH"] = flag
    sims.append(api.Simulation(T(W["vx"]), T(W["vy"]), T(W["vz"]), x=T(W["x"]), shock=W["setup"], **W["kw"]))
ok = True
for k in range(steps):
    for s in sims:
        s.step(1)
    a, b = sims[0].particles(), sims[1].particles()
    sa, sb = sims[0].stats(), sims[1].stats()
    diff = {f: int(np.sum(a[f] != b[f])) for f in ("x", "vx", "vy", "vz")}
    sd = {f: int(np.sum(sa[f] != sb[f])) for f in sa.dtype.names if np.any(sa[f] != sb[f])}
    print(k, "particle diffs", diff, "stat diffs", sd, flush=True)
    ok = ok and not any(diff.values()) and not sd
print("IDENTICAL" if ok else "DIFFERENT")
