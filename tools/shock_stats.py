"""Per-cell statistics summary of a shock workload after a few steps."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_1009_2768_b200 import api

wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
eps = float(sys.argv[3]) if len(sys.argv) > 3 else None
W = bench.workload(wl, eps_override=eps)
T = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=torch.float32)
sim = api.Simulation(T(W["vx"]), T(W["vy"]), T(W["vz"]), x=T(W["x"]), shock=W["setup"], **W["kw"])
sim.step(steps)
st = sim.stats()
n = st["n"]
print("cells", len(n), "particles", n.sum())
for f in ["n", "p", "leaves", "untouched", "thermalised", "proposals", "accepted", "m_used", "m_next", "attempts",
          "depth", "E1"]:
    v = st[f]
    print(f"{f:12s} mean {v.mean():10.4f}  min {v.min():10.4f}  max {v.max():10.4f}  sum/n {v.sum() / n.sum():8.4f}")
q = np.quantile(n, [0.01, 0.1, 0.5, 0.9, 0.99])
print("n quantiles", q)
for f in ("attempts", "m_used", "depth"):
    u, c = np.unique(st[f], return_counts=True)
    print(f, "histogram", dict(zip(u.tolist(), c.tolist())))
