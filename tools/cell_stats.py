"""Statistics rows of a homogeneous bench workload after a few steps."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_1009_2768_b200 import api

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
W = bench.workload(wl)
td = torch.float32 if W["dtype"] == np.float32 else torch.float64
T = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=td)
sim = api.Simulation(T(W["vx"]), T(W["vy"]), T(W["vz"]), offsets=W["offsets"], **W["kw"])
for k in range(steps):
    sim.step(1)
    st = sim.stats()
    print(k, {f: float(st[f].mean()) for f in ("n", "p", "depth", "attempts", "m_used", "m_next", "proposals",
                                              "accepted", "leaves", "thermalised", "E1")}, flush=True)
