"""Small driver for ncu captures: build a workload, run a few steps."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_1009_2768_b200 import api

wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
W = bench.workload(wl)
td = torch.float32 if W["dtype"] == np.float32 else torch.float64
T = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=td)
if W["kind"] == "hom":
    sim = api.Simulation(T(W["vx"]), T(W["vy"]), T(W["vz"]), offsets=W["offsets"], **W["kw"])
else:
    sim = api.Simulation(T(W["vx"]), T(W["vy"]), T(W["vz"]), x=T(W["x"]), shock=W["setup"], **W["kw"])
for _ in range(steps):
    sim.step(1)
torch.cuda.synchronize()
print("ok", sim.launch_count)
