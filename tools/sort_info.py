"""Print the scatter-sort diagnostics of the first steps of a shock workload."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_1009_2768_b200 import api

wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
W = bench.workload(wl)
T = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=torch.float32)
sim = api.Simulation(T(W["vx"]), T(W["vy"]), T(W["vz"]), x=T(W["x"]), shock=W["setup"], **W["kw"])
for k in range(steps):
    sim.step(1)
    print(k, sim.sort_info(), flush=True)
