"""How persistent is a shock cell's number of RAD attempts from one step to the
next (would grouping cells by last step's attempts even out a lock-step group)?"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench
from paper_1009_2768_b200 import api

wl = sys.argv[1] if len(sys.argv) > 1 else "c5"
W = bench.workload(wl)
T = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=torch.float32)
sim = api.Simulation(T(W["vx"]), T(W["vy"]), T(W["vz"]), x=T(W["x"]), shock=W["setup"], **W["kw"])
sim.step(30)
prev = None
for k in range(6):
    sim.step(1)
    st = sim.stats()
    a = st["attempts"].astype(int)
    cost = st["proposals"]
    if prev is not None:
        same = (a == prev).mean()
        # idle of groups of 4 neighbours: max - mean of attempts, natural order vs sorted by previous attempts
        def idle(order):
            g = a[order][: len(a) // 4 * 4].reshape(-1, 4)
            return (g.max(1) - g.mean(1)).mean()
        nat = idle(np.arange(len(a)))
        srt = idle(np.argsort(prev, kind="stable"))
        orc = idle(np.argsort(a, kind="stable"))
        print(f"step {k}: P(same attempts) {same:.3f}  hist {np.bincount(a)[:8]}  group idle (attempts): natural {nat:.3f} by-prev {srt:.3f} oracle {orc:.3f}")
    prev = a
