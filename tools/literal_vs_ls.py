"""The LS reformulation against the paper's own layout on the GPU.

Same cells, same kernel, same truncation: `literal=True` runs Alg 4.3/4.4 literally
(one thread per cell, recursive builds, one sequential stream per cell); the default
runs the level-synchronous plan (warp / CTA per cell, collisions of a level in
parallel).  Prints one JSON line per (workload, layout) with ms/step and particle-
updates/s, device-timed with CUDA events after warm-up.
usage: python tools/literal_vs_ls.py [steps]
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_1009_2768_b200 import api  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
# (name, cells, ppc, eps, dt, m): thermal HS cells; x = mu dt / eps per cell
CASES = [
    ("C3 shape, eps=1 (x~0.8: ~0.4 n collisions/cell)", 16_384, 1024, 1.0, 0.1, 16),
    ("C3 shape, eps=0.3 (x~2.7: deep trees)", 16_384, 1024, 0.3, 0.1, 16),
    ("C4-like cells: 2000 x 500, eps=1", 2_000, 500, 1.0, 0.1, 16),
]
for name, nc, ppc, eps, dt, m in CASES:
    vx, vy, vz, off = synth.uniform_cells(nc, ppc, seed=1, dtype=np.float32)
    for literal in (False, True):
        T = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=torch.float32)
        sim = api.Simulation(T(vx), T(vy), T(vz), offsets=off, model=api.HARD_SPHERE, m_fixed=m, eps=eps, dt=dt,
                             seed=1, literal=literal)
        sim.step(3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sim.step(steps)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        st = sim.stats()
        print(json.dumps(dict(workload=name, layout="literal (Alg 4.3/4.4, thread per cell)" if literal
                              else "LS plan (this framework)", cells=nc, ppc=ppc, eps=eps, dt=dt, m=m,
                              ms_per_step=round(ms, 4), updates_per_s=nc * ppc / ms * 1e3,
                              proposals_per_cell=float(st["proposals"].mean()),
                              depth=float(st["depth"].mean()))), flush=True)
        del sim
