import sys, numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_1009_2768_b200 import api, dist
setup = synth.shock_setup(mach=3.0, ncells=60, n_total=30_000, x_min=-6.0, x_max=6.0)
x, vx, vy, vz = synth.shock_particles(setup, seed=3)
inv = setup["ncells"] / (setup["x_max"] - setup["x_min"])
cell = np.clip(np.floor((x - setup["x_min"]) * inv), 0, 59)
o = np.argsort(cell, kind="stable"); x, vx, vy, vz = x[o], vx[o], vy[o], vz[o]
counts = np.bincount(cell.astype(int), minlength=60)
T = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=torch.float64)
kw = dict(model=1, adaptive=True, m_init=2, m_cap=64, eps=0.3, dt=setup["dt"], seed=5)
full = api.Simulation(T(vx), T(vy), T(vz), x=T(x), shock=setup, **kw)
cuts = dist.slab_cuts(counts, 2); print(cuts)
slabs = [dist.ShockSlab(api, setup, f, n, *[T(a) for a in dist.slab_particles(x, vx, vy, vz, setup, f, n)], device="cuda", exchange_capacity=4096, **kw) for f, n in cuts]
for step in range(6):
    full.step(1)
    for s in slabs: s.sim.shock_begin()
    dist.host_exchange(slabs)
    for s in slabs: s.sim.shock_finish()
    cnt = lambda t: int(t[:4].view(torch.int32)[0].item())
    print(step, full.num_particles(), [s.sim.num_particles() for s in slabs],
          "send_r0", cnt(slabs[0].send_r), "send_l1", cnt(slabs[1].send_l))
    g = full.particles(); off = g["offsets"]
    p0 = slabs[0].sim.particles(); p1 = slabs[1].sim.particles()
    c0 = cuts[1][0]
    print("   full cells", off[c0-2:c0+3] - off[c0-2], " slab0 tail", np.diff(p0["offsets"])[-2:], "slab1 head", np.diff(p1["offsets"])[:3], "full", np.diff(off)[c0-2:c0+3])
