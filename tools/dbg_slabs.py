import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, torch, synth
from paper_1009_2768_b200 import api, dist
from test_gpu_slabs import _sorted_shock
world, dtype = 3, np.float32
for fz in ("1", "0"):
    os.environ["TRMCR_SHOCK_FUSED"] = fz
    setup = synth.shock_setup(mach=3.0, ncells=60, n_total=30_000, x_min=-6.0, x_max=6.0)
    x, vx, vy, vz, counts = _sorted_shock(setup, 3, dtype)
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=torch.float32)
    kw = dict(model=1, adaptive=True, m_init=2, m_cap=64, eps=0.3, dt=setup["dt"], seed=5)
    full = api.Simulation(T(vx), T(vy), T(vz), x=T(x), shock=setup, **kw)
    cuts = dist.slab_cuts(counts, world)
    slabs = []
    for first, nc in cuts:
        px, pvx, pvy, pvz = dist.slab_particles(x, vx, vy, vz, setup, first, nc)
        slabs.append(dist.ShockSlab(api, setup, first, nc, T(pvx), T(pvy), T(pvz), x=T(px), device="cuda", exchange_capacity=4096, **kw))
    for step in range(12):
        full.step(1)
        for s in slabs: s.sim.shock_begin()
        dist.host_exchange(slabs)
        for s in slabs: s.sim.shock_finish()
        st = np.concatenate([s.sim.stats() for s in slabs]); sf = full.stats()
        bad = np.nonzero(st["p"] != sf["p"])[0]
        if len(bad):
            print("fused", fz, "step", step, "cells", bad)
            for c in bad[:3]:
                print(" slab", {f: st[f][c] for f in st.dtype.names})
                print(" full", {f: sf[f][c] for f in sf.dtype.names})
            break
    else:
        print("fused", fz, "all equal")
    print("cuts", cuts, [s.sim.sort_info() for s in slabs], full.sort_info())
