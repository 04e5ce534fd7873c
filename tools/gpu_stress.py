"""Randomised fp64 GPU-vs-oracle decision/velocity parity over many configurations."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
from oracle import oracle as O
from paper_1009_2768_b200 import api

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
fails = 0
t0 = time.time()
for it in range(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    ncell = int(rng.integers(1, 20)); maxp = int(rng.choice([64, 300, 700, 1500, 2500]))
    v = synth.ragged_cells(ncell, maxp, seed=int(rng.integers(1, 10**6)))
    model = int(rng.integers(0, 2)); adaptive = int(rng.integers(0, 2))
    kw = dict(model=model, adaptive=adaptive, m_fixed=int(rng.choice([1, 2, 4, 16, 64])),
              m_init=int(rng.choice([1, 2, 4])), m_cap=int(rng.choice([4, 16, 64])),
              eps=float(10 ** rng.uniform(-2.5, 0.5)), dt=float(rng.choice([0.05, 0.1, 0.3])),
              seed=int(rng.integers(1, 1000)), indicator=int(rng.integers(0, 2)))
    o = O.HomogeneousState(O.Config(**kw), v[0], v[1], v[2], v[3], log_cap=2_000_000)
    d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda").contiguous()
    sim = api.Simulation(d(v[0]), d(v[1]), d(v[2]), offsets=v[3], **kw)
    sim.set_log(2_000_000)
    ok = True
    msg = ""
    for s in range(3):
        o.step(1)
        try:
            sim.step(1)
            st = sim.stats()
        except Exception as e:
            ok, msg = False, str(e); break
        for f in ("proposals", "accepted", "leaves", "thermalised", "m_next", "attempts"):
            if not np.array_equal(st[f], o.stats[f]):
                ok, msg = False, f"step {s} stat {f}"; break
        if not ok: break
    if ok:
        g = sim.particles()
        err = max(np.abs(g["vx"] - o.vx).max(initial=0), np.abs(g["vz"] - o.vz).max(initial=0))
        if err > 1e-10:
            ok, msg = False, f"velocity err {err}"
    if not ok:
        fails += 1
        print("FAIL", it, kw, ncell, maxp, msg, flush=True)
print(f"stress done: {fails} failures, {time.time()-t0:.1f}s", flush=True)
