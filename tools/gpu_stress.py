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
    if rng.random() < 0.25:          # far from equilibrium: majorant violations happen
        v = synth.cold_beams(ncell, int(rng.choice([100, 400, 900])), seed=int(rng.integers(1, 10**6)))
    else:
        v = synth.ragged_cells(ncell, maxp, seed=int(rng.integers(1, 10**6)))
    model = int(rng.integers(0, 3)); adaptive = int(rng.integers(0, 2))
    literal = int(rng.random() < 0.15)
    if literal:
        adaptive = 0
    wb = int(rng.integers(0, 4)) if (not adaptive and not literal and rng.random() < 0.3) else 0
    kw = dict(model=model, adaptive=adaptive, m_fixed=int(rng.choice([1, 2, 4, 16, 64])),
              m_init=int(rng.choice([1, 2, 4])), m_cap=int(rng.choice([4, 16, 64])),
              eps=float(10 ** rng.uniform(-2.5, 0.5)), dt=float(rng.choice([0.05, 0.1, 0.3])),
              seed=int(rng.integers(1, 1000)), indicator=int(rng.integers(0, 2)),
              alpha=float(rng.uniform(0.0, 1.0)), sigma_update=int(rng.integers(0, 2)), wb=wb,
              wb_max=int(rng.integers(0, 6)), literal=literal)
    o = O.HomogeneousState(O.Config(**kw), v[0], v[1], v[2], v[3], log_cap=2_000_000)
    d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda").contiguous()
    sim = api.Simulation(d(v[0]), d(v[1]), d(v[2]), offsets=v[3], **kw)
    sim.set_log(2_000_000)
    ok = True
    msg = ""
    for s in range(3):
        oerr = gerr = None
        try:
            o.step(1)
        except RuntimeError as e:
            oerr = str(e)
        try:
            sim.step(1)
            st = sim.stats()
        except Exception as e:
            gerr = str(e)
        if oerr or gerr:                 # literal mode without a finite-N guard: both must fail
            if not (oerr and gerr):
                ok, msg = False, f"step {s}: oracle {oerr} / gpu {gerr}"
            break
        for f in ("proposals", "accepted", "violations", "leaves", "thermalised", "maxw", "m_next", "attempts"):
            if not np.array_equal(st[f], o.stats[f]):
                ok, msg = False, f"step {s} stat {f}"; break
        if not ok: break
    if ok and not (oerr or gerr):
        g = sim.particles()
        err = max(np.abs(g["vx"] - o.vx).max(initial=0), np.abs(g["vz"] - o.vz).max(initial=0))
        if err > 1e-10:
            ok, msg = False, f"velocity err {err}"
    if not ok:
        fails += 1
        print("FAIL", it, kw, ncell, maxp, msg, flush=True)
print(f"stress done: {fails} failures, {time.time()-t0:.1f}s", flush=True)
