import os, subprocess, sys, time
BODY = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_1009_2768_b200 import api
from oracle import oracle as O
n = int(sys.argv[1]); kw = eval(sys.argv[2])
vx, vy, vz = synth.two_maxwellians(2*n, seed=1)
d = lambda a: torch.as_tensor(a).to(device="cuda", dtype=torch.float64).contiguous()
sim = api.Simulation(d(vx), d(vy), d(vz), offsets=[0, n, 2*n], **kw)
sim.set_log(200000)
sim.step(1)
o = O.HomogeneousState(O.Config(**kw), vx, vy, vz, [0, n, 2*n], log_cap=200000); o.step(1)
try:
    st = sim.stats(); print("gpu", st[["attempts","leaves","thermalised","proposals"]].tolist(), flush=True)
except Exception as e:
    print("ERR", e, flush=True); sys.exit(0)
print("orc", o.stats[["attempts","leaves","thermalised","proposals"]].tolist(), flush=True)
g = sim.particles()
dv = np.abs(g["vx"] - o.vx)
print("max dv", dv.max(), "n bad", (dv > 1e-9).sum(), "first bad", np.nonzero(dv > 1e-9)[0][:10])
lg = sim.collisions(); lo = o.collisions()
key = lambda r: (int(r["cell"]), int(r["attempt"]), int(r["level"]), int(r["j"]))
G = {key(r): (int(r["slot_i"]), int(r["slot_k"]), int(r["accepted"])) for r in lg}
Ob = {key(r): (int(r["slot_i"]), int(r["slot_k"]), int(r["accepted"])) for r in lo}
bad = sorted(k for k in set(G) | set(Ob) if G.get(k) != Ob.get(k))
print("log", len(lg), len(lo), "mismatch", len(bad), bad[:3], [G.get(k) for k in bad[:3]], [Ob.get(k) for k in bad[:3]])
'''
cases = [
 (600, "dict(model=1, m_fixed=8, eps=0.5, dt=0.1)"),
 (600, "dict(model=0, m_fixed=8, eps=0.5, dt=0.3)"),
 (600, "dict(model=1, m_fixed=8, eps=1e-3, dt=0.1)"),
 (600, "dict(model=1, adaptive=1, m_init=2, m_cap=4, eps=0.5, dt=0.1)"),
 (600, "dict(model=1, adaptive=1, m_init=2, m_cap=8, eps=0.5, dt=0.1)"),
 (600, "dict(model=0, adaptive=1, m_init=2, m_cap=8, eps=0.5, dt=0.1)"),
 (100, "dict(model=1, adaptive=1, m_init=2, m_cap=64, eps=0.5, dt=0.1)"),
]
for n, kw in cases:
    t = time.time()
    try:
        r = subprocess.run([sys.executable, "-u", "-c", BODY, str(n), kw], capture_output=True, text=True, timeout=60)
        print(f"== {kw} n={n}: rc={r.returncode} {time.time()-t:.1f}s\n", r.stdout[-3000:], r.stderr[-1500:], flush=True)
    except subprocess.TimeoutExpired as ex:
        print(f"== {kw}: TIMEOUT", (ex.stdout or b"")[-2000:], flush=True)
