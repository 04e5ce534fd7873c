import os, subprocess, sys, time
BODY = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_1009_2768_b200 import api
from oracle import oracle as O
n = int(sys.argv[1]); dt_ = torch.float64
vx, vy, vz = synth.two_maxwellians(2*n, seed=1)
d = lambda a: torch.as_tensor(a).to(device="cuda", dtype=dt_).contiguous()
kw = dict(model=1, adaptive=1, m_init=2, m_cap=64, eps=0.5, dt=0.1)
sim = api.Simulation(d(vx), d(vy), d(vz), offsets=[0, n, 2*n], **kw)
sim.set_log(200000)
sim.step(1)
o = O.HomogeneousState(O.Config(**kw), vx, vy, vz, [0, n, 2*n], log_cap=200000); o.step(1)
try:
    st = sim.stats(); print("gpu stats", st[["attempts","leaves","untouched","thermalised","proposals"]], flush=True)
except Exception as e:
    print("ERR", e, flush=True)
print("orc stats", o.stats[["attempts","leaves","untouched","thermalised","proposals"]], flush=True)
lg = sim.collisions(); lo = o.collisions()
print("log sizes", len(lg), len(lo))
key = lambda r: (r["cell"], r["attempt"], r["level"], r["j"])
G = {key(r): (r["slot_i"], r["slot_k"], r["accepted"]) for r in lg}
Ob = {key(r): (r["slot_i"], r["slot_k"], r["accepted"]) for r in lo}
bad = sorted(k for k in set(G) | set(Ob) if G.get(k) != Ob.get(k))
print("n mismatches", len(bad))
for k in bad[:15]: print(k, G.get(k), Ob.get(k))
'''
for env, n in [({"TRMCR_SMEM_KCAP": "4096"}, 2000), ({"TRMCR_FORCE_GMEM": "1"}, 2000), ({}, 2000), ({}, 600)]:
    e = dict(os.environ); e.update(env)
    t = time.time()
    try:
        r = subprocess.run([sys.executable, "-u", "-c", BODY, str(n)], capture_output=True, text=True, timeout=60, env=e)
        print(f"== {env} n={n}: rc={r.returncode} {time.time()-t:.1f}s\n", r.stdout[-3000:], r.stderr[-2000:], flush=True)
    except subprocess.TimeoutExpired as ex:
        print(f"== {env}: TIMEOUT", (ex.stdout or b"")[-2000:], flush=True)
