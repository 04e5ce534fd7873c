import os, subprocess, sys, time
BODY = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_1009_2768_b200 import api
from oracle import oracle as O
n = 600; kw = eval(sys.argv[1])
vx, vy, vz = synth.two_maxwellians(2*n, seed=1)
d = lambda a: torch.as_tensor(a).to(device="cuda", dtype=torch.float64).contiguous()
sim = api.Simulation(d(vx), d(vy), d(vz), offsets=[0, n, 2*n], **kw)
sim.set_log(200000)
sim.step(1)
o = O.HomogeneousState(O.Config(**kw), vx, vy, vz, [0, n, 2*n], log_cap=200000); o.step(1)
st = sim.stats(); print("gpu", st[["attempts","leaves","untouched","thermalised","proposals", "E1", "S_est"]].tolist(), flush=True)
print("orc", o.stats[["attempts","leaves","untouched","thermalised","proposals", "E1", "S_est"]].tolist(), flush=True)
g = sim.particles()
lo = o.collisions()
groups = {}
for r in lo[lo["cell"] == 0]:
    for s in (r["slot_i"], r["slot_k"]):
        groups.setdefault(int(s), set()).add(int(r["attempt"]))
bad = np.abs(g["vx"][:n] - o.vx[:n]) > 1e-9
untouched = [i for i in range(n) if i not in groups]
a0 = [i for i in groups if groups[i] == {0}]
a1 = [i for i in groups if 1 in groups[i]]
print("untouched/theta bad", bad[untouched].sum(), "of", len(untouched))
print("attempt0-only bad", bad[a0].sum(), "of", len(a0))
print("attempt1 bad", bad[a1].sum(), "of", len(a1))
v0 = np.array(vx[:n])
print("gpu==initial for bad", np.sum(np.abs(g["vx"][:n][bad] - v0[bad]) < 1e-12), "orc==initial for bad", np.sum(np.abs(o.vx[:n][bad]-v0[bad])<1e-12))
'''
for env in [{"TRMCR_FORCE_GMEM": "1", "TRMCR_GMEM_THREADS": "256"}, {"TRMCR_FORCE_GMEM": "1", "TRMCR_GMEM_THREADS": "64"}, {"TRMCR_SMEM_KCAP": "2048"}]:
  for kw in ["dict(model=1, adaptive=1, m_init=2, m_cap=4, eps=0.5, dt=0.1)", "dict(model=1, adaptive=1, m_init=2, m_cap=2, eps=0.5, dt=0.1)"]:
    e = dict(os.environ); e.update(env)
    try:
        r = subprocess.run([sys.executable, "-u", "-c", BODY, kw], capture_output=True, text=True, timeout=60, env=e)
        print(f"== {env} {kw}: rc={r.returncode}\n", r.stdout[-3000:], r.stderr[-1500:], flush=True)
    except subprocess.TimeoutExpired as ex:
        print(f"== {kw}: TIMEOUT", (ex.stdout or b"")[-2000:], flush=True)
