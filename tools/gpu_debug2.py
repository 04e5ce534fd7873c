import os, subprocess, sys, time
BODY = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_1009_2768_b200 import api
vx, vy, vz = synth.two_maxwellians(4000, seed=1)
d = lambda a: torch.as_tensor(a).to(device="cuda", dtype=torch.float64).contiguous()
sim = api.Simulation(d(vx), d(vy), d(vz), offsets=[0, 2000, 4000], model=1, adaptive=True, m_init=2, m_cap=64, eps=0.5, dt=0.1)
print("init ok", flush=True)
sim.step(1)
try:
    st = sim.stats(); print("stats", st, flush=True)
except Exception as e:
    print("ERR", e, flush=True)
'''
for env in [{"TRMCR_SMEM_KCAP": "16384"}, {"TRMCR_FORCE_GMEM": "1"}, {}]:
    e = dict(os.environ); e.update(env)
    t = time.time()
    try:
        r = subprocess.run([sys.executable, "-u", "-c", BODY], capture_output=True, text=True, timeout=60, env=e)
        print(f"== {env}: rc={r.returncode} {time.time()-t:.1f}s\n", r.stdout[-3000:], r.stderr[-2000:], flush=True)
    except subprocess.TimeoutExpired as ex:
        print(f"== {env}: TIMEOUT", (ex.stdout or b"")[-2000:], flush=True)
