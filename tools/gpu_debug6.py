import os, subprocess, sys, time
BODY = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_1009_2768_b200 import api
n = 600; kw = dict(model=1, adaptive=1, m_init=2, m_cap=4, eps=0.5, dt=0.1)
vx, vy, vz = synth.two_maxwellians(2*n, seed=1)
d = lambda a: torch.as_tensor(a).to(device="cuda", dtype=torch.float64).contiguous()
sim = api.Simulation(d(vx), d(vy), d(vz), offsets=[0, n, 2*n], **kw)
sim.set_log(100000)
sim.step(1)
g = sim.particles()
lg = sim.collisions()
np.savez(sys.argv[1], vx=g["vx"], vy=g["vy"], vz=g["vz"], log=lg)
print("saved", len(lg))
'''
for env, tag in [({"TRMCR_DEBUG_STOP": "-1"}, "smem"), ({"TRMCR_DEBUG_STOP": "-1", "TRMCR_FORCE_GMEM": "1"}, "gmem"), ({}, "smemfull"), ({"TRMCR_FORCE_GMEM": "1"}, "gmemfull")]:
    e = dict(os.environ); e.update(env)
    r = subprocess.run([sys.executable, "-u", "-c", BODY, f"gpurun_out/dump_{tag}.npz"], capture_output=True, text=True, timeout=60, env=e)
    print(tag, r.returncode, r.stdout[-500:], r.stderr[-1500:], flush=True)
