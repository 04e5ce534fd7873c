"""Staged GPU debug runner: each case in its own subprocess with a timeout."""
import subprocess
import sys
import time

CASES = {
 "maxwell_tiny": "model=0, m_fixed=4, eps=1.0, dt=0.1", 
 "hs_tiny": "model=1, m_fixed=4, eps=1.0, dt=0.1",
 "hs_rad": "model=1, adaptive=True, m_init=2, m_cap=64, eps=0.5, dt=0.1",
 "hs_therm": "model=1, m_fixed=64, eps=0.01, dt=0.1",
}
BODY = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_1009_2768_b200 import api
n = int(sys.argv[2]); ncell = int(sys.argv[3]); dtype = torch.float64 if sys.argv[4] == "64" else torch.float32
vx, vy, vz = synth.two_maxwellians(n * ncell, seed=1)
d = lambda a: torch.as_tensor(a).to(device="cuda", dtype=dtype).contiguous()
off = np.arange(ncell + 1) * n
t = time.time()
sim = api.Simulation(d(vx), d(vy), d(vz), offsets=off, %s)
print("init ok", time.time() - t, flush=True)
sim.step(1); torch.cuda.synchronize(); print("step1 ok", time.time() - t, flush=True)
st = sim.stats(); print("stats", st[0], flush=True)
sim.step(2); m = sim.moments(); print("moments", m[0], flush=True)
'''
for name, kw in CASES.items():
    for (n, nc, dt) in [(100, 1, "64"), (2000, 2, "64"), (1024, 64, "32")]:
        t = time.time()
        try:
            r = subprocess.run([sys.executable, "-u", "-c", BODY % kw, name, str(n), str(nc), dt],
                               capture_output=True, text=True, timeout=90)
            print(f"== {name} n={n} cells={nc} fp{dt}: rc={r.returncode} {time.time()-t:.1f}s", flush=True)
            print(r.stdout[-1500:], r.stderr[-1500:], flush=True)
        except subprocess.TimeoutExpired as e:
            print(f"== {name} n={n} cells={nc} fp{dt}: TIMEOUT", flush=True)
            print((e.stdout or b"")[-1500:], flush=True)
