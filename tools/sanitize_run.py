"""Small runs of every kernel family, for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck).  usage: sanitize_run.py CASE [steps]
  c1      config 1 (10^4 fp64, one cell, Maxwell): CTA / global-memory kernels
  thermal 256 cells x 1024 fp32 at eps 0.01: thermal warp kernel + idle CTA kernel
  warp    256 cells x 500 fp32 at eps 1: warp-per-cell general kernel + deferrals
  giant   one 40,000-particle HS cell, RAD: grid-cooperative giant-cell kernel
  shock   C4-shaped shock, 80 cells x 40,000: transport, scan, edge/scatter sort,
          lock-step collision kernel (hard-sphere instantiation), CTA fallback
  batch   the same shock through the pooled-batch kernel (TRMCR_SHOCK_BATCH=1)
  fused   the same shock through the fused pass (TRMCR_SHOCK_FUSED=2)
  wb      TRMC-WB + majorant update on cold beams (extended warp / CTA kernels)
  literal Alg 4.3/4.4 literally (thread per cell)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402

case = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if case == "batch":
    os.environ["TRMCR_SHOCK_BATCH"] = "1"
if case == "fused":
    os.environ["TRMCR_SHOCK_FUSED"] = "2"
from paper_1009_2768_b200 import api  # noqa: E402


def dev(a, dt):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dt)


f32, f64 = torch.float32, torch.float64
if case == "c1":
    vx, vy, vz = synth.two_maxwellians(10_000, seed=1)
    sim = api.Simulation(dev(vx, f64), dev(vy, f64), dev(vz, f64), offsets=[0, 10_000], model=api.MAXWELL,
                         m_fixed=64, eps=1.0, dt=0.1, seed=1)
elif case in ("thermal", "warp"):
    v = synth.bimodal_cells(256, 1024 if case == "thermal" else 500, seed=1)
    sim = api.Simulation(dev(v[0], f32), dev(v[1], f32), dev(v[2], f32), offsets=v[3], model=api.HARD_SPHERE,
                         m_fixed=64, eps=0.01 if case == "thermal" else 1.0, dt=0.1, seed=1)
elif case == "giant":
    vx, vy, vz = synth.anisotropic_gaussian(40_000, seed=1)
    sim = api.Simulation(dev(vx, f64), dev(vy, f64), dev(vz, f64), offsets=[0, 40_000], model=api.HARD_SPHERE,
                         adaptive=True, m_init=2, m_cap=4096, eps=0.1, dt=0.05, seed=1)
elif case in ("shock", "batch", "fused"):
    setup = synth.shock_setup(mach=3.0, ncells=80, n_total=40_000, x_min=-8.0, x_max=8.0)
    x, vx, vy, vz = synth.shock_particles(setup, seed=1, dtype=np.float32)
    inv = setup["ncells"] / (setup["x_max"] - setup["x_min"])
    o = np.argsort(np.clip(np.floor((x.astype(np.float64) - setup["x_min"]) * inv), 0, 79), kind="stable")
    sim = api.Simulation(dev(vx[o], f32), dev(vy[o], f32), dev(vz[o], f32), x=dev(x[o], f32), shock=setup,
                         model=api.HARD_SPHERE, adaptive=True, m_init=2, m_cap=64, eps=0.3, dt=setup["dt"], seed=1)
elif case == "wb":
    v = synth.cold_beams(64, 400, seed=1)
    sim = api.Simulation(dev(v[0], f64), dev(v[1], f64), dev(v[2], f64), offsets=v[3], model=api.HARD_SPHERE,
                         m_fixed=8, eps=0.3, dt=0.1, seed=1, wb=2, wb_max=3, sigma_update=1)
elif case == "literal":
    v = synth.ragged_cells(64, 600, seed=1)
    sim = api.Simulation(dev(v[0], f64), dev(v[1], f64), dev(v[2], f64), offsets=v[3], model=api.HARD_SPHERE,
                         m_fixed=16, eps=1.0, dt=0.1, seed=1, literal=1)
else:
    raise SystemExit(f"unknown case {case}")
sim.step(steps)
sim.moments()
torch.cuda.synchronize()
print(case, "ok", sim.launch_count)
