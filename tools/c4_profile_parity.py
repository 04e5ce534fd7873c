"""Config-4 shock-profile statistical parity at full size:
Mach 3, 2,000 cells x 500 particles, eps = 1, RAD; fp32 GPU runs against the
fp64 CPU oracle, STEPS steps per seed, per-cell rho, u_x, T averaged over the
last STEPS/2 steps, over SEEDS seeds; z = |mean_g - mean_o| / sqrt(se_g^2 +
se_o^2) over seeds.  The oracle runs as POOL concurrent processes.
usage: c4_profile_parity.py [steps=2000] [seeds=16] [pool=8] [out.json]"""
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402

STEPS = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
SEEDS = int(sys.argv[2]) if len(sys.argv) > 2 else 16
POOL = int(sys.argv[3]) if len(sys.argv) > 3 else 8
OUT = sys.argv[4] if len(sys.argv) > 4 else "gpurun_out/c4_profile_parity.json"
SETUP = synth.shock_setup(mach=3.0, ncells=2000, n_total=1_000_000, x_min=-20, x_max=20)
KW = dict(model=1, m_init=2, m_cap=64, eps=1.0, dt=SETUP["dt"])
OBS = [1, 2, 5]          # moment columns: rho, u_x, T


def initial(seed, dtype):
    """The same initial state for both sides: fp32 values (the GPU's), binned
    by their own cell (an fp32 position can round across a cell edge)."""
    x, vx, vy, vz = synth.shock_particles(SETUP, seed=seed, dtype=np.float32)
    inv = SETUP["ncells"] / (SETUP["x_max"] - SETUP["x_min"])
    cell = np.clip(np.floor((x.astype(np.float64) - SETUP["x_min"]) * inv), 0, SETUP["ncells"] - 1)
    o = np.argsort(cell, kind="stable")
    return [np.ascontiguousarray(a[o], dtype=dtype) for a in (x, vx, vy, vz)]


def oracle_run(seed):
    from oracle import oracle as O
    x, vx, vy, vz = initial(seed, np.float64)
    s = O.ShockState(O.Config(**KW, adaptive=1, seed=seed), SETUP, x, vx, vy, vz)
    acc = np.zeros((SETUP["ncells"], len(OBS)))
    for k in range(STEPS):
        s.step(1)
        if k >= STEPS // 2:
            acc += s.moments()[:, OBS]
    return acc / (STEPS - STEPS // 2)


def gpu_runs():
    import torch
    from paper_1009_2768_b200 import api
    out = []
    for seed in range(1, SEEDS + 1):
        x, vx, vy, vz = (torch.as_tensor(a, device="cuda") for a in initial(seed, np.float32))
        sim = api.Simulation(vx, vy, vz, x=x, shock=SETUP, adaptive=True, seed=seed, **KW)
        acc = np.zeros((SETUP["ncells"], len(OBS)))
        for k in range(STEPS):
            sim.step(1)
            if k >= STEPS // 2:
                acc += sim.moments()[:, OBS]
        out.append(acc / (STEPS - STEPS // 2))
    return out


def main():
    t0 = time.time()
    from oracle import oracle as O
    O.build()
    with mp.get_context("spawn").Pool(POOL) as pool:
        ores = pool.map_async(oracle_run, range(1, SEEDS + 1))
        G = np.array(gpu_runs())
        t_gpu = time.time() - t0
        Ov = np.array(ores.get())
    t_all = time.time() - t0
    mg, mo = G.mean(0), Ov.mean(0)
    se = np.sqrt(G.var(0, ddof=1) / SEEDS + Ov.var(0, ddof=1) / SEEDS)
    z = np.abs(mg - mo) / np.where(se > 0, se, np.inf)
    rep = dict(config="configs[3] Mach-3 shock, 2000 cells x 500, eps=1, RAD m_init=2 m_cap=64, fp32 GPU vs fp64 oracle",
               steps=STEPS, averaged_over=STEPS - STEPS // 2, seeds=SEEDS, oracle_processes=POOL,
               frac_z_le_3={n: float(np.mean(z[:, k] <= 3)) for k, n in enumerate(["rho", "u_x", "T"])},
               z_max={n: float(z[:, k].max()) for k, n in enumerate(["rho", "u_x", "T"])},
               frac_z_le_3_all=float(np.mean(z <= 3)), z_max_all=float(z.max()),
               plateaus_gpu=dict(rho_L=float(mg[:100, 0].mean()), rho_R=float(mg[-100:, 0].mean()),
                                 T_L=float(mg[:100, 2].mean()), T_R=float(mg[-100:, 2].mean())),
               rankine_hugoniot=dict(rho_L=SETUP["rho_L"], rho_R=SETUP["rho_R"], T_L=SETUP["T_L"], T_R=SETUP["T_R"]),
               seconds=dict(gpu_side=round(t_gpu, 1), total=round(t_all, 1)), cpu_count=os.cpu_count())
    print(json.dumps(rep, indent=1))
    os.makedirs(os.path.dirname(OUT) or ".", exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(rep, f, indent=1)
    ok = rep["frac_z_le_3_all"] >= 0.99 and rep["z_max_all"] <= 5
    print("PASS" if ok else "FAIL")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
