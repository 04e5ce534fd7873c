#!/usr/bin/env python
"""TRMC-R benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5|c3|c4|c2|c1]
                    [--secondary c3|none] [--impl trmcr|reference]

Prints ONE JSON line (rank 0).  Metric: particle-updates/s of the TRMC-R
step (BASELINE.json).  Default workload: configs[4], the large Mach-5 1D
shock (65,536 cells, 65.5 M fp32 particles, eps = 0.01, RAD): the north
star's "large shock workload" - a full step is reservoirs + transport (A1),
the counting sort by cell (A2) and the collision step (A3-A8); its 1.05 GB of
state exceeds L2 (126 MB), so no flush is needed.  Slab-partitioned across
GPUs (strong scaling) with a neighbour exchange.  The same line carries
configs[2] (16,384 independent hard-sphere cells x 1,024, eps = 0.01) as the
"secondary" record (sharded by cell, strong scaling, NCCL all-reduce of the
global moments every step).

--gpus N > 1 without torchrun: the script re-launches itself under
torch.distributed.run (one process per GPU, 127.0.0.1 rendezvous).
--impl reference times the CPU oracle (oracle/, single-threaded, fp64) on a
bounded sample of the same workload (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "TRMC-R particle-updates/s"
UNIT = "particle-updates/s"


# ----------------------------------------------------------------------------- workloads
def workload(name: str, rank: int = 0, world: int = 1, eps_override=None):
    """Synthetic inputs shaped like BASELINE.json configs."""
    if name in ("c3", "c3weak"):
        # configs[2]: ONE 16,384-cell ensemble sharded across the GPUs by contiguous
        # global cell ranges (strong scaling; RNG keyed by global cell id, so a
        # cell's result does not depend on the GPU count).  c3weak: every GPU owns
        # a full ensemble of its own (weak scaling, secondary).
        ncells, ppc = 16_384, 1024
        vx, vy, vz, off = synth.bimodal_cells(ncells, ppc, seed=1)
        weak = name == "c3weak"
        if weak:
            lo, cells_here, base = 0, ncells, rank * ncells
        else:
            from paper_1009_2768_b200 import dist as D
            off, base, sl = D.shard_homogeneous(off, rank, world)
            vx, vy, vz = vx[sl], vy[sl], vz[sl]
            cells_here = len(off) - 1
        return dict(kind="hom", vx=vx, vy=vy, vz=vz, offsets=off, cell_base=base, dtype=np.float32,
                    kw=dict(model=1, m_fixed=64, eps=eps_override or 0.01, dt=0.1, seed=1),
                    cfg=dict(workload="configs[2] batched homogeneous hard spheres", cells_per_gpu=cells_here,
                             ppc=ppc, cells=ncells * (world if weak else 1),
                             particles=ncells * ppc * (world if weak else 1),
                             eps=eps_override or 0.01, dt=0.1, truncation="TRMC-R m=64",
                             sharding=("cells (weak: 16,384 cells per GPU)" if weak else
                                       "one 16,384-cell ensemble sharded by cell (strong)"),
                             global_moments="allreduce/step"),
                    global_cells=ncells * (world if weak else 1), scaling="weak" if weak else "strong")
    if name in ("c4", "c5"):
        if name == "c4":
            setup = synth.shock_setup(mach=3.0, ncells=2000, n_total=1_000_000, x_min=-20, x_max=20)
            eps = eps_override or 1.0
        else:
            setup = synth.shock_setup(mach=5.0, ncells=65_536, n_total=65_536_000, x_min=-50, x_max=50)
            eps = eps_override or 0.01
        x, vx, vy, vz = synth.shock_particles(setup, seed=1, dtype=np.float32)
        inv = setup["ncells"] / (setup["x_max"] - setup["x_min"])
        cell = np.clip(np.floor((x.astype(np.float64) - setup["x_min"]) * inv), 0, setup["ncells"] - 1)
        order = np.argsort(cell, kind="stable")
        x, vx, vy, vz = x[order], vx[order], vy[order], vz[order]
        first, ncl = 0, setup["ncells"]
        if world > 1:     # slabs balanced by particle count
            from paper_1009_2768_b200 import dist as D
            counts = np.bincount(cell.astype(np.int64), minlength=setup["ncells"])
            first, ncl = D.slab_cuts(counts, world)[rank]
            x, vx, vy, vz = D.slab_particles(x, vx, vy, vz, setup, first, ncl)
        return dict(kind="shock", x=x, vx=vx, vy=vy, vz=vz, setup=setup, first=first, local_cells=ncl,
                    dtype=np.float32,
                    kw=dict(model=1, adaptive=True, m_init=2, m_cap=64, eps=eps, dt=setup["dt"], seed=1),
                    cfg=dict(workload=f"configs[{3 if name == 'c4' else 4}] 1D Mach-{setup['mach']:g} shock",
                             cells=setup["ncells"], particles=len(x), eps=eps, dt=setup["dt"],
                             truncation="TRMC-RAD m_init=2 m_cap=64",
                             sharding="slabs balanced by particle count, neighbour exchange over NCCL"),
                    global_cells=setup["ncells"])
    if name == "c2":
        n = 1_000_000
        vx, vy, vz = synth.anisotropic_gaussian(n, seed=1)
        eps = eps_override or 1.0
        return dict(kind="hom", vx=vx.astype(np.float32), vy=vy.astype(np.float32),
                    vz=vz.astype(np.float32), offsets=np.array([0, n]), cell_base=rank, dtype=np.float32,
                    kw=dict(model=1, adaptive=True, m_init=2, m_cap=4096, eps=eps, dt=0.05, seed=1),
                    cfg=dict(workload="configs[1] homogeneous hard spheres, one cell", cells=1,
                             particles=n, eps=eps, dt=0.05, truncation="TRMC-RAD"), global_cells=world,
                    scaling="weak")
    if name == "c1":
        vx, vy, vz = synth.two_maxwellians(10_000, seed=1)
        return dict(kind="hom", vx=vx, vy=vy, vz=vz, offsets=np.array([0, 10_000]), cell_base=rank,
                    dtype=np.float64, kw=dict(model=0, m_fixed=64, eps=1.0, dt=0.1, seed=1),
                    cfg=dict(workload="configs[0] Maxwell molecules, one cell", cells=1, particles=10_000,
                             eps=1.0, dt=0.1, truncation="TRMC-R m=64"), global_cells=world, scaling="weak")
    raise SystemExit(f"unknown workload {name}")


# ----------------------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()            # start timing only once sampling runs
            while not self.rows and time.time() - t0 < 3.0:
                time.sleep(0.01)
            self.rows.clear()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
            except (ValueError, IndexError):
                continue
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def ncu_issue(workload_name):
    """Executed warp instructions per launch of the dominant kernel (committed ncu summary)."""
    path = os.path.join(ROOT, "profiles", "ncu_issue.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload_name)
    except (OSError, ValueError):
        return None


def measured_clock_mhz():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["sm_max_mhz"])
    except (OSError, KeyError, ValueError):
        return 1965.0


def ncu_traffic(workload_name):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(workload_name)
    except (OSError, ValueError):
        return None


def oracle_rate(W, seconds=12.0, min_steps=1, max_steps=10**9):
    """Time the CPU oracle (as it stands) on a bounded sample of workload W."""
    from oracle import oracle as O
    kw = dict(W["kw"])
    cfg = O.Config(model=kw.get("model", 1), adaptive=int(bool(kw.get("adaptive", 0))),
                   m_fixed=kw.get("m_fixed", 64), m_init=kw.get("m_init", 2), m_cap=kw.get("m_cap", 4096),
                   eps=kw["eps"], dt=kw["dt"], seed=kw.get("seed", 1))
    if W["kind"] == "hom":
        off = W["offsets"]
        ncs = len(off) - 1
        take = ncs
        # bounded sample: the first cells, about 1 M particles
        while take > 1 and off[take] > 1_000_000:
            take //= 2
        o = O.HomogeneousState(cfg, W["vx"][: off[take]].astype(np.float64),
                               W["vy"][: off[take]].astype(np.float64),
                               W["vz"][: off[take]].astype(np.float64), off[: take + 1],
                               gcell0=W.get("cell_base", 0))
        per_step = int(off[take])
        sample = f"first {take} of {ncs} cells ({per_step} particles), same per-cell workload"
    else:
        s = dict(W["setup"])
        # a 1,024-cell window of the same grid (same dx, dt, w, ppc) around the shock
        cells = min(1024, s["ncells"])
        half = cells * s["dx"] / 2
        s.update(ncells=cells, x_min=-half, x_max=half)
        x, vx, vy, vz = synth.shock_particles(s, seed=1)
        o = O.ShockState(cfg, s, x, vx, vy, vz)
        per_step = o.n
        sample = f"{cells}-cell window of the same grid around the shock ({per_step} particles)"
    t0 = time.perf_counter()
    steps = 0
    parts = 0
    while (steps < min_steps or time.perf_counter() - t0 < seconds) and steps < max_steps:
        n_before = o.n if W["kind"] == "shock" else per_step
        o.step(1)
        parts += n_before
        steps += 1
    dt = time.perf_counter() - t0
    return parts / dt, dict(sample=f"{sample}; {steps} steps, {dt:.1f} s", cores=1, steps=steps,
                            seconds=dt)


# ----------------------------------------------------------------------------- arms
def full_cfg(W, world):
    """The config record of a workload at `world` GPUs - the same dict on both arms."""
    cfg = dict(W["cfg"])
    rs = 4 if W["dtype"] == np.float32 else 8
    n_local = len(W["vx"])
    cfg.update(parallelism=f"{'cells' if W['kind'] == 'hom' else 'slabs'}x{world}",
               l2="inputs larger than L2 (no flush)" if n_local * 3 * rs > 126e6 else "inputs L2-resident")
    return cfg


def run_reference(args, rank):
    if rank != 0:
        return
    W = workload(args.workload, 0, 1, args.eps)
    # warmup steps then K timed steps, each step a bounded sample of the workload
    from oracle import oracle as O  # noqa: F401
    rate_w, _ = oracle_rate(W, seconds=0.0, min_steps=args.warmup, max_steps=args.warmup)
    rate, info = oracle_rate(W, seconds=0.0, min_steps=args.steps, max_steps=args.steps)
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "ms_per_step": 1e3 * info["seconds"] / max(info["steps"], 1), "dtype": "f64",
            "data": "synthetic", "config": full_cfg(workload(args.workload, 0, args.gpus, args.eps), args.gpus)
            if args.gpus > 1 else full_cfg(W, 1),
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": info["sample"]},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def measure(args, wl_name, rank, world, local_rank, cpu_seconds):
    """Time K steps of workload wl_name on this rank's GPU; the JSON record (rank 0)."""
    import torch
    import torch.distributed as dist
    from paper_1009_2768_b200 import api

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    W = workload(wl_name, rank, world, args.eps if wl_name == args.workload else None)
    td = torch.float32 if W["dtype"] == np.float32 else torch.float64
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(device=dev, dtype=td)
    stream = torch.cuda.current_stream(dev)
    from paper_1009_2768_b200 import dist as D
    # the library's own NCCL communicator (all-reduce of the global moments,
    # slab neighbour exchange); torch.distributed only broadcasts its id
    comm = D.library_comm(api) if world > 1 else None
    ckw = dict(nccl_id=comm[0], rank=comm[1], nranks=comm[2]) if comm else {}
    if W["kind"] == "hom":
        sim = api.Simulation(T(W["vx"]), T(W["vy"]), T(W["vz"]), offsets=W["offsets"],
                             cell_base=W["cell_base"], stream=stream.cuda_stream, **ckw, **W["kw"])
        n_local = int(W["offsets"][-1])
        slab = None
    else:
        slab = D.ShockSlab(api, W["setup"], W["first"], W["local_cells"], T(W["vx"]), T(W["vy"]), T(W["vz"]),
                           x=T(W["x"]), device=dev, stream=stream.cuda_stream, comm=comm, **W["kw"])
        sim = slab.sim
        n_local = sim.num_particles()
    # global moments every step (configs[2]: "NCCL allreduce of global moments"):
    # two buffers; the library all-reduces step k's sums on its communication
    # stream while step k + 1 collides, and orders a buffer's reuse after its
    # all-reduce
    gms = [torch.zeros(len(api.GLOBAL_FIELDS), dtype=torch.float64, device=dev) for _ in range(2)]
    counter = [0]
    xchg = None

    def one_step():
        if W["kind"] == "hom":
            sim.step(1)
            k = counter[0] & 1
            counter[0] += 1
            if not os.environ.get("TRMCR_BENCH_NO_GM"):   # experiment switch (not a bench mode)
                sim.global_moments(gms[k], all_ranks=world > 1)
        else:
            slab.step(xchg)

    def drain():
        if world > 1 and W["kind"] == "hom":
            sim.comm_wait()

    for _ in range(args.warmup):
        one_step()
    drain()
    torch.cuda.synchronize()
    # identify the dominant kernel on a short profiled segment (all launches
    # bracketed), then time the K steps bracketing only that kernel
    sim.set_profiling(True)
    for _ in range(min(20, max(args.steps, 1))):
        one_step()
    drain()
    probe = sim.kernel_times()
    dom_name = max(probe.items(), key=lambda kv: kv[1][0])[0] if probe else None
    torch.cuda.synchronize()
    n_before = sim.num_particles()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = sim.launch_count
    if dom_name:
        sim.set_profiling_kernels([dom_name])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            one_step()
        drain()                                   # every all-reduce inside the timed region
        e1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_local = e0.elapsed_time(e1)
    ktimes = sim.kernel_times()
    sim.set_profiling(False)
    kernel_ms_probe = {k: round(v[0] / max(v[1], 1), 4) for k, v in probe.items()}
    launches = sim.launch_count - launches0
    n_after = sim.num_particles()
    updates_local = 0.5 * (n_before + n_after) * args.steps
    t = torch.tensor([ms_local, updates_local], dtype=torch.float64, device=dev)
    if world > 1:
        tm = t[:1].clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        tu = t[1:].clone()
        dist.all_reduce(tu, op=dist.ReduceOp.SUM)
        ms, updates = float(tm.item()), float(tu.item())
    else:
        ms, updates = ms_local, updates_local
    value = updates / (ms * 1e-3)

    # ---- roofline of the dominant kernel (algorithmic bytes) ----
    dom, (dom_ms, dom_n) = max(ktimes.items(), key=lambda kv: kv[1][0])
    rs = 4 if td == torch.float32 else 8
    if dom in ("cell_step_smem", "cell_step_gmem", "thermal_warp_kernel", "cell_step_warp"):
        bytes_per = 2 * 3 * rs            # read v, write v (f_chg = 1: fluid regime)
    elif dom == "shock_collide_warp" and W["kind"] == "shock" and sim.fused:
        # the fused pass: transport + sort + collisions, reading and
        # writing (x, v) once: SURVEY 8(d) D3's fused minimum, 8 rs per particle
        bytes_per = 8 * rs
    elif dom in ("shock_collide_smem", "shock_collide_gmem", "shock_collide_warp"):
        # SURVEY 8(d) D3, collision step: read every v, write the changed ones:
        # 3 rs (1 + f_chg), f_chg = 1 - untouched / n of this run's last step
        st = sim.stats()
        f_chg = 1.0 - float(st["untouched"].sum()) / max(float(st["n"].sum()), 1.0)
        bytes_per = 3 * rs * (1.0 + f_chg)
    elif dom == "scatter_sorted":
        bytes_per = 2 * 4 * rs            # the sort: read (x, v), write (x, v)
    elif dom == "transport_kernel":
        bytes_per = 3 * rs                # read x, v_x; write x
    else:
        bytes_per = 3 * rs
    peak, peak_kind = measured_peaks()
    n_mean = 0.5 * (n_before + n_after)
    achieved = bytes_per * n_mean / (dom_ms / dom_n * 1e-3) / 1e9
    traffic = ncu_traffic(wl_name)
    # the whole step against its fused minimum: homogeneous
    # read + write v (6 rs), shock read + write (x, v) (8 rs) per particle
    step_bytes = (6 if W["kind"] == "hom" else 8) * rs
    step_gbs = step_bytes * n_mean * args.steps / (ms_local * 1e-3) / 1e9
    roof = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
            "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
            "traffic": traffic, "algorithmic_bytes_per_particle": round(bytes_per, 3),
            "kernel_share_of_step": round(dom_ms / ms_local, 4),
            "step": {"algorithmic_bytes_per_particle": step_bytes, "achieved": round(step_gbs, 1),
                     "frac": round(step_gbs / peak, 4)},
            "kernel_ms_probe": kernel_ms_probe}
    issue = ncu_issue(wl_name)
    if issue:
        # the collision kernel is bound by instruction issue and latency, not by
        # HBM: its executed warp instructions per launch (ncu --set full, the
        # committed summary) per second of this run, against the SM issue peak
        # (4 warp instructions per clock per SM x 148 SMs x the max SM clock)
        clk_hz = 1e6 * float(measured_clock_mhz())
        ipeak = 4.0 * 148 * clk_hz
        ach = issue["warp_instructions"] / (dom_ms / dom_n * 1e-3)
        roof["issue"] = {"kernel": issue["kernel"], "warp_instructions_per_launch": issue["warp_instructions"],
                         "achieved": round(ach / 1e9, 1), "peak": round(ipeak / 1e9, 1),
                         "unit": "G warp-instructions/s", "frac": round(ach / ipeak, 4)}

    # ---- e2e: host buffers through the public API, every step ----
    ke = max(3, min(args.steps, 20))
    out = np.zeros((sim.ncells, len(api.MOMENT_FIELDS)))
    if W["kind"] == "hom":
        hv = [torch.as_tensor(np.ascontiguousarray(W[k])).to(td).pin_memory().numpy() for k in ("vx", "vy", "vz")]

        def e2e_step():
            sim.step_host(*hv, out=out)
        h2d = 3 * rs * n_local
        path = "Simulation.step_host (trmcr_step_host): pinned host velocities in, per-cell moments out"
    else:
        hv = [torch.as_tensor(np.ascontiguousarray(W[k])).to(td).pin_memory().numpy()
              for k in ("x", "vx", "vy", "vz")]
        h2d = 4 * rs * len(hv[0])
        if slab.neighbors == 0:
            def e2e_step():
                sim.step_host_particles(*hv, out=out)
            path = ("Simulation.step_host_particles (trmcr_step_host_particles): pinned host (x, v) in, "
                    "rebinned on the device, one step, per-cell moments out")
        else:
            def e2e_step():
                sim.set_particles(hv[1], hv[2], hv[3], x=hv[0])
                slab.step(xchg)
                out[:] = sim.moments()
            path = ("Simulation.set_particles + ShockSlab.step + Simulation.moments: pinned host (x, v) of the "
                    "slab in, one step with the neighbour exchange, per-cell moments out")
    e2e_step()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(ke):
        e2e_step()
    t_e2e = time.perf_counter() - t0
    tt = torch.tensor([t_e2e, float(h2d), float(out.nbytes)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(tt[1:], op=dist.ReduceOp.SUM)
    e2e_updates = updates / args.steps        # particles per step, all ranks (state at the timed steps)
    if W["kind"] == "shock":
        tn = torch.tensor([float(sum(len(a) for a in hv[:1]))], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tn)
        e2e_updates = float(tn.item())
    e2e = {"value": e2e_updates * ke / float(tt[0].item()), "unit": UNIT,
           "h2d_bytes_per_step": int(tt[1].item()), "d2h_bytes_per_step": int(tt[2].item()), "steps": ke,
           "path": path}

    if rank != 0:
        sim.close()
        return None
    cpu = None
    if world == 1 and cpu_seconds > 0:
        rate, info = oracle_rate(W, seconds=cpu_seconds)
        cpu = {"value": rate, "unit": UNIT, "cores": info["cores"], "kind": "oracle",
               "sample": info["sample"]}
    clocks = clk.summary()
    cfg = full_cfg(W, world)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": W.get("scaling", "strong"), "vs_baseline": None,
            "dtype": "f32" if td == torch.float32 else "f64", "data": "synthetic", "config": cfg,
            "roofline": roof, "cpu_baseline": cpu, "clocks": clocks, "e2e": e2e,
            "gpu_launches": int(launches), "impl": "trmcr"}
    sim.close()
    return line


def run_trmcr(args, rank, world, local_rank):
    line = measure(args, args.workload, rank, world, local_rank,
                   0.0 if args.no_cpu_baseline else args.cpu_seconds)
    sec = None
    if args.secondary != "none" and args.secondary != args.workload:
        import torch
        torch.cuda.empty_cache()
        sec = measure(args, args.secondary, rank, world, local_rank, 0.0)
    if rank == 0:
        if sec is not None:
            sec.pop("cpu_baseline", None)
            sec.pop("impl", None)
            line["secondary"] = sec
        print(json.dumps(line), flush=True)


def self_launch(args):
    """--gpus N > 1 outside torchrun: one process per GPU under torch.distributed.run."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c5", choices=["c1", "c2", "c3", "c3weak", "c4", "c5"])
    ap.add_argument("--secondary", default="c3", choices=["none", "c1", "c2", "c3", "c3weak", "c4", "c5"])
    ap.add_argument("--eps", type=float, default=None)
    ap.add_argument("--impl", default="trmcr", choices=["trmcr", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    run_trmcr(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
