"""Per-phase wall cycles of the pooled-batch shock kernel (debug build
libtrmcr_dbg.so, -DTRMCR_PHASE_TIMING).  usage: batch_phases.py wl steps"""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1009_2768_b200 import api
api.LIB_PATH = os.path.join(os.path.dirname(api.__file__), "libtrmcr_dbg.so")
import bench
wl = sys.argv[1]; steps = int(sys.argv[2])
W = bench.workload(wl)
T = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=torch.float32)
sim = api.Simulation(T(W["vx"]), T(W["vy"]), T(W["vz"]), x=T(W["x"]), shock=W["setup"], **W["kw"])
L = api.lib(); L.trmcr_debug_phase_cycles.argtypes = [ctypes.POINTER(ctypes.c_double)]
out = np.zeros(16)
sim.step(3); torch.cuda.synchronize(); L.trmcr_debug_phase_cycles(out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
sim.step(steps); torch.cuda.synchronize(); L.trmcr_debug_phase_cycles(out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
names = ["stage", "moments+split", "round setup", "plan levels", "guard", "pass1", "pass2+prefix", "pass3",
         "rad+decision", "maxwellian", "write-back"]
nb = out[14]
print("batches", nb / steps, "rounds per batch", out[15] / nb)
print("per batch cycles:", {names[k]: round(out[k] / nb) for k in range(11)}, "total", round(out[:11].sum() / nb))
