import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1009_2768_b200 import api
api.LIB_PATH = os.environ.get("TRMCR_DBG_LIB", os.path.join(os.path.dirname(api.__file__), "libtrmcr_dbg.so"))
import bench
wl = sys.argv[1]; steps = int(sys.argv[2])
W = bench.workload(wl)
td = torch.float32 if W["dtype"] == np.float32 else torch.float64
T = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=td)
if W["kind"] == "hom":
    sim = api.Simulation(T(W["vx"]), T(W["vy"]), T(W["vz"]), offsets=W["offsets"], **W["kw"])
else:
    sim = api.Simulation(T(W["vx"]), T(W["vy"]), T(W["vz"]), x=T(W["x"]), shock=W["setup"], **W["kw"])
L = api.lib(); L.trmcr_debug_phase_cycles.argtypes = [ctypes.POINTER(ctypes.c_double)]
out = np.zeros(16)
sim.step(3); torch.cuda.synchronize(); L.trmcr_debug_phase_cycles(out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
sim.step(steps); torch.cuda.synchronize(); L.trmcr_debug_phase_cycles(out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
names = ["moments+split", "plan_counts", "plan_execute", "rad_estimate", "rad_retries", "pre-maxw", "maxwellian", "store", "gather", "load_sums(lock)", "barrier_begin(lock)", "barrier_end(lock)", "pe_pass2", "pe_pass3"]
cells = sim.ncells * steps
st = sim.stats()
print("per cell-step cycles:", {names[k]: round(out[k] / cells) for k in range(14)})
print("mean depth", st["depth"].mean(), "attempts", st["attempts"].mean(), "proposals", st["proposals"].mean(), "thermalised", st["thermalised"].mean(), "n", st["n"].mean(), "m_used", st["m_used"].mean())
