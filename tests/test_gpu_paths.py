"""Which kernels run: the scheduling decisions of trmcr_step on a B200.

Results do not depend on these decisions (parity tests cover every path);
these tests guard the launch choices that set the speed."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _sim(api, v, **kw):
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=torch.float32)
    return api.Simulation(T(v[0]), T(v[1]), T(v[2]), offsets=v[3], **kw)


def test_collisional_cells_run_the_warp_kernel():
    """Cells outside the fluid regime must go to the warp-per-cell kernel every
    step (a step that skipped the thermal kernel once read its deferral count
    as zero and sent every cell to a single CTA)."""
    from paper_1009_2768_b200 import api
    sim = _sim(api, synth.uniform_cells(2000, 500, seed=1, dtype=np.float32), model=api.HARD_SPHERE,
               m_fixed=16, eps=1.0, dt=0.1, seed=1)
    sim.step(4)
    sim.set_profiling(True)
    sim.step(12)
    kt = sim.kernel_times()
    sim.set_profiling(False)
    assert kt.get("cell_step_warp", (0, 0))[1] == 12, kt
    assert kt["cell_step_smem"][0] / 12 < 0.05, kt          # ms per step: nothing left for the CTA kernel


def test_deep_trees_stay_parallel():
    """Deep trees (x ~ 2.7 at m = 16: ~0.75 n collisions per cell) fit the warp
    slabs; the global-memory kernel is not the bottleneck."""
    from paper_1009_2768_b200 import api
    sim = _sim(api, synth.uniform_cells(4096, 1024, seed=2, dtype=np.float32), model=api.HARD_SPHERE,
               m_fixed=16, eps=0.3, dt=0.1, seed=2)
    sim.step(3)
    sim.set_profiling(True)
    sim.step(5)
    kt = sim.kernel_times()
    sim.set_profiling(False)
    assert kt["cell_step_warp"][1] == 5, kt
    assert kt.get("cell_step_gmem", (0.0, 1))[0] / 5 < 0.1, kt


def test_fluid_cells_run_the_thermal_kernel_only():
    from paper_1009_2768_b200 import api
    sim = _sim(api, synth.uniform_cells(2048, 1024, seed=3, dtype=np.float32), model=api.HARD_SPHERE,
               m_fixed=64, eps=0.01, dt=0.1, seed=3)
    sim.step(20)
    sim.set_profiling(True)
    sim.step(8)
    kt = sim.kernel_times()
    sim.set_profiling(False)
    assert kt["thermal_warp_kernel"][1] == 8 and "cell_step_warp" not in kt, kt


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_pooled_batch_kernel_equals_lock_step_kernel(dtype, monkeypatch):
    """The pooled-batch shock collision kernel (batch.cuh, TRMCR_SHOCK_BATCH=1)
    and the lock-step warp kernel run the same keyed draws in the same
    per-lane reduction orders: positions, velocities and every statistic are
    bitwise identical, step after step, while both kernels take every cell
    (eps 1: RAD retries, no cell over either kernel's capacity - a cell one of
    them defers is stepped by the CTA kernel, whose fp32 sums round
    differently).  tools/batch_vs_lock.py runs the same check on C4 / C5."""
    from paper_1009_2768_b200 import api
    setup = synth.shock_setup(mach=3.0, ncells=64, n_total=40_000, x_min=-6.0, x_max=6.0)
    x, vx, vy, vz = synth.shock_particles(setup, seed=2, dtype=dtype)
    inv = setup["ncells"] / (setup["x_max"] - setup["x_min"])
    o = np.argsort(np.clip(np.floor((x.astype(np.float64) - setup["x_min"]) * inv), 0, 63), kind="stable")
    td = torch.float32 if dtype == np.float32 else torch.float64
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a[o])).to(device="cuda", dtype=td)
    kw = dict(model=1, adaptive=True, m_init=2, m_cap=64, eps=1.0, dt=setup["dt"], seed=9)
    sims = []
    for flag in ("0", "1"):
        monkeypatch.setenv("TRMCR_SHOCK_BATCH", flag)
        sims.append(api.Simulation(T(vx), T(vy), T(vz), x=T(x), shock=setup, **kw))
    for _ in range(6):
        for s in sims:
            s.step(1)
        a, b = sims[0].particles(), sims[1].particles()
        for f in ("x", "vx", "vy", "vz", "offsets"):
            np.testing.assert_array_equal(a[f], b[f], err_msg=f)
        sa, sb = sims[0].stats(), sims[1].stats()
        for f in sa.dtype.names:
            np.testing.assert_array_equal(sa[f], sb[f], err_msg=f)
    assert sims[0].stats()["proposals"].sum() > 0
