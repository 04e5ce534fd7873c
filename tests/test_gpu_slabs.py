"""Slab decomposition of the 1D shock: a run split into 2 or 3
slabs (emulated in one process on one GPU, exchange by device copies between
trmcr_shock_begin and trmcr_shock_finish; no kernel waits on another) is
bitwise identical to the single-slab run — positions, velocities, offsets and
per-cell statistics — because the RNG is keyed by global cell id and the
immigrants are gathered in the global canonical order."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _sorted_shock(setup, seed, dtype):
    x, vx, vy, vz = synth.shock_particles(setup, seed=seed, dtype=dtype)
    inv = setup["ncells"] / (setup["x_max"] - setup["x_min"])
    cell = np.clip(np.floor((x.astype(np.float64) - setup["x_min"]) * inv), 0, setup["ncells"] - 1)
    o = np.argsort(cell, kind="stable")
    return x[o], vx[o], vy[o], vz[o], np.bincount(cell.astype(int), minlength=setup["ncells"])


@pytest.mark.parametrize("world,dtype,fused_full,fused_slabs",
                         [(2, np.float64, "1", "1"), (3, np.float64, "1", "1"), (3, np.float32, "1", "1"),
                          (2, np.float64, "0", "0"), (3, np.float32, "0", "0"), (3, np.float64, "0", "1")])
def test_slabs_match_single_domain(world, dtype, fused_full, fused_slabs, monkeypatch):
    """fused_*: the fused pass (1) or the three-pass step (0) for the single
    domain and for the slabs - the last case cross-checks the two step
    structures (and the two emigrant packers) against each other."""
    _run_slabs(world, dtype, fused_full, fused_slabs, monkeypatch, ncells=60, n_total=30_000, half_width=6.0)


@pytest.mark.parametrize("world,dtype", [(2, np.float64), (3, np.float32)])
def test_slabs_edge_first_transport(world, dtype, monkeypatch):
    """Slabs wider than the emigrant window (64 cells from a neighbour): the
    transport runs in two launches - the edge tiles, whose emigrants are packed
    (and, on the NCCL path, exchanged on the communication stream meanwhile),
    then the bulk tiles.  Same bitwise result as the single domain."""
    _run_slabs(world, dtype, "0", "0", monkeypatch, ncells=720, n_total=72_000, half_width=36.0)


def _run_slabs(world, dtype, fused_full, fused_slabs, monkeypatch, ncells, n_total, half_width):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1009_2768_b200 import api, dist
    setup = synth.shock_setup(mach=3.0, ncells=ncells, n_total=n_total, x_min=-half_width, x_max=half_width)
    x, vx, vy, vz, counts = _sorted_shock(setup, 3, dtype)
    td = torch.float64 if dtype == np.float64 else torch.float32
    T = lambda a: torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=td)
    kw = dict(model=1, adaptive=True, m_init=2, m_cap=64, eps=0.3, dt=setup["dt"], seed=5)
    monkeypatch.setenv("TRMCR_SHOCK_FUSED", fused_full)
    full = api.Simulation(T(vx), T(vy), T(vz), x=T(x), shock=setup, **kw)
    assert full.fused == (fused_full == "1")
    monkeypatch.setenv("TRMCR_SHOCK_FUSED", fused_slabs)
    cuts = dist.slab_cuts(counts, world)
    slabs = []
    for first, nc in cuts:
        px, pvx, pvy, pvz = dist.slab_particles(x, vx, vy, vz, setup, first, nc)
        slabs.append(dist.ShockSlab(api, setup, first, nc, T(pvx), T(pvy), T(pvz), x=T(px), device="cuda",
                                    exchange_capacity=4096, **kw))
    for step in range(12):
        full.step(1)
        for s in slabs:
            s.sim.shock_begin()
        dist.host_exchange(slabs)
        for s in slabs:
            s.sim.shock_finish()
        for sim in [full] + [s.sim for s in slabs]:     # the scatter sort ran (no gather fallback)
            info = sim.sort_info()
            assert info["scatter_enabled"] and not info["gathered"]
    g = full.particles()
    parts = [s.sim.particles() for s in slabs]
    for k in ("x", "vx", "vy", "vz"):
        np.testing.assert_array_equal(np.concatenate([p[k] for p in parts]), g[k], err_msg=k)
    off = np.concatenate([[0]] + [np.diff(p["offsets"]) for p in parts]).cumsum()
    np.testing.assert_array_equal(off, g["offsets"])
    st = np.concatenate([s.sim.stats() for s in slabs])
    for f in ("n", "proposals", "accepted", "thermalised", "m_next", "p"):
        np.testing.assert_array_equal(st[f], full.stats()[f], err_msg=f)
