"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

fp64: every discrete decision identical (collision records: cell, attempt,
level, j, slots, accept bit; split/plan/RAD stats; m_max), velocities within
1e-12 relative (north star).  The two sides compute transcendental functions
and sums in different orders, so fp64 values can differ by a few ulps; a
decision flips only if a uniform lands within those ulps of its threshold
(probability ~1e-15 per decision).
fp32: statistical agreement over 16 seeds (|z| <= 3 for >= 99 % of the
observables, all |z| <= 5) and conservation to 1e-6.
"""
import math

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def api():
    from paper_1009_2768_b200 import api as A
    return A


def _dev(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype).contiguous()


def _dedupe(log):
    """Canonical order of a GPU log.  A cell handed from one kernel to a larger one
    (overflow) is re-run from its unmodified input, so the records its first kernel
    wrote before handing it over reappear; such duplicates must be IDENTICAL (same
    keyed draws on the same data) - any difference fails here instead of being
    dropped silently."""
    if len(log) == 0:
        return log
    keys = np.stack([log["cell"], log["attempt"], log["level"], log["j"]], 1)
    _, idx, inv = np.unique(keys, axis=0, return_index=True, return_inverse=True)
    inv = inv.reshape(-1)
    for f in ("slot_i", "slot_k", "accepted"):
        first = log[f][idx][inv]
        bad = np.nonzero(log[f] != first)[0]
        assert len(bad) == 0, ("duplicate GPU records differ", f, log[bad[:4]])
    out = log[np.sort(idx)]
    order = np.lexsort((out["j"], out["level"], out["attempt"], out["cell"]))
    return out[order]


def _cmp_logs(lg, lo):
    lg, lo = _dedupe(lg), _dedupe(lo)
    assert len(lg) == len(lo), (len(lg), len(lo))
    for f in ("cell", "attempt", "level", "j", "slot_i", "slot_k", "accepted"):
        np.testing.assert_array_equal(lg[f], lo[f], err_msg=f)


def _cmp_v(g, vx, vy, vz, offsets, rel=1e-12):
    V = np.stack([vx, vy, vz], 1)
    G = np.stack([g["vx"], g["vy"], g["vz"]], 1).astype(np.float64)
    err = np.linalg.norm(G - V, axis=1)
    for c in range(len(offsets) - 1):
        a, b = offsets[c], offsets[c + 1]
        if b <= a:
            continue
        scale = np.sqrt((V[a:b] ** 2).sum(1).mean()) + np.linalg.norm(V[a:b], axis=1)
        assert np.all(err[a:b] <= rel * scale), (c, (err[a:b] / scale).max())


STAT_EXACT = ["n", "depth", "attempts", "leaves", "untouched", "thermalised", "proposals", "accepted",
              "violations", "maxw", "m_used", "m_next"]


def _cmp_stats(sg, so):
    for f in STAT_EXACT:
        np.testing.assert_array_equal(sg[f], so[f], err_msg=f)
    for f in ("p", "mu", "sigma", "S0"):
        np.testing.assert_allclose(sg[f], so[f], rtol=1e-12, atol=1e-300, err_msg=f)


def _parity(orc, api, v, offsets, steps, log_cap=400_000, **kw):
    ocfg = orc.Config(**{k: kw[k] for k in kw if k in orc.Config.__dataclass_fields__})
    o = orc.HomogeneousState(ocfg, v[0], v[1], v[2], offsets, log_cap=log_cap)
    gkw = dict(kw)
    sim = api.Simulation(_dev(v[0]), _dev(v[1]), _dev(v[2]), offsets=offsets, **gkw)
    sim.set_log(log_cap)
    for s in range(steps):
        o.step(1)
        sim.step(1)
        _cmp_logs(sim.collisions(), o.collisions())
        _cmp_stats(sim.stats(), o.stats)
    g = sim.particles()
    _cmp_v(g, o.vx, o.vy, o.vz, offsets)
    mg, mo = sim.moments(), o.moments()
    np.testing.assert_allclose(mg[:, 11], mo[:, 11])
    np.testing.assert_allclose(mg[:, 2:11], mo[:, 2:11], rtol=1e-11, atol=1e-11)
    return sim, o


def test_homogeneous_fp64_maxwell_ragged(orc, api):
    v = synth.ragged_cells(60, 300, seed=3)
    _parity(orc, api, v[:3], v[3], 5, model=0, m_fixed=6, eps=0.3, dt=0.2, seed=4)


def test_homogeneous_fp64_hs_rad_ragged(orc, api):
    v = synth.ragged_cells(60, 400, seed=5)
    _parity(orc, api, v[:3], v[3], 6, model=1, adaptive=1, m_init=2, m_cap=64, eps=0.5, dt=0.1, seed=6)


@pytest.mark.parametrize("alpha", [0.35, 0.8])
def test_homogeneous_fp64_vhs_rad_ragged(orc, api, alpha):
    """VHS molecules, B = K|q|^alpha (sec. VHS): Sigma' = (2 dv)^alpha, accept iff
    xi Sigma' < |q|^alpha; every decision and velocity as the oracle's."""
    v = synth.ragged_cells(50, 400, seed=12)
    _parity(orc, api, v[:3], v[3], 5, model=2, alpha=alpha, adaptive=1, m_init=2, m_cap=64, eps=0.5, dt=0.1,
            seed=13)


@pytest.mark.parametrize("wb,warp_path", [(1, "1"), (2, "1"), (3, "1"), (1, "0")])
def test_homogeneous_fp64_trmc_wb(orc, api, monkeypatch, wb, warp_path):
    """TRMC-WB (Alg 4.6): tree lengths under eqs. def:2, def:3, def:1 in the
    LS plan, rejected final samples join the Maxwellian; warp and CTA kernels."""
    monkeypatch.setenv("TRMCR_WARP_PATH", warp_path)
    v = synth.ragged_cells(40, 500, seed=16)
    _parity(orc, api, v[:3], v[3], 3, model=1, m_fixed=10, wb=wb, wb_max=2, eps=2.0, dt=0.3, seed=17)


@pytest.mark.parametrize("model,alpha,warp_path", [(1, 1.0, "1"), (2, 0.5, "1"), (1, 1.0, "0")])
def test_majorant_update_fp64(orc, api, monkeypatch, model, alpha, warp_path):
    """Majorant raised after each collision [R33] on counter-streaming
    cold beams (violations happen): levels with a violation run in canonical
    order on one lane / thread, the others in parallel; RAD attempts carry the
    raised bound.  Every decision, counter and velocity as the oracle's."""
    monkeypatch.setenv("TRMCR_WARP_PATH", warp_path)
    v = synth.cold_beams(24, 400, seed=4)
    sim, o = _parity(orc, api, v[:3], v[3], 1, model=model, alpha=alpha, adaptive=1, m_init=4, m_cap=64,
                     eps=0.15, dt=0.1, seed=5, sigma_update=1)
    assert o.stats["violations"].sum() > 10 and o.stats["attempts"].max() > 1


def test_majorant_update_giant_cell_fp64(orc, api):
    """The same variant on the grid-cooperative kernel (one 40,000-particle cell)."""
    v = synth.cold_beams(1, 40_000, seed=22)
    _, o = _parity(orc, api, v[:3], v[3], 1, log_cap=400_000, model=1, m_fixed=24, eps=0.3, dt=0.1, seed=23,
                   sigma_update=1)
    assert o.stats["violations"][0] > 0


@pytest.mark.parametrize("model,kw", [(1, dict(eps=0.5, dt=0.1)), (0, dict(eps=1.0, dt=0.2)),
                                      (2, dict(alpha=0.6, eps=0.5, dt=0.1))])
def test_literal_layout_fp64(orc, api, model, kw):
    """The paper's own layout (Alg 4.3/4.4 literally: recursive builds, stored
    siblings, one sequential keyed stream per cell; one GPU thread per cell)
    against the oracle's literal mode: every counter and velocity."""
    # the literal algorithm has no finite-N guard: Maxwell cells stay large
    v = synth.ragged_cells(40, 400, seed=24) if model else synth.uniform_cells(32, 300, seed=24)
    _parity(orc, api, v[:3], v[3], 3, model=model, m_fixed=12, seed=25, literal=1, **kw)


def test_literal_layout_majorant_update_fp64(orc, api):
    v = synth.cold_beams(12, 300, seed=26)
    _, o = _parity(orc, api, v[:3], v[3], 1, model=1, m_fixed=32, eps=0.15, dt=0.1, seed=27, literal=1,
                   sigma_update=1)
    assert o.stats["violations"].sum() > 0


def test_giant_cell_parallel_ranks_fp64(orc, api):
    """One 60,000-particle cell (global-memory CTA path) whose low levels hold
    thousands of collisions: in-level ranks computed by all warps (chunk
    histograms) must equal the serial definition - every record and velocity
    as the oracle's."""
    v = synth.anisotropic_gaussian(60_000, seed=18)
    v = tuple(np.asarray(a, dtype=np.float64) for a in v)
    sim, o = _parity(orc, api, v, np.array([0, 60_000]), 2, log_cap=200_000, model=1, m_fixed=24, eps=1.0,
                     dt=0.1, seed=19)
    assert o.stats["proposals"][0] > 8000


def test_giant_cell_deep_rad_config2_eps01_fp64(orc, api):
    """Config 2's deep regime: a 40,000-particle hard-sphere
    cell with the (2, 1/2, 1/2) anisotropic Gaussian, eps = 0.1, dt = 0.05
    (x = mu dt / eps ~ 6-7: p ~ 1e-3, depth limited only by RAD), RAD with
    m_init = 2 and m_cap = 4096, on the grid-cooperative giant-cell kernel:
    every decision (incl. the RAD retries and m_next) and every velocity as the
    oracle's, over 2 steps (measured: m = 4096, 2,858 levels, 113,625 proposals)."""
    v = synth.anisotropic_gaussian(40_000, seed=31)
    v = tuple(np.asarray(a, dtype=np.float64) for a in v)
    sim, o = _parity(orc, api, v, np.array([0, 40_000]), 2, log_cap=3_000_000, model=1, adaptive=1, m_init=2,
                     m_cap=4096, eps=0.1, dt=0.05, seed=31)
    st = o.stats
    x = st["mu"][0] * 0.05 / 0.1
    assert 4.0 < x < 10.0, x
    # RAD doubled m far past the default 64 (step 1) and the trees are thousands of levels deep
    assert st["m_used"][0] >= 256 and st["depth"][0] >= 256 and st["proposals"][0] > 10_000, (
        st["m_used"][0], st["depth"][0], st["proposals"][0])


def test_giant_cell_vhs_wb_fp64(orc, api):
    """A 40,000-particle cell on the grid-cooperative kernel with VHS molecules
    (alpha = 0.6) and TRMC-WB (1 + mean, m_max = 2): every decision and
    velocity as the oracle's."""
    v = synth.anisotropic_gaussian(40_000, seed=20)
    v = tuple(np.asarray(a, dtype=np.float64) for a in v)
    _, o = _parity(orc, api, v, np.array([0, 40_000]), 2, log_cap=200_000, model=2, alpha=0.6, m_fixed=12,
                   wb=2, wb_max=2, eps=1.0, dt=0.1, seed=21)
    assert o.stats["maxw"][0] > 0 and o.stats["proposals"][0] > 4000


def test_homogeneous_fp64_hs_m4_indicator(orc, api):
    v = synth.ragged_cells(30, 500, seed=9)
    _parity(orc, api, v[:3], v[3], 4, model=1, adaptive=1, m_init=4, m_cap=32, indicator=1, eps=0.2,
            dt=0.05, seed=10, delta1=0.001, delta2=0.004)


def test_config1_full_fp64_parity(orc, api):
    """Config 1 (BASELINE.json configs[0]): 10^4 Maxwell particles, one cell, fp64, 20 steps;
    240 KB of velocities exceed shared memory: the global-memory path runs."""
    v = synth.two_maxwellians(10_000, seed=1)
    sim, o = _parity(orc, api, v, [0, 10_000], 20, model=0, m_fixed=64, eps=1.0, dt=0.1, seed=1)
    assert sim.stats()["proposals"][0] > 0


def test_overflowing_tree_takes_global_path(orc, api):
    """Deep trees (x ~ 8) overflow the shared-memory plan: the cell is redone in global memory."""
    v = synth.uniform_cells(8, 256, seed=2)
    _parity(orc, api, v[:3], v[3], 2, model=1, m_fixed=64, eps=0.05, dt=0.05, seed=3)


def test_full_thermalisation_and_identity(orc, api):
    v = synth.uniform_cells(16, 128, seed=4)
    _parity(orc, api, v[:3], v[3], 2, model=1, m_fixed=8, eps=1e-7, dt=0.1, seed=5)   # tau = 1
    _parity(orc, api, v[:3], v[3], 2, model=1, m_fixed=8, eps=1.0, dt=1e-14, seed=5)  # tau -> 0


def test_empty_cells_only(api):
    off = np.zeros(5, dtype=np.int64)
    e = torch.zeros(0, dtype=torch.float64, device="cuda")
    sim = api.Simulation(e, e, e, offsets=off, eps=1.0, dt=0.1)
    sim.step(3)
    assert np.all(sim.stats()["n"] == 0)


def test_invalid_arguments(api):
    v = _dev(np.zeros(4))
    with pytest.raises(api.TrmcrError) as ei:
        api.Simulation(v, v, v, offsets=[0, 4], eps=0.0, dt=0.1)
    assert ei.value.status == api.EINVAL
    with pytest.raises(api.TrmcrError):
        api.Simulation(v, v, v, offsets=[0, 3, 2, 4], eps=1.0, dt=0.1)
    with pytest.raises(api.TrmcrError):
        api.Simulation(v, v, v, offsets=[0, 4], eps=1.0, dt=0.1, adaptive=True, delta1=0.02, delta2=0.01)


def _zstats(a, b):
    a, b = np.asarray(a), np.asarray(b)
    se = np.sqrt(a.var(0, ddof=1) / len(a) + b.var(0, ddof=1) / len(b)) + 1e-300
    return np.abs(a.mean(0) - b.mean(0)) / se


@pytest.mark.parametrize("eps,dt", [(0.01, 0.1), (1.0, 0.05)])
def test_fp32_statistical_parity(orc, api, eps, dt):
    """fp32 production mode vs the fp64 oracle: per-cell T, Pxx, M4 after 3 steps, 16 seeds."""
    ncells, ppc, steps = 256, 1024, 3
    G, O = [], []
    for seed in range(1, 17):
        vx, vy, vz, off = synth.bimodal_cells(ncells, ppc, seed=seed)
        sim = api.Simulation(_dev(vx, torch.float32), _dev(vy, torch.float32), _dev(vz, torch.float32),
                             offsets=off, model=1, m_fixed=64, eps=eps, dt=dt, seed=seed)
        sim.step(steps)
        G.append(sim.moments()[:, [5, 8, 9]])
        o = orc.HomogeneousState(orc.Config(model=1, m_fixed=64, eps=eps, dt=dt, seed=seed),
                                 vx.astype(np.float64), vy.astype(np.float64), vz.astype(np.float64), off)
        o.step(steps)
        O.append(o.moments()[:, [5, 8, 9]])
    z = _zstats(G, O).ravel()
    assert np.mean(z <= 3) >= 0.99 and z.max() <= 5, (np.mean(z <= 3), z.max())


def test_fp32_conservation(api):
    vx, vy, vz, off = synth.bimodal_cells(512, 1024, seed=3)
    sim = api.Simulation(_dev(vx, torch.float32), _dev(vy, torch.float32), _dev(vz, torch.float32),
                         offsets=off, model=1, adaptive=True, m_init=2, m_cap=64, eps=0.5, dt=0.1, seed=3)
    m0 = sim.moments()
    sim.step(1)
    m1 = sim.moments()
    np.testing.assert_array_equal(m0[:, 0], m1[:, 0])
    scale = np.sqrt(2 * m0[:, 6])
    assert np.all(np.abs(m1[:, 2:5] - m0[:, 2:5]).max(1) <= 1e-6 * scale)
    assert np.all(np.abs(m1[:, 6] - m0[:, 6]) <= 1e-6 * m0[:, 6])


# ---------------------------------------------------------------- shock
def _shock_pair(orc, api, mach, ncells, ntot, steps, eps, dtype, seed=1, x_min=-4.0, x_max=4.0, cfl=0.5):
    setup = synth.shock_setup(mach=mach, ncells=ncells, n_total=ntot, x_min=x_min, x_max=x_max, cfl=cfl)
    x, vx, vy, vz = synth.shock_particles(setup, seed=seed)
    inv = setup["ncells"] / (setup["x_max"] - setup["x_min"])
    cell = np.clip(np.floor((x - setup["x_min"]) * inv), 0, ncells - 1)
    order = np.argsort(cell, kind="stable")
    x, vx, vy, vz = x[order], vx[order], vy[order], vz[order]
    td = torch.float64 if dtype == np.float64 else torch.float32
    sim = api.Simulation(_dev(vx, td), _dev(vy, td), _dev(vz, td), x=_dev(x, td), shock=setup,
                         model=1, adaptive=True, m_init=2, m_cap=64, eps=eps, dt=setup["dt"], seed=seed)
    o = orc.ShockState(orc.Config(model=1, adaptive=1, m_init=2, m_cap=64, eps=eps, dt=setup["dt"],
                                  seed=seed), setup, x, vx, vy, vz)
    return setup, sim, o


@pytest.mark.parametrize("fused,scatter", [("1", "1"), ("0", "1"), ("0", "0")])
def test_shock_fp64_parity(orc, api, monkeypatch, fused, scatter):
    """Every step structure: the fused pass (default at CFL < 1: transport, sort
    and collisions in one kernel, fused.cuh), the three-pass step with
    scatter_sorted + edge_place, and the gather inside the collision kernels
    (TRMCR_SHOCK_SCATTER=0)."""
    monkeypatch.setenv("TRMCR_SHOCK_FUSED", fused)
    monkeypatch.setenv("TRMCR_SHOCK_SCATTER", scatter)
    setup, sim, o = _shock_pair(orc, api, 3.0, 40, 8000, 0, 0.2, np.float64)
    assert sim.fused == (fused == "1")
    for s in range(8):
        sim.step(1)
        o.step(1)
        info = sim.sort_info()
        assert info["scatter_enabled"] == (scatter == "1") and not info["gathered"]
        g = sim.particles()
        np.testing.assert_array_equal(g["offsets"], o.offsets)
        n = o.n
        np.testing.assert_allclose(g["x"], o.x[:n], rtol=0, atol=1e-12)
        _cmp_v(g, o.vx[:n], o.vy[:n], o.vz[:n], o.offsets)
        _cmp_stats(sim.stats(), o.stats)
    assert o.counts[0] > 0     # reservoir particles entered


def test_shock_fp64_parity_many_cells(orc, api):
    """10,000 cells: the offsets scan spans three CTAs (decoupled look-back over
    4096-cell tiles) and the sort many tiles; every position, offset and
    velocity as the oracle's."""
    setup, sim, o = _shock_pair(orc, api, 3.0, 10_000, 200_000, 0, 0.5, np.float64, x_min=-20.0, x_max=20.0)
    for s in range(3):
        sim.step(1)
        o.step(1)
        assert not sim.sort_info()["gathered"]
        g = sim.particles()
        np.testing.assert_array_equal(g["offsets"], o.offsets)
        n = o.n
        np.testing.assert_allclose(g["x"], o.x[:n], rtol=0, atol=1e-12)
        _cmp_v(g, o.vx[:n], o.vy[:n], o.vz[:n], o.offsets)
        _cmp_stats(sim.stats(), o.stats)


@pytest.mark.parametrize("cfl", [1.6, 2.5])
def test_shock_fp64_parity_fused_far_movers(orc, api, monkeypatch, cfl):
    """The fused pass forced at CFL > 1 (TRMCR_SHOCK_FUSED=2): particles moving two
    or more cells in a step go through the far-mover list, ranked by source
    index into their destination's canonical order - still the oracle's stable
    sort, position for position."""
    monkeypatch.setenv("TRMCR_SHOCK_FUSED", "2")
    setup, sim, o = _shock_pair(orc, api, 3.0, 40, 8000, 0, 0.2, np.float64, cfl=cfl)
    assert sim.fused
    for s in range(5):
        sim.step(1)
        o.step(1)
        g = sim.particles()
        np.testing.assert_array_equal(g["offsets"], o.offsets)
        n = o.n
        np.testing.assert_allclose(g["x"], o.x[:n], rtol=0, atol=1e-12)
        _cmp_v(g, o.vx[:n], o.vy[:n], o.vz[:n], o.offsets)
        _cmp_stats(sim.stats(), o.stats)


def test_shock_fp64_parity_dense_edges(orc, api):
    """20000 particles per cell, CFL 4: each step's entering reservoir
    particles span several edge_place rounds (512 per round, ranks chained
    warp by warp) and scatter_sorted looks back over many tiles."""
    setup, sim, o = _shock_pair(orc, api, 3.0, 40, 800_000, 0, 0.2, np.float64, cfl=4.0)
    for s in range(6):
        sim.step(1)
        o.step(1)
        assert not sim.sort_info()["gathered"]
        g = sim.particles()
        np.testing.assert_array_equal(g["offsets"], o.offsets)
        n = o.n
        np.testing.assert_allclose(g["x"], o.x[:n], rtol=0, atol=1e-12)
        _cmp_v(g, o.vx[:n], o.vy[:n], o.vz[:n], o.offsets)
        _cmp_stats(sim.stats(), o.stats)
    print("entered per step (L, R):", o.counts[0] / 6, o.counts[1] / 6)
    assert o.counts[0] / 6 > 2 * 512     # left-edge segment: more than two rounds per step


def test_shock_fp32_mass_accounting_and_sort(api):
    setup = synth.shock_setup(mach=3.0, ncells=2000, n_total=1_000_000)
    x, vx, vy, vz = synth.shock_particles(setup, seed=1, dtype=np.float32)
    inv = setup["ncells"] / (setup["x_max"] - setup["x_min"])
    cell = np.clip(np.floor((x.astype(np.float64) - setup["x_min"]) * inv), 0, 1999)
    order = np.argsort(cell, kind="stable")
    sim = api.Simulation(_dev(vx[order], torch.float32), _dev(vy[order], torch.float32),
                         _dev(vz[order], torch.float32), x=_dev(x[order], torch.float32), shock=setup,
                         model=1, adaptive=True, eps=1.0, dt=setup["dt"], seed=1)
    sim.step(5)
    g = sim.particles()
    off = g["offsets"]
    assert np.all(np.diff(off) >= 0) and off[-1] == len(g["x"])
    c = np.clip(np.floor((g["x"].astype(np.float64) - setup["x_min"]) * inv), 0, 1999).astype(int)
    np.testing.assert_array_equal(c, np.repeat(np.arange(2000), np.diff(off)))
    st = sim.stats()
    assert np.all(st["leaves"] + st["untouched"] + st["thermalised"] == st["n"])
    assert abs(len(g["x"]) / 1_000_000 - 1) < 0.01


def test_shock_fp32_statistical_parity(orc, api):
    """fp32 production shock vs the fp64 oracle: time-averaged rho, u_x, T of
    every cell over 16 seeds (|z| <= 3 for >= 99 %, all <= 5)."""
    setup = synth.shock_setup(mach=3.0, ncells=40, n_total=8000, x_min=-4.0, x_max=4.0)
    G, O = [], []
    for seed in range(1, 17):
        x, vx, vy, vz = synth.shock_particles(setup, seed=seed)
        inv = setup["ncells"] / (setup["x_max"] - setup["x_min"])
        cell = np.clip(np.floor((x - setup["x_min"]) * inv), 0, 39)
        o = np.argsort(cell, kind="stable")
        x, vx, vy, vz = x[o], vx[o], vy[o], vz[o]
        kw = dict(model=1, adaptive=True, m_init=2, m_cap=64, eps=0.3, dt=setup["dt"], seed=seed)
        sim = api.Simulation(_dev(vx, torch.float32), _dev(vy, torch.float32), _dev(vz, torch.float32),
                             x=_dev(x, torch.float32), shock=setup, **kw)
        orc_s = orc.ShockState(orc.Config(**{k: v for k, v in kw.items() if k != "adaptive"}, adaptive=1),
                               setup, x, vx, vy, vz)
        ag, ao = [], []
        for k in range(60):
            sim.step(1)
            orc_s.step(1)
            if k >= 20:
                ag.append(sim.moments()[:, [1, 2, 5]])
                ao.append(orc_s.moments()[:, [1, 2, 5]])
        G.append(np.mean(ag, 0))
        O.append(np.mean(ao, 0))
    z = _zstats(G, O).ravel()
    assert np.mean(z <= 3) >= 0.99 and z.max() <= 5, (np.mean(z <= 3), z.max())


def test_shock_step_host_particles_parity(orc, api):
    """The shock e2e call (trmcr_step_host_particles): host (x, v) in, rebinned on the
    device, one step, per-cell moments out - equals the oracle's step of the same
    state (step counter 0, then 1 on a fresh upload of the same state); a bad
    upload (unsorted) is EINVAL and leaves the context usable."""
    setup, sim, o = _shock_pair(orc, api, 3.0, 40, 8000, 0, 0.2, np.float64)
    x, vx, vy, vz = (np.ascontiguousarray(a[:o.n]) for a in (o.x, o.vx, o.vy, o.vz))
    mstate = None
    for s in range(2):
        out = sim.step_host_particles(x, vx, vy, vz)
        ref = orc.ShockState(o.cfg, setup, x, vx, vy, vz)
        ref.step_count = s
        if mstate is not None:           # RAD's m_max per cell carries over (context state)
            ref.m_state[:] = mstate
        ref.step(1)
        mstate = ref.m_state.copy()
        mo = ref.moments()
        np.testing.assert_array_equal(out[:, 0], mo[:, 0])
        np.testing.assert_allclose(out[:, 1:11], mo[:, 1:11], rtol=1e-11, atol=1e-11)
        g = sim.particles()
        np.testing.assert_array_equal(g["offsets"], ref.offsets)
        _cmp_v(g, ref.vx[:ref.n], ref.vy[:ref.n], ref.vz[:ref.n], ref.offsets)
        _cmp_stats(sim.stats(), ref.stats)
    bad = x[::-1].copy()
    with pytest.raises(api.TrmcrError) as e:
        sim.step_host_particles(bad, vx, vy, vz)
    assert e.value.status == api.EINVAL
    sim.set_particles(vx, vy, vz, x=x)
    assert sim.num_particles() == len(x)
    with pytest.raises(TypeError):
        sim.set_particles(vx.astype(np.float32), vy, vz, x=x)
    with pytest.raises(ValueError):
        sim.set_particles(vx[:-1], vy, vz, x=x)
