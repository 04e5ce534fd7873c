"""Checks at BASELINE.json's full sizes, in the launch configuration bench.py
times, on outputs the oracle can compute one by one (cells are independent and
keyed by global cell id) or via properties that hold at any size."""
import os
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _dev(a, dt):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dt)


def test_config3_full_fp64_sampled_cells_match_oracle(orc):
    """Config 3 at full size (16,384 x 1,024) in fp64: 24 sampled cells equal the
    oracle run on those cells alone (decisions and velocities)."""
    from paper_1009_2768_b200 import api
    vx, vy, vz, off = synth.bimodal_cells(16_384, 1024, seed=1, dtype=np.float64)
    kw = dict(model=1, m_fixed=64, eps=0.01, dt=0.1, seed=1)
    sim = api.Simulation(_dev(vx, torch.float64), _dev(vy, torch.float64), _dev(vz, torch.float64),
                         offsets=off, **kw)
    sim.step(2)
    g = sim.particles()
    st = sim.stats()
    rng = np.random.default_rng(0)
    for c in rng.choice(16_384, 24, replace=False):
        a, b = off[c], off[c + 1]
        o = orc.HomogeneousState(orc.Config(**kw), vx[a:b], vy[a:b], vz[a:b], [0, b - a], gcell0=int(c))
        o.step(2)
        for k, want in (("vx", o.vx), ("vy", o.vy), ("vz", o.vz)):
            err = np.abs(g[k][a:b] - want).max()
            assert err <= 1e-12 * (1 + np.abs(want).max()), (c, k, err)
        for f in ("thermalised", "proposals", "m_next"):
            assert st[f][c] == o.stats[f][0]


def test_config3_full_fp32_bench_configuration():
    """Config 3 exactly as bench.py runs it (fp32, thermal warp path): every cell
    is in the fluid regime, count/momentum/energy conserved per cell (1e-6), the
    Maxwellian has the cell's temperature, global sums match the per-cell rows."""
    from paper_1009_2768_b200 import api
    vx, vy, vz, off = synth.bimodal_cells(16_384, 1024, seed=1)
    sim = api.Simulation(_dev(vx, torch.float32), _dev(vy, torch.float32), _dev(vz, torch.float32),
                         offsets=off, model=1, m_fixed=64, eps=0.01, dt=0.1, seed=1)
    m0 = sim.moments()
    sim.step(3)
    m1 = sim.moments()
    st = sim.stats()
    assert np.all(st["thermalised"] == 1024) and np.all(st["proposals"] == 0)
    assert np.all(st["p"] * 1024 < 2.0**-53)
    np.testing.assert_array_equal(m1[:, 0], m0[:, 0])
    scale = np.sqrt(2 * m0[:, 6])
    assert np.all(np.abs(m1[:, 2:5] - m0[:, 2:5]).max(1) <= 1e-6 * scale)
    assert np.all(np.abs(m1[:, 6] - m0[:, 6]) <= 1e-6 * m0[:, 6])
    # isotropic after thermalisation: Pxx = T within sampling error (1024 particles)
    z = (m1[:, 8] - m1[:, 5]) / (m1[:, 5] * np.sqrt(2 / 1024))
    assert abs(z.mean()) < 4 / np.sqrt(len(z)) * 1.5 and np.mean(np.abs(z) < 4.5) > 0.999
    gm = torch.zeros(len(api.GLOBAL_FIELDS), dtype=torch.float64, device="cuda")
    sim.global_moments(gm)
    gm = gm.cpu().numpy()
    assert gm[0] == 16_384 * 1024 and gm[api.GLOBAL_FIELDS.index("maxw")] == 16_384 * 1024
    np.testing.assert_allclose(gm[1], st["px"].sum(), rtol=1e-9, atol=1e-6)
    # the device's deterministic two-level sums against the correctly rounded ones
    from paper_1009_2768_b200 import dist as D
    ex = D.global_sums_exact(D.global_rows(st), 0)
    np.testing.assert_allclose(gm, ex, rtol=1e-12, atol=1e-9)


def test_config2_full_single_cell_rad():
    """Config 2 at full size (10^6 fp32 particles in one cell, RAD, eps = 1): the
    global-memory path; conservation, RAD decisions and the HS majorant hold."""
    from paper_1009_2768_b200 import api
    vx, vy, vz = synth.anisotropic_gaussian(1_000_000, seed=1)
    sim = api.Simulation(_dev(vx, torch.float32), _dev(vy, torch.float32), _dev(vz, torch.float32),
                         offsets=[0, 1_000_000], model=1, adaptive=True, m_init=2, m_cap=4096, eps=1.0,
                         dt=0.05, seed=1)
    m0 = sim.moments()[0]
    sim.step(2)
    m1 = sim.moments()[0]
    st = sim.stats()[0]
    assert st["proposals"] > 0.2 * 1e6 and 0 < st["accepted"] < st["proposals"]
    assert st["leaves"] + st["untouched"] + st["thermalised"] == 1e6
    assert abs(m1[6] - m0[6]) <= 1e-6 * m0[6]
    assert np.abs(m1[2:5] - m0[2:5]).max() <= 1e-6 * np.sqrt(2 * m0[6])
    assert m1[8] < m0[8]                 # Pxx relaxes towards T = 1
    assert st["m_used"] >= 2 and st["m_next"] >= 1


def test_config5_full_shock_two_steps():
    """Config 5 at full size (65,536 cells, 65.5 M fp32 particles, Mach 5,
    eps = 0.01) as bench.py runs it: particle accounting, sorted cells."""
    from paper_1009_2768_b200 import api
    setup = synth.shock_setup(mach=5.0, ncells=65_536, n_total=65_536_000, x_min=-50, x_max=50)
    x, vx, vy, vz = synth.shock_particles(setup, seed=1, dtype=np.float32)
    inv = setup["ncells"] / (setup["x_max"] - setup["x_min"])
    cell = np.clip(np.floor((x.astype(np.float64) - setup["x_min"]) * inv), 0, 65_535)
    o = np.argsort(cell, kind="stable")
    n0 = len(x)
    sim = api.Simulation(_dev(vx[o], torch.float32), _dev(vy[o], torch.float32), _dev(vz[o], torch.float32),
                         x=_dev(x[o], torch.float32), shock=setup, model=1, adaptive=True, m_init=2,
                         m_cap=64, eps=0.01, dt=setup["dt"], seed=1)
    del x, vx, vy, vz
    sim.step(2)
    g = sim.particles()
    off = g["offsets"]
    assert np.all(np.diff(off) >= 0) and off[-1] == len(g["x"])
    assert abs(len(g["x"]) / n0 - 1) < 1e-3
    c = np.clip(np.floor((g["x"].astype(np.float64) - setup["x_min"]) * inv), 0, 65_535).astype(np.int64)
    np.testing.assert_array_equal(c, np.repeat(np.arange(65_536), np.diff(off)))
    st = sim.stats()
    assert np.all(st["leaves"] + st["untouched"] + st["thermalised"] == st["n"])
    assert st["proposals"].sum() > 0


@pytest.mark.slow
def test_c4_shock_profile_statistical_parity_full_size():
    """Config 4 at full size (north star: fp32 shock profiles
    within 3 standard errors over 16 seeds): Mach 3, 2,000 cells x 500, eps 1,
    RAD, 2,000 steps, rho / u_x / T of every cell averaged over the last 1,000
    steps; fp32 GPU against the fp64 oracle run as concurrent processes
    (tools/c4_profile_parity.py; ~90 s on 16 host cores)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    pool = str(max(1, min(15, (os.cpu_count() or 2) - 1)))
    out = os.path.join(root, "gpurun_out", "c4_profile_parity_test.json")
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "c4_profile_parity.py"), "2000", "16", pool, out],
                       cwd=root, capture_output=True, text=True, timeout=3600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
