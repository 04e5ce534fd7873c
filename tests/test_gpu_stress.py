"""Randomised fp64 decision/velocity parity (GPU vs oracle) over many small
configurations: models, RAD on/off, indicators, truncation orders, eps over
three decades, ragged / empty / singleton cells.  Exercises both the
shared-memory and the global-memory (overflow) paths."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.mark.parametrize("seed,warp_path", [(1, "1"), (2, "1"), (3, "1"), (4, "0")])
def test_random_configs(orc, seed, warp_path, monkeypatch):
    """warp_path "0" routes the general cells through the CTA kernel instead of
    the warp-per-cell kernel (TRMCR_WARP_PATH, read at init)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    monkeypatch.setenv("TRMCR_WARP_PATH", warp_path)
    from paper_1009_2768_b200 import api
    rng = np.random.default_rng(seed)
    for it in range(20):
        ncell = int(rng.integers(1, 20))
        maxp = int(rng.choice([64, 300, 700, 1500, 2500]))
        v = synth.ragged_cells(ncell, maxp, seed=int(rng.integers(1, 10**6)))
        kw = dict(model=int(rng.integers(0, 2)), adaptive=int(rng.integers(0, 2)),
                  m_fixed=int(rng.choice([1, 2, 4, 16, 64])), m_init=int(rng.choice([1, 2, 4])),
                  m_cap=int(rng.choice([4, 16, 64])), eps=float(10 ** rng.uniform(-2.5, 0.5)),
                  dt=float(rng.choice([0.05, 0.1, 0.3])), seed=int(rng.integers(1, 1000)),
                  indicator=int(rng.integers(0, 2)))
        o = orc.HomogeneousState(orc.Config(**kw), v[0], v[1], v[2], v[3])
        d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda").contiguous()
        sim = api.Simulation(d(v[0]), d(v[1]), d(v[2]), offsets=v[3], **kw)
        for s in range(3):
            o.step(1)
            sim.step(1)
            st = sim.stats()
            for f in ("proposals", "accepted", "leaves", "thermalised", "m_next", "attempts"):
                np.testing.assert_array_equal(st[f], o.stats[f], err_msg=f"{it} {kw} step {s} {f}")
        g = sim.particles()
        for a, b in ((g["vx"], o.vx), (g["vy"], o.vy), (g["vz"], o.vz)):
            scale = 1.0 + np.abs(b)
            assert np.all(np.abs(a - b) <= 1e-12 * scale * 10), (it, kw)
