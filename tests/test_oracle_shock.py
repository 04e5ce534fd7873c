"""Pins of the oracle's shock pieces (A1 transport + reservoirs, A2 stable sort).

The interior shock profile has no closed form (the paper's figures are
absent): PARITY UNPINNED there; we pin the plateaus (Rankine-Hugoniot,
P:975-985), the boundary inflow (one-sided Maxwellian flux) and the sort."""
import math

import numpy as np
import pytest

import synth


def _state(orc, setup, x, vx, vy, vz, **cfg):
    c = orc.Config(model=1, adaptive=cfg.pop("adaptive", 1), m_init=2, m_cap=64,
                   eps=cfg.pop("eps", 1.0), dt=setup["dt"], seed=cfg.pop("seed", 1), **cfg)
    return orc.ShockState(c, setup, x, vx, vy, vz)


def test_stable_bin_brute_force(orc):
    """A2: cell = floor((x - x_min)/dx) clamped; stable order (Python's sort is stable)."""
    setup = synth.shock_setup(mach=3.0, ncells=37, n_total=3000)
    x, vx, vy, vz = synth.shock_particles(setup, seed=2)
    st = _state(orc, setup, x, vx, vy, vz)
    inv = setup["ncells"] / (setup["x_max"] - setup["x_min"])
    cell = np.clip(np.floor((x - setup["x_min"]) * inv), 0, setup["ncells"] - 1).astype(int)
    order = sorted(range(len(x)), key=lambda i: cell[i])
    np.testing.assert_array_equal(st.x[: len(x)], x[order])
    np.testing.assert_array_equal(st.vy[: len(x)], vy[order])
    np.testing.assert_array_equal(np.diff(st.offsets), np.bincount(cell, minlength=setup["ncells"]))


def test_transport_sort_is_stable_in_source_order(orc):
    """After one step with no collisions (tau -> 0), particles appear grouped by
    destination cell, in (source cell, source position) order (canonical A2)."""
    setup = synth.shock_setup(mach=3.0, ncells=20, n_total=2000)
    x, vx, vy, vz = synth.shock_particles(setup, seed=3)
    st = _state(orc, setup, x, vx, vy, vz, adaptive=0, eps=1e30)
    x0, vx0 = st.x[: st.n].copy(), st.vx[: st.n].copy()
    n0 = st.n
    st.step(1)
    xn = x0 + vx0 * setup["dt"]
    keep = (xn >= setup["x_min"]) & (xn < setup["x_max"])
    inv = setup["ncells"] / (setup["x_max"] - setup["x_min"])
    cell = np.clip(np.floor((xn - setup["x_min"]) * inv), 0, setup["ncells"] - 1).astype(int)
    inj_L, inj_R = int(st.counts[0]), int(st.counts[1])
    assert st.n == n0 - int(st.counts[2]) + inj_L + inj_R
    interior = st.x[: st.n]
    # remove injected particles (they have positions within dt*|v| of the ends), compare the rest
    idx = [i for i in range(n0) if keep[i]]
    order = sorted(idx, key=lambda i: cell[i])
    got = [v for v in interior if v in set(xn[idx])]
    np.testing.assert_array_equal(np.array(got), xn[order])


def _flux(rho, u, T, inward_sign):
    """One-sided Maxwellian number flux across a wall, per unit area and time."""
    s = inward_sign * u / math.sqrt(2 * T)
    return rho * (math.sqrt(T / (2 * math.pi)) * math.exp(-s * s) + inward_sign * u * (1 + math.erf(s)) / 2)


def test_reservoir_inflow_matches_one_sided_flux(orc):
    """A1 ghost-slab reservoirs: injected count per step = flux * dt / w (textbook)."""
    setup = synth.shock_setup(mach=3.0, ncells=10, n_total=4000)
    setup = dict(setup)
    setup["dt"] = 0.02
    x, vx, vy, vz = synth.shock_particles(setup, seed=4)
    st = _state(orc, setup, x, vx, vy, vz, adaptive=0, eps=1e30)
    inj = []
    for _ in range(300):
        st.step(1)
        inj.append(st.counts[:2].copy())
    inj = np.array(inj)
    w, dt = setup["weight"], setup["dt"]
    want_L = _flux(setup["rho_L"], setup["u_L"], setup["T_L"], +1) * dt / w
    want_R = _flux(setup["rho_R"], setup["u_R"], setup["T_R"], -1) * dt / w
    for k, want in ((0, want_L), (1, want_R)):
        se = inj[:, k].std() / math.sqrt(len(inj))
        assert abs(inj[:, k].mean() - want) < 4 * se + 0.02 * want


def test_shock_plateaus_rankine_hugoniot(orc):
    """Mach-3 shock, eps = 0.1: far upstream/downstream cells keep the RH states."""
    setup = synth.shock_setup(mach=3.0, ncells=80, n_total=24_000, x_min=-8, x_max=8)
    x, vx, vy, vz = synth.shock_particles(setup, seed=5)
    st = _state(orc, setup, x, vx, vy, vz, eps=0.1)
    acc = []
    for k in range(150):
        st.step(1)
        if k >= 50:
            acc.append(st.moments())
    m = np.mean(acc, 0)
    up, down = m[2:10], m[-10:-2]
    assert up[:, 1].mean() == pytest.approx(setup["rho_L"], rel=0.05)
    assert up[:, 2].mean() == pytest.approx(setup["u_L"], rel=0.03)
    assert up[:, 5].mean() == pytest.approx(setup["T_L"], rel=0.06)
    assert down[:, 1].mean() == pytest.approx(setup["rho_R"], rel=0.06)
    assert down[:, 2].mean() == pytest.approx(setup["u_R"], rel=0.06)
    assert down[:, 5].mean() == pytest.approx(setup["T_R"], rel=0.06)
    # conservation in each cell's collision step is exact; the temperature rises monotonically
    # on average through the shock
    T = m[:, 5]
    assert T[-10:].mean() > T[35:45].mean() > T[:10].mean()
