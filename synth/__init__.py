"""Seeded synthetic initial data for the TRMC-R configurations (BASELINE.json).

This module holds NONE of the method's arithmetic: it only draws initial
particle velocities/positions (step 1 of Alg 4.3/4.4, P:481-482 — "compute
the initial velocity of the particles by sampling them from f_0"), which is
the caller's job.  It uses numpy's own Philox bit generator, independent of
the method's keyed Philox4x32-10 streams.  Both the oracle-based tests and
the CUDA path consume the arrays it returns, so they start from identical
data.  Recipes are documented in DESIGN.md §6.
"""
from __future__ import annotations

import math

import numpy as np


def _rng(seed: int, tag: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[seed & 0xFFFFFFFFFFFFFFFF, tag]))


def two_maxwellians(n: int = 10_000, seed: int = 1, shift: float = 2.0, T: float = 1.0):
    """Config 1: equal mix of M((+shift,0,0),T) and M((-shift,0,0),T).

    Particles 0..n/2-1 come from the + Maxwellian, the rest from the - one."""
    g = _rng(seed, 1)
    v = g.standard_normal((3, n)) * math.sqrt(T)
    h = n // 2
    v[0, :h] += shift
    v[0, h:] -= shift
    return v[0].copy(), v[1].copy(), v[2].copy()


def anisotropic_gaussian(n: int = 1_000_000, seed: int = 1, temps=(2.0, 0.5, 0.5)):
    """Config 2: v_x ~ N(0, Tx), v_y ~ N(0, Ty), v_z ~ N(0, Tz) (T = 1, Pxx0 = 2)."""
    g = _rng(seed, 2)
    v = g.standard_normal((3, n))
    return tuple((v[k] * math.sqrt(temps[k])).copy() for k in range(3))


def maxwellian(n: int, seed: int = 1, u=(0.0, 0.0, 0.0), T: float = 1.0):
    """Equilibrium data M(u, T) for invariance tests."""
    g = _rng(seed, 3)
    v = g.standard_normal((3, n)) * math.sqrt(T)
    return tuple((v[k] + u[k]).copy() for k in range(3))


def bimodal_cells(ncells: int = 16_384, ppc: int = 1024, seed: int = 1, dtype=np.float32):
    """Config 3: per cell two ppc/2-particle Maxwellians, each with its own drift
    ~ U(-1,1)^3 and temperature ~ U(0.5, 2).  Returns (vx, vy, vz, offsets)."""
    g = _rng(seed, 4)
    half = ppc // 2
    drift = g.uniform(-1.0, 1.0, size=(ncells, 2, 3))
    temp = g.uniform(0.5, 2.0, size=(ncells, 2))
    z = g.standard_normal((3, ncells, 2, half))
    v = z * np.sqrt(temp)[None, :, :, None] + np.moveaxis(drift, 2, 0)[:, :, :, None]
    v = v.reshape(3, ncells * ppc)
    offsets = np.arange(ncells + 1, dtype=np.int64) * ppc
    return (v[0].astype(dtype), v[1].astype(dtype), v[2].astype(dtype), offsets)


def uniform_cells(ncells: int, ppc: int, seed: int = 1, T: float = 1.0, dtype=np.float64):
    """Many small homogeneous cells with anisotropic data (tests)."""
    g = _rng(seed, 5)
    v = g.standard_normal((3, ncells * ppc))
    v[0] *= math.sqrt(2.0 * T)
    v[1] *= math.sqrt(0.5 * T)
    v[2] *= math.sqrt(0.5 * T)
    offsets = np.arange(ncells + 1, dtype=np.int64) * ppc
    return v[0].astype(dtype), v[1].astype(dtype), v[2].astype(dtype), offsets


def ragged_cells(ncells: int, max_ppc: int, seed: int = 1, dtype=np.float64, empty_frac=0.1):
    """Cells of random sizes in [0, max_ppc] (some empty, some of size 1)."""
    g = _rng(seed, 6)
    sizes = g.integers(0, max_ppc + 1, size=ncells)
    sizes[g.random(ncells) < empty_frac] = 0
    if ncells > 2:
        sizes[1] = 1
        sizes[2] = 2
    offsets = np.zeros(ncells + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(sizes)
    n = int(offsets[-1])
    v = g.standard_normal((3, n))
    v[0] *= 1.5
    v[0] += g.uniform(-1, 1, size=n) * 0.5
    return v[0].astype(dtype), v[1].astype(dtype), v[2].astype(dtype), offsets


def cold_beams(ncells: int, ppc: int, seed: int = 1, speed: float = 2.0, spread: float = 0.05,
               dtype=np.float64):
    """Counter-streaming cold beams (a two-Maxwellian mix far from equilibrium,
    T_beam = spread^2): per cell, even particles at +speed, odd at -speed along
    x.  Collisions between beam and scattered particles push relative speeds
    above the pre-step bound 2 max|v - u|, so majorant violations
    actually occur.  Offsets: ncells equal cells of ppc particles."""
    g = _rng(seed, 8)
    n = ncells * ppc
    v = g.standard_normal((3, n)) * spread
    v[0] += np.where(np.arange(n) % 2 == 0, speed, -speed)
    offsets = np.arange(ncells + 1, dtype=np.int64) * ppc
    return v[0].astype(dtype), v[1].astype(dtype), v[2].astype(dtype), offsets


def rankine_hugoniot(mach: float, gamma: float = 5.0 / 3.0, rho_L: float = 1.0, T_L: float = 1.0):
    """Upstream/downstream states of a normal shock, p = rho T.

    Returns dict rho_L, u_L, T_L, rho_R, u_R, T_R; the upstream gas enters at
    x_min moving in +x (mirror of P:984's u_xL = -M sqrt(gamma T_L), [R25])."""
    if not mach > 1.0:
        raise ValueError("no shock for Mach <= 1")
    M2 = mach * mach
    u_L = mach * math.sqrt(gamma * T_L)
    rho_R = rho_L * (gamma + 1) * M2 / ((gamma - 1) * M2 + 2)
    p_R = rho_L * T_L * (2 * gamma * M2 - (gamma - 1)) / (gamma + 1)
    return dict(rho_L=rho_L, u_L=u_L, T_L=T_L, rho_R=rho_R, u_R=rho_L * u_L / rho_R, T_R=p_R / rho_R)


def shock_setup(mach: float = 3.0, ncells: int = 2000, n_total: int = 1_000_000,
                x_min: float = -20.0, x_max: float = 20.0, cfl: float = 0.5):
    """Geometry of configs 4/5: states from Rankine-Hugoniot, weight w from the
    total mass over the domain with a step initial condition at x = 0, and
    dt = cfl * dx / (|u_L| + 4 sqrt(T_R)) ([R26])."""
    st = rankine_hugoniot(mach)
    mass = st["rho_L"] * (0.0 - x_min) + st["rho_R"] * (x_max - 0.0)
    w = mass / n_total
    dx = (x_max - x_min) / ncells
    dt = cfl * dx / (abs(st["u_L"]) + 4.0 * math.sqrt(st["T_R"]))
    return dict(ncells=ncells, x_min=x_min, x_max=x_max, weight=w, dt=dt, dx=dx, mach=mach, **st)


def shock_particles(setup: dict, seed: int = 1, dtype=np.float64):
    """Step initial condition: upstream M(rho_L,u_L,T_L) on [x_min,0), downstream
    M(rho_R,u_R,T_R) on [0,x_max); particle counts rho * length / w (rounded),
    positions uniform.  Returned in random (unsorted) order."""
    g = _rng(seed, 7)
    w = setup["weight"]
    nL = int(round(setup["rho_L"] * (0.0 - setup["x_min"]) / w))
    nR = int(round(setup["rho_R"] * (setup["x_max"] - 0.0) / w))
    x = np.concatenate([g.uniform(setup["x_min"], 0.0, nL), g.uniform(0.0, setup["x_max"], nR)])
    z = g.standard_normal((3, nL + nR))
    sL, sR = math.sqrt(setup["T_L"]), math.sqrt(setup["T_R"])
    vx = np.concatenate([setup["u_L"] + sL * z[0, :nL], setup["u_R"] + sR * z[0, nL:]])
    vy = np.concatenate([sL * z[1, :nL], sR * z[1, nL:]])
    vz = np.concatenate([sL * z[2, :nL], sR * z[2, nL:]])
    x = np.clip(x, setup["x_min"], np.nextafter(setup["x_max"], -np.inf))
    return (x.astype(dtype), vx.astype(dtype), vy.astype(dtype), vz.astype(dtype))
