"""Pins of the CPU oracle's primitives against things other than the oracle itself.

Each test names the paper passage (P:nnn = PAPER.md line) or the external
fact it checks.  No GPU needed.
"""
import math
import os
import shutil
import subprocess

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


def _kat():
    rows = []
    with open(os.path.join(HERE, "golden", "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            w = [int(t, 16) for t in line.split()]
            rows.append((w[:4], w[4:6], w[6:10]))
    return rows


def test_philox_known_answers(orc):
    """Random123 KAT vectors (Salmon et al., SC'11)."""
    for ctr, key, out in _kat():
        assert list(orc.philox(ctr, key)) == out


@pytest.fixture(scope="module")
def curand_host(tmp_path_factory):
    gxx = shutil.which("g++")
    inc = "/usr/local/cuda/include"
    if gxx is None or not os.path.exists(os.path.join(inc, "curand_philox4x32_x.h")):
        pytest.skip("cuRAND headers / g++ unavailable")
    exe = str(tmp_path_factory.mktemp("kat") / "kat")
    subprocess.check_call([gxx, "-O1", "-I", inc, "-o", exe,
                           os.path.join(HERE, "helpers", "curand_philox_host.cpp")])
    return exe


def test_philox_matches_curand(orc, curand_host):
    """Library routine: cuRAND's curand_Philox4x32_10 on 2000 random (ctr, key)."""
    rng = np.random.default_rng(7)
    rows = rng.integers(0, 2**32, size=(2000, 6), dtype=np.uint64)
    inp = "\n".join(" ".join(f"{int(v):08x}" for v in r) for r in rows) + "\n"
    res = subprocess.run([curand_host], input=inp, capture_output=True, text=True, check=True)
    ref = [[int(t, 16) for t in l.split()] for l in res.stdout.strip().splitlines()]
    for r, want in zip(rows, ref):
        assert list(orc.philox(r[:4], r[4:6])) == want


def test_u53_exact_open_interval(orc):
    assert orc.u53(0, 0) == 0.5 * 2.0**-52
    assert orc.u53(0xFFFFFFFF, 0xFFFFFFFF) == 1.0 - 0.5 * 2.0**-52
    assert 0.0 < orc.u53(0x80000000, 0) < 1.0
    # k = hi<<20 | lo>>12: exactly (k + 1/2) 2^-52
    assert orc.u53(1, 0) == (2**20 + 0.5) * 2.0**-52


def test_ir_two_point_law(orc):
    """IR(x) = [x] w.p. [x]+1-x, [x]+1 w.p. x-[x]; SPEC example 2.3."""
    assert orc.ir(3.0, 1e-12) == 3 and orc.ir(3.0, 1 - 1e-12) == 3
    assert orc.ir(2.3, 0.29) == 3 and orc.ir(2.3, 0.31) == 2
    assert orc.ir(0.0, 1e-16) == 0
    us = (np.arange(100_000) + 0.5) / 100_000          # exact quadrature of u in (0,1)
    vals = np.array([orc.ir(2.3, u) for u in us[::10]])
    assert abs(vals.mean() - 2.3) < 1e-3
    assert set(np.unique(vals)) == {2, 3}


def test_feistel_is_bijection(orc):
    rk = [0x12345678, 0x9ABCDEF0, 0x0F1E2D3C, 0x4B5A6978]
    # includes C = 1 (N = 2), perfect squares, A C = N exactly, A C - N = A - 1
    for N in [1, 2, 3, 4, 5, 7, 9, 16, 17, 40, 42, 100, 1000, 1023, 1025, 4097]:
        img = [orc.feistel(x, N, rk) for x in range(N)]
        assert sorted(img) == list(range(N))


def test_feistel_adjacent_images_not_favoured(orc):
    """P(|pi(x) - pi(x+1)| = 1) over 20000 keys equals 2/N for N = 100 and 1000
    (z < 4.5).  A 4-round Feistel fails this (z ~ 70 at N = 100 with 2M keys:
    the two outputs of one collision would be re-paired too often)."""
    rng = np.random.default_rng(11)
    for N in (100, 1000):
        K = 20000
        hit = 0
        for _ in range(K):
            rk = rng.integers(0, 2**32, size=4, dtype=np.uint64)
            hit += abs(orc.feistel(N // 3, N, rk) - orc.feistel(N // 3 + 1, N, rk)) == 1
        p0 = 2 / N
        z = (hit / K - p0) / np.sqrt(p0 * (1 - p0) / K)
        assert abs(z) < 4.5, (N, z)


def test_feistel_pairs_uniform_over_keys(orc):
    """Ordered pair (pi(0), pi(1)) over 9000 keys is uniform on the 90 pairs of
    distinct values of [0, 10) (chi^2, 89 dof): a uniform draw without
    replacement, not just uniform marginals."""
    rng = np.random.default_rng(5)
    hits = np.zeros((10, 10))
    for _ in range(9000):
        rk = rng.integers(0, 2**32, size=4, dtype=np.uint64)
        hits[orc.feistel(0, 10, rk), orc.feistel(1, 10, rk)] += 1
    assert np.trace(hits) == 0
    off = hits[~np.eye(10, dtype=bool)]
    chi2 = ((off - 100) ** 2 / 100).sum()
    assert chi2 < 135.0     # p ~ 0.001 for 89 dof


def test_feistel_uniform_over_keys(orc):
    """Position of element 0 over 4000 keys is uniform on [0, 10) (chi^2, 9 dof)."""
    rng = np.random.default_rng(3)
    hits = np.zeros(10)
    for _ in range(4000):
        rk = rng.integers(0, 2**32, size=4, dtype=np.uint64)
        hits[orc.feistel(0, 10, rk)] += 1
    chi2 = ((hits - 400) ** 2 / 400).sum()
    assert chi2 < 27.9      # p = 0.001


def test_collide_pair_worked_example(orc):
    """(1,0,0),(-1,0,0) with xi1 = 1: theta = 0, sigma = (0,0,1) -> (0,0,+-1) (eq. n3d)."""
    a, b = orc.collide_pair([1, 0, 0], [-1, 0, 0], 1.0, 0.37)
    np.testing.assert_allclose(a, [0, 0, 1], atol=1e-15)
    np.testing.assert_allclose(b, [0, 0, -1], atol=1e-15)
    # identical velocities are unchanged for any xi (|q| = 0)
    a, b = orc.collide_pair([0.3, -1, 2], [0.3, -1, 2], 0.2, 0.9)
    np.testing.assert_array_equal(a, [0.3, -1, 2])
    np.testing.assert_array_equal(b, [0.3, -1, 2])


def test_collide_pair_invariants_and_isotropy(orc):
    """Momentum/energy identity and sigma uniform on S^2 (E s = 0, E ss^T = I/3)."""
    rng = np.random.default_rng(11)
    S = []
    for _ in range(20000):
        vi, vj = rng.normal(size=3) * 2, rng.normal(size=3) * 2
        a, b = orc.collide_pair(vi, vj, rng.random(), rng.random())
        np.testing.assert_allclose(a + b, vi + vj, rtol=0, atol=1e-13)
        e0 = vi @ vi + vj @ vj
        assert abs(a @ a + b @ b - e0) <= 1e-13 * e0
        q = np.linalg.norm(vi - vj)
        S.append((a - (vi + vj) / 2) / (q / 2))
    S = np.array(S)
    assert np.all(np.abs(np.linalg.norm(S, axis=1) - 1) < 1e-12)
    assert np.linalg.norm(S.mean(0)) < 4 / math.sqrt(len(S))
    np.testing.assert_allclose(S.T @ S / len(S), np.eye(3) / 3, atol=0.012)


def test_split_expectations_closed_form(orc):
    """E[N_k] = (1-tau) tau^k n for k <= m, E[N_{m+1}] = tau^{m+1} n (eq. WST, Alg 4.2)."""
    n, m, tau = 10_000, 3, 0.5
    p = 1 - tau
    Ns = np.array([orc.split(p, n, m, seed=s)[0] for s in range(1, 1001)])
    assert np.all(Ns.sum(1) == n)
    want = [(1 - tau) * tau**k * n for k in range(m + 1)] + [tau ** (m + 1) * n]
    mean, se = Ns.mean(0), Ns.std(0) / math.sqrt(len(Ns)) + 1e-9
    assert np.all(np.abs(mean - want) < 4 * se + 1e-9), (mean, want, se)


def test_split_limits(orc):
    """tau = 0 -> N_0 = n (no collisions); tau = 1 -> all thermalised;
    n = 1 -> exactly one set is 1 (SPEC split example)."""
    N, rem, d = orc.split(1.0, 1000, 8)
    assert N[0] == 1000 and rem == 0 and d == 0
    N, rem, d = orc.split(0.0, 1000, 8)
    assert N[:9].sum() == 0 and rem == 1000 and N[9] == 1000
    for s in range(1, 200):
        N, rem, d = orc.split(0.1, 1, 5, seed=s)
        assert N.sum() == 1


def _enum_split_pmf(n, p, m):
    """Exact law of (N_0..N_m, rem) by enumerating both IR branches per level."""
    out = {}

    def rec(k, rem, hist, prob):
        if prob == 0:
            return
        if rem == 0 or k > m:
            key = tuple(hist + [0] * (m + 1 - len(hist)) + [rem])
            out[key] = out.get(key, 0) + prob
            return
        y = p * rem
        fl = math.floor(y)
        for q, pr in ((fl, fl + 1 - y), (fl + 1, y - fl)):
            if pr > 0:
                rec(k + 1, rem - q, hist + [q], prob * pr)

    rec(0, n, [], 1.0)
    return out


def test_split_exact_pmf_small_n(orc):
    """Brute-force enumeration of Alg 4.2's IR branches (n = 4, m = 2) vs 20000 oracle splits."""
    n, m, p = 4, 2, 0.45
    pmf = _enum_split_pmf(n, p, m)
    assert abs(sum(pmf.values()) - 1) < 1e-12
    counts = {}
    T = 20000
    for s in range(T):
        N, rem, d = orc.split(p, n, m, seed=s + 1)
        key = tuple(int(v) for v in N[: m + 1]) + (rem,)
        counts[key] = counts.get(key, 0) + 1
    assert set(counts) <= set(pmf)
    chi2 = sum((counts.get(k, 0) - T * v) ** 2 / (T * v) for k, v in pmf.items())
    dof = len(pmf) - 1
    assert chi2 < dof + 5 * math.sqrt(2 * dof)


def test_maxwellian_exact_moments_and_law(orc):
    """Prescribed momentum/energy exactly; Gaussian law (KS) and isotropy."""
    from scipy import stats
    rng = np.random.default_rng(5)
    n = 20000
    vx, vy, vz = rng.normal(1, 1.3, n), rng.normal(2, 0.7, n), rng.normal(3, 1.0, n)
    slots = np.arange(n)
    P0 = np.array([vx.sum(), vy.sum(), vz.sum()])
    E0 = (vx**2 + vy**2 + vz**2).sum()
    orc.maxwellian(slots, vx, vy, vz, seed=9)
    np.testing.assert_allclose([vx.sum(), vy.sum(), vz.sum()], P0, rtol=1e-12)
    assert abs((vx**2 + vy**2 + vz**2).sum() - E0) <= 1e-12 * E0
    T = ((vx - vx.mean())**2 + (vy - vy.mean())**2 + (vz - vz.mean())**2).mean() / 3
    for v in (vx, vy, vz):
        z = (v - v.mean()) / math.sqrt(T)
        assert stats.kstest(z, "norm").pvalue > 1e-3
    # one particle is kept (cannot match two moments)
    a, b, c = np.array([1.0]), np.array([2.0]), np.array([3.0])
    orc.maxwellian([0], a, b, c)
    assert (a[0], b[0], c[0]) == (1.0, 2.0, 3.0)


def _golden_rh():
    rows = []
    with open(os.path.join(HERE, "golden", "rankine_hugoniot.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            rows.append([float(t) for t in line.split()])
    return rows


def test_rankine_hugoniot_states(orc):
    """Mach 3 and 5 normal shocks."""
    for mach, rho_R, p_R, T_R, u_L in _golden_rh():
        s = orc.rankine_hugoniot(mach)
        assert s[1] == pytest.approx(u_L, rel=1e-14)
        assert s[3] == pytest.approx(rho_R, rel=1e-14)
        assert s[3] * s[5] == pytest.approx(p_R, rel=1e-14)
        assert s[5] == pytest.approx(T_R, rel=1e-14)
        # the three conservation laws themselves
        rL, uL, TL, rR, uR, TR = s
        g = 5.0 / 3.0
        assert rL * uL == pytest.approx(rR * uR, rel=1e-14)
        assert rL * uL**2 + rL * TL == pytest.approx(rR * uR**2 + rR * TR, rel=1e-14)
        EL = rL * TL / (g - 1) + 0.5 * rL * uL**2
        ER = rR * TR / (g - 1) + 0.5 * rR * uR**2
        assert uL * (EL + rL * TL) == pytest.approx(uR * (ER + rR * TR), rel=1e-13)
    with pytest.raises(ValueError):
        orc.rankine_hugoniot(1.0)


def test_tree_lengths_table1(orc):
    """Alg 4.5 lengths of the two trees of Table 1 under eqs.
    (def:1)-(def:3): tests/golden/table1_tree_lengths.txt."""
    from fractions import Fraction
    import pathlib
    rows = [l for l in (pathlib.Path(__file__).parent / "golden" / "table1_tree_lengths.txt").read_text()
            .splitlines() if l.strip() and not l.startswith("#")]
    assert len(rows) == 2
    for row in rows:
        name, path, d1, d2, d3 = [f.strip() for f in row.split("|")]
        path = [int(t) for t in path.split()]
        for definition, want in ((3, d1), (1, d2), (2, d3)):   # oracle codes: 3 = def:1, 1 = def:2, 2 = def:3
            assert orc.tree_length(path, definition) == float(Fraction(want)), (name, definition)
    with pytest.raises(ValueError):
        orc.tree_length([3, 1, 0, 0, 0], 1)                    # j + h + 1 != k
