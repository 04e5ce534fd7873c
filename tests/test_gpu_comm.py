"""The multi-GPU surface of the C ABI (include/trmcr.h, comm.cuh) on one GPU:
an NCCL communicator of one rank (nranks = 1 is what a single B200 can host -
NCCL refuses two ranks on one device).  The all-reduced global moments, the
partition-independent global sums (all-gather + exactly rounded sums on the
host) and the all-gathered per-cell moments must equal the local results; a
shock context with a communicator steps bit for bit like one without."""
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


def test_nccl_id(api):
    a, b = api.get_nccl_id(), api.get_nccl_id()
    assert len(a) == 128 and len(b) == 128 and a != b


def test_homogeneous_comm_one_rank(api):
    from paper_1009_2768_b200 import dist
    vx, vy, vz, off = synth.ragged_cells(300, 400, seed=5)
    kw = dict(offsets=off, model=1, adaptive=True, m_init=2, m_cap=64, eps=0.5, dt=0.1, seed=5)
    sim = api.Simulation(_dev(vx), _dev(vy), _dev(vz), nccl_id=api.get_nccl_id(), rank=0, nranks=1, **kw)
    ref = api.Simulation(_dev(vx), _dev(vy), _dev(vz), **kw)
    assert sim.comm_size == 1 and ref.comm_size == 1
    bufs = [torch.zeros(10, dtype=torch.float64, device="cuda") for _ in range(2)]
    rb = torch.zeros(10, dtype=torch.float64, device="cuda")
    for k in range(4):
        sim.step(1)
        ref.step(1)
        sim.global_moments(bufs[k & 1], all_ranks=True)
        ref.global_moments(rb)
    sim.comm_wait()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(bufs[1].cpu().numpy(), rb.cpu().numpy())
    gs = sim.global_sums()
    rows = dist.global_rows(sim.stats())
    np.testing.assert_array_equal(gs, [math.fsum(rows[:, k]) for k in range(rows.shape[1])])
    np.testing.assert_array_equal(ref.global_sums(), gs)
    np.testing.assert_allclose(gs, rb.cpu().numpy(), rtol=1e-12, atol=1e-9)
    np.testing.assert_array_equal(sim.moments(global_cells=len(off) - 1), sim.moments())
    g, r = sim.particles(), ref.particles()
    for f in ("vx", "vy", "vz"):
        np.testing.assert_array_equal(g[f], r[f])


def test_shock_comm_one_rank(api):
    setup = synth.shock_setup(mach=3.0, ncells=40, n_total=8000, x_min=-4.0, x_max=4.0)
    x, vx, vy, vz = synth.shock_particles(setup, seed=2)
    inv = setup["ncells"] / (setup["x_max"] - setup["x_min"])
    o = np.argsort(np.clip(np.floor((x - setup["x_min"]) * inv), 0, 39), kind="stable")
    x, vx, vy, vz = x[o], vx[o], vy[o], vz[o]
    kw = dict(shock=setup, model=1, adaptive=True, m_init=2, m_cap=64, eps=0.2, dt=setup["dt"], seed=2)
    a = api.Simulation(_dev(vx), _dev(vy), _dev(vz), x=_dev(x), nccl_id=api.get_nccl_id(), rank=0, nranks=1, **kw)
    b = api.Simulation(_dev(vx), _dev(vy), _dev(vz), x=_dev(x), **kw)
    a.step(5)
    b.step(5)
    pa, pb = a.particles(), b.particles()
    for f in ("x", "vx", "vy", "vz", "offsets"):
        np.testing.assert_array_equal(pa[f], pb[f])
    np.testing.assert_array_equal(a.moments(global_cells=40), b.moments())


def test_comm_argument_errors(api):
    vx, vy, vz, off = synth.ragged_cells(8, 50, seed=1)
    with pytest.raises(api.TrmcrError) as e:
        api.Simulation(_dev(vx), _dev(vy), _dev(vz), offsets=off, eps=1.0, dt=0.1, rank=1, nranks=1)
    assert e.value.status == api.EINVAL
    with pytest.raises(api.TrmcrError) as e:
        api.Simulation(_dev(vx), _dev(vy), _dev(vz), offsets=off, eps=1.0, dt=0.1, rank=0, nranks=2)
    assert e.value.status == api.EINVAL
    with pytest.raises(ValueError):
        api.Simulation(_dev(vx), _dev(vy), _dev(vz), offsets=off, eps=1.0, dt=0.1, nccl_id=b"x" * 7)
