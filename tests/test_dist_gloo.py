"""Multi-process (world_size 2, gloo, CPU) tests of the host-side multi-GPU
logic in paper_1009_2768_b200/dist.py: the neighbour exchange protocol of the
shock slabs and the cell sharding + all-reduce of the homogeneous ensembles
(per-cell work done by the CPU oracle here; the CUDA kernels are the same
per-cell computation, checked against the oracle by the -m gpu tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from paper_1009_2768_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(fn, world, *args):
    # a fresh port per attempt; one retry guards against a port grabbed in between
    for attempt in range(2):
        port = _free_port()
        try:
            mp.spawn(_entry, args=(fn, world, port, args), nprocs=world, join=True)
            return
        except mp.ProcessRaisedException as e:
            if attempt == 1 or "address already in use" not in str(e).lower():
                raise


def _entry(rank, fn, world, port, args):
    import datetime
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            timeout=datetime.timedelta(seconds=120))
    try:
        fn(rank, world, *args)
    finally:
        dist.destroy_process_group()


def _exchange_case(rank, world):
    n = 64
    sl = torch.full((n,), 100 * rank + 1, dtype=torch.uint8)
    sr = torch.full((n,), 100 * rank + 2, dtype=torch.uint8)
    rl = torch.zeros(n, dtype=torch.uint8)
    rr = torch.zeros(n, dtype=torch.uint8)
    D.exchange_p2p(sl, sr, rl, rr, rank, world)
    if rank > 0:
        assert torch.all(rl == 100 * (rank - 1) + 2)     # left neighbour's send_right
    else:
        assert torch.all(rl == 0)
    if rank < world - 1:
        assert torch.all(rr == 100 * (rank + 1) + 1)     # right neighbour's send_left
    else:
        assert torch.all(rr == 0)


@pytest.mark.parametrize("world", [2, 3])
def test_neighbour_exchange_protocol(world):
    _run(_exchange_case, world)


def _shard_case(rank, world, outdir):
    from oracle import oracle as O
    O.build()
    vx, vy, vz, off = synth.bimodal_cells(48, 256, seed=4, dtype=np.float64)
    local, base, sl = D.shard_homogeneous(off, rank, world)
    cfg = O.Config(model=O.HARD_SPHERE, m_fixed=16, eps=0.5, dt=0.1, seed=9)
    st = O.HomogeneousState(cfg, vx[sl], vy[sl], vz[sl], local, gcell0=base)
    st.step(2)
    m = st.moments()
    sums = torch.tensor([m[:, 0].sum(), (m[:, 0] * m[:, 2]).sum(), (m[:, 0] * m[:, 6]).sum(),
                         st.stats["proposals"].sum()], dtype=torch.float64)
    dist.all_reduce(sums)
    np.save(os.path.join(outdir, f"vx{rank}.npy"), st.vx)
    if rank == 0:
        np.save(os.path.join(outdir, "sums.npy"), sums.numpy())


def test_cell_sharding_is_partition_independent(orc, tmp_path):
    world = 2
    _run(_shard_case, world, str(tmp_path))
    vx, vy, vz, off = synth.bimodal_cells(48, 256, seed=4, dtype=np.float64)
    cfg = orc.Config(model=orc.HARD_SPHERE, m_fixed=16, eps=0.5, dt=0.1, seed=9)
    st = orc.HomogeneousState(cfg, vx, vy, vz, off)
    st.step(2)
    got = np.concatenate([np.load(tmp_path / f"vx{r}.npy") for r in range(world)])
    np.testing.assert_array_equal(got, st.vx)          # keys are global cell ids
    m = st.moments()
    want = np.array([m[:, 0].sum(), (m[:, 0] * m[:, 2]).sum(), (m[:, 0] * m[:, 6]).sum(),
                     st.stats["proposals"].sum()])
    np.testing.assert_allclose(np.load(tmp_path / "sums.npy"), want, rtol=1e-12)


def test_slab_cuts_balance_particles():
    setup = synth.shock_setup(mach=5.0, ncells=400, n_total=200_000, x_min=-10, x_max=10)
    x, *_ = synth.shock_particles(setup, seed=1)
    inv = setup["ncells"] / (setup["x_max"] - setup["x_min"])
    counts = np.bincount(np.clip(np.floor((x - setup["x_min"]) * inv), 0, 399).astype(int), minlength=400)
    for world in (2, 4, 8):
        cuts = D.slab_cuts(counts, world)
        assert cuts[0][0] == 0 and sum(c[1] for c in cuts) == 400
        load = [counts[a:a + n].sum() for a, n in cuts]
        assert max(load) / (counts.sum() / world) < 1.05     # equal-cell slabs would be ~1.56 at P = 2
        assert all(n >= 4 for _, n in cuts)


def _exact_sums_case(rank, world, out_dir):
    rng = np.random.default_rng(7)
    rows = rng.standard_normal((101, 10)) * 10.0 ** rng.integers(-8, 9, (101, 1))
    lo, hi = D.shard_range(101, rank, world)
    tot = D.global_sums_exact(rows[lo:hi], lo)
    np.save(os.path.join(out_dir, f"sums_{world}_{rank}.npy"), tot)


@pytest.mark.parametrize("world", [1, 2, 3])
def test_global_sums_exact_are_partition_independent(world, tmp_path):
    """All-gather + correctly rounded sums: every rank of every world size gets
    the same bits, equal to math.fsum over all rows."""
    import math
    _run(_exact_sums_case, world, str(tmp_path))
    rng = np.random.default_rng(7)
    rows = rng.standard_normal((101, 10)) * 10.0 ** rng.integers(-8, 9, (101, 1))
    ref = np.array([math.fsum(rows[:, k]) for k in range(10)])
    for r in range(world):
        np.testing.assert_array_equal(np.load(tmp_path / f"sums_{world}_{r}.npy"), ref)
