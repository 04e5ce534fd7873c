"""Host-side multi-GPU logic (one process per GPU, torch.distributed).

* Homogeneous ensembles shard by contiguous global cell ranges; the RNG is
  keyed by global cell id so per-cell results do not depend on the number of
  GPUs.  The only collective is the all-reduce of the global sums (per step,
  asynchronous); `global_sums_exact` gives sums that are bitwise the same for
  any number of GPUs (report steps).
* The 1D shock is split into slabs of contiguous cells balanced by particle
  count; each step every slab sends the particles that moved into a
  neighbouring slab to rank +- 1 (fixed-capacity buffers with a count header,
  one message per direction, no size round trip) between
  trmcr_shock_begin and trmcr_shock_finish.
* On GPUs the collectives run inside the library on its own NCCL communicator
  (comm.cuh; `library_comm` only broadcasts the unique id); the
  torch.distributed exchange below (`exchange_p2p`) is the same protocol for
  gloo (CPU tensors, tests) and for callers that manage the buffers.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np


def shard_range(n: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous near-equal partition of [0, n)."""
    return rank * n // world, (rank + 1) * n // world


GLOBAL_FIELDS = ["n", "px", "py", "pz", "energy", "nPxx", "proposals", "accepted", "maxw", "cost"]


def global_rows(stats: np.ndarray) -> np.ndarray:
    """Per-cell rows of GLOBAL_FIELDS from a statistics table (Simulation.stats()):
    the quantities trmcr_global_moments sums (cost = proposals + maxw / 2)."""
    return np.stack([stats["n"], stats["px"], stats["py"], stats["pz"], stats["energy"],
                     stats["n"] * stats["S0"], stats["proposals"], stats["accepted"], stats["maxw"],
                     stats["proposals"] + 0.5 * stats["maxw"]], axis=1) if len(stats) else np.zeros((0, 10))


def global_sums_exact(rows: np.ndarray, first_cell: int, group=None) -> np.ndarray:
    """Global sums that do not depend on the partition: every rank
    contributes its per-cell rows (host float64 [local cells x k], global cells
    first_cell...) to an all-gather, and every rank adds all rows with
    math.fsum - the correctly rounded sum, independent of order, so the result is
    bitwise identical for any number of GPUs.  Report steps only: the per-step
    path uses the asynchronous all-reduce of trmcr_global_moments."""
    import math
    import torch.distributed as dist
    rows = np.ascontiguousarray(rows, dtype=np.float64)
    if dist.is_available() and dist.is_initialized():
        parts = [None] * dist.get_world_size(group)
        dist.all_gather_object(parts, (int(first_cell), rows), group=group)
    else:
        parts = [(int(first_cell), rows)]
    parts.sort(key=lambda p: p[0])
    allr = np.concatenate([p[1] for p in parts], axis=0) if parts else np.zeros((0, rows.shape[1]))
    return np.array([math.fsum(allr[:, k]) for k in range(allr.shape[1])])


def shard_homogeneous(offsets: np.ndarray, rank: int, world: int):
    """Local offsets (starting at 0), global id of the first local cell and the
    particle slice of this rank."""
    offsets = np.asarray(offsets, dtype=np.int64)
    lo, hi = shard_range(len(offsets) - 1, rank, world)
    local = offsets[lo:hi + 1] - offsets[lo]
    return local, lo, slice(int(offsets[lo]), int(offsets[hi]))


def slab_cuts(counts: Sequence[int], world: int, min_cells: int = 4) -> List[Tuple[int, int]]:
    """(first cell, number of cells) per rank: contiguous slabs with about
    n / world particles each (the shock's density jump makes equal-cell slabs
    unbalanced), at least `min_cells` cells each."""
    counts = np.asarray(counts, dtype=np.int64)
    C = len(counts)
    if world * min_cells > C:
        raise ValueError("too many ranks for the grid")
    cum = np.concatenate([[0], np.cumsum(counts)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        target = total * r / world
        c = int(np.searchsorted(cum, target))
        c = max(c, cuts[-1] + min_cells)
        c = min(c, C - (world - r) * min_cells)
        cuts.append(c)
    cuts.append(C)
    return [(cuts[r], cuts[r + 1] - cuts[r]) for r in range(world)]


def library_comm(api, group=None):
    """(nccl_id, rank, nranks) for Simulation(...): rank 0 draws the NCCL unique id
    in the library (trmcr_get_nccl_id) and torch.distributed broadcasts its 128
    bytes - process-group plumbing only; the collectives themselves run inside
    the library on its own NCCL communicator."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(api.get_nccl_id()), dtype=torch.uint8))
    dist.broadcast(buf, src=0, group=group)
    return bytes(buf.cpu().numpy().tobytes()), rank, world


def exchange_p2p(send_left, send_right, recv_left, recv_right, rank: int, world: int, group=None):
    """Send send_left to rank-1 (its recv_right) and send_right to rank+1 (its
    recv_left); receive symmetrically.  Buffers are torch tensors (CUDA over
    NCCL, CPU over gloo); missing neighbours are skipped."""
    import torch.distributed as dist
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, send_left, rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, recv_left, rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, send_right, rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, recv_right, rank + 1, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def slab_particles(x, vx, vy, vz, setup: dict, first: int, ncells: int):
    """The (cell-sorted) particles of global cells [first, first + ncells)."""
    inv = setup["ncells"] / (setup["x_max"] - setup["x_min"])
    cell = np.clip(np.floor((np.asarray(x, dtype=np.float64) - setup["x_min"]) * inv), 0,
                   setup["ncells"] - 1).astype(np.int64)
    lo = np.searchsorted(cell, first, side="left")
    hi = np.searchsorted(cell, first + ncells, side="left")
    return x[lo:hi], vx[lo:hi], vy[lo:hi], vz[lo:hi]


class ShockSlab:
    """One rank's slab of the 1D shock: a Simulation over global cells
    [first, first + ncells) plus its exchange buffers."""

    def __init__(self, api, setup: dict, first: int, ncells: int, vx, vy, vz, *, x, device,
                 exchange_capacity: int = 1 << 13, comm=None, **kw):
        # capacity: particles crossing one slab edge in one step (a few hundred at
        # CFL 0.5 on C5; the whole buffer travels, so it is kept small: 8192 x 20 B)
        # comm = (nccl_id, rank, nranks) from library_comm(): the library exchanges
        # with the neighbours itself (NCCL send/recv inside trmcr_step); else the
        # caller's exchange function moves this object's buffers.
        import torch
        self.first, self.ncells = first, ncells
        C = setup["ncells"]
        neighbors = (1 if first > 0 else 0) | (2 if first + ncells < C else 0)
        sh = dict(setup)
        sh.update(local_cells=ncells, neighbors=neighbors)
        self.neighbors = neighbors
        self.library_comm = comm is not None
        if comm is not None:
            nid, rank, nranks = comm
            self.sim = api.Simulation(vx, vy, vz, x=x, shock=sh, cell_base=first, nccl_id=nid, rank=rank,
                                      nranks=nranks, **kw)
            return
        self.sim = api.Simulation(vx, vy, vz, x=x, shock=sh, cell_base=first, **kw)
        nb = self.sim.exchange_bytes(exchange_capacity)
        mk = lambda: torch.zeros(nb, dtype=torch.uint8, device=device)
        self.send_l, self.send_r, self.recv_l, self.recv_r = mk(), mk(), mk(), mk()
        self.sim.set_exchange(self.send_l if neighbors & 1 else None, self.send_r if neighbors & 2 else None,
                              self.recv_l if neighbors & 1 else None, self.recv_r if neighbors & 2 else None,
                              exchange_capacity)
        self.neighbors = neighbors

    def step(self, exchange: Optional[Callable[["ShockSlab"], None]] = None):
        """begin (transport, pack) -> exchange(self) -> finish (gather, collide); with
        the library's communicator one trmcr_step does all three."""
        if self.neighbors == 0 or self.library_comm:
            self.sim.step(1)
            return
        self.sim.shock_begin()
        exchange(self)
        self.sim.shock_finish()


def host_exchange(slabs: List[ShockSlab]):
    """In-process exchange between slabs of one GPU (tests): copy each send
    buffer into its neighbour's receive buffer (device copies on the current
    stream; no kernel waits on another)."""
    for a, b in zip(slabs[:-1], slabs[1:]):
        b.recv_l.copy_(a.send_r)
        a.recv_r.copy_(b.send_l)
