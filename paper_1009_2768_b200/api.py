"""Thin Python binding of the C ABI in include/trmcr.h (argument marshalling only).

Every step of the TRMC-R path runs in the CUDA kernels of libtrmcr.so; this
module only converts arguments (torch CUDA tensors, numpy arrays) to pointers
and back.  There is no CPU fallback: a missing library raises at import.
PyTorch supplies device memory and the stream (P:nnn references: PAPER.md).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TRMCR_LIB") or os.path.join(HERE, "libtrmcr.so")   # override: experiments

OK, EINVAL, ENOMEM, ECUDA, ENCCL, ECAPACITY, ESTATE = range(7)
MAXWELL, HARD_SPHERE, VHS = 0, 1, 2
F32, F64 = 0, 1
HOMOGENEOUS, SHOCK_1D = 0, 1
IND_PXX, IND_M4 = 0, 1

STAT_FIELDS = ["n", "p", "mu", "sigma", "S0", "S_est", "E1", "m_used", "m_next", "depth",
               "attempts", "leaves", "untouched", "thermalised", "proposals", "accepted",
               "violations", "maxw", "px", "py", "pz", "energy"]
GLOBAL_FIELDS = ["n", "px", "py", "pz", "energy", "nPxx", "proposals", "accepted", "maxw", "cost"]
MOMENT_FIELDS = ["n", "rho", "ux", "uy", "uz", "T", "E", "p", "Pxx", "M4", "M4c", "m_max"]
KERNELS = ["cell_step_smem", "cell_step_gmem", "moments_kernel", "shock_prologue", "ghost_gen",
           "transport_kernel", "scan_offsets", "shock_collide_smem", "shock_collide_gmem",
           "thermal_warp_kernel", "cell_step_warp", "shock_collide_warp", "scatter_sorted",
           "literal_step_kernel"]
STATS_DTYPE = np.dtype([(f, "<f8") for f in STAT_FIELDS])
COLL_DTYPE = np.dtype([("cell", "<i4"), ("attempt", "<i4"), ("level", "<i4"), ("accepted", "<i4"),
                       ("j", "<i8"), ("slot_i", "<i8"), ("slot_k", "<i8")])


class TrmcrError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"trmcr status {status}: {msg}")
        self.status = status


class _Particles(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("host", C.c_int32), ("n", C.c_int64), ("capacity", C.c_int64),
                ("vx", C.c_void_p), ("vy", C.c_void_p), ("vz", C.c_void_p), ("x", C.c_void_p)]


class _Cells(C.Structure):
    _fields_ = [("geometry", C.c_int32), ("n_cells", C.c_int32), ("cell_base", C.c_int32),
                ("pad", C.c_int32), ("offsets", C.POINTER(C.c_int64)),
                ("x_min", C.c_double), ("x_max", C.c_double), ("weight", C.c_double),
                ("rho_L", C.c_double), ("u_L", C.c_double), ("T_L", C.c_double),
                ("rho_R", C.c_double), ("u_R", C.c_double), ("T_R", C.c_double),
                ("n_cells_global", C.c_int32), ("neighbors", C.c_int32)]


class _Kernel(C.Structure):
    _fields_ = [("model", C.c_int32), ("adaptive", C.c_int32), ("m_fixed", C.c_int32),
                ("m_init", C.c_int32), ("m_cap", C.c_int32), ("indicator", C.c_int32),
                ("delta1", C.c_double), ("delta2", C.c_double), ("seed", C.c_uint64), ("alpha", C.c_double),
                ("wb", C.c_int32), ("wb_max", C.c_int32), ("sigma_update", C.c_int32),
                ("literal", C.c_int32)]


_lib = None


def lib():
    """Load libtrmcr.so (built by __graft_entry__.build() / build.py).  Fails loudly."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1009_2768_b200.build` "
                              "(no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        vp, P = C.c_void_p, C.POINTER
        L.trmcr_init.argtypes = [P(vp), P(_Particles), P(_Cells), C.c_double, C.c_double, P(_Kernel), vp, vp,
                                 C.c_int32, C.c_int32]
        L.trmcr_step.argtypes = [vp, C.c_int32]
        L.trmcr_moments.argtypes = [vp, P(C.c_double), C.c_int32]
        L.trmcr_get_nccl_id.argtypes = [vp]
        L.trmcr_get_nccl_id.restype = C.c_int
        L.trmcr_comm_size.argtypes = [vp]
        L.trmcr_comm_size.restype = C.c_int32
        L.trmcr_comm_wait.argtypes = [vp]
        L.trmcr_comm_wait.restype = C.c_int
        L.trmcr_global_sums.argtypes = [vp, P(C.c_double)]
        L.trmcr_global_sums.restype = C.c_int
        L.trmcr_stats.argtypes = [vp, P(C.c_double)]
        L.trmcr_num_particles.argtypes = [vp, P(C.c_int64)]
        L.trmcr_copy_particles.argtypes = [vp, vp, vp, vp, vp, vp, C.c_int32]
        L.trmcr_set_velocities.argtypes = [vp, vp, vp, vp, C.c_int32]
        L.trmcr_step_host.argtypes = [vp, vp, vp, vp, P(C.c_double)]
        L.trmcr_set_particles.argtypes = [vp, vp, vp, vp, vp, C.c_int64, C.c_int32]
        L.trmcr_step_host_particles.argtypes = [vp, vp, vp, vp, vp, C.c_int64, P(C.c_double)]
        L.trmcr_set_log.argtypes = [vp, C.c_int64]
        L.trmcr_get_log.argtypes = [vp, vp, P(C.c_int64)]
        L.trmcr_shock_sort_info.argtypes = [C.c_void_p, C.c_void_p]
        L.trmcr_shock_sort_info.restype = C.c_int
        L.trmcr_exchange_bytes.argtypes = [C.c_int32, C.c_int64]
        L.trmcr_exchange_bytes.restype = C.c_int64
        L.trmcr_shock_fused.argtypes = [vp]
        L.trmcr_shock_fused.restype = C.c_int32
        L.trmcr_shock_set_exchange.argtypes = [vp, vp, vp, vp, vp, C.c_int64]
        L.trmcr_shock_set_exchange.restype = C.c_int
        L.trmcr_shock_begin.argtypes = [vp]
        L.trmcr_shock_begin.restype = C.c_int
        L.trmcr_shock_finish.argtypes = [vp]
        L.trmcr_shock_finish.restype = C.c_int
        L.trmcr_global_moments.argtypes = [vp, vp, C.c_int32]
        L.trmcr_global_moments.restype = C.c_int
        L.trmcr_set_profiling_mask.argtypes = [vp, C.c_uint32]
        L.trmcr_set_profiling_mask.restype = C.c_int
        L.trmcr_set_profiling.argtypes = [vp, C.c_int32]
        L.trmcr_set_profiling.restype = C.c_int
        L.trmcr_kernel_times.argtypes = [vp, P(C.c_double), P(C.c_int64)]
        L.trmcr_kernel_times.restype = C.c_int
        L.trmcr_launch_count.argtypes = [vp]
        L.trmcr_launch_count.restype = C.c_int64
        L.trmcr_last_error.argtypes = [vp]
        L.trmcr_last_error.restype = C.c_char_p
        L.trmcr_version.restype = C.c_char_p
        L.trmcr_destroy.argtypes = [vp]
        for f in ("trmcr_init", "trmcr_step", "trmcr_moments", "trmcr_stats", "trmcr_num_particles",
                  "trmcr_copy_particles", "trmcr_set_velocities", "trmcr_step_host", "trmcr_set_log",
                  "trmcr_get_log", "trmcr_set_particles", "trmcr_step_host_particles"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _ptr(a):
    """(pointer, is_host, dtype) of a torch tensor or numpy array (contiguous)."""
    try:
        import torch
        if isinstance(a, torch.Tensor):
            assert a.is_contiguous(), "tensor must be contiguous"
            return a.data_ptr(), (0 if a.is_cuda else 1), {torch.float32: F32, torch.float64: F64}.get(a.dtype)
    except ImportError:  # pragma: no cover
        pass
    assert isinstance(a, np.ndarray) and a.flags.c_contiguous, "numpy array must be contiguous"
    return a.ctypes.data, 1, {np.dtype(np.float32): F32, np.dtype(np.float64): F64}.get(a.dtype)


def _arrays(arrays, dtype_code=None, n=None, host=None):
    """Pointers of same-kind arrays: one dtype (= dtype_code if given), all host or
    all device, one length (= n if given).  Raises instead of letting the library
    read past a short array or misread its bytes."""
    ptrs, kinds, codes, lens = [], set(), set(), set()
    for a in arrays:
        p, h, code = _ptr(a)
        ptrs.append(p)
        kinds.add(h)
        codes.add(code)
        lens.add(int(a.shape[0]))
    if len(codes) != 1 or None in codes:
        raise TypeError("particle arrays must share one dtype (float32 or float64)")
    if dtype_code is not None and codes != {dtype_code}:
        raise TypeError("particle arrays must have the context's dtype")
    if len(kinds) != 1:
        raise TypeError("particle arrays must be all host or all device memory")
    if host is not None and kinds != {host}:
        raise TypeError("host arrays required" if host else "device arrays required")
    if len(lens) != 1:
        raise ValueError("particle arrays must have one length")
    if n is not None and lens != {n}:
        raise ValueError(f"particle arrays must have length {n}")
    return ptrs, kinds.pop(), codes.pop(), lens.pop()


class Simulation:
    """A TRMC-R simulation on the current CUDA device (one context per device/stream).

    Homogeneous: pass `offsets` (cells of independent gases, rho = 1).
    Shock: pass `shock` = dict(ncells, x_min, x_max, weight, rho_L, u_L, T_L,
    rho_R, u_R, T_R) and positions `x` sorted by cell.
    """

    def __init__(self, vx, vy, vz, *, eps: float, dt: float, offsets=None, shock: Optional[dict] = None,
                 x=None, model: int = HARD_SPHERE, adaptive: bool = False, m_fixed: int = 64,
                 m_init: int = 2, m_cap: int = 4096, delta1: float = 0.005, delta2: float = 0.01,
                 indicator: int = IND_PXX, seed: int = 1, cell_base: int = 0, capacity: int = 0,
                 stream=None, alpha: float = 1.0, wb: int = 0, wb_max: int = 0, sigma_update: bool = False,
                 literal: bool = False, nccl_id: Optional[bytes] = None, rank: int = 0, nranks: int = 1):
        L = lib()
        self._keep = [vx, vy, vz, x]
        (pvx, pvy, pvz, *rest), host, dt_code, n = _arrays([vx, vy, vz] + ([x] if x is not None else []))
        self.dtype = dt_code
        self.host_init = host
        px = rest[0] if x is not None else None
        part = _Particles(dt_code, host, n, int(capacity), pvx, pvy, pvz, px)
        if shock is None:
            off = np.ascontiguousarray(offsets, dtype=np.int64)
            self._off = off
            self.ncells = len(off) - 1
            cells = _Cells(HOMOGENEOUS, self.ncells, cell_base, 0,
                           off.ctypes.data_as(C.POINTER(C.c_int64)), 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0)
            self.geometry = HOMOGENEOUS
        else:
            self.ncells = int(shock.get("local_cells", shock["ncells"]))
            self.neighbors = int(shock.get("neighbors", 0))
            cells = _Cells(SHOCK_1D, self.ncells, cell_base, 0, None, shock["x_min"], shock["x_max"],
                           shock["weight"], shock["rho_L"], shock["u_L"], shock["T_L"],
                           shock["rho_R"], shock["u_R"], shock["T_R"], int(shock["ncells"]),
                           self.neighbors)
            self.geometry = SHOCK_1D
        kern = _Kernel(model, int(bool(adaptive)), m_fixed, m_init, m_cap, indicator, delta1, delta2,
                       seed & 0xFFFFFFFFFFFFFFFF, float(alpha), int(wb), int(wb_max), int(bool(sigma_update)),
                       int(bool(literal)))
        if stream is None:
            try:
                import torch
                stream = torch.cuda.current_stream().cuda_stream if torch.cuda.is_available() else 0
            except ImportError:  # pragma: no cover
                stream = 0
        self.stream = stream
        h = C.c_void_p()
        idbuf = None
        if nccl_id is not None:
            if len(nccl_id) != 128:
                raise ValueError("nccl_id must be the 128 bytes of get_nccl_id()")
            idbuf = C.create_string_buffer(bytes(nccl_id), 128)
        st = L.trmcr_init(C.byref(h), C.byref(part), C.byref(cells), float(eps), float(dt),
                          C.byref(kern), C.c_void_p(stream), idbuf, int(rank), int(nranks))
        if st != OK:
            raise TrmcrError(st, L.trmcr_last_error(None).decode())
        self._h = h
        self.n_init = n

    # ------------------------------------------------------------------ helpers
    def _check(self, st):
        if st != OK:
            raise TrmcrError(st, lib().trmcr_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            lib().trmcr_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ ABI
    def step(self, n: int = 1):
        self._check(lib().trmcr_step(self._h, int(n)))
        return self

    def moments(self, global_cells: Optional[int] = None) -> np.ndarray:
        """Per-cell moments of this context's cells, or (global_cells = the grid's
        cell count) of every rank's cells in global order (collective)."""
        rows = self.ncells if global_cells is None else int(global_cells)
        out = np.zeros((rows, len(MOMENT_FIELDS)))
        self._check(lib().trmcr_moments(self._h, out.ctypes.data_as(C.POINTER(C.c_double)),
                                        int(global_cells is not None)))
        return out

    @property
    def comm_size(self) -> int:
        return int(lib().trmcr_comm_size(self._h))

    def global_sums(self) -> np.ndarray:
        """Partition-independent global sums (GLOBAL_FIELDS) over every rank (collective)."""
        out = np.zeros(len(GLOBAL_FIELDS))
        self._check(lib().trmcr_global_sums(self._h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def comm_wait(self):
        """Order the context stream after every global all-reduce in flight."""
        self._check(lib().trmcr_comm_wait(self._h))

    def stats(self) -> np.ndarray:
        out = np.zeros(self.ncells, dtype=STATS_DTYPE)
        self._check(lib().trmcr_stats(self._h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def num_particles(self) -> int:
        n = C.c_int64()
        self._check(lib().trmcr_num_particles(self._h, C.byref(n)))
        return n.value

    def particles(self) -> dict:
        n = self.num_particles()
        dt = np.float64 if self.dtype == F64 else np.float32
        vx, vy, vz, x = (np.zeros(max(n, 1), dtype=dt) for _ in range(4))
        off = np.zeros(self.ncells + 1, dtype=np.int64)
        self._check(lib().trmcr_copy_particles(self._h, vx.ctypes.data, vy.ctypes.data, vz.ctypes.data,
                                               x.ctypes.data, off.ctypes.data, 1))
        out = dict(vx=vx[:n], vy=vy[:n], vz=vz[:n], offsets=off)
        if self.geometry == SHOCK_1D:
            out["x"] = x[:n]
        return out

    def _moments_out(self, out):
        if out is None:
            out = np.zeros((self.ncells, len(MOMENT_FIELDS)))
        if out.dtype != np.float64 or out.size < self.ncells * len(MOMENT_FIELDS) or not out.flags.c_contiguous:
            raise ValueError("out must be a contiguous float64 array of ncells x 12")
        return out

    def set_velocities(self, vx, vy, vz):
        (p, q, r), host, _, _ = _arrays([vx, vy, vz], self.dtype, self.num_particles())
        self._check(lib().trmcr_set_velocities(self._h, p, q, r, host))

    def step_host(self, vx, vy, vz, out: Optional[np.ndarray] = None) -> np.ndarray:
        """e2e path (homogeneous): host velocities in, one step, host per-cell moments out."""
        out = self._moments_out(out)
        (p, q, r), _, _, _ = _arrays([vx, vy, vz], self.dtype, self.num_particles(), host=1)
        self._check(lib().trmcr_step_host(self._h, p, q, r, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def set_particles(self, vx, vy, vz, x=None):
        """Replace the particle state (shock: positions sorted by cell; rebinned on the device)."""
        arrs = [x, vx, vy, vz] if x is not None else [vx, vy, vz]
        ptrs, host, _, n = _arrays(arrs, self.dtype)
        px, (p, q, r) = (ptrs[0], ptrs[1:]) if x is not None else (None, ptrs)
        self._check(lib().trmcr_set_particles(self._h, px, p, q, r, n, host))

    def step_host_particles(self, x, vx, vy, vz, out: Optional[np.ndarray] = None) -> np.ndarray:
        """e2e path (any geometry): host particles in (shock: x sorted by cell), one step,
        host per-cell moments out (trmcr_step_host_particles)."""
        out = self._moments_out(out)
        arrs = [x, vx, vy, vz] if x is not None else [vx, vy, vz]
        ptrs, _, _, n = _arrays(arrs, self.dtype, host=1)
        px, (p, q, r) = (ptrs[0], ptrs[1:]) if x is not None else (None, ptrs)
        self._check(lib().trmcr_step_host_particles(self._h, px, p, q, r, n,
                                                    out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def set_log(self, capacity: int):
        self._check(lib().trmcr_set_log(self._h, int(capacity)))
        self._log_cap = int(capacity)

    def collisions(self) -> np.ndarray:
        cnt = C.c_int64()
        cap = getattr(self, "_log_cap", 0)
        buf = np.zeros(max(cap, 1), dtype=COLL_DTYPE)
        self._check(lib().trmcr_get_log(self._h, buf.ctypes.data, C.byref(cnt)))
        if cnt.value > cap:
            raise TrmcrError(ECAPACITY, f"log overflow: {cnt.value} > {cap}")
        return buf[: cnt.value].copy()

    def global_moments(self, dev_out, all_ranks: bool = False):
        """Asynchronously write the global sums (GLOBAL_FIELDS) into a device float64
        tensor; all_ranks: all-reduced over the communicator (overlapping the next steps)."""
        p, host, _ = _ptr(dev_out)
        if host or dev_out.numel() < len(GLOBAL_FIELDS) or dev_out.dtype.itemsize != 8:
            raise ValueError("dev_out must be a device float64 tensor of >= 10 entries")
        self._check(lib().trmcr_global_moments(self._h, C.c_void_p(p), int(bool(all_ranks))))

    # ---- slab decomposition of the shock (see include/trmcr.h) ----
    def sort_info(self) -> dict:
        """Scatter-sort diagnostics of the last shock step (trmcr_shock_sort_info)."""
        out = np.zeros(4, dtype=np.int64)
        self._check(lib().trmcr_shock_sort_info(self._h, out.ctypes.data))
        return {"W": int(out[0]), "emigrant_width": int(out[1]), "gathered": bool(out[2]),
                "scatter_enabled": bool(out[3])}

    @property
    def fused(self) -> bool:
        """The shock context steps with the fused pass (trmcr_shock_fused)."""
        return bool(lib().trmcr_shock_fused(self._h))

    def exchange_bytes(self, capacity: int) -> int:
        return int(lib().trmcr_exchange_bytes(self.dtype, int(capacity)))

    def set_exchange(self, send_left, send_right, recv_left, recv_right, capacity: int):
        """Register caller-owned device buffers (torch uint8 tensors of exchange_bytes())."""
        p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
        self._xbufs = (send_left, send_right, recv_left, recv_right)
        self._check(lib().trmcr_shock_set_exchange(self._h, p(send_left), p(send_right), p(recv_left),
                                                   p(recv_right), int(capacity)))

    def shock_begin(self):
        self._check(lib().trmcr_shock_begin(self._h))

    def shock_finish(self):
        self._check(lib().trmcr_shock_finish(self._h))

    def set_profiling(self, on: bool = True):
        self._check(lib().trmcr_set_profiling(self._h, int(bool(on))))

    def set_profiling_kernels(self, names):
        """Bracket only the named kernels with events (see KERNELS)."""
        mask = 0
        for nm in names:
            mask |= 1 << KERNELS.index(nm)
        self._check(lib().trmcr_set_profiling_mask(self._h, mask))

    def kernel_times(self) -> dict:
        """{kernel name: (total ms, launches)} since the last call (device events)."""
        ms = np.zeros(len(KERNELS))
        cnt = np.zeros(len(KERNELS), dtype=np.int64)
        self._check(lib().trmcr_kernel_times(self._h, ms.ctypes.data_as(C.POINTER(C.c_double)),
                                             cnt.ctypes.data_as(C.POINTER(C.c_int64))))
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNELS) if cnt[i] > 0}

    @property
    def launch_count(self) -> int:
        return int(lib().trmcr_launch_count(self._h))


def get_nccl_id() -> bytes:
    """A fresh NCCL unique id (128 bytes) for Simulation(..., nccl_id=, rank=, nranks=)."""
    buf = C.create_string_buffer(128)
    st = lib().trmcr_get_nccl_id(buf)
    if st != OK:
        raise TrmcrError(st, lib().trmcr_last_error(None).decode())
    return buf.raw


def version() -> str:
    return lib().trmcr_version().decode()
