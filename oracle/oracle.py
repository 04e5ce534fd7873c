"""ctypes wrapper of the CPU oracle (oracle/trmcr_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module; the product
package (paper_1009_2768_b200) never does.  Everything here is argument
marshalling around the C oracle plus numpy conveniences.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "trmcr_oracle.c")
LIB = os.path.join(HERE, "liborc.so")

MAXWELL, HARD_SPHERE, VHS = 0, 1, 2
IND_PXX, IND_M4 = 0, 1
P_SPLIT, P_TYPE, P_PERM, P_COLL, P_COLL2, P_MAXW, P_MAXW2, P_RESV, P_RESV2, P_LITERAL = range(1, 11)


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
        os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "trmcr_oracle.h"))
    ):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
             "-Wall", "-o", tmp, SRC, "-lm"]
        )
        os.replace(tmp, LIB)
    return LIB


class Params(C.Structure):
    _fields_ = [
        ("model", C.c_int32), ("adaptive", C.c_int32), ("m_fixed", C.c_int32),
        ("m_init", C.c_int32), ("m_cap", C.c_int32), ("indicator", C.c_int32),
        ("delta1", C.c_double), ("delta2", C.c_double), ("eps", C.c_double), ("dt", C.c_double),
        ("seed", C.c_uint64), ("literal", C.c_int32), ("pad", C.c_int32), ("alpha", C.c_double),
        ("wb", C.c_int32), ("wb_max", C.c_int32), ("sigma_update", C.c_int32),
    ]


STAT_FIELDS = ["n", "p", "mu", "sigma", "S0", "S_est", "E1", "m_used", "m_next", "depth",
               "attempts", "leaves", "untouched", "thermalised", "proposals", "accepted",
               "violations", "maxw"]


class CellStats(C.Structure):
    _fields_ = [(f, C.c_double) for f in STAT_FIELDS]


class CollRec(C.Structure):
    _fields_ = [("cell", C.c_int32), ("attempt", C.c_int32), ("level", C.c_int32),
                ("accepted", C.c_int32), ("j", C.c_int64), ("slot_i", C.c_int64),
                ("slot_k", C.c_int64)]


COLL_DTYPE = np.dtype([("cell", "<i4"), ("attempt", "<i4"), ("level", "<i4"), ("accepted", "<i4"),
                       ("j", "<i8"), ("slot_i", "<i8"), ("slot_k", "<i8")])
STATS_DTYPE = np.dtype([(f, "<f8") for f in STAT_FIELDS])


class Shock(C.Structure):
    _fields_ = [("ncells", C.c_int32), ("pad", C.c_int32), ("x_min", C.c_double),
                ("x_max", C.c_double), ("weight", C.c_double),
                ("rho_L", C.c_double), ("u_L", C.c_double), ("T_L", C.c_double),
                ("rho_R", C.c_double), ("u_R", C.c_double), ("T_R", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.POINTER
        L.orc_philox4x32_10.argtypes = [P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]
        L.orc_u53.argtypes = [C.c_uint32, C.c_uint32]
        L.orc_u53.restype = C.c_double
        L.orc_ir.argtypes = [C.c_double, C.c_double]
        L.orc_ir.restype = C.c_int64
        L.orc_feistel.argtypes = [C.c_uint64, C.c_uint64, P(C.c_uint32)]
        L.orc_feistel.restype = C.c_int64
        L.orc_collide_pair.argtypes = [P(C.c_double), P(C.c_double), C.c_double, C.c_double]
        L.orc_split.argtypes = [C.c_double, C.c_int64, C.c_int32, C.c_uint64, C.c_uint32,
                                C.c_uint32, P(C.c_int64), P(C.c_int64)]
        L.orc_split.restype = C.c_int32
        L.orc_maxwellian.argtypes = [C.c_int64, P(C.c_int64), P(C.c_double), P(C.c_double),
                                     P(C.c_double), C.c_uint64, C.c_uint32, C.c_uint32]
        L.orc_step_cells.argtypes = [P(Params), C.c_int64, P(C.c_int64), C.c_uint32,
                                     P(C.c_double), C.c_uint32, P(C.c_double), P(C.c_double),
                                     P(C.c_double), P(C.c_int32), P(CellStats), P(CollRec),
                                     C.c_int64, P(C.c_int64)]
        L.orc_step_cells.restype = C.c_int32
        L.orc_moments.argtypes = [C.c_int64, P(C.c_int64), P(C.c_double), P(C.c_double),
                                  P(C.c_double), P(C.c_double), P(C.c_int32), P(C.c_double)]
        L.orc_shock_step.argtypes = [P(Params), P(Shock), C.c_uint32, P(C.c_int64), C.c_int64,
                                     P(C.c_double), P(C.c_double), P(C.c_double), P(C.c_double),
                                     P(C.c_int64), P(C.c_int32), P(CellStats), P(C.c_double)]
        L.orc_shock_step.restype = C.c_int32
        L.orc_shock_bin.argtypes = [P(Shock), C.c_int64, P(C.c_double), P(C.c_double),
                                    P(C.c_double), P(C.c_double), P(C.c_int64)]
        L.orc_shock_bin.restype = C.c_int32
        L.orc_rankine_hugoniot.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double,
                                           P(C.c_double)]
        L.orc_rankine_hugoniot.restype = C.c_int32
        L.orc_tree_length.argtypes = [P(C.c_int32), C.c_int64, C.c_int32, P(C.c_int64)]
        L.orc_tree_length.restype = C.c_double
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


# ---------------------------------------------------------------- primitives
def philox(ctr, key):
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(c, C.c_uint32), _p(k, C.c_uint32), _p(out, C.c_uint32))
    return out


def u53(hi, lo):
    return lib().orc_u53(int(hi), int(lo))


def ir(y, u):
    return lib().orc_ir(float(y), float(u))


def feistel(x, N, rk):
    r = np.ascontiguousarray(rk, dtype=np.uint32)
    return lib().orc_feistel(int(x), int(N), _p(r, C.c_uint32))


def tree_length(path, definition):
    """Alg 4.5 length of the tree given by its path list; definition 1 = 1 + min
    (eq. def:2), 2 = 1 + mean (eq. def:3), 3 = the coefficient k (eq. def:1)."""
    a = np.ascontiguousarray(path, dtype=np.int32)
    used = C.c_int64(0)
    L = lib().orc_tree_length(_p(a, C.c_int32), len(a), int(definition), C.byref(used))
    if used.value != len(a):
        raise ValueError("malformed path list")
    return L


def collide_pair(vi, vj, xi1, xi2):
    a = np.array(vi, dtype=np.float64)
    b = np.array(vj, dtype=np.float64)
    lib().orc_collide_pair(_p(a, C.c_double), _p(b, C.c_double), float(xi1), float(xi2))
    return a, b


def split(p, n, m, seed=1, gcell=0, step=0):
    N = np.zeros(m + 2, dtype=np.int64)
    rem = np.zeros(1, dtype=np.int64)
    d = lib().orc_split(float(p), int(n), int(m), int(seed), int(gcell), int(step),
                        _p(N, C.c_int64), _p(rem, C.c_int64))
    return N, int(rem[0]), d


def maxwellian(slots, vx, vy, vz, seed=1, gcell=0, step=0):
    s = np.ascontiguousarray(slots, dtype=np.int64)
    lib().orc_maxwellian(len(s), _p(s, C.c_int64), _p(vx, C.c_double), _p(vy, C.c_double),
                         _p(vz, C.c_double), int(seed), int(gcell), int(step))


def rankine_hugoniot(mach, gamma=5.0 / 3.0, rho_L=1.0, T_L=1.0):
    out = np.zeros(6)
    rc = lib().orc_rankine_hugoniot(float(mach), float(gamma), float(rho_L), float(T_L),
                                    _p(out, C.c_double))
    if rc != 0:
        raise ValueError("no shock for Mach <= 1")
    return out


# ---------------------------------------------------------------- steps
@dataclass
class Config:
    model: int = MAXWELL
    adaptive: int = 0
    m_fixed: int = 64
    m_init: int = 2
    m_cap: int = 4096
    indicator: int = IND_PXX
    delta1: float = 0.005
    delta2: float = 0.01
    eps: float = 1.0
    dt: float = 0.1
    seed: int = 1
    literal: int = 0
    alpha: float = 1.0          # VHS exponent (model = VHS)
    wb: int = 0                 # TRMC-WB length: 0 off, 1 min (def:2), 2 mean (def:3), 3 level (def:1)
    wb_max: int = 0             # TRMC-WB threshold m_max
    sigma_update: int = 0       # 1: majorant raised after each collision

    def c(self) -> Params:
        return Params(self.model, self.adaptive, self.m_fixed, self.m_init, self.m_cap,
                      self.indicator, self.delta1, self.delta2, self.eps, self.dt, self.seed,
                      self.literal, 0, self.alpha, self.wb, self.wb_max, self.sigma_update)


class HomogeneousState:
    """Cells of independent space-homogeneous gases (rho = 1 each)."""

    def __init__(self, cfg: Config, vx, vy, vz, offsets, gcell0=0, rho=None, log_cap=0):
        self.cfg = cfg
        self.vx = np.array(vx, dtype=np.float64)
        self.vy = np.array(vy, dtype=np.float64)
        self.vz = np.array(vz, dtype=np.float64)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.ncells = len(self.offsets) - 1
        self.gcell0 = gcell0
        self.rho = np.ones(self.ncells) if rho is None else np.ascontiguousarray(rho, np.float64)
        m0 = cfg.m_init if cfg.adaptive else cfg.m_fixed
        self.m_state = np.full(self.ncells, m0, dtype=np.int32)
        self.step_count = 0
        self.stats = np.zeros(self.ncells, dtype=STATS_DTYPE)
        self.log_cap = log_cap
        self.log = np.zeros(max(log_cap, 1), dtype=COLL_DTYPE)
        self.log_n = 0

    def step(self, nsteps=1):
        P = self.cfg.c()
        for _ in range(nsteps):
            st = np.zeros(self.ncells, dtype=STATS_DTYPE)
            ln = np.zeros(1, dtype=np.int64)
            rc = lib().orc_step_cells(
                C.byref(P), self.ncells, _p(self.offsets, C.c_int64), self.gcell0,
                _p(self.rho, C.c_double), self.step_count, _p(self.vx, C.c_double),
                _p(self.vy, C.c_double), _p(self.vz, C.c_double), _p(self.m_state, C.c_int32),
                st.ctypes.data_as(C.POINTER(CellStats)),
                self.log.ctypes.data_as(C.POINTER(CollRec)) if self.log_cap else None,
                self.log_cap, _p(ln, C.c_int64))
            if rc != 0:
                raise RuntimeError(f"oracle step failed rc={rc}")
            self.stats = st
            self.log_n = int(ln[0])
            self.step_count += 1
        return self

    def moments(self):
        out = np.zeros((self.ncells, 12))
        lib().orc_moments(self.ncells, _p(self.offsets, C.c_int64), _p(self.rho, C.c_double),
                          _p(self.vx, C.c_double), _p(self.vy, C.c_double),
                          _p(self.vz, C.c_double), _p(self.m_state, C.c_int32),
                          _p(out, C.c_double))
        return out

    def collisions(self):
        n = min(self.log_n, self.log_cap)
        return self.log[:n].copy()


class ShockState:
    """1D stationary shock (reservoirs + transport + stable sort + collisions)."""

    def __init__(self, cfg: Config, shock: dict, x, vx, vy, vz, capacity=None):
        self.cfg = cfg
        self.S = Shock(int(shock["ncells"]), 0, shock["x_min"], shock["x_max"], shock["weight"],
                       shock["rho_L"], shock["u_L"], shock["T_L"], shock["rho_R"], shock["u_R"],
                       shock["T_R"])
        n = len(x)
        self.cap = capacity or int(2 * n + 1024)
        self.x = np.zeros(self.cap); self.vx = np.zeros(self.cap)
        self.vy = np.zeros(self.cap); self.vz = np.zeros(self.cap)
        self.x[:n] = x; self.vx[:n] = vx; self.vy[:n] = vy; self.vz[:n] = vz
        self.n = n
        self.ncells = self.S.ncells
        self.offsets = np.zeros(self.ncells + 1, dtype=np.int64)
        rc = lib().orc_shock_bin(C.byref(self.S), n, _p(self.x, C.c_double),
                                 _p(self.vx, C.c_double), _p(self.vy, C.c_double),
                                 _p(self.vz, C.c_double), _p(self.offsets, C.c_int64))
        if rc != 0:
            raise ValueError("particle outside the domain")
        m0 = cfg.m_init if cfg.adaptive else cfg.m_fixed
        self.m_state = np.full(self.ncells, m0, dtype=np.int32)
        self.step_count = 0
        self.stats = np.zeros(self.ncells, dtype=STATS_DTYPE)
        self.counts = np.zeros(4)

    def step(self, nsteps=1):
        P = self.cfg.c()
        for _ in range(nsteps):
            nn = np.array([self.n], dtype=np.int64)
            st = np.zeros(self.ncells, dtype=STATS_DTYPE)
            rc = lib().orc_shock_step(
                C.byref(P), C.byref(self.S), self.step_count, _p(nn, C.c_int64), self.cap,
                _p(self.x, C.c_double), _p(self.vx, C.c_double), _p(self.vy, C.c_double),
                _p(self.vz, C.c_double), _p(self.offsets, C.c_int64),
                _p(self.m_state, C.c_int32), st.ctypes.data_as(C.POINTER(CellStats)),
                _p(self.counts, C.c_double))
            if rc != 0:
                raise RuntimeError(f"oracle shock step failed rc={rc}")
            self.n = int(nn[0])
            self.stats = st
            self.step_count += 1
        return self

    def rho(self):
        dx = (self.S.x_max - self.S.x_min) / self.ncells
        return np.diff(self.offsets) * self.S.weight / dx

    def moments(self):
        out = np.zeros((self.ncells, 12))
        rho = np.ascontiguousarray(self.rho())
        lib().orc_moments(self.ncells, _p(self.offsets, C.c_int64), _p(rho, C.c_double),
                          _p(self.vx, C.c_double), _p(self.vy, C.c_double),
                          _p(self.vz, C.c_double), _p(self.m_state, C.c_int32),
                          _p(out, C.c_double))
        return out
