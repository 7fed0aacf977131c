"""solver -- the LUT consumer: a D3Q27 BGK
collide/stream step of one grid level with SBB / interpolated bounce-back
walls read from the cut-link LUT.

SPEC ops:
  equilibrium(rho, u)
  collide_stream_level(state, grid, L, links, flow) SPEC.md:398-411
  accumulate_forces -> LbmLevel.step(...) returns the wall momentum exchange
                                                    SPEC.md:436-440
The kernel is csrc/vf_lbm.cu (one thread per cell, pull streaming, Bouzidi
linear IBB with q_w = LUT[contraction_map[b]][q][t]); the CPU checker is
oracle/lbm_oracle.c.  Lattice units throughout.  Interface exchange between
levels is not built: GHOST cells are held, as the op's
precondition ("ghost cells of L up to date") allows.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import Optional

import numpy as np

from . import _lib
from .datatypes import ForestGrid, LinkTable
from .lattice import D3Q27

CS2 = 1.0 / 3.0


class VfFlow(C.Structure):
    _fields_ = [("tau", C.c_double), ("u_in", C.c_double * 3), ("ibb", C.c_int32),
                ("open_x", C.c_int32)]


@dataclasses.dataclass
class FlowConfig:
    """SPEC.md FlowConfig in lattice units of the stepped level: ``u_in``
    inlet speed (|u| < c_s), ``D_s`` body size in cells, ``Re`` ->
    nu = u_in D_s / Re, tau = nu / c_s^2 + 1/2 (PAPER §4)."""
    Re: float = 20.0
    u_in: float = 0.05
    D_s: float = 8.0
    bc_scheme: str = "IBB"   # "IBB" | "SBB"
    open_x: bool = True      # inlet / outlet on the x faces, else a closed SBB box

    @property
    def tau(self) -> float:
        tau = self.u_in * self.D_s / self.Re / CS2 + 0.5
        if not tau > 0.5:
            raise ValueError("tau_L <= 0.5: unstable configuration (SPEC.md:410)")
        return tau


def equilibrium(rho, u):
    """f_q^eq = w_q rho (1 + c.u/c_s^2 + (c.u)^2/(2 c_s^4) - u.u/(2 c_s^2))
    (SPEC.md:392-397), host numpy, any leading shape of rho / u[..., 3]."""
    vs = D3Q27
    c = np.asarray(vs.c, dtype=np.float64)
    w = np.asarray(vs.w, dtype=np.float64)
    rho = np.asarray(rho, dtype=np.float64)
    u = np.asarray(u, dtype=np.float64)
    cu = u @ c.T
    uu = (u * u).sum(-1, keepdims=True)
    return w * rho[..., None] * (1.0 + cu / CS2 + cu * cu / (2 * CS2 * CS2) - uu / (2 * CS2))


class LbmLevel:
    """State of one level: post-collision populations f[27, (e-s)*64] (f32,
    two buffers) over the level's blocks [s, e)."""

    def __init__(self, grid: ForestGrid, level: int, table: Optional[LinkTable], flow: FlowConfig,
                 tau: Optional[float] = None):
        import torch
        self.lib = _lib.require_cuda()
        self.grid, self.level, self.table, self.flow = grid, int(level), table, flow
        self.s, self.e = grid.level_range(level)
        n = (self.e - self.s) * 64
        self.f = [torch.empty((27, n), dtype=torch.float32, device="cuda") for _ in range(2)]
        self.cur = 0
        self.force = torch.zeros(3, dtype=torch.float64, device="cuda")
        self.scratch = torch.zeros(self.e - self.s + 1, dtype=torch.int32, device="cuda")
        self.c = _lib.make_config(grid.cfg)
        self.vf = VfFlow()
        self.vf.tau = float(tau if tau is not None else flow.tau)
        self.vf.u_in[:] = [float(flow.u_in), 0.0, 0.0]
        self.vf.ibb = int(flow.bc_scheme.upper() == "IBB" and table is not None)
        self.vf.open_x = int(bool(flow.open_x))
        if self.vf.ibb:
            cm = table.contraction_map
            if cm.numel() < grid.capacity:
                full = torch.full((grid.capacity,), -1, dtype=torch.int32, device="cuda")
                full[:cm.numel()] = cm
                cm = full
            self.cmap = cm
        else:
            self.cmap = None

    @property
    def state(self):
        return self.f[self.cur]

    def init_equilibrium(self, rho: float = 1.0, u=(0.0, 0.0, 0.0)):
        u = (C.c_double * 3)(*[float(x) for x in u])
        _lib.check(self.lib.vf_lbm_init(C.byref(self.grid._struct()), self.s, self.e, float(rho), u,
                                        _lib.ptr(self.state), _lib.stream_ptr()), "lbm init")
        return self

    def step(self, n: int = 1, force: bool = True):
        """n collide/stream steps; returns the wall momentum exchange summed
        over them (lattice units, device tensor) when ``force``."""
        gs = self.grid._struct()
        if force:
            self.force.zero_()
        lengths = _lib.ptr(self.table.lengths) if self.vf.ibb else None
        for _ in range(n):
            _lib.check(self.lib.vf_lbm_step(
                C.byref(self.c), C.byref(gs), self.level, self.s, self.e, _lib.ptr(self.cmap), lengths,
                _lib.ptr(self.f[self.cur]), _lib.ptr(self.f[self.cur ^ 1]), C.byref(self.vf),
                _lib.ptr(self.force) if force else None, _lib.ptr(self.scratch), _lib.stream_ptr()),
                "collide_stream_level")
            self.cur ^= 1
        return self.force

    def macroscopic(self):
        """(rho, u) per cell from the post-collision populations (BGK keeps
        rho and u)."""
        import torch
        c = torch.tensor(np.asarray(D3Q27.c), dtype=torch.float32, device="cuda")
        f = self.state
        rho = f.sum(0)
        u = (c.T @ f) / rho
        return rho, u


def collide_stream_level(state: LbmLevel, grid: ForestGrid, level: int, links: LinkTable,
                         flow: FlowConfig) -> LbmLevel:
    """SPEC.md:398-411 on the GPU (state must be an LbmLevel of that level)."""
    if state.level != level or state.grid is not grid:
        raise ValueError("state belongs to another grid level")
    state.step(1)
    return state
