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
oracle/lbm_oracle.c.  Lattice units throughout.

Multi-level:
  interface_exchange(state, grid, order)
  step_hierarchy(state, grid, links, flow)
LbmHierarchy holds one LbmLevel per level with acoustic scaling (SPEC.md:473:
nu_L = 2^L nu_0, tau_L = 3 nu_L + 1/2).  One coarse step advances level L
once and, recursively, level L+1 twice: before each fine substep the fine
GHOST cells (A14) are filled from level L by tensor-product interpolation
(cubic or linear, cell-centred 2:1 layout) of L's post-collision populations
at theta = 0 and 1/2 between L's old and new states (vf_lbm_fill_ghosts);
after the two substeps the covered cells of L's refined blocks (not
INTERFACE: those stay coupled to L's own dynamics) are restricted from
their 8 children (vf_lbm_restrict).  Non-equilibrium parts are rescaled by
(tau_f - 1) / (2 (tau_c - 1)) coarse -> fine and its inverse fine -> coarse
(post-collision Dupuis-Chopard factor).  The CPU checker of the
same schedule is oracle.lbm_step_hierarchy.
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
        self.scratch = torch.zeros(7 * (self.e - self.s) + 4, dtype=torch.int32, device="cuda")
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


def level_taus(tau0: float, n_levels: int):
    """Acoustic scaling: nu_L = 2^L nu_0, tau_L = 3 nu_L + 1/2."""
    nu0 = (tau0 - 0.5) / 3.0
    return [3.0 * nu0 * 2 ** L + 0.5 for L in range(n_levels)]


def neq_factors(tau_c: float, tau_f: float):
    """(alpha, beta): post-collision non-equilibrium rescale coarse -> fine
    (tau_f - 1) / (2 (tau_c - 1)) and fine -> coarse (its inverse)."""
    if abs(tau_c - 1.0) < 1e-9 or abs(tau_f - 1.0) < 1e-9:
        raise ValueError("tau_L = 1 loses the non-equilibrium part of post-collision populations")
    a = (tau_f - 1.0) / (2.0 * (tau_c - 1.0))
    return a, 1.0 / a


class LbmHierarchy:
    """State of every level of an embedded grid (SPEC.md:389 LbmState): one
    LbmLevel per level, tau_L by acoustic scaling from ``flow.tau`` at level
    0; ``order`` 3 (cubic) or 1 (linear) ghost interpolation."""

    def __init__(self, grid: ForestGrid, table: Optional[LinkTable], flow: FlowConfig, order: int = 3,
                 rescale: bool = True):
        import torch
        if order not in (0, 1, 3):
            raise ValueError("interp order must be 1 (linear) or 3 (cubic)")
        self.lib = _lib.require_cuda()
        self.grid, self.table, self.flow, self.order = grid, table, flow, int(order)
        self.taus = level_taus(flow.tau, grid.n_levels)
        for t in self.taus:
            if not t > 0.5:
                raise ValueError("tau_L <= 0.5: unstable configuration (SPEC.md:410)")
        self.factors = [neq_factors(self.taus[L], self.taus[L + 1]) if rescale else (1.0, 1.0)
                        for L in range(grid.n_levels - 1)]
        self.levels = [LbmLevel(grid, L, table, flow, tau=self.taus[L]) for L in range(grid.n_levels)]
        n = grid.n_used
        self.parent = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
        _lib.check(self.lib.vf_lbm_parents(C.byref(grid._struct()), n, _lib.ptr(self.parent), _lib.stream_ptr()),
                   "lbm parents")
        self.substeps = [0] * grid.n_levels

    def init_equilibrium(self, rho: float = 1.0, u=(0.0, 0.0, 0.0)):
        for lv in self.levels:
            lv.init_equilibrium(rho, u)
        return self

    def fill_ghosts(self, L: int, old, new, theta: float):
        """Ghost cells of level L+1 from level L (old/new post-collision
        states of L, time weight theta)."""
        fine, coarse = self.levels[L + 1], self.levels[L]
        _lib.check(self.lib.vf_lbm_fill_ghosts(
            C.byref(self.grid._struct()), fine.s, fine.e, coarse.s, coarse.e, _lib.ptr(self.parent), _lib.ptr(old),
            _lib.ptr(new), float(theta), float(self.factors[L][0]), self.order, _lib.ptr(fine.state),
            _lib.stream_ptr()), "interface_exchange (fill ghosts)")

    def restrict(self, L: int):
        """Covered cells of level L from level L+1."""
        fine, coarse = self.levels[L + 1], self.levels[L]
        _lib.check(self.lib.vf_lbm_restrict(
            C.byref(self.grid._struct()), coarse.s, coarse.e, fine.s, fine.e, _lib.ptr(self.parent),
            _lib.ptr(fine.state), float(self.factors[L][1]), _lib.ptr(coarse.state), _lib.stream_ptr()), "interface_exchange (restrict)")

    def _advance(self, L: int, force: bool):
        lv = self.levels[L]
        old = lv.state
        lv.step(1, force=force)
        self.substeps[L] += 1
        if L + 1 < len(self.levels):
            for theta in (0.0, 0.5):
                self.fill_ghosts(L, old, lv.state, theta)
                self._advance(L + 1, force)
            self.restrict(L)

    def step(self, n: int = 1, force: bool = False):
        """n coarse steps (level L takes 2^L substeps each)."""
        for _ in range(n):
            self._advance(0, force)
        return self

    def graph(self):
        """A CUDA graph of two coarse steps (every level then takes an even
        number of substeps, so the ping-pong buffers are back in place after
        each replay); the launch-bound host loop of step() is captured once."""
        import torch
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.step(2)
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step(2)
        return g

    def mass(self) -> float:
        """sum over leaf cells (not SOLID / GHOST, block not refined) of
        rho (dx_L / dx_0)^3 -- the conservation audit of SPEC.md:434."""
        import torch
        g = self.grid
        total = 0.0
        for L, lv in enumerate(self.levels):
            m = g.masks[lv.s:lv.e].reshape(-1)
            leaf = (g.child[lv.s:lv.e] < 0).repeat_interleave(64)
            keep = leaf & (m != 1) & (m != 3)
            rho = lv.state.sum(0, dtype=torch.float64)
            total += float(rho[keep].sum()) / 8.0 ** L
        return total


def interface_exchange(state: LbmHierarchy, grid: ForestGrid, order: int = 3, level: int = 0,
                       theta: float = 0.0) -> LbmHierarchy:
    """SPEC.md:417-425 between levels ``level`` and ``level + 1``: fine
    ghosts <- coarse (current state, time weight theta against itself), then
    coarse covered cells <- fine."""
    if state.grid is not grid:
        raise ValueError("state belongs to another grid")
    state.order = int(order)
    cur = state.levels[level].state
    state.fill_ghosts(level, cur, cur, theta)
    state.restrict(level)
    return state


def step_hierarchy(state: LbmHierarchy, grid: ForestGrid, links: Optional[LinkTable] = None,
                   flow: Optional[FlowConfig] = None) -> LbmHierarchy:
    """one coarse step of the whole hierarchy."""
    if state.grid is not grid:
        raise ValueError("state belongs to another grid")
    return state.step(1)
