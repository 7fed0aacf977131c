"""forest -- block-based forest-of-octrees on the GPU.

Drop-in for the SPEC ops of ``voxforest.forest``:
  init_forest(config)
  adapt(grid, marks)                       SPEC.md:219-227 (refine-only)
  index_maps(I, c)                         SPEC.md:228-236 (host, pure integer math)
  block_of_point(grid, point, level)       SPEC.md:237-245 (host test utility)

Block ids are grouped by level and appended in creation order; children of one
parent occupy 8 consecutive ids.  The gap set is [n_used,
capacity): coarsening/defragmentation are out of scope for a static geometry.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Tuple

import numpy as np

from . import _lib, _ws
from .config import EmbedConfig
from .datatypes import ForestGrid
from .lattice import D3Q27_C


def init_forest(cfg: EmbedConfig, capacity: Optional[int] = None,
                surface_area: float = 1.0) -> ForestGrid:
    """Root grid of N_B^3 blocks, full-halo links, all cells fluid."""
    lib = _lib.require_cuda()
    cap = int(capacity if capacity is not None else cfg.block_capacity(surface_area))
    g = ForestGrid.allocate(cfg, cap)
    gs = g._struct()
    c = _lib.make_config(cfg)
    _lib.check(lib.vf_init_forest(C.byref(c), C.byref(gs), _lib.stream_ptr()), "init_forest")
    g.n_levels = gs.n_levels
    return g


def adapt(grid: ForestGrid, marks=None) -> ForestGrid:
    """Refine the finest level's marked blocks (8-step procedure of
    PAPER.md:261-271, refine-only).  ``marks``: None = the grid's MARK bits
    (set by mark_near_wall_refinement), or a bool tensor over the finest
    level's blocks."""
    import torch
    lib = _lib.require_cuda()
    L = grid.n_levels - 1
    if marks is not None:
        s, e = grid.level_range(L)
        m = torch.as_tensor(marks, device="cuda").to(torch.bool).reshape(-1)
        if m.numel() != e - s:
            raise ValueError("marks must cover the finest level's blocks")
        f = grid.bflags[s:e]
        grid.bflags[s:e] = torch.where(m, f | _lib.BF_MARK, f & ~_lib.BF_MARK)
    gs = grid._struct()
    c = _lib.make_config(grid.cfg)
    ws = _ws.get("adapt", lib.vf_adapt_workspace_size(C.byref(gs)))
    _lib.check(lib.vf_adapt_refine(C.byref(c), C.byref(gs), L, _lib.ptr(ws), ws.numel(),
                                   _lib.stream_ptr()), "adapt")
    grid.n_levels = gs.n_levels
    _lib.check(lib.vf_check_status(C.byref(gs), _lib.stream_ptr()), "adapt")
    return grid


def index_maps(I, c) -> Tuple[int, int, Tuple[int, int, int], bool]:
    """(t, t_h, I', violation) of SPEC.md:228-236, literally:

    t = LINEAR(I,4), t_h = LINEAR(I+1,6), I'_d = mod(4+mod(I_d+c_d,4),4)
    (PAPER.md:949 adds c twice, pin A15) and the violation flag
    AND_d ((I'_d != I_d + c_d) or c_d = 0) of SPEC.md:229 / PAPER.md:954.
    That flag is true only when the step leaves the block along EVERY
    non-zero axis of c (and for c = 0); the kernels read a neighbour cell
    through the general neighbour-block direction of neighbour_direction()
    (pin A15), which also covers steps that leave along some axes only."""
    I = tuple(int(v) for v in I)
    c = tuple(int(v) for v in c)
    t = I[0] + 4 * I[1] + 16 * I[2]
    th = (I[0] + 1) + 6 * (I[1] + 1) + 36 * (I[2] + 1)
    Ip = tuple((4 + ((I[d] + c[d]) % 4)) % 4 for d in range(3))
    viol = all(Ip[d] != I[d] + c[d] or c[d] == 0 for d in range(3))
    return t, th, Ip, viol


def neighbor_direction(I, c) -> Tuple[int, int, int]:
    """Pin A15: the neighbour block holding cell I + c is the block in
    direction (c_d if the step wraps axis d else 0)_d -- (0, 0, 0) = the
    block itself.  This is what the boundary-cell and LBM kernels use."""
    return tuple(int(c[d]) if not (0 <= int(I[d]) + int(c[d]) < 4) else 0 for d in range(3))


def neighbor_slot(c) -> int:
    """D3Q27 slot of a direction (lattice.py:19-39 order)."""
    for q, v in enumerate(D3Q27_C):
        if tuple(v) == tuple(int(x) for x in c):
            return q
    raise ValueError(f"not a D3Q27 direction: {c}")


def block_of_point(grid: ForestGrid, point, level: Optional[int] = None) -> Optional[int]:
    """Leaf (or level-L) block containing ``point``: root-grid indexing plus
    child descent; ties at faces go to the lower index."""
    cfg = grid.cfg
    h = grid.to_numpy()
    p = np.asarray(point, dtype=np.float64)
    if np.any(p < 0) or np.any(p > np.asarray(cfg.domain)):
        return None
    nb = cfg.nb
    h0 = 4.0 * cfg.dx0

    def cell(x, hh, n):  # block index along an axis; a point on a face -> lower index
        return min(max(int(np.ceil(x / hh)) - 1, 0), n - 1)

    ijk = [cell(p[d], h0, nb[d]) for d in range(3)]
    b = ijk[0] + nb[0] * (ijk[1] + nb[1] * ijk[2])
    L = 0
    while (level is None or L < level) and h["child"][b] >= 0:
        hL1 = h0 / 2 ** (L + 1)
        sub = [cell(p[d], hL1, nb[d] << (L + 1)) & 1 for d in range(3)]
        b = int(h["child"][b] + sub[0] + 2 * sub[1] + 4 * sub[2])
        L += 1
    if level is not None and L != level:
        return None
    return int(b)
