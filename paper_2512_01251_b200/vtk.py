"""Outputs (SPEC.md write_outputs kind=voxels, legacy
ASCII VTK chosen for diff-stable goldens): one unstructured-grid file per
level, every cell of the level's blocks a VTK_VOXEL tagged with its cell mask,
plus the block id and a link count (cut links of the cell in the LUT).

Host-side formatting of device results (numpy, vectorised); byte-stable for a
fixed grid.
"""
from __future__ import annotations

import os
from typing import Dict, List, Optional

import numpy as np

VTK_VOXEL = 11


def level_cells(coords, masks, s, e, dx):
    """(origins (n,3), masks (n,), block ids (n,)) of the cells of blocks
    [s, e): cell t = I + 4J + 16K of block (i, j, k) at ((4i+I)dx, ...)."""
    blk = np.arange(s, e)
    t = np.arange(64)
    I, J, K = t & 3, (t >> 2) & 3, t >> 4
    c = coords[s:e, :3].astype(np.int64)
    gi = (4 * c[:, 0:1] + I[None, :]).reshape(-1)
    gj = (4 * c[:, 1:2] + J[None, :]).reshape(-1)
    gk = (4 * c[:, 2:3] + K[None, :]).reshape(-1)
    org = np.stack([gi, gj, gk], axis=1).astype(np.float64) * dx
    return org, masks[s:e].reshape(-1), np.repeat(blk, 64)


def write_voxels_vtk(path: str, origins, dx: float, cell_data: Dict[str, np.ndarray],
                     title: str = "voxforest level") -> None:
    """Legacy ASCII VTK unstructured grid of axis-aligned voxels."""
    n = len(origins)
    off = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0], [0, 0, 1], [1, 0, 1], [0, 1, 1], [1, 1, 1]],
                   dtype=np.float64) * dx  # VTK_VOXEL corner order
    pts = (origins[:, None, :] + off[None, :, :]).reshape(-1, 3)
    with open(path, "w", newline="\n") as fh:
        fh.write(f"# vtk DataFile Version 3.0\n{title}\nASCII\nDATASET UNSTRUCTURED_GRID\n")
        fh.write(f"POINTS {8 * n} double\n")
        np.savetxt(fh, pts, fmt="%.17g")
        fh.write(f"CELLS {n} {9 * n}\n")
        conn = np.concatenate([np.full((n, 1), 8, np.int64), np.arange(8 * n, dtype=np.int64).reshape(n, 8)], 1)
        np.savetxt(fh, conn, fmt="%d")
        fh.write(f"CELL_TYPES {n}\n")
        np.savetxt(fh, np.full(n, VTK_VOXEL, np.int64), fmt="%d")
        fh.write(f"CELL_DATA {n}\n")
        for name, arr in cell_data.items():
            fh.write(f"SCALARS {name} int 1\nLOOKUP_TABLE default\n")
            np.savetxt(fh, np.asarray(arr, dtype=np.int64), fmt="%d")


def write_levels(out_dir: str, grid_np: dict, cfg, lengths=None, cmap=None,
                 levels: Optional[List[int]] = None) -> List[str]:
    """One VTK file per level (SPEC.md write_outputs: 'sphere embedding
    snapshot per level -> one file per level 0..L_max-1')."""
    os.makedirs(out_dir, exist_ok=True)
    ls = grid_np["level_start"]
    paths = []
    Lf = cfg.l_max - 1
    for L in (range(cfg.l_max) if levels is None else levels):
        s, e = int(ls[L]), int(ls[L + 1])
        if e <= s:
            continue
        org, msk, blk = level_cells(grid_np["coords"], grid_np["masks"], s, e, cfg.dx(L))
        data = {"mask": msk, "block": blk}
        if L == Lf and lengths is not None and cmap is not None:
            slot = np.repeat(cmap[s:e], 64)
            t = np.tile(np.arange(64), e - s)
            links = np.zeros(len(slot), np.int64)
            ok = slot >= 0
            if ok.any():
                links[ok] = (lengths[slot[ok], 1:, t[ok]] > 0).sum(1)
            data["links"] = links
        p = os.path.join(out_dir, f"level_{L}.vtk")
        write_voxels_vtk(p, org, cfg.dx(L), data, title=f"voxforest level {L}")
        paths.append(p)
    return paths


def read_vtk_cell_data(path: str) -> Dict[str, np.ndarray]:
    """Minimal reader of the files above (round-trip tests)."""
    with open(path) as fh:
        toks = fh.read().split()
    out, i = {}, 0
    while i < len(toks):
        if toks[i] == "CELL_DATA":
            n = int(toks[i + 1])
            i += 2
            while i < len(toks) and toks[i] == "SCALARS":
                name = toks[i + 1]
                i += 6  # SCALARS name int 1 LOOKUP_TABLE default
                out[name] = np.array(toks[i:i + n], dtype=np.int64)
                i += n
            break
        i += 1
    return out
