"""Command line (SPEC.md run_cli / load_config):

  python -m paper_2512_01251_b200 voxelize --config run.cfg | [--stl F | --primitive sphere|torus]
                                          [--nx 64 --lmax 4 --nspec 2 --dspec 0.05 --out DIR]
  python -m paper_2512_01251_b200 bench    (same options) [--reps 20]

voxelize: embed the geometry on the GPU, write one legacy ASCII VTK file per
level (cell masks; cut-link counts on the finest level) and a JSON summary of
the grid and the LinkTable.  bench: repeat the embedding and print the
TimingReport (mean and 95% confidence half-width per stage group, the paper's
Table 2 grouping).  simulate: embed, then run iters_total coarse steps of the
multi-level LBM (solver.step_hierarchy: D3Q27 BGK, IBB/SBB walls from the LUT,
inlet/outlet on the x faces, cubic/linear interface exchange) and write the
wall-force samples (finest level, lattice units) to forces.csv with a JSON
summary (mean F_x and the drag coefficient C_D = 2 F_x / (rho u_in^2 A),
A = pi D_s^2 / 4 in finest cells, for the sphere primitive).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
from typing import Dict

KEYS = {"stl": str, "primitive": str, "subdivisions": int, "torus_m": int, "torus_n": int,
        "diameter": float, "N_x": int, "L_max": int, "N_spec": int, "d_spec": float, "out": str, "reps": int,
        "Re": float, "u_in": float, "bc_scheme": str, "interp_order": str, "iters_total": int,
        "sample_start": int, "sample_stride": int}
DEFAULTS = {"primitive": "sphere", "subdivisions": 4, "torus_m": 280, "torus_n": 200, "diameter": 0.5,
            "N_x": 64, "L_max": 3, "N_spec": 2, "d_spec": 0.05, "out": "voxforest_out", "reps": 20,
            "Re": 20.0, "u_in": 0.05, "bc_scheme": "IBB", "interp_order": "cubic", "iters_total": 100,
            "sample_start": 50, "sample_stride": 10}


class ConfigError(ValueError):
    pass


def load_config(path: str) -> Dict:
    """Plain-text key=value (SPEC.md load_config); '#' comments; unknown keys
    and unparsable values are errors naming the key and the line."""
    cfg = dict(DEFAULTS)
    with open(path) as fh:
        for ln, line in enumerate(fh, 1):
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            if "=" not in line:
                raise ConfigError(f"line {ln}: expected key=value")
            k, v = (x.strip() for x in line.split("=", 1))
            if k not in KEYS:
                raise ConfigError(f"line {ln}: unknown key '{k}'")
            try:
                cfg[k] = KEYS[k](v)
            except ValueError:
                raise ConfigError(f"line {ln}: bad value for '{k}': '{v}'") from None
    if cfg["L_max"] < 1:
        raise ConfigError("L_max must be >= 1")
    return cfg


def _mesh(c):
    from . import make_icosphere, make_torus
    if c.get("stl"):
        from .stl import parse_stl
        with open(c["stl"], "rb") as fh:
            return parse_stl(fh.read())
    if c["primitive"] == "torus":
        return make_torus(c["torus_m"], c["torus_n"])
    return make_icosphere((0.5, 0.5, 0.5), c["diameter"], c["subdivisions"])


def _embed_cfg(c):
    from .config import EmbedConfig
    return EmbedConfig(n_x=c["N_x"], l_max=c["L_max"], n_spec=c["N_spec"], d_spec=c["d_spec"])


def cmd_voxelize(c) -> int:
    import numpy as np
    from .vtk import write_levels
    from .voxelizer import EmbedEngine
    mesh, cfg = _mesh(c), _embed_cfg(c)
    grid, table = EmbedEngine(mesh, cfg).run()
    g = grid.to_numpy()
    lengths, _, cmap = table.to_numpy()
    paths = write_levels(c["out"], g, cfg, lengths, cmap)
    q = lengths[lengths >= 0]
    summary = {"faces": int(mesh.n_faces), "levels": [int(x) for x in np.diff(g["level_start"][:cfg.l_max + 1])],
               "blocks": int(grid.n_used), "boundary_blocks": int(table.n_b), "links": int(q.size),
               "q_min": float(q.min()) if q.size else None, "q_max": float(q.max()) if q.size else None,
               "files": [os.path.basename(p) for p in paths]}
    with open(os.path.join(c["out"], "summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary))
    return 0


def cmd_bench(c) -> int:
    import numpy as np
    import torch
    from .voxelizer import EmbedEngine
    mesh, cfg = _mesh(c), _embed_cfg(c)
    eng = EmbedEngine(mesh, cfg)
    for _ in range(3):
        eng.run(timed=True)
    rows = []
    for _ in range(max(1, c["reps"])):
        eng.run(timed=True)
        torch.cuda.synchronize()
        rows.append(eng.timings())
    rep = {}
    for k in ("refinement", "binning", "voxelization", "boundary", "links", "total"):
        x = np.array([getattr(r, k) for r in rows])
        hw = 1.96 * x.std(ddof=1) / math.sqrt(len(x)) if len(x) > 1 else 0.0
        rep[k] = {"mean_ms": float(x.mean()), "ci95_ms": float(hw)}
    print(json.dumps({"faces": int(mesh.n_faces), "reps": len(rows), "timing": rep}))
    return 0


def cmd_simulate(c) -> int:
    import numpy as np
    import torch
    from .solver import FlowConfig, LbmHierarchy
    from .voxelizer import EmbedEngine
    if c["bc_scheme"].upper() not in ("IBB", "SBB") or c["interp_order"] not in ("linear", "cubic"):
        raise ConfigError("bc_scheme must be IBB|SBB and interp_order linear|cubic")
    mesh, cfg = _mesh(c), _embed_cfg(c)
    grid, table = EmbedEngine(mesh, cfg).run()
    L = grid.n_levels - 1
    d0 = c["diameter"] / cfg.dx0  # body size in level-0 cells (sphere primitive / bounding box)
    if c.get("stl") or c["primitive"] != "sphere":
        lo, hi = np.asarray(mesh.vertices).min(0), np.asarray(mesh.vertices).max(0)
        d0 = float((hi - lo).max()) / cfg.dx0
    flow = FlowConfig(Re=c["Re"], u_in=c["u_in"], D_s=d0, bc_scheme=c["bc_scheme"].upper(), open_x=True)
    h = LbmHierarchy(grid, table, flow, order=3 if c["interp_order"] == "cubic" else 1)
    h.init_equilibrium(1.0, (c["u_in"], 0.0, 0.0))
    fine = h.levels[L]
    os.makedirs(c["out"], exist_ok=True)
    rows = []
    for it in range(c["iters_total"]):
        h.step(1, force=True)
        if it >= c["sample_start"] and (it - c["sample_start"]) % max(1, c["sample_stride"]) == 0:
            f = fine.force.cpu().numpy()
            if not np.all(np.isfinite(f)):
                raise FloatingPointError(f"non-finite wall force at coarse step {it}")
            rows.append((it, *map(float, f)))
    torch.cuda.synchronize()
    with open(os.path.join(c["out"], "forces.csv"), "w") as fh:
        fh.write("coarse_step,F_x,F_y,F_z\n")
        for r in rows:
            fh.write(",".join(str(x) for x in r) + "\n")
    fx = float(np.mean([r[1] for r in rows])) if rows else None
    d_f = d0 * 2 ** L
    # C_D = 2 F_x / (u^2 A_ref): the frontal disc pi d^2 / 4 is the sphere's
    # reference area; for other bodies (d = largest bounding-box extent) the
    # same disc is only a convention, so C_D is reported for spheres alone
    sphere = not c.get("stl") and c["primitive"] == "sphere"
    area = np.pi * d_f * d_f / 4.0
    cd = 2.0 * fx / (c["u_in"] ** 2 * area) if (fx is not None and sphere) else None
    summary = {"levels": grid.n_levels, "taus": h.taus, "substeps": h.substeps, "samples": len(rows),
               "F_x_mean_lattice": fx, "C_D": cd, "D_s_finest_cells": d_f,
               "reference_area_finest_cells2": area,
               "area_convention": "pi D^2/4 (sphere frontal disc)" if sphere else
               "C_D not reported: non-sphere body; F_x / (u^2 A / 2) with A = pi d^2/4, d = largest extent"}
    print(json.dumps(summary))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2512_01251_b200")
    ap.add_argument("command", choices=["voxelize", "bench", "simulate"])
    ap.add_argument("--config")
    ap.add_argument("--stl")
    ap.add_argument("--primitive", choices=["sphere", "torus"])
    ap.add_argument("--nx", type=int)
    ap.add_argument("--lmax", type=int)
    ap.add_argument("--nspec", type=int)
    ap.add_argument("--dspec", type=float)
    ap.add_argument("--out")
    ap.add_argument("--reps", type=int)
    a = ap.parse_args(argv)
    try:
        c = load_config(a.config) if a.config else dict(DEFAULTS)
    except (OSError, ConfigError) as ex:
        print(f"config error: {ex}", file=sys.stderr)
        return 2
    for k, v in (("stl", a.stl), ("primitive", a.primitive), ("N_x", a.nx), ("L_max", a.lmax),
                 ("N_spec", a.nspec), ("d_spec", a.dspec), ("out", a.out), ("reps", a.reps)):
        if v is not None:
            c[k] = v
    try:
        if a.command == "simulate":
            return cmd_simulate(c)
        return cmd_voxelize(c) if a.command == "voxelize" else cmd_bench(c)
    except Exception as ex:  # non-zero exit with a message on any pipeline error
        print(f"{a.command}: {type(ex).__name__}: {ex}", file=sys.stderr)
        return 1
