"""Command line (SPEC.md run_cli / load_config):

  python -m paper_2512_01251_b200 voxelize --config run.cfg | [--stl F | --primitive sphere|torus]
                                          [--nx 64 --lmax 4 --nspec 2 --dspec 0.05 --out DIR]
  python -m paper_2512_01251_b200 bench    (same options) [--reps 20]

voxelize: embed the geometry on the GPU, write one legacy ASCII VTK file per
level (cell masks; cut-link counts on the finest level) and a JSON summary of
the grid and the LinkTable.  bench: repeat the embedding and print the
TimingReport (mean and 95% confidence half-width per stage group, the paper's
Table 2 grouping).  simulate (the full multi-level LBM) is not built: exit 2.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
from typing import Dict

KEYS = {"stl": str, "primitive": str, "subdivisions": int, "torus_m": int, "torus_n": int,
        "N_x": int, "L_max": int, "N_spec": int, "d_spec": float, "out": str, "reps": int}
DEFAULTS = {"primitive": "sphere", "subdivisions": 4, "torus_m": 280, "torus_n": 200, "N_x": 64,
            "L_max": 3, "N_spec": 2, "d_spec": 0.05, "out": "voxforest_out", "reps": 20}


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
    return make_icosphere((0.5, 0.5, 0.5), 0.5, c["subdivisions"])


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
    if a.command == "simulate":
        print("simulate: the multi-level LBM solver is not built (only the single-level LUT "
              "consumer, solver.py)", file=sys.stderr)
        return 2
    try:
        return cmd_voxelize(c) if a.command == "voxelize" else cmd_bench(c)
    except Exception as ex:  # non-zero exit with a message on any pipeline error
        print(f"{a.command}: {type(ex).__name__}: {ex}", file=sys.stderr)
        return 1
