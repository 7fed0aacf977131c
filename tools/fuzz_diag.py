"""Diagnose GPU-vs-oracle mismatches of the margin fuzz (tests/fuzz_meshes.py):
for each case print the differing grid keys and LUT entries (block, coords,
q, cell, GPU value, oracle value) as JSON lines.

  python tools/fuzz_diag.py nx24_l4:0 nx32:3 ..."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402
from fuzz_meshes import fuzz_case  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2512_01251_b200.lattice import D3Q27_C  # noqa: E402
from paper_2512_01251_b200.voxelizer import EmbedEngine  # noqa: E402


def diag(name, seed, small_ext=None):
    from paper_2512_01251_b200 import _lib
    lib = _lib.require_cuda()
    old = lib.vf_set_link_small_ext(small_ext) if small_ext is not None else None
    mesh, cfg = fuzz_case(name, seed)
    grid, table = EmbedEngine(mesh, cfg).run()
    torch.cuda.synchronize()
    if old is not None:
        lib.vf_set_link_small_ext(old)
    ref = O.embed(mesh.faces_coord, mesh.normals, cfg, capacity=grid.capacity)
    g = grid.to_numpy()
    out = {"case": f"{name}:{seed}", "small_ext": small_ext, "faces": mesh.n_faces}
    n = ref.grid.n_used
    out["n_used"] = [int(g["level_start"][grid.n_levels]), n]
    for k in ("coords", "nbr", "nbr_child", "child", "bflags", "masks"):
        a, b = g[k][:n], getattr(ref.grid, k)[:n]
        if a.shape != b.shape or not np.array_equal(a, b):
            bad = np.argwhere(a != b) if a.shape == b.shape else []
            out[k] = {"n": len(bad), "first": [list(map(int, x)) for x in bad[:10]]}
    lg = table.lengths.cpu().numpy()
    lr = ref.lengths
    cmap = ref.contraction_map
    inv = np.full(max(ref.n_b, 1), -1)
    inv[cmap[cmap >= 0]] = np.nonzero(cmap >= 0)[0]
    if lg.shape == lr.shape:
        neg = lr < 0
        bad = np.argwhere((lg < 0) != neg)
        pos = ~neg & (lg >= 0)
        rel = np.zeros_like(lr)
        rel[pos] = np.abs(lg[pos] - lr[pos]) / np.abs(lr[pos])
        bad2 = np.argwhere(rel > 1e-5)
        Lf = cfg.l_max - 1
        dx = cfg.dx(Lf)
        ent = []
        for s, q, t in list(bad[:20]) + list(bad2[:10]):
            b = int(inv[s])
            c = ref.grid.coords[b]
            cell = (4 * c[:3] + np.array([t % 4, (t // 4) % 4, t // 16]) + 0.5) * dx
            ent.append({"slot": int(s), "block": b, "coords": c.tolist(), "q": int(q), "t": int(t),
                        "c": D3Q27_C[q].tolist(), "cell": cell.tolist(), "gpu": float(lg[s, q, t]),
                        "oracle": float(lr[s, q, t]), "mask": int(ref.grid.masks[b, t])})
        out["lut_pattern_bad"] = int(len(bad))
        out["lut_value_bad"] = int(len(bad2))
        out["entries"] = ent
    else:
        out["lut_shape"] = [list(lg.shape), list(lr.shape)]
    return out


if __name__ == "__main__":
    for a in sys.argv[1:]:
        parts = a.split(":")
        se = float(parts[2]) if len(parts) > 2 else None
        print(json.dumps(diag(parts[0], int(parts[1]), se)), flush=True)
