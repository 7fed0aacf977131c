"""Shared LBM test cases: an embedded sphere (oracle embed) and a perturbed
initial state of its finest level."""
import numpy as np

from paper_2512_01251_b200 import EmbedConfig, make_icosphere


def sphere_case(O, l_max=3, n_x=32, sub=3):
    mesh = make_icosphere((0.5, 0.5, 0.5), 0.4, sub)
    cfg = EmbedConfig(n_x=n_x, l_max=l_max)
    cap = cfg.block_capacity(float(mesh.face_areas().sum()))
    ref = O.embed(mesh.faces_coord, mesh.normals, cfg, cap)
    return mesh, cfg, ref


def level_arrays(ref, L):
    g = ref.grid
    s, e = int(g.level_start[L]), int(g.level_start[L + 1])
    return g, s, e


def perturbed_state(masks, s, e, rng, u=(0.03, 0.0, 0.0), amp=1e-3):
    from paper_2512_01251_b200.solver import equilibrium
    n = (e - s) * 64
    feq = equilibrium(np.ones(n), np.broadcast_to(np.asarray(u), (n, 3)))  # (n, 27)
    f = (feq * (1.0 + amp * rng.standard_normal(feq.shape))).T.astype(np.float32)
    solid = np.asarray(masks).reshape(-1)[64 * s:64 * e] == 1
    f[:, solid] = 0.0
    return np.ascontiguousarray(f)


# ---- interface exchange cases ----------------------------
W3 = (-7 / 128, 105 / 128, 35 / 128, -5 / 128)


def level_cells(g, s, e):
    """Global cell coordinates (n, 3) of the blocks [s, e) in state order."""
    c = np.asarray(g["coords"])[s:e, :3].astype(np.int64)
    t = np.arange(64)
    loc = np.stack([t & 3, (t >> 2) & 3, t >> 4], 1)
    return (4 * c[:, None, :] + loc[None]).reshape(-1, 3)


def poly_field(cells, n_cells, kind):
    """(27, n) float32 field f_q = (1 + q/100) P(x), x = (cell + 1/2) / n_cells:
    P trilinear ("linear") or tensor-cubic ("cubic"), "const" = 1."""
    x = (cells + 0.5) / n_cells
    X, Y, Z = x[:, 0], x[:, 1], x[:, 2]
    if kind == "const":
        P = np.ones(len(x))
    elif kind == "linear":
        P = 1.0 + 0.3 * X - 0.2 * Y + 0.25 * Z + 0.1 * X * Y * Z
    else:
        P = 1.0 + 0.3 * X - 0.2 * Y + 0.25 * Z + 0.4 * X ** 3 - 0.3 * Y ** 2 * Z + 0.2 * X * Y ** 3 * Z ** 2
    q = np.arange(27)[:, None]
    return np.ascontiguousarray(((1.0 + q / 100.0) * P[None]).astype(np.float32))


def exact_ghosts(g, sf, ef, sc, ec, order):
    """Fine ghost cells (state indices) of blocks [sf, ef) whose full stencil
    of the given order lies on non-SOLID cells of coarse blocks [sc, ec)."""
    masks = np.asarray(g["masks"]).reshape(-1, 64)
    cc = level_cells(g, sc, ec)
    size = cc.max(0) + 8
    dense = np.full(tuple(size), 255, np.uint8)
    dense[cc[:, 0], cc[:, 1], cc[:, 2]] = masks[sc:ec].reshape(-1)
    fc = level_cells(g, sf, ef)
    fm = masks[sf:ef].reshape(-1)
    ks = (-1, 0, 1, 2) if order == 3 else (0, 1)
    off = np.array([(a, b, c) for c in ks for b in ks for a in ks])
    x = np.nonzero(fm == 3)[0]
    G = fc[x] >> 1
    sd = np.where(fc[x] & 1, 1, -1)
    p = G[:, None, :] + sd[:, None, :] * off[None]
    inside = ((p >= 0) & (p < size)).all(-1)
    pc = np.clip(p, 0, size - 1)
    m = dense[pc[..., 0], pc[..., 1], pc[..., 2]]
    ok = (inside & (m != 1) & (m != 255)).all(1)
    out = x[ok]
    return np.asarray(out, dtype=np.int64)
