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
