"""Adversarial meshes for the FP32 fast-accept classifiers.

The GPU decides most x-row and cut-link SAT outcomes with FP32 edge
functions (`RowClass`, vf_common.cuh; `point_class` / `link_fast`,
vf_linklen.cu) and hands only a margin band to the exact FP64 SAT of
geometry.py:441-500.  These generators put triangle features exactly where
those margins are tight:

  * vertices and edges at {0, eps/2, eps, 2 eps, 0.1 tol, tol, 10 tol} from
    the x-rows (y_j, z_k) of every level and from the 13 cut-link lines
    through finest-level nodes (tol = 1e-5 (ext + dx) + 6 eps, the margin the
    classifiers use);
  * slivers (third vertex 1e-9 .. 1e-4 of the edge off the line);
  * normals with |n_x| within 1e-6 of 1e-3 (the fast-accept conditioning
    threshold) and near-x-parallel faces;
  * faces touching x = 0 and x = l_x, and in the 1e-6 l_x end band;
  * faces from 0.2 to ~5 finest cells (both cut-link enumeration kernels).

The features are anchored at lattice nodes within a shell around a closed
icosphere, which is part of the mesh, so near-wall refinement carries them
down to the finest level (where the link lines live).  The result is an
open triangle soup plus one closed surface: the embed is deterministic for
it, and the oracle is the checker.
"""
from __future__ import annotations

import numpy as np

from paper_2512_01251_b200 import EmbedConfig, make_icosphere
from paper_2512_01251_b200.lattice import D3Q27_C
from paper_2512_01251_b200.mesh import TriangleMesh

_DIRS = np.array([D3Q27_C[q] for q in range(1, 27, 2)], dtype=np.float64)  # 13 representatives


def _unit(rng, n=3):
    v = rng.normal(size=n)
    return v / np.linalg.norm(v)


def _perp(rng, c):
    """random unit vector orthogonal to c"""
    c = c / np.linalg.norm(c)
    w = _unit(rng)
    w = w - np.dot(w, c) * c
    return w / np.linalg.norm(w)


def margin_soup(cfg: EmbedConfig, seed: int, n_feat: int = 2500, radius: float = 0.28):
    rng = np.random.default_rng(seed)
    L_f = cfg.l_max - 1
    dxf = cfg.dx(L_f)
    lx = float(cfg.domain[0])
    eps = cfg.eps
    center = np.array([0.5 * float(d) for d in cfg.domain])
    l_spec = min(cfg.domain) * 0.95 * cfg.n_spec / (2 ** (cfg.l_max - 1) * cfg.nb[0])
    tris = []

    def node(L):
        """a level-L lattice node near the sphere shell"""
        dx = cfg.dx(L)
        p = center + (radius + rng.uniform(-0.6, 0.6) * 4 * dxf) * _unit(rng)
        g = np.floor(p / dx)
        return (g + 0.5) * dx

    def delta(ext, dx):
        tol = 1e-5 * (ext + dx) + 6 * eps
        return rng.choice([0.0, 0.5 * eps, eps, 2 * eps, 0.1 * tol, tol, 10 * tol]) * rng.choice([-1.0, 1.0])

    def size():
        return dxf * (rng.uniform(0.2, 1.5) if rng.random() < 0.6 else rng.uniform(1.5, 5.0))

    def tri_from(v1, s):
        """v1 + two random edges of length ~s"""
        a, b = _unit(rng), _unit(rng)
        return [v1, v1 + s * a, v1 + s * rng.uniform(0.5, 1.0) * b]

    for _ in range(n_feat):
        kind = rng.integers(0, 9)
        s = size()
        L = int(rng.integers(0, cfg.l_max))
        dx = cfg.dx(L)
        if kind == 0:    # vertex near an x-row (y_j, z_k) of level L
            p = node(L)
            u = _unit(rng, 2)
            v1 = np.array([p[0] + rng.uniform(-0.5, 0.5) * dx, p[1] + delta(s, dx) * u[0],
                           p[2] + delta(s, dx) * u[1]])
            t = tri_from(v1, s)
        elif kind == 1:  # edge passing delta from an x-row (yz projection)
            p = node(L)
            ang = rng.uniform(0, 2 * np.pi)
            tyz = np.array([np.cos(ang), np.sin(ang)])
            nyz = np.array([-tyz[1], tyz[0]])
            m = np.array([p[0], *(p[1:] + delta(s, dx) * nyz)])
            e = np.array([rng.uniform(-1, 1), *tyz])
            a, b = rng.uniform(0.2, 0.8) * s, rng.uniform(0.2, 0.8) * s
            third = m + s * rng.uniform(0.3, 1.0) * np.array([rng.uniform(-1, 1), *(nyz * rng.choice([-1, 1]))])
            t = [m - a * e, m + b * e, third]
        elif kind == 2:  # vertex near a finest-level node (13 link lines through it)
            p = node(L_f)
            t = tri_from(p + delta(s, dxf) * _unit(rng), s)
        elif kind == 3:  # edge passing delta from a link line through a node
            p = node(L_f)
            c = _DIRS[rng.integers(0, 13)]
            w = _perp(rng, c)
            e = np.cross(c, w)
            e = e / np.linalg.norm(e)
            e = e + rng.uniform(-0.3, 0.3) * c / np.linalg.norm(c)   # stay off-parallel
            m = p + delta(s, dxf) * w + rng.uniform(-0.5, 0.5) * dxf * c
            a, b = rng.uniform(0.2, 0.8) * s, rng.uniform(0.2, 0.8) * s
            t = [m - a * e, m + b * e, m + s * rng.uniform(0.3, 1.0) * w * rng.choice([-1, 1])]
        elif kind == 4:  # sliver
            v1 = node(L) + rng.uniform(-0.5, 0.5, 3) * dx
            v2 = v1 + s * _unit(rng)
            h = rng.choice([1e-9, 1e-7, 1e-5, 1e-4]) * s
            t = [v1, v2, 0.5 * (v1 + v2) + h * _perp(rng, v2 - v1)]
        elif kind == 5:  # |n_x| within 1e-6 of 1e-3, or nearly x-parallel
            nx = rng.choice([1e-3, 1e-3 + 1e-6, 1e-3 - 1e-6, 1e-3 * (1 + 1e-9), 1e-12, 2e-12, 0.0])
            r = np.sqrt(1 - nx * nx)
            ang = rng.uniform(0, 2 * np.pi)
            n = np.array([nx * rng.choice([-1, 1]), r * np.cos(ang), r * np.sin(ang)])
            a = _perp(rng, n)
            b = np.cross(n, a)
            p = node(L)
            p = p + delta(s, dx) * _unit(rng)
            t = [p, p + s * a, p + s * (0.3 * a + 0.9 * b)]
        elif kind == 6:  # touching a domain face, just outside it, or in the 1e-6 l_x end band
            p = node(L)
            ax = 0 if rng.random() < 0.6 else int(rng.integers(1, 3))
            la = float(cfg.domain[ax])
            ta = 1e-6 * la
            x0 = rng.choice([0.0, la, ta, la - ta, ta * (1 + 1e-3), la - ta * (1 - 1e-3),
                             -0.3 * dxf, la + 0.3 * dxf, -eps, la + eps, -2 * dxf, la + 1.1 * dxf])
            v1 = p.copy()
            v1[ax] = x0
            v1[(ax + 1) % 3] += delta(s, dx) * rng.choice([-1, 1])
            t = tri_from(v1, s)
            if rng.random() < 0.5:   # an edge lying in the boundary plane
                t[1][ax] = x0
        elif kind == 7:  # vertex exactly on a node / row, edges along lattice axes
            p = node(L)
            ax = rng.permutation(3)
            t = [p, p + s * np.eye(3)[ax[0]], p + s * (np.eye(3)[ax[0]] * rng.uniform(0, 1) + np.eye(3)[ax[1]])]
        else:            # generic interior crossing
            t = tri_from(node(L) + rng.uniform(-0.5, 0.5, 3) * dx, s)
        t = np.array(t, dtype=np.float64)
        if rng.random() < 0.5:
            t = t[::-1].copy()                   # both orientations
        e = np.linalg.norm(np.roll(t, -1, axis=0) - t, axis=1)
        if e.max() >= 0.9 * l_spec or np.linalg.norm(np.cross(t[1] - t[0], t[2] - t[0])) == 0.0:
            continue
        tris.append(t)
    sph = make_icosphere(tuple(center), 2 * radius, 3)
    V = np.concatenate([sph.vertices, np.concatenate(tris)])
    F = np.concatenate([sph.faces_indexed, len(sph.vertices) + np.arange(3 * len(tris)).reshape(-1, 3)])
    return TriangleMesh(V, F)


def soup_capacity(cfg: EmbedConfig) -> int:
    """every block refined at every level: an upper bound on the forest"""
    return sum(cfg.n_root * 8 ** L for L in range(cfg.l_max))


FUZZ_CONFIGS = {
    "nx32": dict(n_x=32, l_max=3),
    "nx48": dict(n_x=48, l_max=3),                          # non-power-of-two dx
    "nx48_1.5x1x1": dict(n_x=48, l_max=3, domain=(1.5, 1.0, 1.0)),
    "nx24_l4": dict(n_x=24, l_max=4),                       # 1/96 dx, deeper
}


def fuzz_case(name: str, seed: int):
    kw = dict(FUZZ_CONFIGS[name])
    base = EmbedConfig(**kw)
    cfg = EmbedConfig(**kw, capacity=soup_capacity(base))
    return margin_soup(cfg, seed), cfg
