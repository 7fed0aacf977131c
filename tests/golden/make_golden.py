"""Generate golden vectors by importing the REFERENCE package (run in the
build container only; /root/reference does not exist on the GPU box).

  PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/vf_numba python tests/golden/make_golden.py

Outputs (committed):
  sat_golden.npz  -- tri (n,9) f64, box (n,6) f64, out (n,) bool from the
                     reference tri_aabb_overlap_3d (geometry.py:484-500).
                     Cases: random pairs, plus the exact box shapes the
                     pipeline builds (x-row slabs, Δx-expanded bin boxes,
                     ε-boxes at link intersection points) around an icosphere
                     and a torus, concentrated on touching / near-miss cases.
  lattice_golden.npz -- D3Q27 c, opposite (lattice.py:19-97).
  mesh_golden.npz -- reference make_primitive sphere k=2 vertices / faces /
                     normals, to pin the local icosphere generator.
"""
import importlib.util
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src/voxforest"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))


def load_ref(name):
    spec = importlib.util.spec_from_file_location("vref_" + name, os.path.join(REF, name + ".py"))
    m = importlib.util.module_from_spec(spec)
    sys.modules["vref_" + name] = m
    spec.loader.exec_module(m)
    return m


def pipeline_cases(rng, fc, nrm, dx, eps, lx, n):
    """(tri, box) pairs shaped like the pipeline's SAT calls."""
    tris, boxes = [], []
    F = len(fc)
    for _ in range(n):
        f = rng.integers(F)
        v = fc[f]
        kind = rng.integers(3)
        lo = np.minimum(np.minimum(v[0:3], v[3:6]), v[6:9])
        hi = np.maximum(np.maximum(v[0:3], v[3:6]), v[6:9])
        if kind == 0:  # x-row slab through a lattice row near the face
            j = np.floor(lo[1] / dx) + rng.integers(-1, 3)
            k = np.floor(lo[2] / dx) + rng.integers(-1, 3)
            y, z = (j + 0.5) * dx, (k + 0.5) * dx
            if rng.random() < 0.3:  # snap the row onto a vertex (touching)
                y, z = v[3 * rng.integers(3) + 1], v[3 * rng.integers(3) + 2]
            box = [0.0, y - eps, z - eps, lx, y + eps, z + eps]
        elif kind == 1:  # expanded bin box
            h = 4 * dx
            b = np.floor(lo / h) + rng.integers(-1, 3, size=3)
            box = list(b * h - dx) + list((b + 1) * h + dx)
        else:  # eps box at a point on / near the face plane
            w = rng.dirichlet([1, 1, 1])
            p = w[0] * v[0:3] + w[1] * v[3:6] + w[2] * v[6:9]
            if rng.random() < 0.5:  # onto an edge
                a, b2 = rng.choice(3, 2, replace=False)
                t = rng.random()
                p = (1 - t) * v[3 * a:3 * a + 3] + t * v[3 * b2:3 * b2 + 3]
            p = p + rng.normal(size=3) * eps * rng.choice([0.0, 0.5, 1.0, 2.0, 10.0])
            box = list(p - eps) + list(p + eps)
        tris.append(v)
        boxes.append(box)
    return np.array(tris), np.array(boxes)


def main():
    geom = load_ref("geometry")
    lat = load_ref("lattice")
    from paper_2512_01251_b200.mesh import make_torus
    rng = np.random.default_rng(20251217)

    # random pairs
    n_rand = 4000
    tri_r = rng.random((n_rand, 9))
    c = rng.random((n_rand, 3))
    s = rng.random((n_rand, 3)) * 0.5
    box_r = np.concatenate([c - s, c + s], axis=1)
    # degenerate-ish: axis aligned / touching boxes built from vertices
    n_t = 2000
    tri_t = rng.integers(0, 8, size=(n_t, 9)) / 8.0
    lo = rng.integers(0, 8, size=(n_t, 3)) / 8.0
    box_t = np.concatenate([lo, lo + rng.integers(0, 4, size=(n_t, 3)) / 8.0], axis=1)

    sph = geom.make_primitive(geom.PrimitiveSpec("sphere", (0.5, 0.5, 0.5), 0.5, 4))
    tor = make_torus(60, 40)
    eps = 1e-9
    parts_t, parts_b = [tri_r, tri_t], [box_r, box_t]
    for mesh, n in ((sph, 7000), (tor, 7000)):
        for dx in (1 / 64, 1 / 256):
            t, b = pipeline_cases(rng, mesh.faces_coord, mesh.normals, dx, eps, 1.0, n // 2)
            parts_t.append(t)
            parts_b.append(b)
    tri = np.concatenate(parts_t)
    box = np.concatenate(parts_b)
    out = np.array([geom.tri_aabb_overlap_3d(*t, *b) for t, b in zip(tri, box)], dtype=bool)
    np.savez_compressed(os.path.join(HERE, "sat_golden.npz"), tri=tri, box=box, out=out)
    print("sat_golden:", len(out), "cases,", int(out.sum()), "true")

    np.savez_compressed(os.path.join(HERE, "lattice_golden.npz"), c=lat.D3Q27.c,
                        opposite=lat.D3Q27.opposite, w=lat.D3Q27.w)
    s2 = geom.make_primitive(geom.PrimitiveSpec("sphere", (0.5, 0.5, 0.5), 0.5, 2))
    np.savez_compressed(os.path.join(HERE, "mesh_golden.npz"), vertices=s2.vertices,
                        faces=s2.faces_indexed, normals=s2.normals,
                        faces_coord=s2.faces_coord)
    print("lattice/mesh golden written")


if __name__ == "__main__":
    main()
