"""Host-side triangle-mesh container and synthetic mesh generators.

The GPU engine only needs the two arrays the reference ``TriangleMesh`` exposes
(``faces_coord`` record-major (F, 9) f64 and unit ``normals`` (F, 3) f64,
/root/reference/pkg/src/voxforest/geometry.py:86-90); any object with those
fields (including the reference class itself) is accepted by the API.  This
module provides a minimal look-alike so the engine runs where the reference is
not installed (the GPU box), plus vectorised generators for the benchmark
meshes: the icosphere of geometry.py:297-327 and the torus grid.

Mesh generation is host preprocessing and is never timed.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import MeshError

__all__ = ["TriangleMesh", "Aabb", "make_icosphere", "make_torus", "translate",
           "l_spec_bound", "refine_faces", "mesh_arrays"]


@dataclass(frozen=True)
class Aabb:
    lo: np.ndarray
    hi: np.ndarray


class TriangleMesh:
    """Duck-type compatible with geometry.py:65-111 (3D only).

    Normals follow ``_face_normals`` (geometry.py:114-124) operation for
    operation: ``np.cross`` of the two edges from vertex 0, divided by the
    row norm.
    """

    def __init__(self, vertices, faces_indexed, dim=3):
        self.vertices = np.ascontiguousarray(vertices, dtype=np.float64)
        self.faces_indexed = np.ascontiguousarray(faces_indexed, dtype=np.int64)
        self.dim = int(dim)
        if self.dim != 3:
            raise NotImplementedError("the B200 engine is 3D only (SURVEY §2)")
        if self.faces_indexed.ndim != 2 or self.faces_indexed.shape[1] != 3:
            raise MeshError("faces_indexed must be (F, 3)")
        if len(self.faces_indexed) == 0:
            raise MeshError("empty mesh (zero faces)")
        if self.faces_indexed.max() >= len(self.vertices):
            raise MeshError("face index out of range")
        fc = self.vertices[self.faces_indexed.reshape(-1)].reshape(len(self.faces_indexed), 9)
        self.faces_coord = np.ascontiguousarray(fc)
        v = self.vertices[self.faces_indexed]
        n = np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0])
        lens = np.linalg.norm(n, axis=1)
        if np.any(lens == 0.0):
            raise MeshError("degenerate face (zero normal)")
        self.normals = n / lens[:, None]

    @classmethod
    def from_arrays(cls, vertices, faces_indexed, faces_coord, normals, dim=3):
        """A mesh whose derived arrays were built elsewhere (GPU STL
        ingestion, stl.py) with the same operations as __init__."""
        m = cls.__new__(cls)
        m.vertices = np.ascontiguousarray(vertices, dtype=np.float64)
        m.faces_indexed = np.ascontiguousarray(faces_indexed, dtype=np.int64)
        m.dim = int(dim)
        m.faces_coord = np.ascontiguousarray(faces_coord, dtype=np.float64)
        m.normals = np.ascontiguousarray(normals, dtype=np.float64)
        return m

    @property
    def faces_coord_cm(self) -> np.ndarray:
        """Column-major copy of faces_coord (geometry.py:88), built on demand."""
        cm = self.__dict__.get("_faces_coord_cm")
        if cm is None:
            cm = self.__dict__["_faces_coord_cm"] = np.ascontiguousarray(self.faces_coord.T)
        return cm

    @property
    def n_faces(self) -> int:
        return len(self.faces_indexed)

    def aabb(self) -> Aabb:
        return Aabb(self.vertices.min(axis=0), self.vertices.max(axis=0))

    def face_areas(self) -> np.ndarray:
        v = self.vertices[self.faces_indexed]
        return 0.5 * np.linalg.norm(np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]), axis=1)

    def max_edge_lengths(self) -> np.ndarray:
        v = self.vertices[self.faces_indexed]
        e = [np.linalg.norm(v[:, (i + 1) % 3] - v[:, i], axis=1) for i in range(3)]
        return np.max(e, axis=0)


def mesh_arrays(mesh):
    """(faces_coord (F,9), normals (F,3)) as contiguous f64 from any mesh
    object exposing the reference TriangleMesh fields (geometry.py:86-90)."""
    if int(getattr(mesh, "dim", 3)) != 3:
        raise NotImplementedError("2D meshes are not supported by the B200 engine (SURVEY §2)")
    fc = np.ascontiguousarray(mesh.faces_coord, dtype=np.float64).reshape(-1, 9)
    nrm = np.ascontiguousarray(mesh.normals, dtype=np.float64).reshape(-1, 3)
    if fc.shape[0] != nrm.shape[0] or fc.shape[0] == 0:
        raise MeshError("faces_coord / normals mismatch or empty mesh")
    return fc, nrm


_T = (1.0 + np.sqrt(5.0)) / 2.0
_ICO_V = np.array([
    [-1, _T, 0], [1, _T, 0], [-1, -_T, 0], [1, -_T, 0],
    [0, -1, _T], [0, 1, _T], [0, -1, -_T], [0, 1, -_T],
    [_T, 0, -1], [_T, 0, 1], [-_T, 0, -1], [-_T, 0, 1]], dtype=np.float64)
_ICO_F = np.array([
    [0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
    [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
    [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
    [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int64)


def _subdivide(verts, faces):
    """One midpoint-subdivision pass with the vertex numbering and face order
    of geometry.py:308-327 (midpoints numbered at first encounter scanning faces
    in order, edges (a,b), (b,c), (c,a); children [a,ab,ca],[b,bc,ab],[c,ca,bc],
    [ab,bc,ca]); vectorised instead of a Python dict walk."""
    a, b, c = faces[:, 0], faces[:, 1], faces[:, 2]
    e = np.stack([np.stack([a, b], 1), np.stack([b, c], 1), np.stack([c, a], 1)], 1).reshape(-1, 2)
    key = np.sort(e, axis=1)
    uniq, first, inv = np.unique(key, axis=0, return_index=True, return_inverse=True)
    order = np.argsort(first, kind="stable")         # first-encounter order
    rank = np.empty_like(order)
    rank[order] = np.arange(len(order))
    ids = len(verts) + rank[inv.reshape(-1)]
    m = (verts[uniq[order, 0]] + verts[uniq[order, 1]]) / 2.0
    m = m / np.sqrt(np.sum(m * m, axis=1))[:, None]
    nv = np.concatenate([verts, m], axis=0)
    ab, bc, ca = ids.reshape(-1, 3).T
    out = np.stack([np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
                    np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)], 1).reshape(-1, 3)
    return nv, out


def make_icosphere(center=(0.5, 0.5, 0.5), diameter=0.5, subdivisions=5) -> TriangleMesh:
    """Icosphere of geometry.py:297-305 (20*4^k faces; k=5 -> 20,480)."""
    verts = _ICO_V / np.sqrt(np.sum(_ICO_V[0] * _ICO_V[0]))
    faces = _ICO_F
    for _ in range(int(subdivisions)):
        verts, faces = _subdivide(verts, faces)
    verts = np.asarray(center, dtype=np.float64) + (diameter / 2.0) * verts
    return TriangleMesh(verts, faces)


def make_torus(m, n, R=0.25, r=0.1, center=(0.5, 0.5, 0.5)) -> TriangleMesh:
    """Torus grid of SURVEY.md §8d: 2*m*n faces, axis z, outward normals.
    m=280,n=200 -> 112,000 faces (C2); m=3000,n=1200 -> 7,200,000 (C4)."""
    i = np.arange(m)
    j = np.arange(n)
    u = 2.0 * np.pi * i / m
    v = 2.0 * np.pi * j / n
    U, V = np.meshgrid(u, v, indexing="ij")
    rr = R + r * np.cos(V)
    verts = np.stack([rr * np.cos(U), rr * np.sin(U), r * np.sin(V)], axis=-1).reshape(-1, 3)
    verts = verts + np.asarray(center, dtype=np.float64)
    I, J = np.meshgrid(i, j, indexing="ij")
    a = (I * n + J).reshape(-1)
    b = (((I + 1) % m) * n + J).reshape(-1)
    c = (((I + 1) % m) * n + (J + 1) % n).reshape(-1)
    d = (I * n + (J + 1) % n).reshape(-1)
    faces = np.concatenate([np.stack([a, b, c], 1), np.stack([a, c, d], 1)], axis=0)
    return TriangleMesh(verts, faces)


def translate(mesh: TriangleMesh, offset) -> TriangleMesh:
    """Rigid translation (robustness variants)."""
    return TriangleMesh(mesh.vertices + np.asarray(offset, dtype=np.float64), mesh.faces_indexed)


def l_spec_bound(domain_lengths, n_spec, l_max, n_b) -> float:
    """geometry.py:406-410 / PAPER.md:393-396."""
    lmin = float(np.min(domain_lengths))
    return lmin * (0.95 * n_spec) / (2 ** (l_max - 1) * n_b)


def refine_faces(mesh: TriangleMesh, l_spec: float) -> TriangleMesh:
    """Midpoint subdivision until every edge < l_spec (geometry.py:355-403),
    with the reference's face AND vertex numbering.

    The reference walks a LIFO stack seeded with the faces in order
    (geometry.py:383-397): it pops the last face, splits it into
    [a,ab,ca], [b,bc,ab], [c,ca,bc], [ab,bc,ca] (pushed in that order, so
    popped last-child first), emits faces that are fine enough, numbers each
    new midpoint at its first creation (deduplicated by exact coordinates,
    including against the input vertices, geometry.py:370-378) and finally
    reverses the emitted list (:399).  Hence:
      * face order = input faces in order, each replaced by the leaves of its
        split tree in natural child order (pre-order, children 0..3);
      * vertex order = input vertices, then midpoints in the order the split
        faces are popped: input faces last to first, children 3..0, pre-order;
        each split face creates ab, bc, ca in that order.
    This is reproduced breadth-first and vectorised: the tree is built level
    by level with provisional midpoint handles, then faces and midpoints are
    renumbered by those two orders.  The per-face test uses the 1-D
    ``np.linalg.norm`` of the reference (a BLAS dot); the vectorised norm is
    recomputed that way wherever it is within 1e-12 relative of l_spec."""
    if l_spec <= 0:
        raise MeshError("l_spec must be positive")
    if np.all(mesh.max_edge_lengths() < l_spec):    # geometry.py:361-362
        return mesh
    V0 = mesh.vertices
    n0 = len(V0)
    # per tree node: vertex handles (h < n0: input vertex; else midpoint
    # handle n0 + 3 * split_index + k), root face, path code, depth
    faces = mesh.faces_indexed.astype(np.int64)
    root = np.arange(len(faces), dtype=np.int64)
    path = np.zeros(len(faces), dtype=np.int64)     # child digits, base 4
    depth = 0
    coords = [V0]                                   # coordinates of every handle
    leaves, splits = [], []                         # (faces, root, path, depth)
    n_split = 0
    while len(faces):
        P = np.concatenate(coords, axis=0) if len(coords) > 1 else coords[0]
        v = P[faces]
        e = np.stack([np.linalg.norm(v[:, (k + 1) % 3] - v[:, k], axis=1) for k in range(3)], 1)
        emax = e.max(axis=1)
        near = np.nonzero(np.abs(emax - l_spec) <= 1e-12 * l_spec)[0]
        for i in near:                              # the reference's own per-face norms
            pa, pb, pc = v[i]
            emax[i] = max(np.linalg.norm(pb - pa), np.linalg.norm(pc - pb), np.linalg.norm(pa - pc))
        big = ~(emax < l_spec)
        leaves.append((faces[~big], root[~big], path[~big], depth))
        if not big.any():
            break
        fb, rb, pb_ = faces[big], root[big], path[big]
        k = len(fb)
        vb = v[big]
        mid = np.stack([(vb[:, 0] + vb[:, 1]) / 2.0, (vb[:, 1] + vb[:, 2]) / 2.0,
                        (vb[:, 2] + vb[:, 0]) / 2.0], 1)            # ab, bc, ca
        h = n0 + 3 * (n_split + np.arange(k, dtype=np.int64))
        ab, bc, ca = h, h + 1, h + 2
        splits.append((rb, pb_, depth, mid.reshape(-1, 3)))
        coords.append(mid.reshape(-1, 3))
        n_split += k
        a, b, c = fb[:, 0], fb[:, 1], fb[:, 2]
        faces = np.stack([np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
                          np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)], 1).reshape(-1, 3)
        root = np.repeat(rb, 4)
        path = (np.repeat(pb_, 4) << 2) | np.tile(np.arange(4, dtype=np.int64), k)
        depth += 1
    dmax = depth + 1

    def code(p, d, flip):
        # pre-order key over paths of mixed depth: digits 1..4, padded with 0
        out = np.zeros(len(p), dtype=np.int64)
        for i in range(dmax):
            sh = d - 1 - i                          # digit i of a depth-d path
            dig = np.where(sh >= 0, (p >> (2 * np.maximum(sh, 0))) & 3, -1)
            if flip:
                dig = np.where(dig >= 0, 3 - dig, -1)
            out = out * 5 + (dig + 1)
        return out

    # midpoints in pop order: roots descending, children 3..0, pre-order
    r_s = np.concatenate([s[0] for s in splits])
    d_s = np.concatenate([np.full(len(s[0]), s[2], np.int64) for s in splits])
    c_s = code(np.concatenate([s[1] for s in splits]), d_s, True)
    pop = np.lexsort((c_s, -r_s))                   # split index in pop order
    cand = np.concatenate([s[3] for s in splits]).reshape(-1, 3, 3)[pop].reshape(-1, 3)
    cand_h = (n0 + 3 * pop[:, None] + np.arange(3)[None, :]).reshape(-1)

    def keys(x):
        x = np.ascontiguousarray(x + 0.0)           # -0.0 == 0.0 as a dict key
        return x.view(np.dtype((np.void, 24))).reshape(-1)

    k0, kc = keys(V0), keys(cand)
    # input vertices: dict built in order, so a duplicated coordinate maps to
    # its LAST index (geometry.py:364)
    u0, inv0 = np.unique(k0[::-1], return_index=True)
    last0 = n0 - 1 - inv0
    pos = np.searchsorted(u0, kc)
    pos_c = np.minimum(pos, len(u0) - 1)
    hit = u0[pos_c] == kc
    lut = np.empty(n0 + 3 * n_split, dtype=np.int64)
    lut[:n0] = np.arange(n0)
    new = ~hit
    kn = kc[new]
    un, first, invn = np.unique(kn, return_index=True, return_inverse=True)
    rank = np.empty(len(un), dtype=np.int64)
    rank[np.argsort(first, kind="stable")] = np.arange(len(un))
    ids = np.empty(len(kc), dtype=np.int64)
    ids[hit] = last0[pos_c[hit]]
    ids[new] = n0 + rank[invn.reshape(-1)]
    lut[cand_h] = ids
    newv = cand[new][np.sort(first)]
    verts = np.concatenate([V0, newv], axis=0)
    # leaves in the reversed emission order: roots ascending, children 0..3
    f_l = np.concatenate([x[0] for x in leaves])
    r_l = np.concatenate([x[1] for x in leaves])
    d_l = np.concatenate([np.full(len(x[0]), x[3], np.int64) for x in leaves])
    c_l = code(np.concatenate([x[2] for x in leaves]), d_l, False)
    out = lut[f_l[np.lexsort((c_l, r_l))]]
    return TriangleMesh(verts, out)
