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
    """Midpoint subdivision until every edge < l_spec (geometry.py:355-403).

    Vectorised breadth-first variant: every face with an edge >= l_spec is
    split into four per pass.  The resulting face set equals the reference's
    depth-first result up to face order (both split exactly the same
    triangles), which the engine does not depend on beyond face ids."""
    if l_spec <= 0:
        raise MeshError("l_spec must be positive")
    verts = mesh.vertices
    faces = mesh.faces_indexed
    done = []
    while True:
        v = verts[faces]
        e = np.stack([np.linalg.norm(v[:, (k + 1) % 3] - v[:, k], axis=1) for k in range(3)], 1)
        big = e.max(axis=1) >= l_spec
        done.append(faces[~big])
        if not big.any():
            break
        verts, faces = _split_plain(verts, faces[big])
    out = np.concatenate(done, axis=0)
    if len(out) == len(mesh.faces_indexed) and np.array_equal(out, mesh.faces_indexed):
        return mesh
    return TriangleMesh(verts, out)


def _split_plain(verts, faces):
    a, b, c = faces[:, 0], faces[:, 1], faces[:, 2]
    e = np.stack([np.stack([a, b], 1), np.stack([b, c], 1), np.stack([c, a], 1)], 1).reshape(-1, 2)
    key = np.sort(e, axis=1)
    uniq, inv = np.unique(key, axis=0, return_inverse=True)
    mid = (verts[uniq[:, 0]] + verts[uniq[:, 1]]) / 2.0
    ids = len(verts) + inv.reshape(-1)
    nv = np.concatenate([verts, mid], axis=0)
    ab, bc, ca = ids.reshape(-1, 3).T
    out = np.stack([np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
                    np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)], 1).reshape(-1, 3)
    return nv, out
