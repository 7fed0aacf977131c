"""SPEC domain types as dataclasses of torch CUDA tensors.

  BinLevel   SPEC.md:111-117   FilterMap SPEC.md:118-121
  ForestGrid SPEC.md:196-203   LinkTable SPEC.md:271-276
  DeviceMesh the uploaded face records (geometry.py:86-90 record-major coords +
             host unit normals, 96 B/face)

Every type has ``to_numpy()`` for oracle comparison.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np

from . import _lib
from .config import MAX_LEVELS, EmbedConfig
from .mesh import mesh_arrays


def _torch():
    import torch
    return torch


@dataclass
class DeviceMesh:
    """Packed device face records [F, 12] f64: v1 v2 v3 n."""
    faces: "object"          # torch.float64 (F, 12) cuda
    n_faces: int
    area: float

    @classmethod
    def upload(cls, mesh, stream=None) -> "DeviceMesh":
        torch = _torch()
        lib = _lib.require_cuda()
        fc, nrm = mesh_arrays(mesh)
        dfc = torch.from_numpy(fc).cuda(non_blocking=False)
        dn = torch.from_numpy(nrm).cuda(non_blocking=False)
        out = torch.empty((len(fc), 12), dtype=torch.float64, device="cuda")
        _lib.check(lib.vf_pack_faces(_lib.ptr(dfc), _lib.ptr(dn), len(fc), _lib.ptr(out),
                                     _lib.stream_ptr(stream)), "pack_faces")
        v = fc.reshape(-1, 3, 3)
        area = float(0.5 * np.linalg.norm(np.cross(v[:, 1] - v[:, 0], v[:, 2] - v[:, 0]), axis=1).sum())
        return cls(out, len(fc), area)

    @classmethod
    def from_packed(cls, faces, area: float = 1.0) -> "DeviceMesh":
        return cls(faces, int(faces.shape[0]), area)


def as_device_mesh(mesh) -> DeviceMesh:
    if isinstance(mesh, DeviceMesh):
        return mesh
    cached = getattr(mesh, "_vf_device_mesh", None)
    if cached is not None:
        return cached
    dm = DeviceMesh.upload(mesh)
    try:
        mesh._vf_device_mesh = dm
    except AttributeError:
        pass
    return dm


@dataclass
class FilterMap:
    """indicators (F,) uint8 and the ascending compact_map."""
    indicators: Optional[object]
    compact_map: object

    def to_numpy(self):
        ind = None if self.indicators is None else self.indicators.cpu().numpy()
        return ind, self.compact_map.cpu().numpy()


@dataclass
class BinLevel:
    """SPEC.md:111-117 (bins_face_ids_3D / _n_3D / _N_3D of PAPER.md:294)."""
    level: int
    bin_density: Tuple[int, int, int]
    face_ids: object
    counts: object
    offsets: object
    filter_map: Optional[FilterMap] = None
    mode: int = 0

    @property
    def n_bins(self) -> int:
        a, b, c = self.bin_density
        return a * b * c

    def to_numpy(self):
        return (self.counts.cpu().numpy(), self.offsets.cpu().numpy(),
                self.face_ids.cpu().numpy())

    def _struct(self, n_face_ids_dev=None, n_map_dev=None) -> _lib.VfBins:
        torch = _torch()
        b = _lib.VfBins()
        b.level = self.level
        b.mode = self.mode
        b.d_counts = self.counts.data_ptr()
        b.d_offsets = self.offsets.data_ptr()
        b.d_face_ids = self.face_ids.data_ptr()
        b.face_ids_cap = int(self.face_ids.numel())
        self._keep = []
        if n_face_ids_dev is None:
            n_face_ids_dev = torch.tensor([self.face_ids.numel()], dtype=torch.int32, device="cuda")
        self._keep.append(n_face_ids_dev)
        b.d_n_face_ids = n_face_ids_dev.data_ptr()
        return b


@dataclass
class ForestGrid:
    """SPEC.md:196-203 as flat device arrays with ids grouped by level:
    level L owns ids [level_start[L], level_start[L+1])."""
    cfg: EmbedConfig
    coords: object          # (cap, 4) int32: i, j, k, level
    nbr: object             # (cap, 27) int32, D3Q27 slot order (lattice.py:19-39)
    nbr_child: object       # (cap, 27) int32
    child: object           # (cap,) int32 first child id / -1  (refinement id)
    bflags: object          # (cap,) uint8 block mask bits
    masks: object           # (cap, 64) uint8 cell masks
    level_start: object     # (17,) int32 device-resident
    status: object          # (4,) int32 latched device errors
    solid64: object = None  # (cap,) int64: bit t = cell t SOLID (set by finalize)
    n_levels: int = 0
    bcount: object = None   # (cap,) int32 boundary-cell counts of the last identify_boundary_cells
    table: object = None    # LinkTable of the last build_boundary_tables (SPEC.md:328-345 chaining)

    @classmethod
    def allocate(cls, cfg: EmbedConfig, capacity: int) -> "ForestGrid":
        torch = _torch()
        dev = "cuda"
        cap = int(capacity)
        return cls(cfg,
                   torch.empty((cap, 4), dtype=torch.int32, device=dev),
                   torch.empty((cap, 27), dtype=torch.int32, device=dev),
                   torch.empty((cap, 27), dtype=torch.int32, device=dev),
                   torch.empty((cap,), dtype=torch.int32, device=dev),
                   torch.zeros((cap,), dtype=torch.uint8, device=dev),
                   torch.empty((cap, 64), dtype=torch.uint8, device=dev),
                   torch.zeros((MAX_LEVELS + 1,), dtype=torch.int32, device=dev),
                   torch.zeros((4,), dtype=torch.int32, device=dev),
                   torch.zeros((cap,), dtype=torch.int64, device=dev), 0)

    @property
    def capacity(self) -> int:
        return int(self.child.shape[0])

    def _struct(self) -> _lib.VfGrid:
        g = _lib.VfGrid()
        g.d_coords = self.coords.data_ptr()
        g.d_nbr = self.nbr.data_ptr()
        g.d_nbr_child = self.nbr_child.data_ptr()
        g.d_child = self.child.data_ptr()
        g.d_bflags = self.bflags.data_ptr()
        g.d_masks = self.masks.data_ptr()
        g.d_level_start = self.level_start.data_ptr()
        g.d_status = self.status.data_ptr()
        g.d_solid64 = self.solid64.data_ptr()
        g.capacity = self.capacity
        g.n_levels = self.n_levels
        return g

    def level_starts(self) -> np.ndarray:
        return self.level_start.cpu().numpy()

    @property
    def n_used(self) -> int:
        return int(self.level_starts()[self.n_levels])

    def level_range(self, L: int) -> Tuple[int, int]:
        ls = self.level_starts()
        return int(ls[L]), int(ls[L + 1])

    def id_sets(self):
        """Active ids grouped by level; the gap set is
        [n_used, capacity) (refine-only)."""
        ls = self.level_starts()
        return [np.arange(ls[L], ls[L + 1]) for L in range(self.n_levels)]

    def to_numpy(self):
        """Host copy in the oracle.Grid layout (dict of arrays)."""
        n = self.n_used
        return dict(coords=self.coords[:n].cpu().numpy(), nbr=self.nbr[:n].cpu().numpy(),
                    nbr_child=self.nbr_child[:n].cpu().numpy(), child=self.child[:n].cpu().numpy(),
                    bflags=self.bflags[:n].cpu().numpy(), masks=self.masks[:n].cpu().numpy(),
                    level_start=self.level_starts(), n_levels=self.n_levels)

    @classmethod
    def from_numpy(cls, cfg: EmbedConfig, g, capacity: Optional[int] = None) -> "ForestGrid":
        """Upload an oracle-layout grid (stage-isolated differential tests)."""
        torch = _torch()
        cap = int(capacity or len(g["child"]))
        fg = cls.allocate(cfg, cap)
        n = len(g["child"])
        fg.coords[:n] = torch.from_numpy(np.ascontiguousarray(g["coords"][:n])).cuda()
        fg.nbr[:n] = torch.from_numpy(np.ascontiguousarray(g["nbr"][:n])).cuda()
        fg.nbr_child[:n] = torch.from_numpy(np.ascontiguousarray(g["nbr_child"][:n])).cuda()
        fg.child[:n] = torch.from_numpy(np.ascontiguousarray(g["child"][:n])).cuda()
        fg.bflags[:n] = torch.from_numpy(np.ascontiguousarray(g["bflags"][:n])).cuda()
        fg.masks[:n] = torch.from_numpy(np.ascontiguousarray(g["masks"][:n])).cuda()
        fg.level_start.copy_(torch.from_numpy(np.ascontiguousarray(g["level_start"], dtype=np.int32)))
        fg.n_levels = int(g["n_levels"])
        # per-block SOLID bitmask (bit t = cell t), as finalize would write it
        bits = (np.asarray(g["masks"][:n]) == 1).astype(np.uint64)
        sm = (bits << np.arange(64, dtype=np.uint64)[None, :]).sum(axis=1, dtype=np.uint64)
        fg.solid64[:n] = torch.from_numpy(sm.view(np.int64)).cuda()
        return fg


@dataclass
class LinkTable:
    """SPEC.md:271-276.  lengths (N_b, 27, 64) f32, layout [slot][q][t]
    (index (slot*27+q)*64+t, pin A16); -1 = no wall within one link."""
    lengths: object
    bc_ids: object
    contraction_map: object
    n_b: int = 0

    def to_numpy(self):
        return (self.lengths.cpu().numpy(), self.bc_ids.cpu().numpy(),
                self.contraction_map.cpu().numpy())


def lengths_from_sparse(n_b: int, link_index, link_q) -> np.ndarray:
    """Host expansion of the sparse LUT download (vf_lut_sparse: unsigned
    32-bit flat indices (slot * 27 + q) * 64 + t and their q) to the SPEC
    layout lengths[N_b][27][64] with -1 where there is no cut link."""
    out = np.full(n_b * 27 * 64, -1.0, dtype=np.float32)
    idx = np.asarray(link_index).view(np.uint32).astype(np.int64)
    out[idx] = np.asarray(link_q, dtype=np.float32)
    return out.reshape(n_b, 27, 64)
