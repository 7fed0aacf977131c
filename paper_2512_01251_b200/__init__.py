"""paper_2512_01251_b200 -- B200-native geometry embedding for block-structured
forest-of-octrees grids (arXiv 2512.01251): spatial-bin hierarchy, per-block
ray-cast voxelization, near-wall refinement with octree split, and the cut-link
LUT for interpolated bounce-back, as hand-written sm_100a CUDA behind the
C-ABI of include/voxforest_b200.h.

The module layout mirrors the reference's SPEC modules:
``binning``, ``forest``, ``voxelizer``; meshes are duck-typed on the reference
``TriangleMesh`` (geometry.py:65-111).
"""
from .config import EmbedConfig
from .errors import BinCapError, CapacityError, CudaError, MeshError, VoxforestError
from .mesh import TriangleMesh, l_spec_bound, make_icosphere, make_torus, refine_faces

__all__ = ["EmbedConfig", "TriangleMesh", "make_icosphere", "make_torus", "refine_faces",
           "l_spec_bound", "MeshError", "CapacityError", "BinCapError", "CudaError",
           "VoxforestError", "binning", "forest", "voxelizer", "solver"]


def __getattr__(name):
    # lazy submodules: importing the package must not require CUDA/torch
    if name in ("binning", "forest", "voxelizer", "datatypes", "solver", "parallel"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
