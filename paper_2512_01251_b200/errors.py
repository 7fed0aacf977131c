"""Exception family.  Mirrors the reference's ``MeshError(ValueError)``
(geometry.py:28-33) and the SPEC's error conditions: capacity exhaustion with
level context and the N_lim pair-cap violation, an internal
error after refine_faces."""


class VoxforestError(RuntimeError):
    """Base class for engine failures that are not input errors."""


class MeshError(ValueError):
    """Invalid mesh input (geometry.py:28)."""


class StlParseError(MeshError):
    """Malformed STL input (geometry.py:32)."""


class CapacityError(VoxforestError, MemoryError):
    """Forest block capacity / scratch capacity exhausted."""


class BinCapError(VoxforestError):
    """A face needed more than N_lim = (2+N_spec)^3 bins."""


class CudaError(VoxforestError):
    """CUDA runtime failure or no device (there is no CPU fallback)."""
