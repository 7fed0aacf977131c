"""Embedding configuration (SPEC.md:277-280 VoxelConfig + the grid keys of
PAPER.md:291) and the derived quantities shared by the CUDA path and the
oracle (SURVEY.md Appendix A pins A1-A2, A12)."""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Sequence, Tuple

EPS_PARALLEL = 1e-12          # geometry.py:25
MAX_LEVELS = 16


@dataclass(frozen=True)
class EmbedConfig:
    """Frozen embedding config.

    n_x        root-grid cells along x (multiple of 4)
    domain     domain lengths (l_x, l_y, l_z), origin at 0
    l_max      number of grid levels L_max (levels 0..l_max-1)
    n_spec     N_spec; per-face pair cap (2+N_spec)^3
    d_spec     near-wall refinement distance
    eps_slab   point-in-face AABB half width, default 1e-9*max(l)
    capacity   block capacity of the forest; None = estimate
    use_filter ray-indicator face filtering on/off (invariant)
    """

    n_x: int = 64
    domain: Tuple[float, float, float] = (1.0, 1.0, 1.0)
    l_max: int = 3
    n_spec: int = 2
    d_spec: float = 0.05
    eps_slab: Optional[float] = None
    eps_parallel: float = EPS_PARALLEL
    capacity: Optional[int] = None
    use_filter: bool = True

    def __post_init__(self):
        if self.n_x % 4 or self.n_x <= 0:
            raise ValueError("n_x must be a positive multiple of 4")
        if not (1 <= self.l_max <= MAX_LEVELS - 1):
            raise ValueError("l_max must be in [1, 15]")
        if self.d_spec < 0:
            raise ValueError("d_spec must be >= 0")
        if self.n_spec < 1:
            raise ValueError("n_spec must be >= 1")
        for d in range(3):
            nd = self.domain[d] / self.dx0
            if abs(nd - round(nd)) > 1e-9 or round(nd) % 4:
                raise ValueError("domain lengths must be multiples of 4*dx0")

    @property
    def dx0(self) -> float:
        return float(self.domain[0]) / self.n_x

    @property
    def nb(self) -> Tuple[int, int, int]:
        """Root blocks per axis N_B (4^3-cell blocks)."""
        return tuple(int(round(self.domain[d] / self.dx0)) // 4 for d in range(3))

    @property
    def n_root(self) -> int:
        a, b, c = self.nb
        return a * b * c

    @property
    def eps(self) -> float:
        return self.eps_slab if self.eps_slab is not None else 1e-9 * max(self.domain)

    def dx(self, L: int) -> float:
        return math.ldexp(self.dx0, -L)

    def bins(self, L: int) -> Tuple[int, int, int]:
        """Bin density B_L per axis, matched to blocks (A4)."""
        return tuple(n << L for n in self.nb)

    def n_bins(self, L: int) -> int:
        a, b, c = self.bins(L)
        return a * b * c

    @property
    def n_lim(self) -> int:
        return (2 + self.n_spec) ** 3

    @property
    def n_prop(self) -> int:
        """N_prop = 1 + floor((1/2^L) d_spec / (sqrt(2) * 4 dx_L));
        level independent because dx_L = dx0 / 2^L exactly (A12)."""
        return 1 + int(math.floor(1.0 * (self.d_spec / (math.sqrt(2.0) * (4.0 * self.dx0)))))

    def block_capacity(self, surface_area: float = 1.0) -> int:
        """Forest capacity: explicit, else a surface-shell estimate with 2x
        head-room (blocks within (N_prop+4) block layers of the surface)."""
        if self.capacity is not None:
            return int(self.capacity)
        cap = self.n_root
        for L in range(self.l_max - 1):
            h = 4.0 * self.dx(L)
            shell = (self.n_prop + 4) * 2.0 * surface_area / (h * h)
            marked = min(shell, float(self.n_bins(L)))
            cap += int(8 * marked)
        return int(min(2 * cap + 4096, 2**31 - 1))
