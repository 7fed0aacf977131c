"""D3Q27 direction convention shared by neighbour slots, ray directions and
the link-length LUT q axis: rest first, then antiparallel pairs (2k-1, 2k)
ordered by number of non-zero components (/root/reference/pkg/src/voxforest/
lattice.py:19-39; pinned by tests/golden/lattice_golden.npz)."""
import numpy as np


def _paired_directions():
    reps, seen = [], set()
    cands = [(x, y, z) for x in (-1, 0, 1) for y in (-1, 0, 1) for z in (-1, 0, 1)
             if (x, y, z) != (0, 0, 0)]
    for c in sorted(cands, key=lambda c: (sum(abs(v) for v in c), tuple(-v for v in c))):
        if c in seen or tuple(-v for v in c) in seen:
            continue
        seen.add(c)
        reps.append(c)
    dirs = [(0, 0, 0)]
    for c in reps:
        dirs += [c, tuple(-v for v in c)]
    return np.array(dirs, dtype=np.int64)


D3Q27_C = _paired_directions()
D3Q27_OPPOSITE = np.array([0] + [q + 1 if q % 2 == 1 else q - 1 for q in range(1, 27)])
REPRESENTATIVES = np.arange(1, 27, 2)

# D3Q27 weights (SPEC.md VelocitySet: sum w = 1, sum w c = 0, sum w c c^T = I/3)
_NZ = np.abs(D3Q27_C).sum(1)
D3Q27_W = np.where(_NZ == 0, 8 / 27, np.where(_NZ == 1, 2 / 27, np.where(_NZ == 2, 1 / 54, 1 / 216)))


class _VelocitySet:
    """SPEC.md:384-386 VelocitySet (D3Q27)."""
    D = 3
    Q = 27
    c = D3Q27_C
    w = D3Q27_W
    opposite = D3Q27_OPPOSITE
    cs2 = 1.0 / 3.0


D3Q27 = _VelocitySet()
