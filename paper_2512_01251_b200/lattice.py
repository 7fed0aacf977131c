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
