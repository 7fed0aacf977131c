"""Adversarial parity for the FP32 fast-accept classifiers:
meshes with vertices and edges at {0, eps/2, eps, 2 eps, 0.1, 1, 10} x the
classifier margins from x-rows and cut-link lines, slivers, |n_x| within 1e-6
of 1e-3, faces touching x = 0 / x = l_x, non-power-of-two dx and a non-cubic
domain (tests/fuzz_meshes.py).  GPU == oracle bitwise (topology, masks,
contraction map, -1 pattern), link lengths <= 1e-5 relative; also with every
face forced through either cut-link enumeration kernel."""
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from fuzz_meshes import FUZZ_CONFIGS, fuzz_case  # noqa: E402
from test_gpu_parity import _embed_compare  # noqa: E402


@pytest.fixture(scope="module")
def O(oracle_mod):
    return oracle_mod


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("name", sorted(FUZZ_CONFIGS))
def test_fuzz_margins(O, name, seed):
    mesh, cfg = fuzz_case(name, seed)
    _embed_compare(O, mesh, cfg)


@pytest.mark.parametrize("small_ext", [-1.0, 1e9])
@pytest.mark.parametrize("seed", [11, 12])
def test_fuzz_margins_link_kernels(O, seed, small_ext):
    from paper_2512_01251_b200 import _lib
    lib = _lib.require_cuda()
    old = lib.vf_set_link_small_ext(small_ext)
    try:
        mesh, cfg = fuzz_case("nx32", seed)
        _embed_compare(O, mesh, cfg)
    finally:
        lib.vf_set_link_small_ext(old)


@pytest.mark.parametrize("seed", [21, 22])
def test_fuzz_margins_no_filter(O, seed):
    """filter off: every face through every level's row classifier"""
    mesh, cfg = fuzz_case("nx48", seed)
    _embed_compare(O, mesh, cfg, use_filter=False)


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("name", sorted(FUZZ_CONFIGS))
def test_fuzz_bins(O, name, seed):
    """The bin-pair classifier (box-axis pruning, vertex fast accept, FP32
    bin_class, exact SAT in the band) against the oracle's per-candidate SAT:
    every level's bins, 1D filter on and off."""
    from paper_2512_01251_b200 import binning
    import numpy as np
    mesh, cfg = fuzz_case(name, seed)
    for L in range(cfg.l_max):
        for use_filter in (True, False):
            bl = binning.build_level(mesh, L, cfg, 0, use_filter)
            c, o, f = bl.to_numpy()
            cr, orr, fr = O.build_bins(mesh.faces_coord, mesh.normals, cfg, L, 0, use_filter)
            assert np.array_equal(c, cr) and np.array_equal(o, orr) and np.array_equal(f, fr), (L, use_filter)
