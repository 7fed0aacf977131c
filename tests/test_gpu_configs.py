"""GPU vs oracle on the BASELINE configs the round-1 suite did not embed
(VERDICT r1 #1): C3 exactly as `bench.py --config c3` runs it, C5 at
L_max=6 (finest bin density 512) on the two smallest sweep tori after
refine_faces, and a small sphere at L_max=7 (finest bin density 1024: the
block-indexed bins, sparse rows and parent-bucketed cut links must hold past
the sizes where the round-1 dense per-level arrays reached 4.3 GB).
Bit-exact topology / masks / contraction map / -1 pattern, link lengths
<= 1e-5 relative (north star)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2512_01251_b200 import EmbedConfig, l_spec_bound, make_icosphere, make_torus, refine_faces  # noqa: E402

from test_gpu_parity import _embed_compare  # noqa: E402


@pytest.fixture(scope="module")
def O(oracle_mod):
    return oracle_mod


def test_embed_c3_bench_config(O):
    """C3 (bench.py WORKLOADS['c3']): icosphere k=5 of diameter 1/64 at the
    centre, N_x=128 (N_B=32), L_max=3, N_spec=2, d_spec=0.05 (N_prop=2)."""
    import bench
    w = bench.WORKLOADS["c3"]
    mesh, cfg = bench.make_mesh(w, 0), bench.make_cfg(w)
    assert cfg.n_x == 128 and cfg.l_max == 3 and cfg.n_prop == 2 and mesh.n_faces == 20480
    _embed_compare(O, mesh, cfg)


@pytest.mark.slow
@pytest.mark.parametrize("m,n,faces", [(100, 50, 640000), (280, 200, 891520)])
def test_embed_c5_lmax6(O, m, n, faces):
    """C5 at L_max=6: torus after refine_faces to
    l_spec(L_max=6) -- 4.94 M blocks, 376 K boundary blocks (2.6 GB LUT)."""
    cfg = EmbedConfig(n_x=64, l_max=6, n_spec=2, d_spec=0.05, capacity=5_200_000)
    mesh = refine_faces(make_torus(m, n), l_spec_bound(cfg.domain, cfg.n_spec, cfg.l_max, cfg.nb[0]))
    assert mesh.n_faces == faces
    eng, grid, table = _embed_compare(O, mesh, cfg)
    assert grid.n_levels == 6 and table.n_b > 300000
    del eng, grid, table
    torch.cuda.empty_cache()


def test_embed_lmax7_small_sphere(O):
    """L_max = 7: an icosphere of diameter 0.1 in a N_x=32
    root (N_B = 8, finest bin density 8 * 2^6 = 512 per axis), refined to
    l_spec(L_max=7): 170 K blocks over 7 levels, 12.5 K boundary blocks,
    against the oracle."""
    mesh = make_icosphere((0.5 + 0.3 / 4096, 0.5 + 0.7 / 4096, 0.5 + 0.2 / 4096), 0.1, 4)
    cfg = EmbedConfig(n_x=32, l_max=7, n_spec=2, d_spec=0.05)
    mesh = refine_faces(mesh, l_spec_bound(cfg.domain, cfg.n_spec, cfg.l_max, cfg.nb[0]))
    eng, grid, table = _embed_compare(O, mesh, cfg)
    assert grid.n_levels == 7 and table.n_b > 10000
    del eng, grid, table
    torch.cuda.empty_cache()
