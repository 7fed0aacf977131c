"""CPU checks of the drop-in boundary: the C-ABI library loads without a GPU
and exports every entry point declared in include/*.h; host-side logic."""
import ctypes
import glob
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        txt = open(h).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        names |= set(re.findall(r"\b(vf_[a-z0-9_]+)\s*\(", txt))
    return names


def test_header_declares_entry_points():
    names = _declared()
    for n in ("vf_ray_indicators", "vf_bin_pairs", "vf_bin_assemble", "vf_voxelize_level",
              "vf_propagate_x", "vf_finalize_level", "vf_mark_level", "vf_adapt_refine",
              "vf_boundary_cells", "vf_link_tables", "vf_link_lengths", "vf_last_error",
              "vf_abi_version", "vf_embed_phase1", "vf_embed_phase2"):
        assert n in names


def test_library_exports_every_declared_symbol():
    from paper_2512_01251_b200 import _lib
    lib = _lib.load()
    for n in sorted(_declared()):
        assert hasattr(lib, n), n
        assert n in _lib.EXPORTED, f"{n} declared but not typed in _lib"
    assert lib.vf_abi_version() == _lib.ABI_VERSION


def test_library_is_sm100a():
    so = os.path.join(ROOT, "paper_2512_01251_b200", "libvoxforest_b200.so")
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_ops_fail_loudly_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    from paper_2512_01251_b200 import CudaError, EmbedConfig, make_icosphere
    from paper_2512_01251_b200 import voxelizer
    with pytest.raises(CudaError):
        voxelizer.embed_geometry(None, make_icosphere(subdivisions=1), EmbedConfig(n_x=16, l_max=1))


def test_config_validation():
    from paper_2512_01251_b200 import EmbedConfig
    with pytest.raises(ValueError):
        EmbedConfig(l_max=0)
    with pytest.raises(ValueError):
        EmbedConfig(n_x=30)
    c = EmbedConfig(n_x=64, l_max=5)
    assert c.nb == (16, 16, 16) and c.bins(4) == (256, 256, 256) and c.n_lim == 64
    assert c.dx(3) == 1 / 512
