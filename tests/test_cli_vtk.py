"""CPU checks of the outputs / CLI plumbing (SPEC.md write_outputs, load_config,
run_cli): VTK voxel files round-trip, config errors name key and line,
unknown subcommands exit 2, pipeline commands without a GPU exit non-zero."""
import os

import numpy as np
import pytest

from paper_2512_01251_b200 import cli
from paper_2512_01251_b200.config import EmbedConfig
from paper_2512_01251_b200.vtk import read_vtk_cell_data, write_levels


def test_vtk_one_block_roundtrip(tmp_path):
    cfg = EmbedConfig(n_x=4, l_max=1)  # one 4^3 block
    coords = np.zeros((1, 4), np.int32)
    masks = np.arange(64, dtype=np.uint8).reshape(1, 64) % 6
    g = {"coords": coords, "masks": masks, "level_start": np.array([0, 1] + [1] * 15, np.int32)}
    paths = write_levels(str(tmp_path), g, cfg)
    assert [os.path.basename(p) for p in paths] == ["level_0.vtk"]
    data = read_vtk_cell_data(paths[0])
    assert np.array_equal(data["mask"], masks.reshape(-1))
    assert np.array_equal(data["block"], np.zeros(64))
    text = open(paths[0]).read()
    assert "CELLS 64 576" in text and "POINTS 512 double" in text
    # byte-stable
    paths2 = write_levels(str(tmp_path / "again"), g, cfg)
    assert open(paths2[0], "rb").read() == open(paths[0], "rb").read()


def test_config_errors(tmp_path):
    p = tmp_path / "a.cfg"
    p.write_text("N_x = 64\nL_max = 4 # comment\nprimitive = torus\n")
    c = cli.load_config(str(p))
    assert c["N_x"] == 64 and c["L_max"] == 4 and c["primitive"] == "torus" and c["N_spec"] == 2
    p.write_text("N_x = 64\nbogus = 1\n")
    with pytest.raises(cli.ConfigError, match="line 2: unknown key 'bogus'"):
        cli.load_config(str(p))
    p.write_text("L_max = four\n")
    with pytest.raises(cli.ConfigError, match="line 1: bad value for 'L_max'"):
        cli.load_config(str(p))
    p.write_text("L_max = 0\n")
    with pytest.raises(cli.ConfigError, match="L_max"):
        cli.load_config(str(p))


def test_cli_exit_codes(capsys):
    import torch
    if not torch.cuda.is_available():  # no CPU fallback: a message and exit 1
        assert cli.main(["simulate", "--nx", "16", "--lmax", "1"]) == 1
    with pytest.raises(SystemExit) as ei:
        cli.main(["frobnicate"])
    assert ei.value.code == 2
