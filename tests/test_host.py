"""Host-side logic and the C-ABI surface (CPU only; no kernel launches)."""

from __future__ import annotations

import ctypes
import os
import re

import numpy as np
import pytest

from paper_2509_24677_b200 import _lib, synth
from paper_2509_24677_b200.froxel import FroxelGrid
from paper_2509_24677_b200.neural import ConvSpec, ModelConfig, TrainConfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    text = open(os.path.join(ROOT, "include", "fpvs.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fpvs_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2509_24677_b200.build import build
    build(verbose=False)
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = header_functions()
    assert len(names) >= 25
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.SIGNATURES), "ctypes table out of sync with include/fpvs.h"
    lib = _lib.load()
    assert lib.fpvs_abi_version() == 4
    # size queries are pure host arithmetic
    assert _lib.size("fpvs_pack_weights_tc_size", 27, 64, 64, 0) == 27 * 64 * 128
    assert _lib.size("fpvs_pack_weights_tc_size", 27, 8, 32, 0) == 4 * 32 * 128
    assert _lib.size("fpvs_pack_weights_tc_size", 27, 256, 256, 64) == 4 * 108 * 64 * 128
    assert _lib.size("fpvs_pack_weights_tc_size", 27, 64, 64, 48) == 0
    assert _lib.size("fpvs_kmap_workspace_size", 1, 64, 64, 64) > 0


def test_argument_errors_map_to_valueerror():
    # rejected before any launch, so no GPU is needed
    with pytest.raises(ValueError, match="divide"):
        _lib.call("fpvs_interleave", 1, 0, 1, 6, 4, 4, 4, 1, 0, None, None)
    with pytest.raises(ValueError):
        _lib.call("fpvs_spconv_tc", 1, 64, 10, None, 27, None, 1, 10, 1, 0, None, 64, 64, 1, 1, 64, 0, None)


def test_round2_entry_points_validate_before_launching():
    """The round-2 entry points reject bad arguments on the host (no GPU)."""
    p = 256  # a non-null dummy address: never dereferenced, the checks fail first
    # the grid writer: d must be 4, N_x a multiple of 32
    with pytest.raises(ValueError, match="d = 4"):
        _lib.call("fpvs_rowbits_to_grid", p, p, 1, 64, 64, 64, 2, p, None)
    with pytest.raises(ValueError, match="N_x"):
        _lib.call("fpvs_rowbits_to_grid", p, p, 1, 48, 64, 64, 4, p, None)
    with pytest.raises(ValueError, match="null"):
        _lib.call("fpvs_rowbits_to_grid", None, p, 1, 64, 64, 64, 4, p, None)
    # column-block up conv: Cout % 32, 8 Cout <= 1024, a child table
    with pytest.raises(ValueError, match="Cout"):
        _lib.call("fpvs_spconv_tc_upblocks", p, 64, 10, p, 10, p, 0, p, 64, 48, 1, p, p, 96, 0, None)
    with pytest.raises(ValueError, match="child_rows"):
        _lib.call("fpvs_spconv_tc_upblocks", p, 64, 10, p, 10, p, 0, p, 64, 64, 1, None, p, 128, 0, None)
    # dataflow consumer without settled tables; producer with a K split
    halo = [p, 64, 10, p, p, p, p, p, p, 10, p, 64, 1, p, 64, 64]
    with pytest.raises(ValueError, match="SETTLED"):
        _lib.call("fpvs_spconv_halo_flow", *halo, 1, p, 64, 0, p, 1 << 20, None, p, None)
    halo_split = halo[:12] + [2] + halo[13:]
    with pytest.raises(ValueError, match="unsplit"):
        _lib.call("fpvs_spconv_halo_flow", *halo_split, 1 | _lib.TABLES_SETTLED, p, 64, 0, p, 1 << 20, p, None,
                  None)
    # gather-GEMM consumer needs the producer's row count
    with pytest.raises(ValueError, match="row count"):
        _lib.call("fpvs_spconv_tc_flow", p, 64, 10, p, 27, p, p, 10, p, 0, p, 64, 64, 1, p, 64, 0, p, None, None)
    # multi-pack: 1..32 jobs
    with pytest.raises(ValueError, match="pack jobs"):
        _lib.call("fpvs_pack_weights_tc_multi", None, 0, None)
    # dense-brick conv: tile width, Cin % 64, a split dividing Cin / 64, the workspace of a split
    brick = [p, 128, 10, p, 1, 16, 16, 16, p]
    with pytest.raises(ValueError, match="tile width"):
        _lib.call("fpvs_spconv_brick", *brick, 96, 1, p, 128, 192, 1, p, 192, 0, None, 0, None)
    with pytest.raises(ValueError, match="Cin"):
        _lib.call("fpvs_spconv_brick", p, 96, 10, p, 1, 16, 16, 16, p, 128, 1, p, 96, 128, 1, p, 128, 0, None, 0,
                  None)
    with pytest.raises(ValueError, match="split"):
        _lib.call("fpvs_spconv_brick", *brick, 128, 3, p, 128, 128, 1, p, 128, 0, p, 1 << 30, None)
    with pytest.raises(ValueError, match="workspace"):
        _lib.call("fpvs_spconv_brick", *brick, 128, 2, p, 128, 128, 1, p, 128, 0, p, 16, None)
    with pytest.raises(ValueError, match="null"):
        _lib.call("fpvs_spconv_brick", None, 128, 10, p, 1, 16, 16, 16, p, 128, 1, p, 128, 128, 1, p, 128, 0, None,
                  0, None)
    assert _lib.size("fpvs_spconv_brick_workspace_size", 1, 16, 16, 16, 256, 128, 2) == \
        256 + 32 * 2 * 2 * 128 * 128 * 4  # 32 bricks x 2 column blocks: counters, then 2 partials each
    assert _lib.size("fpvs_spconv_brick_workspace_size", 1, 16, 16, 16, 256, 96, 1) == 0


# -------------------------------------------------------- FPVS boundary format


def test_bit_packing_layout():
    # reference KAT pkg/tests/test_froxel.py:33-37
    g = FroxelGrid((16, 4, 4))
    g.set(0, 0, 0)
    g.set(3, 0, 0)
    assert g.bits[0] == 0b00001001


def test_dense_round_trip_and_file(tmp_path, rng):
    dense = rng.random((24, 8, 5)) < 0.3
    g = FroxelGrid.from_dense(dense, role="gt_pvs", supersample=3)
    assert np.array_equal(g.to_dense(), dense)
    p = tmp_path / "g.fpvs"
    g.save(p)
    raw = p.read_bytes()
    assert raw[:4] == b"FPVS" and len(raw) == 24 + 24 * 8 * 5 // 8
    h = FroxelGrid.load(p)
    assert h == g and h.supersample == 3
    with pytest.raises(ValueError):
        FroxelGrid((12, 4, 4))
    with pytest.raises(IndexError):
        g.set(24, 0, 0)


# -------------------------------------------------------- configs and synthesis


def test_model_config_validation():
    ModelConfig.config1()
    with pytest.raises(ValueError):
        ModelConfig(2, [ConvSpec(3, 4, 8, "relu"), ConvSpec(1, 8, 8, "sigmoid")])
    with pytest.raises(ValueError):
        ModelConfig(2, [ConvSpec(3, 8, 8, "relu"), ConvSpec(1, 8, 8, "relu")])
    with pytest.raises(ValueError):
        ConvSpec(2, 8, 8)
    with pytest.raises(ValueError):
        TrainConfig(alpha=1.5)
    with pytest.raises(ValueError):
        TrainConfig(optimizer="lion")


def test_synthetic_grids_are_seeded():
    a = synth.config1_grid(0)
    assert a.shape == (64, 64, 32) and np.array_equal(a, synth.config1_grid(0))
    assert 0.03 < a.mean() < 0.10
    occ = synth.box_grid((32, 32, 32), 40, 1, 6, 9)
    lab = synth.first_hit_labels(occ)
    assert not (lab & ~occ).any() and lab.any()
    # brute-force the label rule on a few columns
    nx, ny, nz = occ.shape
    zf = np.where(occ.any(2), occ.argmax(2), nz)
    for x, y in [(3, 4), (10, 10), (0, 31), (31, 0)]:
        for z in range(nz):
            want = occ[x, y, z] and any(
                zf[xx, yy] == z for xx in range(max(0, x - 2), min(nx, x + 3))
                for yy in range(max(0, y - 2), min(ny, y + 3)))
            assert lab[x, y, z] == want


def test_density_bisection_hits_target():
    occ, n = synth.box_grid_density((64, 64, 64), 0.02, 1, 6, 3)
    assert 0.02 <= occ.mean() < 0.022
