"""(1) interleave / deinterleave kernels vs the reference golden vectors (bit-exact)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import sparse as osp
from paper_2509_24677_b200 import synth
from paper_2509_24677_b200.froxel import FroxelGrid

pytestmark = pytest.mark.gpu


def test_interleave_reference_golden(golden):
    from paper_2509_24677_b200.interleave import ChannelTensor, deinterleave, interleave
    g = golden("interleave.npz")
    for ci in range(int(g["ncases"])):
        dims, d = tuple(g[f"c{ci}_dims"]), int(g[f"c{ci}_d"])
        grid = FroxelGrid(dims, bits=g[f"c{ci}_bits"])
        t = interleave(grid, d)                                   # packed bits -> float64
        assert t.values.dtype == np.float64
        assert np.array_equal(t.values, g[f"c{ci}_il_bits"])
        tf = interleave(g[f"c{ci}_f32"], d)                        # f32 ndarray keeps dtype
        assert tf.values.dtype == np.float32
        assert np.array_equal(tf.values, g[f"c{ci}_il_f32"])
        back = deinterleave(ChannelTensor(g[f"c{ci}_il_f32"], d), d)
        assert np.array_equal(back, g[f"c{ci}_deil_f32"])
        if f"c{ci}_thr_bits" in g:
            thr = deinterleave(ChannelTensor(g[f"c{ci}_il_f32"], d), d, threshold=0.5)
            assert np.array_equal(thr.bits, g[f"c{ci}_thr_bits"]) and thr.role == "predicted_pvs"


def test_interleave_kats_and_errors():
    from paper_2509_24677_b200.interleave import ChannelTensor, deinterleave, interleave
    g = FroxelGrid((8, 4, 4))
    g.set(3, 3, 3)
    t = interleave(g, 2).values
    assert t[1, 1, 1, 7] == 1 and t.sum() == 1
    assert interleave(np.zeros((32, 32, 32), np.float32), 8).values.shape == (4, 4, 4, 512)
    assert deinterleave(ChannelTensor(np.full((4, 2, 2, 8), 0.5, np.float32), 2), threshold=0.5).bits.all()
    assert not deinterleave(ChannelTensor(np.full((4, 2, 2, 8), 0.49, np.float32), 2), threshold=0.5).bits.any()
    with pytest.raises(ValueError):
        interleave(np.zeros((6, 4, 4), np.float32), 4)
    with pytest.raises(ValueError):
        interleave(np.zeros((4, 4)), 2)
    with pytest.raises(ValueError):
        ChannelTensor(np.zeros((2, 2, 2, 7)), 2)


@pytest.mark.parametrize("d", [2, 4, 8])
def test_interleave_round_trip_100_grids(d):
    """deinterleave(interleave(G, d)) == G for 100 random grids, d in {2,4,8}."""
    import torch
    from paper_2509_24677_b200.interleave import deinterleave_device, interleave_device
    rng = np.random.default_rng(d)
    occ = rng.random((100, 32, 16, 32)) < 0.1
    dev = torch.from_numpy(occ.astype(np.uint8)).cuda()
    cells = interleave_device(dev, d, torch.float32)
    back = deinterleave_device(cells, d)
    assert torch.equal(back.to(torch.uint8), dev)
    bits = deinterleave_device(cells, d, 0.5)
    want = np.concatenate([FroxelGrid.from_dense(o).bits for o in occ])
    assert np.array_equal(bits.cpu().numpy(), want)
    # packed input path gives the same cells, bf16 output is exact for 0/1
    cells_p = interleave_device(torch.from_numpy(want).cuda(), d, torch.bfloat16, packed_dims=(100, 32, 16, 32))
    assert torch.equal(cells_p.float(), cells)


def test_interleave_config_sizes_bit_exact():
    """cfg1 (64x64x32, d=2) and cfg2 (256^3, d=4): device interleave == oracle, plus active mask."""
    import torch
    from paper_2509_24677_b200.interleave import interleave_device
    for occ, d in ((synth.config1_grid(0), 2), (synth.config2_grid(1), 4)):
        bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
        cells, act = interleave_device(bits, d, torch.bfloat16, packed_dims=(1,) + occ.shape, want_active=True)
        ref = osp.interleave(occ.astype(np.float32), d)
        assert np.array_equal(cells[0].float().cpu().numpy(), ref)
        assert np.array_equal(act[0].cpu().numpy().astype(bool), ref.any(-1))
        dense = torch.from_numpy(occ.astype(np.float32)).cuda()[None]
        cells2, act2 = interleave_device(dense, d, torch.float32, want_active=True)
        assert np.array_equal(cells2[0].cpu().numpy(), ref)
        assert torch.equal(act2, act)
