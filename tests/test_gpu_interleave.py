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


def _np_interleave(a, d):
    nx, ny, nz = a.shape[-3:]
    lead = a.shape[:-3]
    t = a.reshape(lead + (nx // d, d, ny // d, d, nz // d, d))
    n = len(lead)
    t = t.transpose(tuple(range(n)) + (n, n + 2, n + 4, n + 5, n + 3, n + 1))  # (X, Y, Z, lz, ly, lx)
    return t.reshape(lead + (nx // d, ny // d, nz // d, d ** 3))


@pytest.mark.parametrize("d", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("kind", ["u8", "f32", "f64"])
def test_tiled_and_generic_paths_exact(d, kind):
    """Every dtype x d on the tiled kernels (d in {1,2,4,8}, aligned) and the
    generic ones (d = 3, odd N_z, misaligned views): exact permutations, exact
    casts, the active mask, and the inverse."""
    import torch
    from paper_2509_24677_b200.interleave import deinterleave_device, interleave_device
    rng = np.random.default_rng(40 + d)
    for dims in ((2, 8 * d, 4 * d, 16 * d), (1, 8 * d, 2 * d, 3 * d)):
        if kind == "u8":
            host = (rng.random(dims) < 0.2).astype(np.uint8)
            tdt = torch.uint8
        elif kind == "f32":
            host = (rng.random(dims) * (rng.random(dims) < 0.3)).astype(np.float32)
            tdt = torch.float32
        else:
            host = rng.standard_normal(dims) * (rng.random(dims) < 0.3)
            tdt = torch.float64
        want = _np_interleave(host, d)
        base = torch.from_numpy(host).cuda()
        flat = torch.empty(base.numel() + 1, dtype=tdt, device="cuda")
        views = [base, flat[1:].view(dims)]  # aligned and 1-element-misaligned (generic kernels)
        views[1].copy_(base)
        for src in views:
            for odt in ((torch.float64,) if kind == "f64" else (torch.float32, torch.bfloat16)):
                cells, act = interleave_device(src, d, odt, want_active=True)
                got = cells.double().cpu().numpy()
                assert np.array_equal(got, torch.from_numpy(want.astype(np.float64)).to(odt).double().numpy())
                assert np.array_equal(act.cpu().numpy().astype(bool), want.any(-1))
            back = deinterleave_device(interleave_device(src, d, torch.float64 if kind == "f64" else torch.float32),
                                       d)
            assert np.array_equal(back.cpu().numpy(), host.astype(back.cpu().numpy().dtype))


def test_float64_threshold_exact_near_tau():
    """float64 cells within 1e-8 of tau keep the reference's float64
    comparison (values just below tau stay clear), and float64 arrays
    interleave to float64 exactly."""
    from paper_2509_24677_b200.interleave import ChannelTensor, deinterleave, interleave
    rng = np.random.default_rng(3)
    vals = 0.5 + rng.choice([-1e-9, -1e-12, 0.0, 1e-12, 5e-9], size=(8, 4, 4, 8))
    for d, shape in ((2, (8, 4, 4, 8)),):
        t = ChannelTensor(vals.reshape(shape), d)
        got = deinterleave(t, d, threshold=0.5).to_dense()
        want = _np_inverse(vals, d) >= 0.5
        assert np.array_equal(got, want) and got.sum() > 0 and (~got).sum() > 0
    dense = rng.standard_normal((16, 8, 24))
    t = interleave(dense, 4)
    assert t.values.dtype == np.float64 and np.array_equal(t.values, _np_interleave(dense, 4))
    assert np.array_equal(deinterleave(t, 4), dense)
    ints = rng.integers(-2 ** 40, 2 ** 40, (8, 8, 8))
    ti = interleave(ints, 2)
    assert ti.values.dtype == ints.dtype and np.array_equal(ti.values, _np_interleave(ints, 2))


def _np_inverse(cells, d):
    X, Y, Z, _ = cells.shape
    t = cells.reshape(X, Y, Z, d, d, d).transpose(0, 5, 1, 4, 2, 3)  # (X, lx, Y, ly, Z, lz)
    return t.reshape(X * d, Y * d, Z * d)


@pytest.mark.parametrize("d", [1, 2, 4, 8])
def test_deinterleave_threshold_word_and_byte_paths(d):
    """Packed [p >= tau] via the 32-bit word kernel (N_x % 32 == 0) and the byte
    kernel (N_x % 32 != 0), bf16 / f32 / f64 cells."""
    import torch
    from paper_2509_24677_b200.interleave import deinterleave_device
    rng = np.random.default_rng(d)
    for nx in (32 * d, 8 * d if d < 4 else 8 * d + 8 * (d == 4)):
        if nx % d:
            continue
        cells = rng.random((2, nx // d, 3, 2, d ** 3))
        dense = np.stack([_np_inverse(c, d) for c in cells])
        for dt in (torch.float32, torch.bfloat16, torch.float64):
            ct = torch.from_numpy(cells).to(dt).cuda()
            bits = deinterleave_device(ct, d, 0.5).cpu().numpy()
            ref_dense = torch.from_numpy(dense).to(dt).double().numpy() >= 0.5
            want = np.concatenate([FroxelGrid.from_dense(g).bits for g in ref_dense])
            assert np.array_equal(bits, want), (nx, dt)
