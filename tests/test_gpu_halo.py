"""Halo-cached tcgen05 submanifold conv (fpvs_kmap_halo + fpvs_spconv_halo).

The halo tables are integer work and must equal a numpy restatement exactly
(sorted distinct neighbour rows per 128-row tile, the tile-local slot table,
-2 for rows the 512-slot cache cannot hold).  The conv is checked against
the float64 oracle on the same bf16 values with the bf16-output tolerance of
test_gpu_conv (half an ulp + fp32 accumulation noise), across tile widths,
K splits, and a table that forces the uncached direct-read path.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import sparse as osp

pytestmark = pytest.mark.gpu

HMAX = 512


def _halo_ref(nbr: np.ndarray, n: int):
    """Per tile: sorted distinct rows (first HMAX), count, local table."""
    tiles = (n + 127) // 128
    out = []
    for t in range(tiles):
        tab = np.full((128, 27), -1, np.int64)
        rows = nbr[t * 128:min(n, (t + 1) * 128)]
        tab[:len(rows)] = rows
        v = tab[tab >= 0]
        if len(v) == 0:
            out.append((np.zeros(0, np.int64), 0, np.full((128, 27), -1)))
            continue
        lo, hi = v.min(), v.max()
        if hi - lo >= 16384:
            loc = np.where(tab >= 0, -2, -1)
            out.append((np.zeros(0, np.int64), 0, loc))
            continue
        u = np.unique(v)
        rank = np.searchsorted(u, tab)
        loc = np.where(tab < 0, -1, np.where(rank < HMAX, rank, -2))
        out.append((u[:HMAX], min(len(u), HMAX), loc))
    return out


def _build(nbr_t, n_t, cap):
    import torch
    from paper_2509_24677_b200 import _lib
    tiles = max(1, (cap + 127) // 128)
    rows = torch.full((tiles, HMAX), -7, dtype=torch.int32, device="cuda")
    hn = torch.full((tiles,), -7, dtype=torch.int32, device="cuda")
    ln = torch.full((tiles, 128 * 27), -7, dtype=torch.int16, device="cuda")
    _lib.call("fpvs_kmap_halo", _lib.ptr(nbr_t), _lib.ptr(n_t), cap, _lib.ptr(rows), _lib.ptr(hn), _lib.ptr(ln), 0)
    return {"rows": rows, "n": hn, "lnbr": ln}


def _check_tables(h, nbr, n):
    rows, hn, ln = h["rows"].cpu().numpy(), h["n"].cpu().numpy(), h["lnbr"].cpu().numpy()
    for t, (u, cnt, loc) in enumerate(_halo_ref(nbr, n)):
        assert hn[t] == cnt, (t, hn[t], cnt)
        assert np.array_equal(rows[t, :cnt], u[:cnt]), t
        assert np.array_equal(ln[t].reshape(128, 27), loc), t


def _level(dims, density, seed, B=1):
    import torch
    from paper_2509_24677_b200 import sparse as sp
    rng = np.random.default_rng(seed)
    mask = rng.random((B,) + dims) < density
    lv = sp.new_level(B, dims)
    lv.active.copy_(torch.from_numpy(mask.reshape(-1).astype(np.uint8)).cuda())
    sp.compact(lv)
    sp.build_subm(lv)
    return lv


def test_halo_tables_config2_levels():
    """Tables of the three config-2 levels (real box geometry) vs numpy."""
    import torch
    from paper_2509_24677_b200 import sparse as sp, synth
    from paper_2509_24677_b200.froxel import FroxelGrid
    from paper_2509_24677_b200.unet import PvsUNet
    occ = synth.config2_grid(1)
    bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
    plan = PvsUNet(seed=1).plan(1, occ.shape)
    plan.build_maps(bits)   # all three levels in one fpvs_kmap_halo_multi launch
    for lv in (plan.L0, plan.L1, plan.L2):
        n = lv.count()
        h = lv.extra["halo"]
        _check_tables(h, lv.nbr[:n].cpu().numpy().astype(np.int64), n)
        tiles = (n + 127) // 128
        multi = {k: v[:tiles].clone() for k, v in h.items()}
        h1 = sp.build_halo(lv)  # the single-level entry point gives the same tables
        for k in ("n", "lnbr"):
            assert torch.equal(multi[k], h1[k][:tiles]), k


def test_halo_tables_overflow_and_window():
    """Synthetic tables: > 512 distinct rows in a tile, a > 16384-row window, empty rows."""
    import torch
    rng = np.random.default_rng(5)
    n, cap = 700, 768
    nbr = rng.integers(0, 3000, size=(n, 27))
    nbr[rng.random((n, 27)) < 0.3] = -1
    nbr[128:256] = rng.integers(0, 200000, size=(128, 27))   # window overflow tile
    nbr[256:384] = -1                                          # a tile with no neighbours
    nbr[256, 13] = 256
    t = torch.zeros((cap, 27), dtype=torch.int32, device="cuda")
    t[:n] = torch.from_numpy(nbr.astype(np.int32)).cuda()
    nt = torch.tensor([n], dtype=torch.int32, device="cuda")
    h = _build(t, nt, cap)
    _check_tables(h, nbr, n)
    assert int(h["n"][0]) == HMAX  # 3000-row range -> far more than 512 distinct rows


def _run_halo(layer, xt, ldx, lv, nbr_t, h, y, ldy, col_off, bn, split, act="relu"):
    import torch
    from paper_2509_24677_b200 import _lib
    from paper_2509_24677_b200.neural import run_conv
    ws = torch.zeros(_lib.size("fpvs_spconv_halo_workspace_size", lv.cap, layer.spec.out_channels, bn, split),
                     dtype=torch.uint8, device="cuda")
    run_conv(layer, xt, ldx, nbr_t, 27, lv.n, lv.cap, y, ldy, col_off, "bf16", act=act,
             masks=lv.nbr_masks, halo=(bn, split, ws), halo_tabs=h)
    return ws


def _layer(cin, cout, seed):
    from paper_2509_24677_b200.neural import Conv3d, ConvSpec
    layer = Conv3d(ConvSpec(3, cin, cout, "relu"), np.random.default_rng(seed), init="kaiming_uniform")
    layer.b.uniform_(-0.1, 0.1)
    return layer


def _rows(n, c, seed, cap):
    import torch
    rng = np.random.default_rng(seed)
    v = osp.bf16_round(np.maximum(rng.normal(size=(n, c)), 0).astype(np.float32)).astype(np.float32)
    t = torch.zeros((cap, c), dtype=torch.bfloat16, device="cuda")
    t[:n] = torch.from_numpy(v).to(torch.bfloat16).cuda()
    return v, t


@pytest.mark.parametrize("cin,cout,bn,split", [(64, 64, 64, 1), (64, 64, 64, 2), (128, 64, 64, 1), (64, 128, 128, 1),
                                               (128, 128, 128, 3), (256, 128, 128, 1), (256, 256, 128, 5),
                                               (256, 256, 64, 2), (128, 128, 64, 8), (256, 256, 256, 1),
                                               (256, 256, 256, 3), (128, 256, 256, 2), (64, 64, 64, 3),
                                               (64, 64, 64, -2), (128, 128, 128, -3),
                                               # Cin = 32: 64-wide K chunks are offset pairs
                                               (32, 32, 32, 1), (32, 32, 32, 2), (32, 32, 32, -2), (32, 64, 64, 1),
                                               (32, 64, 32, 3), (32, 128, 128, 1)])
def test_halo_conv_vs_oracle(cin, cout, bn, split):
    import torch
    from paper_2509_24677_b200 import sparse as sp
    lv = _level((24, 20, 18), 0.25, cin + 3 * cout + split)
    n = lv.count()
    h = sp.build_halo(lv)
    xv, xt = _rows(n, cin, 1, lv.cap)
    layer = _layer(cin, cout, cout + split)
    w = osp.bf16_round(layer.w.cpu().numpy())
    b = layer.b.cpu().numpy().astype(np.float64)
    y = torch.zeros((lv.cap, cout), dtype=torch.bfloat16, device="cuda")
    ws = _run_halo(layer, xt, cin, lv, lv.nbr, h, y, cout, 0, bn, split, act="none")
    nbr = lv.nbr[:n].cpu().numpy().astype(np.int64)
    z = osp.gather_conv(xv.astype(np.float64), nbr, w, b)
    got = y[:n].float().cpu().numpy()
    assert np.all(np.abs(got - z) <= np.abs(z) * 2.0 ** -8 + 1e-4), np.abs(got - z).max()
    # counters left at zero; a second launch (graph replay) gives the identical result
    if split > 1:
        tiles = (lv.cap + 127) // 128
        assert not ws[:tiles * (cout // bn) * 4].any()
    y2 = torch.zeros_like(y)
    _run_halo(layer, xt, cin, lv, lv.nbr, h, y2, cout, 0, bn, split, act="none")
    assert torch.equal(y, y2)
    # relu epilogue into the right half of a concat buffer
    y3 = torch.zeros((lv.cap, 2 * cout), dtype=torch.bfloat16, device="cuda")
    _run_halo(layer, xt, cin, lv, lv.nbr, h, y3, 2 * cout, cout, bn, split)
    assert torch.equal(y3[:n, cout:], torch.relu(y[:n]))
    assert not y3[:n, :cout].any()


def test_halo_conv_tail_balancing_more_tiles_than_sms():
    """split = -2 with > 148 tiles: whole waves stay whole, only the tail tiles are cut."""
    import torch
    from paper_2509_24677_b200 import sparse as sp
    lv = _level((40, 40, 40), 0.3, 77)
    n = lv.count()
    assert (n + 127) // 128 > 148
    h = sp.build_halo(lv)
    xv, xt = _rows(n, 64, 6, lv.cap)
    layer = _layer(64, 64, 12)
    w = osp.bf16_round(layer.w.cpu().numpy())
    b = layer.b.cpu().numpy().astype(np.float64)
    ya = torch.zeros((lv.cap, 64), dtype=torch.bfloat16, device="cuda")
    yb = torch.zeros_like(ya)
    _run_halo(layer, xt, 64, lv, lv.nbr, h, ya, 64, 0, 64, -2, act="none")
    _run_halo(layer, xt, 64, lv, lv.nbr, h, yb, 64, 0, 64, 1, act="none")
    z = osp.gather_conv(xv.astype(np.float64), lv.nbr[:n].cpu().numpy().astype(np.int64), w, b)
    got = ya[:n].float().cpu().numpy()
    assert np.all(np.abs(got - z) <= np.abs(z) * 2.0 ** -8 + 1e-4), np.abs(got - z).max()
    # whole tiles are bit-identical to the unsplit run (same accumulation order)
    full = 148 * 128
    assert torch.equal(ya[:full], yb[:full])


@pytest.mark.parametrize("cin,bn", [(64, 64), (32, 32)])
def test_halo_conv_direct_read_path(cin, bn):
    """Tiles whose halo overflows the cache read uncached rows straight from HBM."""
    import torch
    from paper_2509_24677_b200 import sparse as sp
    rng = np.random.default_rng(11)
    n, cap, cout = 600, 640, 64
    nbr = rng.integers(0, n, size=(n, 27))
    nbr[rng.random((n, 27)) < 0.4] = -1
    nbr[:, 13] = np.arange(n)
    lv = sp.new_level(1, (16, 8, 5))   # shape only carries cap; tables are injected below
    lv.cap = cap
    lv.n = torch.tensor([n], dtype=torch.int32, device="cuda")
    lv.nbr = torch.full((cap, 27), -1, dtype=torch.int32, device="cuda")
    lv.nbr[:n] = torch.from_numpy(nbr.astype(np.int32)).cuda()
    lv.nbr_masks = sp.tile_masks(lv.nbr, 27, lv.n, cap)
    h = sp.build_halo(lv)
    assert (h["lnbr"][:(n + 127) // 128] == -2).any()
    xv, xt = _rows(n, cin, 4, cap)
    layer = _layer(cin, cout, 9)
    w = osp.bf16_round(layer.w.cpu().numpy())
    b = layer.b.cpu().numpy().astype(np.float64)
    y = torch.zeros((cap, cout), dtype=torch.bfloat16, device="cuda")
    _run_halo(layer, xt, cin, lv, lv.nbr, h, y, cout, 0, bn, 1, act="none")
    z = osp.gather_conv(xv.astype(np.float64), nbr.astype(np.int64), w, b)
    got = y[:n].float().cpu().numpy()
    assert np.all(np.abs(got - z) <= np.abs(z) * 2.0 ** -8 + 1e-4), np.abs(got - z).max()


def test_halo_plan_matches_plain_plan():
    """Config-2 U-Net (64^3 grid) with the halo kernel vs FPVS_HALO=0 plain gather: same mask."""
    import torch
    from paper_2509_24677_b200 import synth
    from paper_2509_24677_b200.froxel import FroxelGrid
    from paper_2509_24677_b200.unet import PvsUNet
    occ = synth.box_grid((64, 64, 64), 60, 1, 8, 5)
    bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
    net = PvsUNet(seed=1)
    a = net.plan(1, occ.shape)
    b = net.plan(1, occ.shape)
    b.use_halo, b.halo_cfg = False, {}
    assert a.use_halo and a.halo_cfg
    la = torch.zeros((a.L0.cap, 64), device="cuda")
    lb = torch.zeros((b.L0.cap, 64), device="cuda")
    oa = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
    ob = torch.empty_like(oa)
    a.run(bits, oa, 0.5, logits=la)
    b.run(bits, ob, 0.5, logits=lb)
    n = a.L0.count()
    assert float((la[:n] - lb[:n]).abs().max()) <= 2e-2
