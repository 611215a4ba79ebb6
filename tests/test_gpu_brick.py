"""Dense-brick tcgen05 submanifold conv (fpvs_spconv_brick).

Checked against the float64 oracle on the same bf16 values with the bf16
tolerance of test_gpu_halo (half an ulp + fp32 accumulation noise): partial
bricks at the grid edge, batches of two, empty bricks, tile widths, channel
splits; against the halo-cached kernel bit for bit (same chunk-outer,
tap-inner accumulation; absent taps add exact zeros); and on the config-2
U-Net's level-2 layer.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import sparse as osp

pytestmark = pytest.mark.gpu


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


def _brick(layer, xt, ldx, lv, y, ldy, col_off, bn, split, act="relu"):
    import torch
    from paper_2509_24677_b200 import _lib
    from paper_2509_24677_b200.neural import run_conv
    X, Y, Z = lv.dims
    nbytes = _lib.size("fpvs_spconv_brick_workspace_size", lv.B, X, Y, Z, layer.spec.out_channels, bn, split)
    ws = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device="cuda")
    run_conv(layer, xt, ldx, None, 27, lv.n, lv.cap, y, ldy, col_off, "bf16", act=act, brick=(bn, split, ws, lv))
    return ws


@pytest.mark.parametrize("dims,density,B,cin,cout,bn,split", [
    ((24, 20, 18), 0.25, 1, 64, 64, 64, 1),
    ((24, 20, 18), 0.8, 1, 128, 128, 128, 1),
    ((24, 20, 18), 0.8, 2, 128, 128, 128, 2),
    ((16, 16, 16), 0.9, 1, 256, 256, 128, 2),
    ((16, 16, 16), 0.9, 1, 256, 256, 256, 4),
    ((9, 33, 7), 0.5, 2, 64, 128, 128, 1),
    ((9, 33, 7), 0.5, 1, 256, 64, 64, 2),
    ((12, 16, 8), 0.02, 1, 128, 256, 256, 1),   # mostly empty bricks
])
def test_brick_conv_vs_oracle(dims, density, B, cin, cout, bn, split):
    import torch
    lv = _level(dims, density, cin + cout + split, B)
    n = lv.count()
    assert n > 0
    xv, xt = _rows(n, cin, 1, lv.cap)
    layer = _layer(cin, cout, cout + split)
    w = osp.bf16_round(layer.w.cpu().numpy())
    b = layer.b.cpu().numpy().astype(np.float64)
    y = torch.full((lv.cap, cout), 7.0, dtype=torch.bfloat16, device="cuda")
    ws = _brick(layer, xt, cin, lv, y, cout, 0, bn, split, act="none")
    nbr = lv.nbr[:n].cpu().numpy().astype(np.int64)
    z = osp.gather_conv(xv.astype(np.float64), nbr, w, b)
    got = y[:n].float().cpu().numpy()
    assert np.all(np.abs(got - z) <= np.abs(z) * 2.0 ** -8 + 1e-4), np.abs(got - z).max()
    assert bool((y[n:] == 7.0).all()), "rows past the active count must not be written"
    if split > 1:  # the arrival counters are back at zero for the next launch
        X, Y, Z = lv.dims
        items = B * X * ((Y + 15) // 16) * ((Z + 7) // 8) * (cout // bn)
        assert not ws[:items * 4].any()
    y2 = torch.zeros_like(y)
    _brick(layer, xt, cin, lv, y2, cout, 0, bn, split, act="none")
    assert torch.equal(y[:n], y2[:n])
    # relu epilogue into the right half of a concat buffer
    y3 = torch.zeros((lv.cap, 2 * cout), dtype=torch.bfloat16, device="cuda")
    _brick(layer, xt, cin, lv, y3, 2 * cout, cout, bn, split)
    assert torch.equal(y3[:n, cout:], torch.relu(y[:n]))
    assert not y3[:n, :cout].any()


@pytest.mark.parametrize("cin,cout,bn,split", [(64, 64, 64, 1), (128, 128, 128, 1), (256, 256, 128, 2),
                                               (128, 128, 128, 2)])
def test_brick_conv_equals_halo_conv(cin, cout, bn, split):
    """Same accumulation order as the halo-cached kernel: bit-identical rows."""
    import torch
    from paper_2509_24677_b200 import _lib
    from paper_2509_24677_b200 import sparse as sp
    from paper_2509_24677_b200.neural import run_conv
    lv = _level((20, 32, 24), 0.6, 5 + cin)
    n = lv.count()
    h = sp.build_halo(lv)
    _, xt = _rows(n, cin, 2, lv.cap)
    layer = _layer(cin, cout, 3)
    ya = torch.zeros((lv.cap, cout), dtype=torch.bfloat16, device="cuda")
    yb = torch.zeros_like(ya)
    ws = torch.zeros(_lib.size("fpvs_spconv_halo_workspace_size", lv.cap, cout, bn, split), dtype=torch.uint8,
                     device="cuda")
    run_conv(layer, xt, cin, lv.nbr, 27, lv.n, lv.cap, ya, cout, 0, "bf16", masks=lv.nbr_masks,
             halo=(bn, split, ws), halo_tabs=h)
    _brick(layer, xt, cin, lv, yb, cout, 0, bn, split)
    assert torch.equal(ya[:n], yb[:n])


def test_brick_conv_unet_level2_equals_halo():
    """The config-2 U-Net's enc2b on its real level-2 rows: brick == halo kernel."""
    import torch
    from paper_2509_24677_b200 import _lib, synth
    from paper_2509_24677_b200.froxel import FroxelGrid
    from paper_2509_24677_b200.neural import run_conv
    from paper_2509_24677_b200.unet import PvsUNet
    occ = synth.config2_grid(1)
    bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
    net = PvsUNet(seed=1)
    plan = net.plan(1, occ.shape)
    plan.tune(bits)
    out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
    plan.run(bits, out, 0.5)
    torch.cuda.synchronize()
    lv = plan.L2
    n = lv.count()
    layer = net.layers["enc2b"]
    x = plan.t2b  # enc2a's output = enc2b's input
    ya = torch.zeros((lv.cap, 256), dtype=torch.bfloat16, device="cuda")
    yb = torch.zeros_like(ya)
    ws = torch.zeros(_lib.size("fpvs_spconv_halo_workspace_size", lv.cap, 256, 128, 2), dtype=torch.uint8,
                     device="cuda")
    run_conv(layer, x, 256, lv.nbr, 27, lv.n, lv.cap, ya, 256, 0, "bf16", masks=lv.nbr_masks,
             halo=(128, 2, ws), halo_tabs=lv.extra["halo"])
    _brick(layer, x, 256, lv, yb, 256, 0, 128, 2)
    assert torch.equal(ya[:n], yb[:n])


def test_unet_frame_with_level2_bricks_equals_default():
    """FPVS_BRICK=2 (the level-2 convs on the brick kernel, 128-wide tiles, a
    2-way channel split as clusters) gives the default frame's bits, eagerly
    and from the captured graph."""
    import os
    import torch
    from paper_2509_24677_b200 import synth
    from paper_2509_24677_b200.froxel import FroxelGrid
    from paper_2509_24677_b200.pipeline import FramePipeline
    from paper_2509_24677_b200.unet import PvsUNet
    occ = synth.config2_grid(1)
    bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
    outs = []
    for flag in ("", "2"):
        os.environ["FPVS_BRICK"] = flag
        try:
            pipe = FramePipeline(PvsUNet(seed=1), 1, occ.shape)
        finally:
            os.environ.pop("FPVS_BRICK", None)
        pipe.load(bits)
        pipe.capture()
        assert bool(pipe.plan.brick_of) == (flag == "2")
        pipe.run_device()
        torch.cuda.synchronize()
        eager = torch.full_like(pipe.out_bits, 0x5A)
        pipe.plan.run(bits, eager, 0.5)
        torch.cuda.synchronize()
        assert torch.equal(eager, pipe.out_bits)
        outs.append(pipe.out_bits.clone())
    assert torch.equal(outs[0], outs[1])
