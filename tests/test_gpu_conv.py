"""(3) sparse convolution kernels (SIMT fp32 and tcgen05 bf16) and the fused head.

Tolerances (north_star): thresholded masks bit-exact except froxels whose
reference probability lies within 1e-3 of tau; logits max-abs <= 1e-4 in the
fp32 mode (vs the float64 oracle) and <= 2e-2 in bf16 (vs the oracle's bf16
emulation, which rounds weights and stored activations exactly as the device).
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import sparse as osp
from paper_2509_24677_b200 import synth
from paper_2509_24677_b200.froxel import FroxelGrid

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FP32_LOGIT_TOL = 1e-4
BF16_LOGIT_TOL = 2e-2
BAND = 1e-3


def _mask_mismatch(got_bits, ref_prob_dense, tau=0.5):
    """Bits that differ from the oracle outside the +-BAND exemption around tau."""
    ref_bits = ref_prob_dense >= tau
    got = FroxelGrid(ref_prob_dense.shape, bits=got_bits).to_dense()
    diff = got != ref_bits
    return int((diff & (np.abs(ref_prob_dense - tau) >= BAND)).sum()), int(diff.sum())


def test_config1_fp32_end_to_end_vs_reference_golden(golden):
    """Config 1 through the drop-in predict_pvs (fp32 SIMT) vs the masked reference."""
    import torch
    from paper_2509_24677_b200 import sparse as sp
    from paper_2509_24677_b200.neural import PvsNet, predict_pvs
    g = golden("config1.npz")
    net = PvsNet.load(os.path.join(GOLDEN, "config1.fpvw"))
    grid = FroxelGrid(tuple(g["dims"]), bits=g["bits"])
    bits = torch.from_numpy(g["bits"]).cuda()
    lv = sp.level_from_bits(bits, 1, grid.dims, 2)
    feats = sp.gather_features(bits, lv, grid.dims, 2, torch.float32)
    logits = torch.zeros((lv.cap, 8), device="cuda")
    net.forward_rows(feats, lv, grid.dims, logits=logits)
    n = lv.count()
    assert np.array_equal(lv.coords[:n].cpu().numpy(), g["coords"])
    err = np.abs(logits[:n].cpu().numpy() - g["logits_active"]).max()
    assert err <= FP32_LOGIT_TOL, err
    pred = predict_pvs(grid, net)
    assert pred.role == "predicted_pvs" and pred.dims == grid.dims
    ref_dense = osp.deinterleave(osp.scatter_cells(g["coords"], g["prob_active"], (1, 32, 32, 16))[0], 2)
    hard, total = _mask_mismatch(pred.bits, ref_dense)
    assert hard == 0, (hard, total)


def test_reference_golden_layers_simt(golden):
    """Each masked reference layer of conv.npz (Cin 8 -> 16 -> 16 -> 8) through fpvs_spconv_simt / head."""
    import torch
    from paper_2509_24677_b200 import sparse as sp
    from paper_2509_24677_b200.neural import Conv3d, ConvSpec, run_conv
    g = golden("conv.npz")
    x, mask = g["x"], g["mask"]
    B = mask.shape[0]
    lv = sp.new_level(B, mask.shape[1:])
    lv.active.copy_(torch.from_numpy(mask.reshape(-1).astype(np.uint8)).cuda())
    sp.compact(lv)
    sp.build_subm(lv)
    n = lv.count()
    coords = lv.coords[:n].cpu().numpy()
    h = torch.zeros((lv.cap, 8), device="cuda")
    h[:n] = torch.from_numpy(x[tuple(coords.T)]).float().cuda()
    specs = [ConvSpec(3, 8, 16, "relu"), ConvSpec(3, 16, 16, "relu"), ConvSpec(1, 16, 8, "sigmoid")]
    for i, s in enumerate(specs):
        layer = Conv3d(s)
        layer.set_weights(g[f"w{i}"], g[f"b{i}"])
        y = torch.zeros((lv.cap, s.out_channels), device="cuda")
        table, K = (lv.nbr, 27) if s.kernel == 3 else (None, 1)
        run_conv(layer, h, h.shape[1], table, K, lv.n, lv.cap, y, y.shape[1])
        ref = g[f"y{i}"][tuple(coords.T)]
        # the golden weights are float64; the device holds their float32 rounding
        np.testing.assert_allclose(y[:n].cpu().numpy(), ref, atol=2e-5, rtol=1e-5)
        h = y


def _rand_level(B, dims, density, seed):
    import torch
    from paper_2509_24677_b200 import sparse as sp
    rng = np.random.default_rng(seed)
    mask = rng.random((B,) + dims) < density
    lv = sp.new_level(B, dims)
    lv.active.copy_(torch.from_numpy(mask.reshape(-1).astype(np.uint8)).cuda())
    sp.compact(lv)
    sp.build_subm(lv)
    return lv, mask


def _bf16_rows(n, c, seed, cap, relu_like=True):
    import torch
    rng = np.random.default_rng(seed)
    v = rng.normal(size=(n, c)).astype(np.float32)
    if relu_like:
        v = np.maximum(v, 0)
    v = osp.bf16_round(v).astype(np.float32)
    t = torch.zeros((cap, c), dtype=torch.bfloat16, device="cuda")
    t[:n] = torch.from_numpy(v).to(torch.bfloat16).cuda()
    return v, t


@pytest.mark.parametrize("cin,cout", [(8, 32), (32, 32), (64, 64), (64, 128), (128, 128), (256, 128), (256, 256),
                                      (128, 64)])
def test_tc_subm_vs_oracle(cin, cout):
    """tcgen05 gather-GEMM (bf16 in, fp32 accumulate) vs float64 on the same bf16 values."""
    import torch
    from paper_2509_24677_b200.neural import Conv3d, ConvSpec, run_conv
    lv, _ = _rand_level(2, (12, 10, 9), 0.3, cin + cout)
    n = lv.count()
    xv, xt = _bf16_rows(n, cin, 1, lv.cap)
    layer = Conv3d(ConvSpec(3, cin, cout, "relu"), np.random.default_rng(cout), init="kaiming_uniform")
    layer.b.uniform_(-0.1, 0.1)
    w = osp.bf16_round(layer.w.cpu().numpy())
    b = layer.b.cpu().numpy().astype(np.float64)
    y = torch.zeros((lv.cap, cout), dtype=torch.bfloat16, device="cuda")
    run_conv(layer, xt, cin, lv.nbr, 27, lv.n, lv.cap, y, cout, 0, "bf16", act="none")
    nbr = lv.nbr[:n].cpu().numpy().astype(np.int64)
    z = osp.gather_conv(xv.astype(np.float64), nbr, w, b)
    got = y[:n].float().cpu().numpy()
    # bf16 output rounding: half an ulp (2^-9 relative) plus fp32-accumulation noise
    assert np.all(np.abs(got - z) <= np.abs(z) * 2.0 ** -8 + 1e-4), np.abs(got - z).max()
    # relu epilogue and a column offset into a wider buffer
    y2 = torch.zeros((lv.cap, 2 * cout), dtype=torch.bfloat16, device="cuda")
    run_conv(layer, xt, cin, lv.nbr, 27, lv.n, lv.cap, y2, 2 * cout, cout, "bf16", act="relu")
    assert torch.equal(y2[:n, cout:], torch.relu(y[:n]))
    assert not y2[:n, :cout].any()


def test_tc_matches_simt_on_bf16_inputs():
    import torch
    from paper_2509_24677_b200.neural import Conv3d, ConvSpec, run_conv
    lv, _ = _rand_level(1, (20, 20, 20), 0.15, 7)
    n = lv.count()
    _, xt = _bf16_rows(n, 64, 2, lv.cap)
    layer = Conv3d(ConvSpec(3, 64, 64, "relu"), np.random.default_rng(3), init="kaiming_uniform")
    layer.w.copy_(layer.w.bfloat16().float())   # same bf16 weights on both paths
    a = torch.zeros((lv.cap, 64), dtype=torch.float32, device="cuda")
    b = torch.zeros((lv.cap, 64), dtype=torch.bfloat16, device="cuda")
    run_conv(layer, xt, 64, lv.nbr, 27, lv.n, lv.cap, a, 64, 0, "fp32")
    run_conv(layer, xt, 64, lv.nbr, 27, lv.n, lv.cap, b, 64, 0, "bf16")
    ref = a[:n]
    assert torch.all((b[:n].float() - ref).abs() <= ref.abs() * 2.0 ** -8 + 1e-4)


@pytest.mark.parametrize("kind,cin,cout", [("down", 64, 128), ("down", 128, 256), ("up", 256, 128), ("up", 128, 64)])
def test_tc_down_up_vs_oracle(kind, cin, cout):
    import torch
    from paper_2509_24677_b200 import sparse as sp
    from paper_2509_24677_b200.unet import SparseLayer
    from paper_2509_24677_b200.neural import run_conv
    fine, mask = _rand_level(1, (16, 12, 10), 0.2, cin * 3 + cout)
    coarse, down, up = sp.coarsen(fine)
    nf, nc = fine.count(), coarse.count()
    rng = np.random.default_rng(5)
    w = rng.uniform(-0.2, 0.2, size=(8 * cin, cout))
    b = rng.uniform(-0.1, 0.1, size=cout)
    layer = SparseLayer("t", kind, cin, cout, w, b)
    wb = osp.bf16_round(w)
    if kind == "down":
        xv, xt = _bf16_rows(nf, cin, 4, fine.cap)
        y = torch.zeros((coarse.cap, cout), dtype=torch.bfloat16, device="cuda")
        run_conv(layer, xt, cin, down, 8, coarse.n, coarse.cap, y, cout, 0, "bf16", act="relu")
        z = osp.gather_conv(xv.astype(np.float64), down[:nc].cpu().numpy().astype(np.int64), wb, b)
        rows = nc
    else:
        xv, xt = _bf16_rows(nc, cin, 4, coarse.cap)
        y = torch.zeros((fine.cap, cout), dtype=torch.bfloat16, device="cuda")
        run_conv(layer, xt, cin, up, 8, fine.n, fine.cap, y, cout, 0, "bf16", act="relu")
        fc = fine.coords[:nf].cpu().numpy().astype(np.int64)
        cc = coarse.coords[:nc].cpu().numpy().astype(np.int64)
        par, parity = osp.kmap_up(fc, cc, coarse.dims)
        z = osp.up_conv(xv.astype(np.float64), par, parity, wb, b)
        rows = nf
    ref = np.maximum(z, 0)
    got = y[:rows].float().cpu().numpy()
    assert np.all(np.abs(got - ref) <= np.abs(ref) * 2.0 ** -8 + 1e-4), np.abs(got - ref).max()


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_head_bits_probs(precision):
    """Fused head: 1x1x1 conv + sigmoid + >= tau + deinterleave bit-pack, d = 2 and 4."""
    import torch
    from paper_2509_24677_b200 import sparse as sp
    from paper_2509_24677_b200.neural import Conv3d, ConvSpec, run_head
    for d, occ in ((2, synth.box_grid((32, 16, 16), 30, 1, 4, 3)), (4, synth.box_grid((64, 32, 32), 40, 1, 6, 4))):
        d3 = d ** 3
        bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
        lv = sp.level_from_bits(bits, 1, occ.shape, d)
        n = lv.count()
        cin = 32 if d == 2 else 64
        xv, xt = _bf16_rows(n, cin, 9, lv.cap)
        x = xt if precision == "bf16" else xt.float()
        layer = Conv3d(ConvSpec(1, cin, d3, "sigmoid"), np.random.default_rng(d), init="kaiming_uniform")
        layer.b.uniform_(-0.2, 0.2)
        w = layer.w.cpu().numpy().astype(np.float64)
        if precision == "bf16":
            w = osp.bf16_round(w)
        z = xv.astype(np.float64) @ w + layer.b.cpu().numpy()
        p = osp.sigmoid(z)
        out = torch.zeros(occ.size // 8, dtype=torch.uint8, device="cuda")
        probs = torch.zeros((lv.cap, d3), device="cuda")
        logits = torch.zeros((lv.cap, d3), device="cuda")
        run_head(layer, x, cin, lv, d, occ.shape, 0.5, out, probs, logits, precision)
        assert np.abs(logits[:n].cpu().numpy() - z).max() < 1e-4
        coords = lv.coords[:n].cpu().numpy()
        dense = osp.deinterleave(osp.scatter_cells(coords, p, (1,) + lv.dims)[0], d)
        hard, _ = _mask_mismatch(out.cpu().numpy(), dense)
        assert hard == 0


def test_config1_bf16_vs_bf16_oracle(golden):
    """Config-1 net on the tcgen05 path vs the oracle's bf16 emulation (mask + logits)."""
    import torch
    from paper_2509_24677_b200 import sparse as sp
    from paper_2509_24677_b200.neural import PvsNet, read_fpvw
    g = golden("config1.npz")
    net = PvsNet.load(os.path.join(GOLDEN, "config1.fpvw"), precision="bf16")
    dims = tuple(g["dims"])
    bits = torch.from_numpy(g["bits"]).cuda()
    lv = sp.level_from_bits(bits, 1, dims, 2)
    feats = sp.gather_features(bits, lv, dims, 2, torch.bfloat16)
    logits = torch.zeros((lv.cap, 8), device="cuda")
    out = torch.zeros(int(np.prod(dims)) // 8, dtype=torch.uint8, device="cuda")
    net.forward_rows(feats, lv, dims, out_bits=out, logits=logits)
    _, specs, arrays = read_fpvw(os.path.join(GOLDEN, "config1.fpvw"))
    layers = [(s.kernel, w.astype(np.float64), b.astype(np.float64), s.activation) for s, (w, b) in zip(specs, arrays)]
    occ = FroxelGrid(dims, bits=g["bits"]).to_dense()
    coords, z16 = osp.chain_forward(osp.interleave(occ.astype(np.float64), 2)[None], layers, bf16=True,
                                    return_logits=True)
    n = lv.count()
    err = np.abs(logits[:n].cpu().numpy() - z16).max()
    assert err <= BF16_LOGIT_TOL, err
    dense = osp.deinterleave(osp.scatter_cells(coords, osp.sigmoid(z16), (1, 32, 32, 16))[0], 2)
    hard, total = _mask_mismatch(out.cpu().numpy(), dense)
    assert hard == 0, (hard, total)


@pytest.mark.parametrize("bn", [32, 64, 128, 256])
def test_tc_n_split_tiles(bn):
    """Output-column blocking (BN < Cout) gives the same result as one block."""
    import torch
    from paper_2509_24677_b200.neural import Conv3d, ConvSpec, run_conv
    lv, _ = _rand_level(1, (14, 12, 10), 0.3, bn)
    n = lv.count()
    _, xt = _bf16_rows(n, 256, 3, lv.cap)
    layer = Conv3d(ConvSpec(3, 256, 256, "relu"), np.random.default_rng(8), init="kaiming_uniform")
    layer.b.uniform_(-0.1, 0.1)
    ref = torch.zeros((lv.cap, 256), dtype=torch.bfloat16, device="cuda")
    got = torch.zeros_like(ref)
    run_conv(layer, xt, 256, lv.nbr, 27, lv.n, lv.cap, ref, 256, 0, "bf16", bn=0)
    run_conv(layer, xt, 256, lv.nbr, 27, lv.n, lv.cap, got, 256, 0, "bf16", bn=bn)
    assert torch.equal(got[:n], ref[:n])
