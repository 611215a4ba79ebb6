"""Tensor-core backward (fpvs_spconv_wgrad_tc, fpvs_spconv_tc_dgrad) vs float64.

Conv3d.backward (pkg/src/froxelpvs/neural.py:221-249) on the active set:
dW = colsᵀ·dz, db = Σ dz, dx = col2im(dz·Wᵀ) masked by relu' of the layer
below.  Inputs are bf16-representable, so the float64 reference sees exactly
the device's operands; tolerances are fp32-accumulation noise for dW / db and
half a bf16 ulp + noise for the bf16 dx.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import sparse as osp

pytestmark = pytest.mark.gpu


def _level(dims, density, seed):
    import torch
    from paper_2509_24677_b200 import sparse as sp
    rng = np.random.default_rng(seed)
    mask = rng.random((1,) + dims) < density
    lv = sp.new_level(1, dims)
    lv.active.copy_(torch.from_numpy(mask.reshape(-1).astype(np.uint8)).cuda())
    sp.compact(lv)
    sp.build_subm(lv)
    return lv


def _bf16(n, c, cap, seed, relu=False):
    import torch
    rng = np.random.default_rng(seed)
    v = rng.normal(size=(n, c)).astype(np.float32)
    if relu:
        v = np.maximum(v, 0) * (rng.random((n, c)) < 0.7)
    v = osp.bf16_round(v).astype(np.float32)
    t = torch.zeros((cap, c), dtype=torch.bfloat16, device="cuda")
    t[:n] = torch.from_numpy(v).to(torch.bfloat16).cuda()
    return v.astype(np.float64), t


@pytest.mark.parametrize("K,cin,cout", [(27, 32, 32), (27, 8, 32), (1, 32, 8), (27, 64, 128), (27, 128, 64)])
def test_wgrad_tc_vs_float64(K, cin, cout):
    import torch
    from paper_2509_24677_b200 import _lib
    lv = _level((20, 18, 16), 0.3, K + cin + cout)
    n = lv.count()
    xv, xt = _bf16(n, cin, lv.cap, 1, relu=True)
    dv, dt = _bf16(n, cout, lv.cap, 2)
    dw = torch.full((K * cin, cout), 7.0, device="cuda")
    db = torch.full((cout,), 7.0, device="cuda")
    ws = torch.empty(_lib.size("fpvs_wgrad_tc_workspace_size", K, cin, cout, lv.cap), dtype=torch.uint8, device="cuda")
    nbr = lv.nbr if K == 27 else None
    _lib.call("fpvs_spconv_wgrad_tc", _lib.ptr(xt), cin, _lib.ptr(dt), cout, _lib.ptr(nbr), K, _lib.ptr(lv.n), lv.cap,
              cin, cout, _lib.ptr(dw), _lib.ptr(db), _lib.ptr(ws), ws.numel(), 0)
    tab = lv.nbr[:n].cpu().numpy().astype(np.int64) if K == 27 else np.arange(n)[:, None]
    ref = np.zeros((K, cin, cout))
    for j in range(K):
        v = tab[:, j] >= 0
        ref[j] = xv[tab[v, j]].T @ dv[v]
    ref = ref.reshape(K * cin, cout)
    got = dw.cpu().numpy()
    scale = np.abs(ref).max()
    assert np.abs(got - ref).max() <= 2e-5 * scale + 1e-4, (np.abs(got - ref).max(), scale)
    assert np.allclose(db.cpu().numpy(), dv.sum(0), rtol=1e-4, atol=1e-3)
    # deterministic: a second run is bit-identical
    dw2 = torch.zeros_like(dw)
    _lib.call("fpvs_spconv_wgrad_tc", _lib.ptr(xt), cin, _lib.ptr(dt), cout, _lib.ptr(nbr), K, _lib.ptr(lv.n), lv.cap,
              cin, cout, _lib.ptr(dw2), None, _lib.ptr(ws), ws.numel(), 0)
    assert torch.equal(dw, dw2)


@pytest.mark.parametrize("K,cin,cout", [(27, 32, 32), (1, 32, 8), (27, 64, 64)])
def test_dgrad_tc_masked_vs_float64(K, cin, cout):
    import torch
    from paper_2509_24677_b200 import _lib
    from paper_2509_24677_b200.neural import Conv3d, ConvSpec, packed_dgrad_cache
    lv = _level((20, 18, 16), 0.3, 5 * K + cin)
    n = lv.count()
    dv, dt = _bf16(n, cout, lv.cap, 3)
    mv, mt = _bf16(n, cin, lv.cap, 4, relu=True)  # the kept output of the layer below
    layer = Conv3d(ConvSpec(3 if K == 27 else 1, cin, cout, "relu"), np.random.default_rng(K + cout),
                   init="kaiming_uniform")
    w = osp.bf16_round(layer.w.cpu().numpy()).reshape(K, cin, cout)
    dx = torch.zeros((lv.cap, cin), dtype=torch.bfloat16, device="cuda")
    nbr = lv.nbr if K == 27 else None
    _lib.call("fpvs_spconv_tc_dgrad", _lib.ptr(dt), cout, lv.cap, _lib.ptr(nbr), K,
              _lib.ptr(lv.nbr_masks if K == 27 else None), _lib.ptr(lv.n), lv.cap,
              _lib.ptr(packed_dgrad_cache(layer)), 0, cin, cout, _lib.ptr(mt), cin, _lib.ptr(dx), cin, 0)
    tab = lv.nbr[:n].cpu().numpy().astype(np.int64) if K == 27 else np.arange(n)[:, None]
    ref = np.zeros((n, cin))
    for j in range(K):
        v = tab[:, j] >= 0
        np.add.at(ref, tab[v, j], dv[v] @ w[j].T)
    ref *= mv > 0
    got = dx[:n].float().cpu().numpy()
    assert np.all(np.abs(got - ref) <= np.abs(ref) * 2.0 ** -8 + 1e-3 * np.abs(ref).max() + 1e-6), \
        np.abs(got - ref).max()
    assert not got[mv <= 0].any()


def test_train_step_tc_backward_matches_simt():
    """Config-1 net, bf16: the tensor-core backward's flat gradient vs the SIMT fp32 backward on the same step."""
    import torch
    from paper_2509_24677_b200 import synth
    from paper_2509_24677_b200.froxel import FroxelGrid
    from paper_2509_24677_b200.neural import ModelConfig, PvsNet, TrainConfig
    from paper_2509_24677_b200.train import TrainStep
    pairs = [synth.config5_pair(0, i) for i in range(2)]
    bits = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(g).bits for g, _ in pairs])).cuda()
    gt = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(l).bits for _, l in pairs])).cuda()
    net = PvsNet(ModelConfig.config1(), np.random.Generator(np.random.PCG64(0)), precision="bf16")
    step = TrainStep(net, 2, (128, 128, 128), TrainConfig(optimizer="adamw"))
    assert step.tc_backward
    step.forward_backward(bits, gt)
    g_tc = step.grads.clone()
    step.tc_backward = False  # same forward caches, SIMT fp32 backward
    step.grads.zero_()
    step.backward()
    g_simt = step.grads.clone()
    o = 0
    for layer in net.layers:
        for t in (layer.w, layer.b):
            a, b = g_tc[o:o + t.numel()], g_simt[o:o + t.numel()]
            rel = float((a - b).norm() / (b.norm() + 1e-30))
            assert rel < 0.02, (layer.spec, t.shape, rel)
            o += t.numel()


@pytest.mark.parametrize("cout,dims,density", [(32, (20, 18, 16), 0.3), (8, (20, 18, 16), 0.3),
                                               (16, (40, 36, 30), 0.25), (32, (64, 64, 32), 0.08)])
def test_wgrad_halo_vs_float64(cout, dims, density):
    """fpvs_spconv_wgrad_halo (27 taps, Cin 32): dW / db vs float64, and vs the gathering wgrad."""
    import torch
    from paper_2509_24677_b200 import _lib, sparse as sp
    lv = _level(dims, density, cout + 7)
    n = lv.count()
    cin = 32
    h = sp.build_halo(lv)
    xv, xt = _bf16(n, cin, lv.cap, 5, relu=True)
    dv, dt = _bf16(n, cout, lv.cap, 6)
    dw = torch.full((27 * cin, cout), 7.0, device="cuda")
    db = torch.full((cout,), 7.0, device="cuda")
    ws = torch.empty(_lib.size("fpvs_wgrad_halo_workspace_size", lv.cap), dtype=torch.uint8, device="cuda")
    _lib.call("fpvs_spconv_wgrad_halo", _lib.ptr(xt), cin, _lib.ptr(dt), cout, _lib.ptr(lv.nbr), _lib.ptr(lv.n),
              lv.cap, _lib.ptr(h["rows"]), _lib.ptr(h["n"]), _lib.ptr(h["lnbr"]), cin, cout, _lib.ptr(dw), _lib.ptr(db),
              _lib.ptr(ws), ws.numel(), 0)
    tab = lv.nbr[:n].cpu().numpy().astype(np.int64)
    ref = np.zeros((27, cin, cout))
    for j in range(27):
        v = tab[:, j] >= 0
        ref[j] = xv[tab[v, j]].T @ dv[v]
    ref = ref.reshape(27 * cin, cout)
    got = dw.cpu().numpy()
    scale = np.abs(ref).max()
    assert np.abs(got - ref).max() <= 2e-5 * scale + 1e-4, (np.abs(got - ref).max(), scale)
    assert np.allclose(db.cpu().numpy(), dv.sum(0), rtol=1e-4, atol=1e-3)
    dw2 = torch.zeros_like(dw)
    _lib.call("fpvs_spconv_wgrad_halo", _lib.ptr(xt), cin, _lib.ptr(dt), cout, _lib.ptr(lv.nbr), _lib.ptr(lv.n),
              lv.cap, _lib.ptr(h["rows"]), _lib.ptr(h["n"]), _lib.ptr(h["lnbr"]), cin, cout, _lib.ptr(dw2), None,
              _lib.ptr(ws), ws.numel(), 0)
    assert torch.equal(dw, dw2)  # deterministic
