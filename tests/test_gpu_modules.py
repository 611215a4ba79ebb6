"""torch autograd face (modules.py) vs the library's own fp32 training step.

``PvsNetModule`` + ``pvs_loss`` + ``loss.backward()`` must give the loss and
the per-parameter gradients of ``train.TrainStep`` (fp32 SIMT backward, the
1e-4 parity mode) on the same batch, and a torch optimizer step must move
the Parameters.  Also: a single ``SparseConv3dFunction`` against float64
(forward and all three gradients via torch.autograd.gradcheck-style finite
sums replaced by the explicit oracle formulas).
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import sparse as osp

pytestmark = pytest.mark.gpu


def test_module_grads_match_train_step():
    import torch
    from paper_2509_24677_b200 import synth
    from paper_2509_24677_b200.froxel import FroxelGrid
    from paper_2509_24677_b200.modules import PvsNetModule
    from paper_2509_24677_b200.neural import ModelConfig, PvsNet, TrainConfig
    from paper_2509_24677_b200.train import TrainStep
    B, dims = 2, (64, 64, 64)
    pairs = [synth.config5_pair(1, i) for i in range(B)]
    pairs = [(g[:64, :64, :64], lb[:64, :64, :64]) for g, lb in pairs]
    bits = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(g).bits for g, _ in pairs])).cuda()
    gt = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(lb).bits for _, lb in pairs])).cuda()
    cfg = ModelConfig.config1()
    tcfg = TrainConfig(optimizer="adamw")
    net = PvsNet(cfg, np.random.Generator(np.random.PCG64(3)), precision="fp32")
    step = TrainStep(net, B, dims, tcfg)
    step.forward_backward(bits, gt)
    torch.cuda.synchronize()
    mod = PvsNetModule(cfg, np.random.Generator(np.random.PCG64(3)))
    loss = mod.loss(bits, gt, B, dims, tcfg)
    loss.backward()
    torch.cuda.synchronize()
    assert abs(float(loss.detach()) - float(step.loss)) <= 1e-6 * max(1.0, abs(float(step.loss)))
    for m, (dw, db) in zip(mod.layers, step.views):
        for got, want in ((m.weight.grad, dw), (m.bias.grad, db)):
            err = float((got - want).abs().max())
            scale = float(want.abs().max()) + 1e-12
            assert err <= 1e-4 * scale + 1e-7, (err, scale)
    opt = torch.optim.AdamW(mod.parameters(), lr=1e-3)
    w0 = mod.layers[1].weight.detach().clone()
    opt.step()
    assert not torch.equal(w0, mod.layers[1].weight)


def test_sparse_conv_function_vs_float64():
    import torch
    from paper_2509_24677_b200 import sparse as sp
    from paper_2509_24677_b200.modules import sparse_conv3d
    rng = np.random.default_rng(4)
    dims = (12, 10, 9)
    mask = rng.random((1,) + dims) < 0.35
    lv = sp.new_level(1, dims)
    lv.active.copy_(torch.from_numpy(mask.reshape(-1).astype(np.uint8)).cuda())
    sp.compact(lv)
    sp.build_subm(lv)
    n, cin, cout = lv.count(), 8, 16
    xv = rng.normal(size=(n, cin))
    wv = rng.normal(size=(27 * cin, cout)) * 0.2
    bv = rng.normal(size=cout) * 0.1
    gv = rng.normal(size=(n, cout))
    x = torch.zeros((lv.cap, cin), device="cuda")
    x[:n] = torch.tensor(xv, dtype=torch.float32)
    x.requires_grad_(True)
    w = torch.tensor(wv, dtype=torch.float32, device="cuda", requires_grad=True)
    b = torch.tensor(bv, dtype=torch.float32, device="cuda", requires_grad=True)
    y = sparse_conv3d(x, w, b, lv, 27, "relu")
    g = torch.zeros_like(y)
    g[:n] = torch.tensor(gv, dtype=torch.float32)
    y.backward(g)
    tab = lv.nbr[:n].cpu().numpy().astype(np.int64)
    xf = xv.astype(np.float32).astype(np.float64)
    wf = wv.astype(np.float32).astype(np.float64)
    z = osp.gather_conv(xf, tab, wf, bv.astype(np.float32).astype(np.float64))
    yr = np.maximum(z, 0)
    assert np.allclose(y[:n].detach().cpu().numpy(), yr, atol=1e-4)
    dz = gv.astype(np.float32).astype(np.float64) * (z > 0)
    dw = np.zeros((27, cin, cout))
    dx = np.zeros((n, cin))
    for j in range(27):
        v = tab[:, j] >= 0
        dw[j] = xf[tab[v, j]].T @ dz[v]
        np.add.at(dx, tab[v, j], dz[v] @ wf.reshape(27, cin, cout)[j].T)
    assert np.allclose(w.grad.cpu().numpy(), dw.reshape(27 * cin, cout), atol=1e-3, rtol=1e-4)
    assert np.allclose(b.grad.cpu().numpy(), dz.sum(0), atol=1e-3, rtol=1e-4)
    assert np.allclose(x.grad[:n].cpu().numpy(), dx, atol=1e-3, rtol=1e-4)
    assert not x.grad[n:].any()


def test_module_bf16_grads_close_to_fp32():
    """bf16 tensor-core autograd path: loss and per-parameter gradients within bf16 noise of fp32."""
    import torch
    from paper_2509_24677_b200 import synth
    from paper_2509_24677_b200.froxel import FroxelGrid
    from paper_2509_24677_b200.modules import PvsNetModule
    from paper_2509_24677_b200.neural import ModelConfig, TrainConfig
    B, dims = 2, (64, 64, 64)
    pairs = [synth.config5_pair(2, i) for i in range(B)]
    pairs = [(g[:64, :64, :64], lb[:64, :64, :64]) for g, lb in pairs]
    bits = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(g).bits for g, _ in pairs])).cuda()
    gt = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(lb).bits for _, lb in pairs])).cuda()
    cfg = ModelConfig.config1()
    mods = {p: PvsNetModule(cfg, np.random.Generator(np.random.PCG64(5)), precision=p) for p in ("fp32", "bf16")}
    losses = {}
    for p, m in mods.items():
        loss = m.loss(bits, gt, B, dims, TrainConfig())
        loss.backward()
        losses[p] = float(loss.detach())
    torch.cuda.synchronize()
    assert abs(losses["bf16"] - losses["fp32"]) <= 0.02 * abs(losses["fp32"]) + 1e-4
    for a, b in zip(mods["bf16"].parameters(), mods["fp32"].parameters()):
        rel = float((a.grad - b.grad).norm() / (b.grad.norm() + 1e-30))
        assert rel < 0.05, (a.shape, rel)
