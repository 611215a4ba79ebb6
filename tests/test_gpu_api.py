"""The reference-shaped layer API on the device:
``Conv3d.forward(x, keep_cache)`` / ``Conv3d.backward(dy, cache)``,
``conv3d_forward`` / ``conv3d_backward``, ``PvsNet.forward`` /
``forward_cached`` / ``backward`` / ``sgd_step``, ``evaluate_pairs(net, x, y,
tau)``, any odd kernel and a 3^3 head (``ModelConfig.default``), and the
reference CLI's own train / infer call pattern (pkg/src/froxelpvs/cli.py:255-282)
with only the imports swapped.

Expected values: ``tests/golden/api.npz`` / ``default_d2.fpvw`` written by the
reference itself (make_api_golden.py: its Conv3d forward/backward and
sgd_step with the submanifold mask), and the float64 oracle where the
reference has no direct counterpart.  Tolerances: fp32 device arithmetic,
so outputs within 1e-5 absolute (probabilities), gradients within 1e-4 of the
largest reference magnitude per tensor.
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
SPECS = {"def": [(3, 8, 8, "relu"), (3, 8, 8, "relu"), (3, 8, 8, "sigmoid")],
         "k5": [(5, 8, 8, "relu"), (3, 8, 8, "sigmoid")]}


def _close(got, want, rel=1e-4):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    scale = max(1.0, float(np.abs(want).max()))
    err = float(np.abs(got - want).max())
    assert err <= rel * scale, f"max err {err} (scale {scale})"


def _net(g, tag):
    from paper_2509_24677_b200.neural import ConvSpec, ModelConfig, PvsNet
    specs = [ConvSpec(*s) for s in SPECS[tag]]
    net = PvsNet(ModelConfig(2, specs))
    for i, L in enumerate(net.layers):
        L.set_weights(g[f"{tag}_w{i}"], g[f"{tag}_b{i}"])
    return net


def test_default_config_is_the_reference_default_and_init_matches_its_fpvw():
    """ModelConfig.default == neural.py:94-99 (3^3 head); He-normal init from
    PCG64(3) equals the reference's own FPVW bytes; PvsNet.load reads it."""
    from paper_2509_24677_b200.neural import ModelConfig, PvsNet, read_fpvw
    cfg = ModelConfig.default(2, 8)
    assert [(s.kernel, s.in_channels, s.out_channels, s.activation) for s in cfg.layers] == SPECS["def"]
    net = PvsNet(cfg, np.random.Generator(np.random.PCG64(3)))
    d, specs, arrays = read_fpvw(os.path.join(GOLDEN, "default_d2.fpvw"))
    assert d == 2 and len(specs) == 3
    for L, (w, b) in zip(net.layers, arrays):
        assert np.array_equal(L.w.cpu().numpy(), w) and np.array_equal(L.b.cpu().numpy(), b)
    loaded = PvsNet.load(os.path.join(GOLDEN, "default_d2.fpvw"))
    assert loaded.cfg.layers[-1].kernel == 3


def test_config1_init_matches_reference_fpvw(golden):
    """PvsNet(config1, PCG64(0)) Kaiming-uniform weights == tests/golden/config1.fpvw
    (written by the reference's save from the same draws, make_golden.py)."""
    from paper_2509_24677_b200.neural import ModelConfig, PvsNet, read_fpvw
    net = PvsNet(ModelConfig.config1(), np.random.Generator(np.random.PCG64(0)))
    _, _, arrays = read_fpvw(os.path.join(GOLDEN, "config1.fpvw"))
    for L, (w, b) in zip(net.layers, arrays):
        assert np.array_equal(L.w.cpu().numpy(), w) and np.array_equal(L.b.cpu().numpy(), b)


@pytest.mark.parametrize("tag", ["def", "k5"])
def test_pvsnet_dense_forward_cached_backward_sgd_match_reference(golden, tag):
    g = golden("api.npz")
    net = _net(g, tag)
    nl = len(SPECS[tag])
    x = g["x"]
    y = net.forward(x)
    assert isinstance(y, np.ndarray) and y.dtype == np.float64 and y.shape == x.shape
    _close(y, g[f"{tag}_y{nl - 1}"], 1e-5)
    pred, caches = net.forward_cached(x)
    _close(pred, g[f"{tag}_y{nl - 1}"], 1e-5)
    grads, dx = net.backward(g[f"{tag}_dy"], caches)
    for i, (dw, db) in enumerate(grads):
        assert dw.shape == g[f"{tag}_dw{i}"].shape
        _close(dw, g[f"{tag}_dw{i}"])
        _close(db, g[f"{tag}_db{i}"])
    _close(dx, g[f"{tag}_dx"])
    net.sgd_step(grads, 0.05)
    for i, L in enumerate(net.layers):
        _close(L.w.cpu().numpy(), g[f"{tag}_w{i}_sgd"], 1e-5)
        _close(L.b.cpu().numpy(), g[f"{tag}_b{i}_sgd"], 1e-5)


def test_conv3d_isolated_forward_backward_and_functions(golden):
    """A single Conv3d on a dense input (active = any nonzero channel):
    forward vs the reference layer, backward vs the oracle; conv3d_forward /
    conv3d_backward are the same calls; torch in -> torch out."""
    import torch
    from paper_2509_24677_b200.neural import Conv3d, ConvSpec, conv3d_backward, conv3d_forward
    g = golden("api.npz")
    x, mask = g["x"], g["mask"]
    layer = Conv3d(ConvSpec(3, 8, 8, "relu"))
    layer.set_weights(g["def_w0"], g["def_b0"])
    y, cache = layer.forward(x, keep_cache=True)
    _close(y, g["def_y0"], 1e-5)
    _close(conv3d_forward(x, layer), y, 1e-6)
    dy = np.random.default_rng(5).normal(size=y.shape) * mask[..., None]
    dx, dw, db = layer.backward(dy, cache)
    coords = np.argwhere(mask)
    dims = mask.shape[1:]
    rows = x[tuple(coords.T)]
    layers = [(3, g["def_w0"], g["def_b0"], "relu")]
    _, caches = osp.chain_forward_cached(rows, osp.kmap_subm(coords, dims), layers)
    [(gw, gb)], gx = osp.chain_backward(dy[tuple(coords.T)], layers, caches)
    _close(dw, gw)
    _close(db, gb)
    _close(dx[tuple(coords.T)], gx)
    assert np.all(dx[~mask] == 0)
    dx2, dw2, db2 = conv3d_backward(layer, dy, cache)
    assert np.array_equal(dx2, dx) and np.array_equal(dw2, dw)
    with pytest.raises(ValueError):
        layer.backward(dy, None)
    with pytest.raises(ValueError):
        layer.forward(x[..., :4])
    yt = layer.forward(torch.as_tensor(x, dtype=torch.float32).cuda())
    assert isinstance(yt, torch.Tensor) and yt.is_cuda
    _close(yt.cpu().numpy(), y, 1e-6)


def test_predict_pvs_with_3cube_head_checkpoint(golden):
    """predict_pvs(grid, path) with the reference default checkpoint: bit-exact
    outside the 1e-3 band around tau."""
    from paper_2509_24677_b200.neural import predict_pvs
    g = golden("api.npz")
    grid = FroxelGrid((16, 16, 16), bits=g["grid_bits"][0])
    pred = predict_pvs(grid, os.path.join(GOLDEN, "default_d2.fpvw"), 0.5)
    assert pred.role == "predicted_pvs" and pred.dims == (16, 16, 16)
    want = FroxelGrid((16, 16, 16), bits=g["def_pred_bits"]).to_dense()
    prob = osp.deinterleave(g["def_pred_prob"], 2)
    bad = (pred.to_dense() != want) & (np.abs(prob - 0.5) >= 1e-3)
    assert not bad.any()
    for precision in ("bf16",):
        from paper_2509_24677_b200.neural import PvsNet
        net = PvsNet.load(os.path.join(GOLDEN, "default_d2.fpvw"), precision=precision)
        p16 = predict_pvs(grid, net, 0.5)
        assert (p16.to_dense() != want).mean() < 0.02


def test_evaluate_pairs_reference_signature(golden):
    """evaluate_pairs(net, x, y, tau) over stacked interleaved tensors (neural.py:429-439)."""
    from paper_2509_24677_b200.neural import _epoch_rates, evaluate_pairs
    g = golden("api.npz")
    net = _net(g, "def")
    x = g["x"]
    y = (np.random.default_rng(9).random(x.shape) < 0.3) * g["mask"][..., None]
    prob = g["def_y2"]
    for tau in (0.3, 0.5, 0.0):
        pred, gt = prob >= tau, y > 0.5
        want = _epoch_rates(int((pred & gt).sum()), int((pred & ~gt).sum()), int((~pred & gt).sum()), int(gt.sum()))
        got = evaluate_pairs(net, x, y, tau)
        assert got == pytest.approx(want, abs=1e-12), tau
    assert _epoch_rates(0, 5, 0, 0) == (0.0, 0.0)


def _write_dataset(root, n):
    """FPVS pairs + manifest in the layout load_pairs reads (scenegen.py:433-446)."""
    lines = ["# frame viewcell geometry gt"]
    for i in range(n):
        occ = synth.box_grid((32, 32, 16), 30, 1, 4, 40 + i)
        lab = synth.first_hit_labels(occ)
        FroxelGrid.from_dense(occ, role="geometry").save(root / f"g{i}.fpvs")
        FroxelGrid.from_dense(lab, role="gt_pvs").save(root / f"t{i}.fpvs")
        lines.append(f"{i} 0 g{i}.fpvs t{i}.fpvs")
    (root / "manifest.txt").write_text("\n".join(lines) + "\n")
    return root / "manifest.txt"


def test_reference_cli_train_and_infer_call_pattern(tmp_path):
    """cmd_train / cmd_infer (cli.py:255-282) with the imports swapped: the
    default 3^3-head estimator trains through train() (two epochs, SGD) to the
    same weights as the float64 oracle restatement of neural.py:442-510, writes
    the checkpoint and the epoch log, and predict_pvs reads the checkpoint."""
    from paper_2509_24677_b200.neural import (ModelConfig, PvsNet, TrainConfig, load_pairs, predict_pvs,
                                              train)
    manifest = _write_dataset(tmp_path, 4)
    out = str(tmp_path / "net.fpvw")
    # ---- cmd_train's body
    pairs = load_pairs(manifest)
    holdout = 1
    eval_pairs = pairs[len(pairs) - holdout:]
    train_pairs = pairs[:len(pairs) - holdout]
    tcfg = TrainConfig(lr=2e-2, epochs=2, batch_size=2, seed=6)
    net, history = train(train_pairs, ModelConfig.default(2), tcfg, eval_pairs=eval_pairs, checkpoint_path=out,
                         log_path=out + ".epochs.csv", verbose=True)
    assert len(history) == 2 and "val_fnr" in history[-1]
    assert (tmp_path / "net.fpvw.epochs.csv").read_text().startswith("epoch,loss,fnr,fpr,val_fnr,val_fpr")
    # ---- cmd_infer's body
    grid = FroxelGrid.load(tmp_path / "g0.fpvs")
    pred = predict_pvs(grid, out, 0.5)
    pred.save(tmp_path / "pred.fpvs")
    assert FroxelGrid.load(tmp_path / "pred.fpvs").dims == grid.dims
    # ---- the same training restated in float64 (oracle)
    from tests.test_gpu_train import oracle_step
    rng = np.random.Generator(np.random.PCG64(tcfg.seed))
    ref = PvsNet(ModelConfig.default(2), rng)
    layers = [(L.spec.kernel, L.w.double().cpu().numpy(), L.b.double().cpu().numpy(), L.spec.activation)
              for L in ref.layers]
    occs = [p[0].to_dense() for p in train_pairs]
    labs = [p[1].to_dense() for p in train_pairs]
    step, n = 0, len(train_pairs)
    losses = []
    for _ in range(tcfg.epochs):
        order = rng.permutation(n)
        tot = 0.0
        for s in range(0, n, tcfg.batch_size):
            b = order[s:s + tcfg.batch_size]
            loss, grads, _, _ = oracle_step([occs[i] for i in b], [labs[i] for i in b], 2, layers)
            lr = tcfg.lr * (1.0 - tcfg.decay) ** step
            layers = [(k, w - lr * gw, bb - lr * gb, a) for (k, w, bb, a), (gw, gb) in zip(layers, grads)]
            step += 1
            tot += loss * len(b)
        losses.append(tot / n)
    for h, want in zip(history, losses):
        assert abs(h["loss"] - want) <= 1e-5 * max(1.0, abs(want))
    for L, (_, w, b, _) in zip(net.layers, layers):
        _close(L.w.double().cpu().numpy(), w, 1e-5)
        _close(L.b.double().cpu().numpy(), b, 1e-5)
    loaded = PvsNet.load(out)
    for a, L in zip(loaded.layers, net.layers):
        assert bool((a.w == L.w).all())
