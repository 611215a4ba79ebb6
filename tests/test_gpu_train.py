"""(4) training path: fused loss, dgrad/wgrad, optimizer steps, hard counts and
the drop-in ``train`` against the float64 oracle (oracle/sparse.py restates
neural.py:221-249 and 353-399 on the active set).

Tolerances: fp32 gradients within 1e-4 of the largest oracle magnitude per
tensor (f32 accumulation vs f64); the loss within 1e-6 relative; bf16 training
gradients (bf16 activations/weights, f32 backward) within 5e-2 of the norm.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import sparse as osp
from paper_2509_24677_b200 import synth
from paper_2509_24677_b200.froxel import FroxelGrid

pytestmark = pytest.mark.gpu

DIMS = (32, 32, 16)


def _batch(seeds):
    occs = [synth.box_grid(DIMS, 30, 1, 4, s) for s in seeds]
    labs = [synth.first_hit_labels(o) for o in occs]
    return occs, labs


def _bits(grids):
    import torch
    return torch.from_numpy(np.concatenate([FroxelGrid.from_dense(g).bits for g in grids])).cuda()


def _layers(net):
    return [(L.spec.kernel, L.w.detach().double().cpu().numpy().reshape(L.w.shape[0], -1),
             L.b.detach().double().cpu().numpy(), L.spec.activation) for L in net.layers]


def oracle_step(occs, labs, d, layers, alpha=0.1, lam=0.99):
    cells = np.stack([osp.interleave(o.astype(np.float64), d) for o in occs])
    gts = np.stack([osp.interleave(g.astype(np.float64), d) for g in labs])
    coords = osp.active_coords(cells)
    dims = cells.shape[1:4]
    x0 = cells[tuple(coords.T)]
    nbr = osp.kmap_subm(coords, dims)
    probs, caches = osp.chain_forward_cached(x0, nbr, layers)
    B = len(occs)
    loss, dp = 0.0, np.zeros_like(probs)
    for b in range(B):
        rows = coords[:, 0] == b
        pd = np.zeros(dims + (probs.shape[1],))
        pd[tuple(coords[rows, 1:].T)] = probs[rows]
        lv, lg = osp.combined_loss(pd, gts[b], alpha, lam)
        loss += lv
        dp[rows] = lg[tuple(coords[rows, 1:].T)] / B
    grads, _ = osp.chain_backward(dp, layers, caches)
    return loss / B, grads, probs, coords


def _net(precision="fp32", seed=0):
    from paper_2509_24677_b200.neural import ModelConfig, PvsNet
    return PvsNet(ModelConfig.config1(), np.random.Generator(np.random.PCG64(seed)), precision=precision)


def test_loss_and_gradients_fp32_vs_oracle():
    from paper_2509_24677_b200.neural import TrainConfig
    from paper_2509_24677_b200.train import TrainStep
    occs, labs = _batch([3, 4])
    net = _net()
    layers = _layers(net)
    plan = TrainStep(net, 2, DIMS, TrainConfig())
    plan.forward_backward(_bits(occs), _bits(labs))
    loss, grads, probs, coords = oracle_step(occs, labs, 2, layers)
    n = len(coords)
    assert plan.lv.count() == n
    assert np.abs(plan.probs[:n].cpu().numpy() - probs).max() < 1e-5
    assert abs(float(plan.loss[0]) - loss) <= 1e-6 * max(1.0, abs(loss))
    for li, ((dw, db), (rw, rb)) in enumerate(zip(plan.views, grads)):
        gw = dw.double().cpu().numpy().reshape(rw.shape)
        assert np.abs(gw - rw).max() <= 1e-4 * np.abs(rw).max() + 1e-9, li
        assert np.abs(db.double().cpu().numpy() - rb).max() <= 1e-4 * np.abs(rb).max() + 1e-9, li
    # hard counts at tau = 0.5 from the packed prediction (exempting the +-1e-3 band)
    cnt = plan.counts.view(-1, 4).cpu().numpy()
    for b in range(2):
        gt = labs[b]
        assert cnt[b, 3] == int(gt.sum())
        assert cnt[b, 0] + cnt[b, 2] == int(gt.sum())


def test_bf16_training_gradients_close_to_fp32():
    from paper_2509_24677_b200.neural import TrainConfig
    from paper_2509_24677_b200.train import TrainStep
    occs, labs = _batch([5, 6, 7])
    net = _net("bf16", seed=1)
    layers = _layers(net)
    plan = TrainStep(net, 3, DIMS, TrainConfig())
    plan.forward_backward(_bits(occs), _bits(labs))
    loss, grads, _, _ = oracle_step(occs, labs, 2, layers)
    assert abs(float(plan.loss[0]) - loss) < 2e-2
    for (dw, db), (rw, rb) in zip(plan.views, grads):
        gw = dw.double().cpu().numpy().reshape(rw.shape)
        assert np.linalg.norm(gw - rw) <= 5e-2 * np.linalg.norm(rw) + 1e-9


def test_sgd_and_adamw_steps():
    import torch
    from paper_2509_24677_b200.neural import TrainConfig
    from paper_2509_24677_b200.train import TrainStep
    occs, labs = _batch([8])
    for opt in ("sgd", "adamw"):
        net = _net()
        tc = TrainConfig(optimizer=opt, weight_decay=0.01)
        plan = TrainStep(net, 1, DIMS, tc)
        p0 = plan.params.double().cpu().numpy().copy()
        m = np.zeros_like(p0)
        v = np.zeros_like(p0)
        p = p0.copy()
        for step in (1, 2):
            plan.forward_backward(_bits(occs), _bits(labs))
            g = plan.grads[:plan.nparams].double().cpu().numpy()
            plan.update(1e-3, step)
            if opt == "sgd":
                p = p - 1e-3 * g
            else:
                m = 0.9 * m + 0.1 * g
                v = 0.999 * v + 0.001 * g * g
                mh, vh = m / (1 - 0.9 ** step), v / (1 - 0.999 ** step)
                p = p - 1e-3 * (mh / (np.sqrt(vh) + 1e-8) + 0.01 * p)
            got = plan.params.double().cpu().numpy()
            assert np.abs(got - p).max() <= 1e-6 + 1e-5 * np.abs(p).max(), (opt, step)
        # the layers read the updated master weights
        assert torch.equal(net.layers[0].w.reshape(-1), plan.params[:net.layers[0].w.numel()])


def test_bits_confusion_counts():
    import torch
    from paper_2509_24677_b200 import _lib
    rng = np.random.default_rng(0)
    for B, nbytes in ((1, 4096), (3, 1000), (2, 16 * 1024 + 5)):
        a = rng.integers(0, 256, B * nbytes, dtype=np.uint8)
        c = rng.integers(0, 256, B * nbytes, dtype=np.uint8)
        ws = torch.empty(_lib.size("fpvs_bits_confusion_workspace_size", B), dtype=torch.uint8, device="cuda")
        out = torch.zeros(4 * B, dtype=torch.int64, device="cuda")
        ta, tc = torch.from_numpy(a).cuda(), torch.from_numpy(c).cuda()  # keep both alive across the call
        _lib.call("fpvs_bits_confusion", _lib.ptr(ta), _lib.ptr(tc), B, nbytes, _lib.ptr(out), _lib.ptr(ws),
                  ws.numel(), _lib.stream_ptr())
        got = out.view(B, 4).cpu().numpy()
        pa = np.unpackbits(a.reshape(B, nbytes), axis=1).astype(bool)
        pc = np.unpackbits(c.reshape(B, nbytes), axis=1).astype(bool)
        want = np.stack([(pa & pc).sum(1), (pa & ~pc).sum(1), (~pa & pc).sum(1), pc.sum(1)], 1)
        assert np.array_equal(got, want), (B, nbytes)


def test_train_api_one_step_matches_oracle(tmp_path):
    """train(): PCG64 init + permutation + one SGD step over the whole set == oracle."""
    from paper_2509_24677_b200.neural import ModelConfig, PvsNet, TrainConfig
    from paper_2509_24677_b200.train import train
    occs, labs = _batch([11, 12, 13])
    pairs = [(FroxelGrid.from_dense(o), FroxelGrid.from_dense(g, role="gt_pvs")) for o, g in zip(occs, labs)]
    tc = TrainConfig(lr=1e-2, epochs=1, batch_size=3, seed=4)
    net, hist = train(pairs, ModelConfig.config1(), tc, checkpoint_path=tmp_path / "w.fpvw",
                      log_path=tmp_path / "log.csv")
    rng = np.random.Generator(np.random.PCG64(4))
    ref = PvsNet(ModelConfig.config1(), rng)
    order = rng.permutation(3)
    layers = _layers(ref)
    loss, grads, _, _ = oracle_step([occs[i] for i in order], [labs[i] for i in order], 2, layers)
    assert len(hist) == 1 and abs(hist[0]["loss"] - loss) <= 1e-6
    for L, (k, w, b, _), (gw, gb) in zip(net.layers, layers, grads):
        assert np.abs(L.w.double().cpu().numpy() - (w - 1e-2 * gw)).max() < 1e-6
        assert np.abs(L.b.double().cpu().numpy() - (b - 1e-2 * gb)).max() < 1e-6
    assert (tmp_path / "w.fpvw").exists()
    assert (tmp_path / "log.csv").read_text().startswith("epoch,loss,fnr,fpr")
    # deterministic: the same call gives the same weights
    net2, hist2 = train(pairs, ModelConfig.config1(), tc)
    assert hist2[0]["loss"] == hist[0]["loss"]
    for a, b in zip(net.layers, net2.layers):
        assert bool((a.w == b.w).all())


def test_train_adamw_bf16_runs_and_learns():
    from paper_2509_24677_b200.neural import ModelConfig, TrainConfig
    from paper_2509_24677_b200.train import train
    occs, labs = _batch(range(20, 26))
    pairs = [(FroxelGrid.from_dense(o), FroxelGrid.from_dense(g)) for o, g in zip(occs, labs)]
    tc = TrainConfig(lr=1e-2, epochs=6, batch_size=4, optimizer="adamw", seed=0)
    _, hist = train(pairs, ModelConfig.config1(), tc, eval_pairs=pairs[:2], precision="bf16")
    losses = [h["loss"] for h in hist]
    assert all(np.isfinite(losses)) and losses[-1] < losses[0]
    assert "val_fnr" in hist[-1]


@pytest.mark.slow
def test_config5_full_size_bf16_step_vs_bf16_oracle():
    """BASELINE config 5 at its stated size: 8 x 128^3 grids (~4 % density), the
    config-1 net in bf16, one forward + fused loss + tcgen05 backward, against
    the oracle's bf16 emulation of the same rounding points
    (osp.chain_train_step_bf16).  Tolerance: loss within 1e-4 relative;
    each gradient tensor within 1e-2 relative (Frobenius) — the device sums in
    fp32 in a different order, which flips occasional bf16 roundings of dz."""
    import torch
    from paper_2509_24677_b200.neural import ModelConfig, PvsNet, TrainConfig
    from paper_2509_24677_b200.train import TrainStep
    pairs = [synth.config5_pair(0, i) for i in range(8)]
    occs, labs = [g for g, _ in pairs], [lb for _, lb in pairs]
    net = PvsNet(ModelConfig.config1(), np.random.Generator(np.random.PCG64(0)), precision="bf16")
    layers = _layers(net)
    step = TrainStep(net, 8, (128, 128, 128), TrainConfig(optimizer="adamw"))
    assert step.tc_backward
    step.forward_backward(_bits(occs), _bits(labs))
    torch.cuda.synchronize()
    cells = np.stack([osp.interleave(o.astype(np.float64), 2) for o in occs])
    gts = np.stack([osp.interleave(g.astype(np.float64), 2) for g in labs])
    loss, grads, coords, _ = osp.chain_train_step_bf16(cells, gts, layers)
    assert step.lv.count() == len(coords)
    got_loss = float(step.loss[0])
    assert abs(got_loss - loss) <= 1e-4 * abs(loss), (got_loss, loss)
    for li, (L, (gw, gb)) in enumerate(zip(net.layers, grads)):
        dw, db = (t.double().cpu().numpy() for t in step.views[li])
        for name, a, b in (("dw", dw.reshape(gw.shape), gw), ("db", db, gb)):
            rel = float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))
            assert rel <= 1e-2, (li, name, rel)


@pytest.mark.parametrize("radius", [0, 1, 2, 3])
def test_first_hit_labels_kernel_matches_host_rule(radius):
    """Row LBL on the device (fpvs_first_hit_labels) == synth.first_hit_labels:
    config-5 grids, a grid with occupancy against every border, an empty grid."""
    from paper_2509_24677_b200.synth import first_hit_labels_bits
    dims = (128, 128, 128)
    grids = [synth.config5_pair(0, i)[0] for i in range(2)]
    edge = np.zeros(dims, bool)
    edge[0, :, 5] = edge[-1, :, 7] = edge[:, 0, 0] = edge[:, -1, -1] = True
    edge[60:70, 60:70, 30:40] = True
    grids += [edge, np.zeros(dims, bool)]
    got = first_hit_labels_bits(_bits(grids), len(grids), dims, radius).cpu().numpy()
    per = dims[0] * dims[1] * dims[2] // 8
    for b, g in enumerate(grids):
        want = FroxelGrid.from_dense(synth.first_hit_labels(g, radius)).bits
        assert np.array_equal(got[b * per:(b + 1) * per], want), b


def test_dropin_losses_match_reference_golden(golden):
    """dice_loss / rvl_loss / combined_loss (neural.py:353-399) on the device vs
    the reference's own values and gradients (tests/golden/loss.npz), numpy in
    -> numpy out and CUDA tensors in -> tensors out; shape mismatch -> ValueError."""
    import torch
    from paper_2509_24677_b200.neural import TrainConfig, combined_loss, dice_loss, rvl_loss
    g = golden("loss.npz")
    cfg = TrainConfig()
    for i in range(int(g["n"])):
        pred, gt = g[f"l{i}_pred"], g[f"l{i}_gt"]
        for fn, key, args in ((dice_loss, "dice", (cfg.alpha,)), (rvl_loss, "rvl", ()), (combined_loss, "comb", (cfg,))):
            v, gr = fn(pred, gt, *args)
            assert abs(float(v) - float(g[f"l{i}_{key}"])) <= 1e-12, (i, key)
            assert isinstance(gr, np.ndarray) and np.abs(gr - g[f"l{i}_{key}_g"]).max() <= 1e-12, (i, key)
            vt, gt_ = fn(torch.as_tensor(pred).cuda(), torch.as_tensor(gt).cuda(), *args)
            assert abs(float(vt) - float(g[f"l{i}_{key}"])) <= 1e-12
            assert isinstance(gt_, torch.Tensor) and float((gt_.cpu() - torch.as_tensor(g[f"l{i}_{key}_g"])).abs().max()) <= 1e-12
    with pytest.raises(ValueError):
        dice_loss(np.zeros(3), np.zeros(4), 0.1)


def test_pack_weights_multi_equals_single_packs():
    """fpvs_pack_weights_tc_multi (the training step's one-launch re-pack) writes
    exactly the bytes of the single fpvs_pack_weights_tc / _dgrad calls."""
    import ctypes as C
    import torch
    from paper_2509_24677_b200 import _lib
    rng = np.random.default_rng(7)
    specs = [(27, 8, 32, 0, 0), (27, 32, 32, 0, 1), (27, 32, 32, 32, 0), (1, 32, 8, 0, 0), (8, 64, 128, 0, 1),
             (27, 64, 64, 64, 1)]
    jobs, refs = [], []
    for K, cin, cout, bn, dg in specs:
        w = torch.from_numpy(rng.standard_normal((K * cin, cout)).astype(np.float32)).cuda()
        fn = "fpvs_pack_weights_tc_dgrad" if dg else "fpvs_pack_weights_tc"
        n = _lib.size("fpvs_pack_weights_tc_size", K, cout, cin, bn) if dg else \
            _lib.size("fpvs_pack_weights_tc_size", K, cin, cout, bn)
        ref = torch.zeros(n, dtype=torch.uint8, device="cuda")
        _lib.call(fn, _lib.ptr(w), K, cin, cout, bn, _lib.ptr(ref), _lib.stream_ptr())
        out = torch.full((n,), 0x7F, dtype=torch.uint8, device="cuda")
        jobs.append((w, K, cin, cout, bn, dg, out))
        refs.append(ref)
    arr = (_lib.PackJob * len(jobs))()
    for e, (w, K, cin, cout, bn, dg, out) in zip(arr, jobs):
        e.w, e.K, e.cin, e.cout, e.bn, e.dgrad, e.packed = _lib.ptr(w), K, cin, cout, bn, dg, _lib.ptr(out)
    _lib.call("fpvs_pack_weights_tc_multi", C.addressof(arr), len(jobs), _lib.stream_ptr())
    torch.cuda.synchronize()
    for (w, K, cin, cout, bn, dg, out), ref in zip(jobs, refs):
        assert torch.equal(out, ref), (K, cin, cout, bn, dg)
