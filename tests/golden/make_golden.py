"""Generate the golden fixtures in this directory by running the REAL reference.

Run in the build container (which has /root/reference):

    python tests/golden/make_golden.py

Every array written here is an output of ``froxelpvs`` itself
(pkg/src/froxelpvs/{froxel,interleave,neural}.py) on seeded inputs; the tests
check the oracle restatement and (on the GPU) the CUDA path against them, so
parity stays pinned on the GPU box where the reference does not exist.
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle import refbridge  # noqa: E402
from oracle import sparse as osp  # noqa: E402
from paper_2509_24677_b200 import synth  # noqa: E402


def _save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def interleave_cases(fp):
    """interleave / deinterleave outputs of the reference (interleave.py:54-85)."""
    il = fp.interleave
    FroxelGrid = fp.froxel.FroxelGrid
    rng = np.random.default_rng(7)
    out = {}
    cases = [((16, 8, 8), 2), ((16, 8, 8), 4), ((32, 16, 8), 2), ((16, 16, 16), 8), ((24, 12, 6), 3),
             ((8, 4, 2), 1)]
    for ci, (dims, d) in enumerate(cases):
        dense = rng.random(dims) < 0.3
        grid = FroxelGrid.from_dense(dense)
        t = il.interleave(grid, d)                        # FroxelGrid input -> float64
        fval = rng.random(dims).astype(np.float32)
        tf = il.interleave(fval, d)                        # ndarray input keeps dtype
        back = il.deinterleave(tf, d)
        thr = il.deinterleave(tf, d, threshold=0.5) if dims[0] % 8 == 0 else None
        out[f"c{ci}_dims"] = np.array(dims)
        out[f"c{ci}_d"] = np.array(d)
        out[f"c{ci}_bits"] = grid.bits
        out[f"c{ci}_il_bits"] = t.values
        out[f"c{ci}_f32"] = fval
        out[f"c{ci}_il_f32"] = tf.values
        out[f"c{ci}_deil_f32"] = back
        if thr is not None:
            out[f"c{ci}_thr_bits"] = thr.bits
    out["ncases"] = np.array(len(cases))
    return out


def conv_cases(fp):
    """Masked reference Conv3d forward/backward (neural.py:187-249) on sparse inputs."""
    nn = fp.neural
    rng = np.random.default_rng(11)
    out = {}
    shape = (2, 6, 5, 7)
    mask = rng.random(shape) < 0.35
    specs = [nn.ConvSpec(3, 8, 16, "relu"), nn.ConvSpec(3, 16, 16, "relu"), nn.ConvSpec(1, 16, 8, "sigmoid")]
    x = (rng.random(shape + (8,)) < 0.5) * mask[..., None]
    x = x.astype(np.float64)
    layers = []
    for i, s in enumerate(specs):
        layer = nn.Conv3d(s)
        layer.w = rng.uniform(-0.5, 0.5, size=layer.w.shape)
        layer.b = rng.uniform(-0.1, 0.1, size=layer.b.shape)
        layers.append(layer)
        out[f"w{i}"] = layer.w
        out[f"b{i}"] = layer.b
    m = mask[..., None].astype(np.float64)
    h = x
    caches = []
    for i, layer in enumerate(layers):
        y, cache = layer.forward(h, keep_cache=True)
        out[f"dense_y{i}"] = y                 # unmasked reference output of this layer
        y = y * m
        out[f"y{i}"] = y
        caches.append(cache)
        h = y
    # backward of the masked chain via the reference's own Conv3d.backward
    dy0 = np.random.default_rng(12).normal(size=h.shape) * m
    dy = dy0
    for i in reversed(range(len(layers))):
        dx, dw, db = layers[i].backward(dy * m, caches[i])
        out[f"dw{i}"] = dw
        out[f"db{i}"] = db
        dy = dx * m
    out["dx"] = dy
    out["dy"] = dy0
    out["x"] = x
    out["mask"] = mask
    return out


def loss_cases(fp):
    """dice / rvl / combined values and gradients (neural.py:353-399)."""
    nn = fp.neural
    rng = np.random.default_rng(13)
    out = {}
    cfg = nn.TrainConfig()
    for i, (n, pg) in enumerate([(1000, 0.1), (4096, 0.02), (64, 0.0), (512, 1.0)]):
        pred = rng.random(n)
        gt = (rng.random(n) < pg).astype(np.float64)
        dv, dg = nn.dice_loss(pred, gt, cfg.alpha)
        rv, rg = nn.rvl_loss(pred, gt)
        cv, cg = nn.combined_loss(pred, gt, cfg)
        out.update({f"l{i}_pred": pred, f"l{i}_gt": gt, f"l{i}_dice": dv, f"l{i}_dice_g": dg,
                    f"l{i}_rvl": rv, f"l{i}_rvl_g": rg, f"l{i}_comb": cv, f"l{i}_comb_g": cg})
    out["n"] = np.array(4)
    return out


def fpvw_case(fp):
    """Reference FPVW bytes for the config-1 net (neural.py:299-346)."""
    nn = fp.neural
    mcfg = nn.ModelConfig(2, [nn.ConvSpec(3, 8, 32, "relu"), nn.ConvSpec(3, 32, 32, "relu"),
                              nn.ConvSpec(3, 32, 32, "relu"), nn.ConvSpec(3, 32, 32, "relu"),
                              nn.ConvSpec(1, 32, 8, "sigmoid")])
    net = nn.PvsNet(mcfg)
    rng = np.random.Generator(np.random.PCG64(0))
    for layer in net.layers:
        s = layer.spec
        layer.w, layer.b = osp.kaiming_uniform(rng, s.kernel ** 3, s.in_channels, s.out_channels,
                                               s.activation)
    with tempfile.TemporaryDirectory() as tmp:
        p = os.path.join(tmp, "c1.fpvw")
        net.save(p)
        raw = open(p, "rb").read()
        net = nn.PvsNet.load(p)          # f32-quantised weights, as both sides read them
    return net, raw


def config1_case(fp, net):
    """Config 1 end to end through the reference arithmetic with the submanifold mask."""
    FroxelGrid = fp.froxel.FroxelGrid
    il = fp.interleave
    occ = synth.config1_grid(0)
    grid = FroxelGrid.from_dense(occ)
    x = il.interleave(grid, 2).values[None]
    mask = x.any(axis=-1)
    outs, _ = refbridge.masked_reference_forward(fp.neural, net, x, mask)
    prob = outs[-1][0]
    pred = il.deinterleave(il.ChannelTensor(prob, 2), 2, threshold=0.5)
    # logits on active cells, for the fp32 tolerance check
    h = outs[-2]
    z = h.reshape(-1, h.shape[-1]) @ net.layers[-1].w + net.layers[-1].b
    coords = np.argwhere(mask)
    logits = z.reshape(h.shape[:-1] + (8,))[tuple(coords.T)]
    return dict(bits=grid.bits, prob_active=prob[tuple(coords[:, 1:].T)], logits_active=logits,
                coords=coords, pred_bits=pred.bits, dims=np.array(occ.shape))


def main():
    fp = refbridge.load()
    if fp is None:
        raise SystemExit("reference not found at " + refbridge.REF_SRC)
    _save("interleave.npz", **interleave_cases(fp))
    _save("conv.npz", **conv_cases(fp))
    _save("loss.npz", **loss_cases(fp))
    net, raw = fpvw_case(fp)
    with open(os.path.join(HERE, "config1.fpvw"), "wb") as fh:
        fh.write(raw)
    print("wrote config1.fpvw", len(raw))
    _save("config1.npz", **config1_case(fp, net))


if __name__ == "__main__":
    main()
