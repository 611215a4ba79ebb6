"""BASELINE configs 3 and 4 through the drop-in chain path vs the oracle.

Config 3: 64 independent 64x64x32 grids in ONE batched frame (the batch index
is the outermost coordinate of the active cells and kernel maps), densities
U(1%, 6%), the config-1 network.  Config 4: 256^3 grids at swept occupancy
with the config-1 network (d = 2 -> 128^3 cells).

Masks are bit-exact against the oracle outside the +-1e-3 band around tau;
logits within 2e-2 (bf16, vs the oracle's bf16 emulation) or 1e-4 (fp32, vs
float64), as north_star states.
"""

from __future__ import annotations

import numpy as np
import pytest

from oracle import sparse as osp
from paper_2509_24677_b200 import synth
from paper_2509_24677_b200.froxel import FroxelGrid

pytestmark = pytest.mark.gpu

BAND = 1e-3


def _net(precision):
    from paper_2509_24677_b200.neural import ModelConfig, PvsNet
    return PvsNet(ModelConfig.config1(), np.random.Generator(np.random.PCG64(0)), precision=precision)


def _layers(net):
    return [(layer.spec.kernel, layer.w.cpu().numpy().astype(np.float64), layer.b.cpu().numpy().astype(np.float64),
             layer.spec.activation) for layer in net.layers]


def _run_batch(net, grids):
    import torch
    from paper_2509_24677_b200.pipeline import ChainPlan
    dims = grids[0].shape
    B = len(grids)
    bits = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(g).bits for g in grids])).cuda()
    plan = ChainPlan(net, B, dims)
    out = torch.empty(B * int(np.prod(dims)) // 8, dtype=torch.uint8, device="cuda")
    logits = torch.zeros((plan.L0.cap, net.cfg.d ** 3), device="cuda")
    plan.run(bits, out, 0.5, logits=logits)
    torch.cuda.synchronize()
    n = plan.L0.count()
    return plan, out.cpu().numpy(), logits[:n].cpu().numpy(), plan.L0.coords[:n].cpu().numpy()


def _check(grids, net, out_bits, logits, coords, bf16, logit_tol):
    d = net.cfg.d
    cells = np.stack([osp.interleave(g.astype(np.float64), d) for g in grids])
    ref_coords, z = osp.chain_forward(cells, _layers(net), bf16=bf16, return_logits=True)
    assert np.array_equal(coords, ref_coords)
    err = float(np.abs(logits - z).max())
    assert err <= logit_tol, err
    prob = osp.scatter_cells(ref_coords, osp.sigmoid(z), cells.shape[:4])
    per = len(out_bits) // len(grids)
    for b, g in enumerate(grids):
        ref = osp.deinterleave(prob[b], d)
        got = FroxelGrid(g.shape, bits=out_bits[b * per:(b + 1) * per]).to_dense()
        diff = got != (ref >= 0.5)
        assert not (diff & (np.abs(ref - 0.5) >= BAND)).any(), (b, int(diff.sum()))
    return err


@pytest.mark.parametrize("precision,tol", [("bf16", 2e-2), ("fp32", 1e-4)])
def test_config3_batch_of_64(precision, tol):
    grids = [synth.config3_grid(i) for i in range(64)]
    dens = [float(g.mean()) for g in grids]
    assert 0.005 < min(dens) and max(dens) < 0.08
    net = _net(precision)
    plan, out, logits, coords = _run_batch(net, grids)
    assert set(np.unique(coords[:, 0])) == set(range(64))  # every grid contributes rows, batch-major order
    _check(grids, net, out, logits, coords, precision == "bf16", tol)


def test_config3_batch_equals_single_grids():
    """A grid's mask does not depend on the other grids of the batch."""
    grids = [synth.config3_grid(i) for i in range(8)]
    net = _net("bf16")
    _, out_b, _, _ = _run_batch(net, grids)
    per = len(out_b) // len(grids)
    for b, g in enumerate(grids):
        _, out_1, _, _ = _run_batch(net, [g])
        assert np.array_equal(out_b[b * per:(b + 1) * per], out_1), b


@pytest.mark.parametrize("density", [0.005, 0.02, 0.08, pytest.param(0.25, marks=pytest.mark.slow)])
def test_config4_density_sweep_full_size(density):
    occ = synth.config4_grid(density)
    assert abs(float(occ.mean()) - density) < 0.25 * density
    net = _net("bf16")
    _, out, logits, coords = _run_batch(net, [occ])
    _check([occ], net, out, logits, coords, True, 2e-2)
