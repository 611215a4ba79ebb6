"""(2) kernel-map builder vs the oracle's canonical maps (bit-exact, integer)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import sparse as osp
from paper_2509_24677_b200 import synth
from paper_2509_24677_b200.froxel import FroxelGrid

pytestmark = pytest.mark.gpu


def _bits(occs):
    import torch
    return torch.from_numpy(np.concatenate([FroxelGrid.from_dense(o).bits for o in occs])).cuda()


def _oracle_level0(occs, d):
    cells = np.stack([osp.interleave(o.astype(np.float32), d) for o in occs])
    return osp.active_coords(cells), cells.shape[1:4]


@pytest.mark.parametrize("case", ["cfg1", "batch", "empty", "full", "edges"])
def test_subm_map_bit_exact(case):
    from paper_2509_24677_b200 import sparse as sp
    rng = np.random.default_rng(0)
    if case == "cfg1":
        occs, d = [synth.config1_grid(0)], 2
    elif case == "batch":
        occs, d = [synth.box_grid((32, 16, 16), 30, 1, 4, s) for s in range(5)], 2
    elif case == "empty":
        occs, d = [np.zeros((16, 16, 16), bool)], 2
    elif case == "full":
        occs, d = [np.ones((16, 8, 8), bool)], 4
    else:  # single froxels on the grid faces and corners
        o = np.zeros((16, 16, 16), bool)
        for p in [(0, 0, 0), (15, 15, 15), (0, 15, 7), (8, 0, 15), (15, 0, 0)]:
            o[p] = True
        occs, d = [o], 2
    dims = occs[0].shape
    lv = sp.level_from_bits(_bits(occs), len(occs), dims, d)
    coords, cdims = _oracle_level0(occs, d)
    n = lv.count()
    assert n == len(coords)
    assert np.array_equal(lv.coords[:n].cpu().numpy(), coords)
    ref = osp.kmap_subm(coords, cdims)
    assert np.array_equal(lv.nbr[:n].cpu().numpy(), ref)
    vol = lv.index_vol.cpu().numpy().reshape((len(occs),) + cdims)
    want = np.full(vol.shape, -1)
    if n:
        want[tuple(coords.T)] = np.arange(n)
    assert np.array_equal(vol, want)
    if n:
        nbr_h = sp.build_subm_hash(lv)
        assert np.array_equal(nbr_h[:n].cpu().numpy(), ref)
    del rng


def test_down_up_maps_bit_exact():
    from paper_2509_24677_b200 import sparse as sp
    occs = [synth.box_grid((64, 64, 64), 80, 1, 10, s) for s in (1, 2)]
    d = 4
    L0 = sp.level_from_bits(_bits(occs), 2, (64, 64, 64), d)
    L1, down, up = sp.coarsen(L0)
    L2, down2, up2 = sp.coarsen(L1)
    c0, dims0 = _oracle_level0(occs, d)
    c1 = osp.coarsen(c0)
    c2 = osp.coarsen(c1)
    dims1 = tuple(v // 2 for v in dims0)
    dims2 = tuple(v // 2 for v in dims1)
    for lv, c, dm in ((L1, c1, dims1), (L2, c2, dims2)):
        n = lv.count()
        assert n == len(c)
        assert np.array_equal(lv.coords[:n].cpu().numpy(), c)
        assert np.array_equal(lv.nbr[:n].cpu().numpy(), osp.kmap_subm(c, dm))
    assert np.array_equal(down[:len(c1)].cpu().numpy(), osp.kmap_down(c0, dims0, c1))
    assert np.array_equal(down2[:len(c2)].cpu().numpy(), osp.kmap_down(c1, dims1, c2))
    par, parity = osp.kmap_up(c0, c1, dims1)
    want = np.full((len(c0), 8), -1)
    want[np.arange(len(c0)), parity] = par
    assert np.array_equal(up[:len(c0)].cpu().numpy(), want)


def test_config2_level0_map_full_size():
    """cfg2 (256^3, d=4): A and P match the oracle; symmetric-map property on the device."""
    import torch
    from paper_2509_24677_b200 import sparse as sp
    occ = synth.config2_grid(1)
    lv = sp.level_from_bits(_bits([occ]), 1, occ.shape, 4)
    coords, cdims = _oracle_level0([occ], 4)
    n = lv.count()
    assert n == len(coords)
    ref = osp.kmap_subm(coords, cdims)
    got = lv.nbr[:n]
    assert np.array_equal(got.cpu().numpy(), ref)
    # property: nbr[nbr[i][j]][26-j] == i for every present pair
    i, j = torch.nonzero(got >= 0, as_tuple=True)
    assert torch.equal(got[got[i, j].long(), 26 - j], i.int())


def _granular(bits, B, dims, d, nlev):
    from paper_2509_24677_b200 import sparse as sp
    levels = [sp.level_from_bits(bits, B, dims, d)]
    downs, ups = [], []
    for _ in range(nlev - 1):
        c, dn, up = sp.coarsen(levels[-1])
        levels.append(c)
        downs.append(dn)
        ups.append(up)
    return levels, downs, ups


FUSED_CASES = {
    "cfg2": (lambda: [synth.config2_grid(1)], 4, 3),
    "batch64": (lambda: [synth.box_grid((64, 64, 64), 80, 1, 10, s) for s in (1, 2)], 4, 3),
    "cfg1": (lambda: [synth.config1_grid(0)], 2, 2),
    "smallz": (lambda: [synth.box_grid((32, 16, 16), 30, 1, 4, s) for s in range(5)], 2, 1),
    "d8": (lambda: [synth.box_grid((64, 64, 128), 60, 1, 12, 3)], 8, 2),
    "d1": (lambda: [synth.box_grid((16, 16, 32), 10, 1, 3, 4)], 1, 3),
    "empty": (lambda: [np.zeros((32, 32, 32), bool)], 4, 2),
}


@pytest.mark.parametrize("case", list(FUSED_CASES))
def test_fused_levels_match_granular(case):
    """fpvs_levels_from_bits == the granular kmap sequence, bit for bit (and
    re-arms its workspace: a second frame on the same plan is exact too)."""
    import torch
    from paper_2509_24677_b200 import sparse as sp
    make, d, nlev = FUSED_CASES[case]
    occs = make()
    B, dims = len(occs), occs[0].shape
    X, Y, Z = (v // d for v in dims)
    lv0 = sp.new_level(B, (X, Y, Z))
    levels, downs, ups = [lv0], [], []
    for _ in range(nlev - 1):
        c, dn, up = sp.new_coarse(levels[-1])
        levels.append(c)
        downs.append(dn)
        ups.append(up)
    maps = sp.LevelMaps(levels, downs, ups, dims, d)
    feat = torch.full((lv0.cap, d ** 3 + 8), 7.0, dtype=torch.bfloat16, device="cuda")
    frames = [occs, [o[::-1].copy() for o in occs]]
    for fr in frames:
        bits = _bits(fr)
        clear = torch.full((bits.numel(),), 255, dtype=torch.uint8, device="cuda")
        maps.run(bits, feat=feat, clear=clear)
        ref, rdowns, rups = _granular(bits, B, dims, d, nlev)
        for lv, rl in zip(levels, ref):
            n = rl.count()
            assert lv.count() == n
            assert torch.equal(lv.coords[:n], rl.coords[:n])
            assert torch.equal(lv.index_vol, rl.index_vol)
            assert torch.equal(lv.nbr[:n], rl.nbr[:n])
            t = (n + 127) // 128
            assert torch.equal(lv.nbr_masks[:t], rl.nbr_masks[:t])
        for i in range(nlev - 1):
            c, f, rc = levels[i + 1], levels[i], ref[i + 1]
            nc, nf = c.count(), f.count()
            assert torch.equal(downs[i][:nc], rdowns[i][:nc])
            assert torch.equal(ups[i][:nf], rups[i][:nf])
            assert torch.equal(c.extra["down_masks"][:(nc + 127) // 128], rc.extra["down_masks"][:(nc + 127) // 128])
            assert torch.equal(c.extra["up_masks"][:(nf + 127) // 128], rc.extra["up_masks"][:(nf + 127) // 128])
        n0 = ref[0].count()
        want = sp.gather_features(bits, ref[0], dims, d, torch.bfloat16)
        assert torch.equal(feat[:n0, :d ** 3], want[:n0])
        assert bool((feat[:n0, d ** 3:] == 7).all())  # columns past d^3 untouched
        assert int(clear.sum()) == 0


@pytest.mark.parametrize("dims,density", [((20, 18, 16), 0.3), ((64, 64, 32), 0.06), ((3, 4, 5), 0.9)])
def test_pair_lists_match_oracle(dims, density):
    """fpvs_kmap_pairs: per-offset (in, out) lists sorted by out and their offsets (row KM) == oracle."""
    import torch
    from oracle import sparse as osp
    from paper_2509_24677_b200 import sparse as sp
    rng = np.random.default_rng(int(density * 1000))
    mask = rng.random((1,) + dims) < density
    lv = sp.new_level(1, dims)
    lv.active.copy_(torch.from_numpy(mask.reshape(-1).astype(np.uint8)).cuda())
    sp.compact(lv)
    sp.build_subm(lv)
    n = lv.count()
    pin, pout, off = sp.pair_lists(lv.nbr, 27, lv.n, lv.cap)
    ins, outs, ref_off = osp.pair_lists(lv.nbr[:n].cpu().numpy())
    assert np.array_equal(off.cpu().numpy(), ref_off)
    assert np.array_equal(pin.cpu().numpy(), ins) and np.array_equal(pout.cpu().numpy(), outs)
