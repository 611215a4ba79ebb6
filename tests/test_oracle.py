"""The oracle restatement pinned against the reference (CPU only).

(a) committed golden vectors written by tests/golden/make_golden.py from the
real reference; (b) the SPEC known-answer examples; (c) when /root/reference
is present (build container only), the reference itself.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import refbridge
from oracle import sparse as osp
from paper_2509_24677_b200 import synth
from paper_2509_24677_b200.froxel import FroxelGrid
from paper_2509_24677_b200.neural import read_fpvw

# ---------------------------------------------------------------- interleave


def test_interleave_matches_reference_golden(golden):
    g = golden("interleave.npz")
    for ci in range(int(g["ncases"])):
        dims, d = tuple(g[f"c{ci}_dims"]), int(g[f"c{ci}_d"])
        dense = FroxelGrid(dims, bits=g[f"c{ci}_bits"]).to_dense().astype(np.float64)
        assert np.array_equal(osp.interleave(dense, d), g[f"c{ci}_il_bits"])
        assert np.array_equal(osp.interleave(g[f"c{ci}_f32"], d), g[f"c{ci}_il_f32"])
        assert np.array_equal(osp.deinterleave(g[f"c{ci}_il_f32"], d), g[f"c{ci}_deil_f32"])
        if f"c{ci}_thr_bits" in g:
            thr = FroxelGrid.from_dense(osp.deinterleave(g[f"c{ci}_il_f32"], d) >= 0.5)
            assert np.array_equal(thr.bits, g[f"c{ci}_thr_bits"])


def test_spec_interleave_kats():
    # 4^3 grid, d=2, bit (3,3,3) -> cell (1,1,1) channel 7
    g = np.zeros((4, 4, 4))
    g[3, 3, 3] = 1
    t = osp.interleave(g, 2)
    assert t.shape == (2, 2, 2, 8) and t[1, 1, 1, 7] == 1 and t.sum() == 1
    assert osp.interleave(np.zeros((32, 32, 32)), 8).shape == (4, 4, 4, 512)
    # SPEC.md:314-316 (N_x divisible by 8 for the packed grid)
    half = np.full((4, 4, 4, 8), 0.5)
    assert (osp.deinterleave(half, 2) >= 0.5).all()
    assert not (osp.deinterleave(np.full((4, 4, 4, 8), 0.49), 2) >= 0.5).any()
    # x-fastest channel order
    g = np.zeros((2, 2, 2))
    g[1, 0, 0] = 1
    assert osp.interleave(g, 2)[0, 0, 0, 1] == 1
    g = np.zeros((2, 2, 2))
    g[0, 0, 1] = 1
    assert osp.interleave(g, 2)[0, 0, 0, 4] == 1


def test_interleave_round_trip_random(rng):
    for d in (2, 4, 8):
        for _ in range(10):
            g = rng.random((16, 8, 16)) < 0.2 if d < 8 else rng.random((16, 16, 8)) < 0.2
            assert np.array_equal(osp.deinterleave(osp.interleave(g, d), d), g)


def test_interleave_rejects_non_divisible():
    with pytest.raises(ValueError):
        osp.interleave(np.zeros((6, 4, 4)), 4)


# ---------------------------------------------------------------- conv / kmap


def _sparse_from_dense(x, mask):
    coords = np.argwhere(mask).astype(np.int64)
    return coords, x[tuple(coords.T)]


def test_sparse_conv_equals_masked_reference(golden):
    g = golden("conv.npz")
    x, mask = g["x"], g["mask"]
    dims = mask.shape[1:]
    coords, rows = _sparse_from_dense(x, mask)
    nbr = osp.kmap_subm(coords, dims)
    centre = np.arange(len(coords))[:, None]
    h = rows
    layers = [(3, "relu"), (3, "relu"), (1, "sigmoid")]
    for i, (k, act) in enumerate(layers):
        z = osp.gather_conv(h, nbr if k == 3 else centre, g[f"w{i}"], g[f"b{i}"])
        h = osp._act(z, act)
        ref = g[f"y{i}"][tuple(coords.T)]
        np.testing.assert_allclose(h, ref, rtol=0, atol=1e-12)
        # masked cells are exactly zero in the reference-with-mask
        assert np.all(g[f"y{i}"][~mask] == 0)


def test_sparse_backward_equals_masked_reference(golden):
    g = golden("conv.npz")
    x, mask = g["x"], g["mask"]
    dims = mask.shape[1:]
    coords, rows = _sparse_from_dense(x, mask)
    nbr = osp.kmap_subm(coords, dims)
    layers = [(3, g["w0"], g["b0"], "relu"), (3, g["w1"], g["b1"], "relu"), (1, g["w2"], g["b2"], "sigmoid")]
    _, caches = osp.chain_forward_cached(rows, nbr, layers)
    dy = g["dy"][tuple(coords.T)]
    grads, dx = osp.chain_backward(dy, layers, caches)
    for i, (dw, db) in enumerate(grads):
        np.testing.assert_allclose(dw, g[f"dw{i}"], rtol=1e-10, atol=1e-10)
        np.testing.assert_allclose(db, g[f"db{i}"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(dx, g["dx"][tuple(coords.T)], rtol=1e-10, atol=1e-10)


def test_kmap_canonical_properties(rng):
    mask = rng.random((2, 7, 6, 5)) < 0.3
    coords = np.argwhere(mask).astype(np.int64)
    nbr = osp.kmap_subm(coords, mask.shape[1:])
    a = len(coords)
    assert np.array_equal(nbr[:, 13], np.arange(a))               # centre tap is self
    for j in range(27):                                             # symmetry: j <-> 26 - j
        i = np.nonzero(nbr[:, j] >= 0)[0]
        assert np.array_equal(nbr[nbr[i, j], 26 - j], i)
    # brute-force check of a few entries
    for i in rng.integers(0, a, 20):
        b, x, y, z = coords[i]
        for j, o in enumerate(osp.SUBM_OFFSETS):
            q = (b, x + o[0], y + o[1], z + o[2])
            inside = all(0 <= q[k + 1] < mask.shape[k + 1] for k in range(3))
            want = -1
            if inside and mask[q]:
                want = int(np.nonzero((coords == q).all(1))[0][0])
            assert nbr[i, j] == want
    ins, outs, off = osp.pair_lists(nbr)
    assert off[-1] == (nbr >= 0).sum() and len(ins) == len(outs) == off[-1]


def test_down_up_maps_are_transposes(rng):
    mask = rng.random((2, 8, 6, 4)) < 0.25
    fine = np.argwhere(mask).astype(np.int64)
    coarse = osp.coarsen(fine)
    down = osp.kmap_down(fine, mask.shape[1:], coarse)
    parent, parity = osp.kmap_up(fine, coarse, (4, 3, 2))
    assert (parent >= 0).all()
    assert (down >= 0).any(axis=1).all()
    for p in range(len(coarse)):
        for j in range(8):
            c = down[p, j]
            if c >= 0:
                assert parent[c] == p and parity[c] == j
    assert (down >= 0).sum() == len(fine)


def test_bf16_round_matches_torch():
    import torch
    v = np.random.default_rng(3).normal(size=10000) * 10
    v[:4] = [1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, -0.0, 65504.0]
    ref = torch.tensor(v, dtype=torch.float32).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(osp.bf16_round(v), ref)


# ---------------------------------------------------------------- losses


def test_losses_match_reference_golden(golden):
    g = golden("loss.npz")
    for i in range(int(g["n"])):
        p, t = g[f"l{i}_pred"], g[f"l{i}_gt"]
        dv, dg = osp.dice_loss(p, t, 0.1)
        rv, rg = osp.rvl_loss(p, t)
        cv, cg = osp.combined_loss(p, t)
        assert dv == pytest.approx(float(g[f"l{i}_dice"]), abs=1e-14)
        assert rv == pytest.approx(float(g[f"l{i}_rvl"]), abs=1e-14)
        assert cv == pytest.approx(float(g[f"l{i}_comb"]), abs=1e-14)
        np.testing.assert_allclose(dg, g[f"l{i}_dice_g"], atol=1e-15)
        np.testing.assert_allclose(rg, g[f"l{i}_rvl_g"], atol=1e-15)
        np.testing.assert_allclose(cg, g[f"l{i}_comb_g"], atol=1e-15)


def test_spec_loss_kats():
    # TP=FP=FN=1, alpha=.5 -> 1/3
    p = np.array([1.0, 1.0, 0.0])
    g = np.array([1.0, 0.0, 1.0])
    assert osp.dice_loss(p, g, 0.5)[0] == pytest.approx(1 / 3)
    # all-positive prediction, GTP=10 of 1000 -> 99
    g = np.zeros(1000)
    g[:10] = 1
    assert osp.rvl_loss(np.ones(1000), g)[0] == pytest.approx(99.0)
    # lambda=1 -> dice, lambda=0 -> rvl
    p = np.random.default_rng(1).random(1000)
    assert osp.combined_loss(p, g, 0.1, 1.0)[0] == pytest.approx(osp.dice_loss(p, g, 0.1)[0])
    assert osp.combined_loss(p, g, 0.1, 0.0)[0] == pytest.approx(osp.rvl_loss(p, g)[0])
    # empty ground truth conventions (neural.py:367-368, 388-389)
    assert osp.dice_loss(np.zeros(5), np.zeros(5), 0.1)[0] == 0.0
    assert osp.rvl_loss(np.ones(5), np.zeros(5))[0] == 0.0


# ---------------------------------------------------------------- config 1 end to end


def _config1_layers():
    d, specs, arrays = read_fpvw(osp_golden_path("config1.fpvw"))
    return d, [(s.kernel, w.astype(np.float64), b.astype(np.float64), s.activation)
               for s, (w, b) in zip(specs, arrays)]


def osp_golden_path(name):
    return os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name)


def test_config1_oracle_matches_masked_reference(golden):
    g = golden("config1.npz")
    d, layers = _config1_layers()
    occ = FroxelGrid(tuple(g["dims"]), bits=g["bits"]).to_dense()
    assert np.array_equal(occ, synth.config1_grid(0))          # generator pinned too
    cells = osp.interleave(occ.astype(np.float64), d)[None]
    coords, logits = osp.chain_forward(cells, layers, return_logits=True)
    assert np.array_equal(coords, g["coords"])
    np.testing.assert_allclose(logits, g["logits_active"], atol=1e-12)
    prob = osp.sigmoid(logits)
    np.testing.assert_allclose(prob, g["prob_active"], atol=1e-12)
    dense = osp.scatter_cells(coords, prob, cells.shape[:4])[0]
    bits = FroxelGrid.from_dense(osp.predict_bits(dense, d, 0.5)).bits
    assert np.array_equal(bits, g["pred_bits"])


def test_fpvw_golden_parses():
    d, specs, arrays = read_fpvw(osp_golden_path("config1.fpvw"))
    assert d == 2 and [s.out_channels for s in specs] == [32, 32, 32, 32, 8]
    assert sum(w.size + b.size for w, b in arrays) == 90248


def test_unet_oracle_bf16_close_to_fp64():
    occ = synth.box_grid((64, 64, 64), 60, 1, 8, 5)
    cells = osp.interleave(occ.astype(np.float64), 4)[None]
    params = osp.unet_init(1)
    c0, z64 = osp.unet_forward(cells, params, bf16=False, return_logits=True)
    _, z16 = osp.unet_forward(cells, params, bf16=True, return_logits=True)
    assert z64.shape == (len(c0), 64)
    assert np.abs(z64 - z16).max() < 5e-2


# ---------------------------------------------------------------- against the live reference


ref = refbridge.load()


@pytest.mark.skipif(ref is None, reason="reference not mounted (GPU box)")
def test_oracle_against_live_reference(rng):
    il = ref.interleave
    for d in (2, 4):
        g = rng.random((16, 8, 8)) < 0.3
        fg = ref.froxel.FroxelGrid.from_dense(g)
        assert np.array_equal(osp.interleave(g.astype(np.float64), d), il.interleave(fg, d).values)
    nn = ref.neural
    layer = nn.Conv3d(nn.ConvSpec(3, 8, 8, "relu"), np.random.Generator(np.random.PCG64(4)))
    mask = rng.random((1, 5, 5, 5)) < 0.4
    x = (rng.random((1, 5, 5, 5, 8)) * mask[..., None])
    y = layer.forward(x) * mask[..., None]
    coords = np.argwhere(mask).astype(np.int64)
    z = osp.gather_conv(x[tuple(coords.T)], osp.kmap_subm(coords, (5, 5, 5)), layer.w, layer.b)
    np.testing.assert_allclose(np.maximum(z, 0), y[tuple(coords.T)], atol=1e-12)


# ---------------------------------------------------------------- froxelize


def test_froxelize_oracle_matches_reference_golden(golden):
    """oracle/froxelize.py vs the reference's froxelize output (froxel.py:387-394)."""
    from oracle import froxelize as ofz
    g = golden("froxelize.npz")
    for i in range(int(g["ncases"])):
        h, n, f = g[f"c{i}_lens"]
        fn = ofz.froxelize_ortho if int(g[f"c{i}_mode"]) == 1 else ofz.froxelize
        bits = fn(g[f"c{i}_verts"], g[f"c{i}_tris"], g[f"c{i}_origin"], g[f"c{i}_basis"], h, n, f,
                  g[f"c{i}_dims"], int(g[f"c{i}_ss"]), "linear" if int(g[f"c{i}_depth"]) == 0 else "log")
        assert np.array_equal(bits, g[f"c{i}_bits"]), str(g[f"c{i}_name"])


def test_froxelize_full_span_quad_is_one_layer(golden):
    """test_froxel.py:148-159: a full-cross-section quad at w = 0.5 fills layer 8 of 16 only (both modes)."""
    g = golden("froxelize.npz")
    for name in ("full_span_quad", "ortho_full_span_quad"):
        i = next(i for i in range(int(g["ncases"])) if str(g[f"c{i}_name"]) == name)
        dense = FroxelGrid((16, 16, 16), bits=g[f"c{i}_bits"]).to_dense()
        assert dense[:, :, 8].all()
        dense[:, :, 8] = False
        assert not dense.any()


@pytest.mark.skipif(ref is None, reason="reference not mounted (GPU box)")
def test_froxelize_oracle_against_live_reference():
    import sys
    from oracle import froxelize as ofz
    sys.path.insert(0, refbridge.REF_SRC)
    from froxelpvs import core, froxel, scenegen
    for seed in (11, 12):
        scene, cell = scenegen.generate_scene(scenegen.SceneGenConfig(seed=seed, count_range=(3, 6)))
        fr = core.build_viewcell_frustum(cell)
        for ss in (1, 2):
            want = froxel.froxelize(scene, fr, (32, 16, 24), froxel.FroxelizeConfig(supersample=ss)).bits
            got = ofz.froxelize(scene.vertices, scene.triangles, fr._o, fr._basis, fr.half_extent, fr.near,
                                fr.far, (32, 16, 24), ss)
            assert np.array_equal(got, want)


# ---------------------------------------------------------------- GT PVS


def _gt_case(g, i):
    return {k[len(f"c{i}_"):]: g[k] for k in g.files if k.startswith(f"c{i}_")}


def test_gtpvs_oracle_and_viewpoints_match_reference_golden(golden):
    """oracle/gtpvs.py and views.sample_viewpoints vs compute_gt_pvs / sample_viewpoints output."""
    from oracle import gtpvs as ogt
    from paper_2509_24677_b200 import views
    g = golden("gtpvs.npz")
    for i in range(int(g["ncases"])):
        c = _gt_case(g, i)
        cams = [(r[0:3], r[3:12].reshape(3, 3), r[12], r[13], r[14]) for r in c["cams"]]
        f = c["frustum"]
        geo = c["geo_in"].copy() if "geo_in" in c else None
        bits = ogt.gt_pvs(c["verts"], c["tris"], cams, (f[0:3], f[3:12].reshape(3, 3), f[12], f[13], f[14]),
                          c["dims"], c["res"], "linear" if int(c["depth"]) == 0 else "log", c["prim_ids"], geo)
        assert np.array_equal(bits, c["bits"]), str(c["name"])
        if geo is not None:
            assert np.array_equal(geo, c["geo_out"])
        cl = c["cell"]
        cell = views.ViewCell(tuple(cl[0:3]), cl[3], cl[4], cl[5], tuple(cl[6:9]), tuple(cl[9:12]),
                              tuple(cl[12:15]), cl[15], cl[16])
        vp, mode, seed, sub = (int(x) for x in c["sampling"])
        vs = views.sample_viewpoints(cell, vp, "uniform-grid" if mode == 0 else "uniform-random", seed)
        vs = vs[:sub] if sub >= 0 else vs
        rows = np.array([np.concatenate([v.position, v.right, v.up, v.forward, [v.half_extent, v.near, v.far]])
                         for v in vs]).reshape(-1, 15)
        assert np.array_equal(rows, c["cams"]), str(c["name"])
        fv = views.build_viewcell_frustum(cell)
        assert np.array_equal(np.concatenate([fv._o, fv._basis.ravel(), [fv.half_extent, fv.near, fv.far]]), f)


def test_gtpvs_occluder_hides_everything_behind(golden):
    """test_oracle.py:113-137: no GT froxel strictly behind a full-cross-section occluder."""
    g = golden("gtpvs.npz")
    i = next(i for i in range(int(g["ncases"])) if str(g[f"c{i}_name"]) == "occluder")
    dense = FroxelGrid((16, 16, 16), bits=g[f"c{i}_bits"]).to_dense()
    assert dense[:, :, :9].sum() > 0 and dense[:, :, 9:].sum() == 0


# ------------------------------------------- any odd kernel, 3^3 head (api.npz)

def _api_layers(g, tag, specs):
    return [(k, g[f"{tag}_w{i}"], g[f"{tag}_b{i}"], act) for i, (k, act) in enumerate(specs)]


API_SPECS = {"def": [(3, "relu"), (3, "relu"), (3, "sigmoid")], "k5": [(5, "relu"), (3, "sigmoid")]}


@pytest.mark.parametrize("tag", ["def", "k5"])
def test_oracle_general_kernels_match_masked_reference(golden, tag):
    """The oracle's k^3 maps and chain (forward, backward) against the reference's
    own Conv3d on the reference default net (3^3 head) and a 5^3 layer."""
    g = golden("api.npz")
    x, mask = g["x"], g["mask"]
    coords, rows = _sparse_from_dense(x, mask)
    layers = _api_layers(g, tag, API_SPECS[tag])
    c, prob = osp.chain_forward(x, layers)
    assert np.array_equal(c, coords)
    np.testing.assert_allclose(prob, g[f"{tag}_y{len(layers) - 1}"][tuple(coords.T)], rtol=0, atol=1e-12)
    dims = mask.shape[1:]
    tables = {k: osp.kmap_subm(coords, dims, k) for k in (3, 5)}
    _, caches = osp.chain_forward_cached(rows, tables[3], layers, tables)
    grads, dx = osp.chain_backward(g[f"{tag}_dy"][tuple(coords.T)], layers, caches)
    for i, (dw, db) in enumerate(grads):
        np.testing.assert_allclose(dw, g[f"{tag}_dw{i}"], rtol=1e-10, atol=1e-10)
        np.testing.assert_allclose(db, g[f"{tag}_db{i}"], rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(dx, g[f"{tag}_dx"][tuple(coords.T)], rtol=1e-10, atol=1e-10)


def test_kmap_subm_general_k_offsets(rng):
    """k^3 maps: centre tap is the identity, k = 3 equals the default table,
    mirror symmetry nbr[nbr[i][j]][K-1-j] == i for k = 5."""
    dims = (6, 7, 5)
    occ = rng.random((1,) + dims) < 0.3
    coords = np.argwhere(occ)
    n3 = osp.kmap_subm(coords, dims)
    assert np.array_equal(osp.kmap_subm(coords, dims, 3), n3)
    assert np.array_equal(osp.kmap_subm(coords, dims, 1)[:, 0], np.arange(len(coords)))
    n5 = osp.kmap_subm(coords, dims, 5)
    assert np.array_equal(n5[:, 62], np.arange(len(coords)))
    for j in range(125):
        m = n5[:, j] >= 0
        assert np.array_equal(n5[n5[m, j], 124 - j], np.nonzero(m)[0])
