"""Parity-sorted k2s2 up conv (fpvs_up_sort + fpvs_spconv_tc_scatter).

The sort is integer work: it must equal a numpy stable counting sort by
parity class with each class padded to 128 rows.  The sorted conv adds the
same products as the unsorted one minus exact zeros, so its output must be
bit-identical to the plain K = 8 gather-GEMM.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ref_sort(up: np.ndarray):
    cls = np.argmax(up >= 0, axis=1)
    parent = up[np.arange(len(up)), cls]
    perm, table, masks = [], [], []
    for c in range(8):
        rows = np.nonzero(cls == c)[0]
        pad = (len(rows) + 127) // 128 * 128
        p = np.full(pad, -1, np.int64)
        p[:len(rows)] = rows
        t = np.full((pad, 8), -1, np.int64)
        t[np.arange(len(rows)), c] = parent[rows]
        perm.append(p)
        table.append(t)
        masks += [1 << c] * (pad // 128)
    return np.concatenate(perm), np.concatenate(table), np.array(masks, np.int64)


def _config2_plan():
    import torch
    from paper_2509_24677_b200 import synth
    from paper_2509_24677_b200.froxel import FroxelGrid
    from paper_2509_24677_b200.unet import PvsUNet
    occ = synth.config2_grid(1)
    bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
    import os
    net = PvsUNet(seed=1)
    # the default frame runs the up convs as dense column-block GEMMs
    # (fpvs_spconv_tc_upblocks) and builds no up tables; the parity-sorted
    # path (up tables + fpvs_up_sort) stays available behind FPVS_UPBLOCKS=0
    os.environ["FPVS_UPBLOCKS"] = "0"
    try:
        plan = net.plan(1, occ.shape)
    finally:
        os.environ.pop("FPVS_UPBLOCKS", None)
    assert plan.use_upsort
    plan.build_maps(bits)
    return net, plan, bits, occ


def test_up_sort_tables_config2():
    _, plan, _, _ = _config2_plan()
    for fine, up in ((plan.L1, plan.up21), (plan.L0, plan.up10)):
        n = fine.count()
        u = fine.extra["upsort"]
        perm, table, masks = _ref_sort(up[:n].cpu().numpy().astype(np.int64))
        npad = int(u["n"].item())
        assert npad == len(perm)
        assert np.array_equal(u["perm"][:npad].cpu().numpy(), perm)
        assert np.array_equal(u["table"][:npad].cpu().numpy(), table)
        assert np.array_equal(u["masks"][:npad // 128].cpu().numpy().astype(np.int64) & 0xffffffff, masks)


def test_up_sort_small_and_empty_classes():
    """A hand-made up table where some parity classes are empty."""
    import torch
    from paper_2509_24677_b200 import sparse as sp
    rng = np.random.default_rng(3)
    n, cap = 300, 512
    up = np.full((n, 8), -1, np.int64)
    cls = rng.choice([0, 3, 5], size=n)
    up[np.arange(n), cls] = rng.integers(0, 50, size=n)
    lv = sp.new_level(1, (8, 8, 8))
    lv.cap = cap
    lv.n = torch.tensor([n], dtype=torch.int32, device="cuda")
    t = torch.full((cap, 8), -1, dtype=torch.int32, device="cuda")
    t[:n] = torch.from_numpy(up.astype(np.int32)).cuda()
    sp.UpSorter([(lv, t)]).run()
    u = lv.extra["upsort"]
    perm, table, masks = _ref_sort(up)
    npad = int(u["n"].item())
    assert npad == len(perm)
    assert np.array_equal(u["perm"][:npad].cpu().numpy(), perm)
    assert np.array_equal(u["table"][:npad].cpu().numpy(), table)


def test_sorted_up_conv_bit_identical():
    import torch
    from paper_2509_24677_b200.neural import run_conv
    net, plan, bits, _ = _config2_plan()
    L1, L0 = plan.L1, plan.L0
    for name, coarse, fine, up, cin, cout in (("up21", plan.L2, L1, plan.up21, 256, 128),
                                              ("up10", L1, L0, plan.up10, 128, 64)):
        layer = net.layers[name]
        nc = coarse.count()
        x = torch.zeros((coarse.cap, cin), dtype=torch.bfloat16, device="cuda")
        x[:nc] = torch.relu(torch.randn((nc, cin), device="cuda")).bfloat16()
        a = torch.zeros((fine.cap, cout), dtype=torch.bfloat16, device="cuda")
        b = torch.zeros_like(a)
        masks = coarse.extra["up_masks"]
        run_conv(layer, x, cin, up, 8, fine.n, fine.cap, a, cout, 0, "bf16", act="relu", masks=masks)
        u = fine.extra["upsort"]
        run_conv(layer, x, cin, u["table"], 8, u["n"], u["cap"], b, cout, 0, "bf16", act="relu", masks=u["masks"],
                 out_rows=u["perm"])
        n = fine.count()
        assert torch.equal(a[:n], b[:n]), name


def test_up_blocks_bit_identical():
    """fpvs_spconv_tc_upblocks (dense coarse-row GEMM, column block j -> child
    in parity class j through the down table) == the gathered up conv."""
    import torch
    from paper_2509_24677_b200 import _lib
    from paper_2509_24677_b200.neural import packed_upblocks_cache, run_conv
    net, plan, bits, _ = _config2_plan()
    for name, coarse, fine, up, down, cin, cout in (("up21", plan.L2, plan.L1, plan.up21, plan.down12, 256, 128),
                                                    ("up10", plan.L1, plan.L0, plan.up10, plan.down01, 128, 64)):
        layer = net.layers[name]
        nc = coarse.count()
        x = torch.zeros((coarse.cap, cin), dtype=torch.bfloat16, device="cuda")
        x[:nc] = torch.relu(torch.randn((nc, cin), device="cuda")).bfloat16()
        a = torch.zeros((fine.cap, 2 * cout), dtype=torch.bfloat16, device="cuda")
        b = torch.full_like(a, 7.0)
        run_conv(layer, x, cin, up, 8, fine.n, fine.cap, a, 2 * cout, cout, "bf16", act="relu",
                 masks=coarse.extra["up_masks"])
        for bn in (256, 128):
            w8, b8 = packed_upblocks_cache(layer, bn)
            _lib.call("fpvs_spconv_tc_upblocks", _lib.ptr(x), cin, x.shape[0], _lib.ptr(coarse.n), coarse.cap,
                      _lib.ptr(w8), bn, _lib.ptr(b8), cin, cout, _lib.ACT["relu"], _lib.ptr(down), _lib.ptr(b),
                      2 * cout, cout, _lib.stream_ptr())
            torch.cuda.synchronize()
            n = fine.count()
            assert torch.equal(a[:n, cout:], b[:n, cout:]), (name, bn)
            assert bool((b[:n, :cout] == 7.0).all())  # columns outside [col_off, col_off + Cout) untouched


def test_unet_with_and_without_up_sort():
    import torch
    from paper_2509_24677_b200.unet import PvsUNet
    net, plan, bits, occ = _config2_plan()
    import os
    os.environ["FPVS_UPBLOCKS"] = "0"  # plain gathered up convs (up tables built by the maps)
    try:
        other = net.plan(1, occ.shape)
    finally:
        os.environ.pop("FPVS_UPBLOCKS", None)
    other.use_upsort = False
    la = torch.zeros((plan.L0.cap, 64), device="cuda")
    lb = torch.zeros_like(la)
    oa = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
    ob = torch.empty_like(oa)
    plan.run(bits, oa, 0.5, logits=la)
    other.run(bits, ob, 0.5, logits=lb)
    n = plan.L0.count()
    assert torch.equal(la[:n], lb[:n])
    assert torch.equal(oa, ob)
