"""Config-2 sparse U-Net on the tcgen05 path vs the oracle's bf16 emulation."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import sparse as osp
from paper_2509_24677_b200 import synth
from paper_2509_24677_b200.froxel import FroxelGrid

pytestmark = pytest.mark.gpu

BF16_LOGIT_TOL = 2e-2
BAND = 1e-3


def _run(occ, seed=1, precision="bf16"):
    import torch
    from paper_2509_24677_b200.unet import PvsUNet
    net = PvsUNet(seed=seed, precision=precision)
    bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
    plan = net.plan(1, occ.shape)
    out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
    logits = torch.zeros((plan.L0.cap, 64), device="cuda")
    plan.run(bits, out, 0.5, logits=logits)
    torch.cuda.synchronize()
    return plan, out, logits


def _check(occ, plan, out, logits, bf16=True):
    cells = osp.interleave(occ.astype(np.float64), 4)[None]
    params = osp.unet_init(1)
    coords, z = osp.unet_forward(cells, params, bf16=bf16, return_logits=True)
    n = plan.L0.count()
    assert n == len(coords)
    assert np.array_equal(plan.L0.coords[:n].cpu().numpy(), coords)
    err = np.abs(logits[:n].cpu().numpy() - z).max()
    prob = osp.sigmoid(z)
    dense = osp.deinterleave(osp.scatter_cells(coords, prob, (1,) + plan.L0.dims)[0], 4)
    got = FroxelGrid(occ.shape, bits=out.cpu().numpy()).to_dense()
    diff = got != (dense >= 0.5)
    hard = int((diff & (np.abs(dense - 0.5) >= BAND)).sum())
    return err, hard, int(diff.sum()), int((dense >= 0.5).sum())


def test_unet_small_grid():
    occ = synth.box_grid((64, 64, 64), 60, 1, 8, 5)
    plan, out, logits = _run(occ)
    err, hard, soft, vis = _check(occ, plan, out, logits)
    assert err <= BF16_LOGIT_TOL, err
    assert hard == 0, (hard, soft)
    assert vis > 0


def test_unet_fp32_mode_small_grid():
    occ = synth.box_grid((64, 64, 64), 60, 1, 8, 6)
    plan, out, logits = _run(occ, precision="fp32")
    err, hard, soft, _ = _check(occ, plan, out, logits, bf16=False)
    assert err <= 1e-4, err
    assert hard == 0, (hard, soft)


def test_unet_empty_and_tiny_grids():
    for occ in (np.zeros((64, 64, 64), bool), _single_froxel()):
        plan, out, logits = _run(occ)
        if not occ.any():
            assert plan.L0.count() == 0 and not out.any()
        else:
            _, hard, _, _ = _check(occ, plan, out, logits)
            assert hard == 0


def _single_froxel():
    o = np.zeros((64, 64, 64), bool)
    o[63, 0, 17] = True
    return o


@pytest.mark.slow
def test_unet_config2_full_size():
    """BASELINE config 2 (256^3, 4000 boxes, seed 1) end to end."""
    occ = synth.config2_grid(1)
    plan, out, logits = _run(occ)
    err, hard, soft, vis = _check(occ, plan, out, logits)
    print(f"cfg2: logits max-abs {err:.3g}, mask diffs {soft} (outside band {hard}), visible {vis}")
    assert err <= BF16_LOGIT_TOL, err
    assert hard == 0, (hard, soft)


@pytest.mark.parametrize("inflight", [1, 2, 3])
def test_streamed_frames_match_eager(inflight):
    """FramePipeline.infer_stream: every streamed frame (distinct inputs, up to
    ``inflight`` computing concurrently on separate buffers) equals the eager frame."""
    import torch
    from paper_2509_24677_b200 import synth
    from paper_2509_24677_b200.froxel import FroxelGrid
    from paper_2509_24677_b200.pipeline import FramePipeline
    from paper_2509_24677_b200.unet import PvsUNet
    dims = (64, 64, 64)
    frames = [FroxelGrid.from_dense(synth.box_grid(dims, 40 + 7 * k, 1, 8, 10 + k)).bits for k in range(5)]
    ins = [torch.from_numpy(b).pin_memory() for b in frames]
    outs = [torch.empty(len(frames[0]), dtype=torch.uint8, pin_memory=True) for _ in range(7)]
    net = PvsUNet(seed=1, precision="bf16")
    pipe = FramePipeline(net, 1, dims, graph=True)
    pipe.load(ins[0].cuda())
    pipe.capture()
    seq = [ins[i % len(ins)] for i in range(7)]
    pipe.infer_stream(seq, outs, inflight=inflight)
    torch.cuda.synchronize()
    ref = FramePipeline(net, 1, dims, graph=False)
    for i, x in enumerate(seq):
        ref.plan.run(x.cuda(), ref.out_bits, 0.5)
        torch.cuda.synchronize()
        assert torch.equal(outs[i], ref.out_bits.cpu()), i


def test_fused_head_equals_standalone_head():
    """dec0b with the head fused into its epilogue (fpvs_spconv_halo_head)
    writes exactly the bits of dec0b + the stand-alone head (same bf16
    activations, same MMA products and K order)."""
    import torch
    from paper_2509_24677_b200 import synth
    from paper_2509_24677_b200.froxel import FroxelGrid
    from paper_2509_24677_b200.unet import PvsUNet
    for seed, dims in ((1, (128, 128, 128)), (3, (256, 256, 256))):
        occ = synth.box_grid(dims, 4000 if dims[0] == 256 else 600, 1, 12, seed)
        bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
        net = PvsUNet(seed=1, precision="bf16")
        plan = net.plan(1, occ.shape)
        plan.tune(bits)
        outs = []
        for fuse in (True, False):
            plan.fuse_head = fuse
            # garbage in the output grid: the fused path writes every word (no clear)
            out = torch.full((occ.size // 8,), 0xA5, dtype=torch.uint8, device="cuda")
            names = [n for n, _ in plan.stages(bits, out, 0.5)]
            # fused only where dec0b runs unsplit 64-wide tiles (the 256^3 frame)
            assert ("head" in names) != (fuse and dims[0] == 256)
            plan.run(bits, out, 0.5)
            torch.cuda.synchronize()
            outs.append(out.cpu().numpy())
        assert np.array_equal(outs[0], outs[1]), (seed, int(np.unpackbits(outs[0] ^ outs[1]).sum()))
        assert np.unpackbits(outs[0]).sum() > 0


def test_rowbits_to_grid_matches_dense_scatter():
    """fpvs_rowbits_to_grid: per-row 64-bit cell masks (bit lx + 4 ly + 16 lz)
    scattered through the level-0 index volume into the packed froxel grid,
    every word written (inactive cells and garbage in the buffer -> 0)."""
    import torch
    from paper_2509_24677_b200 import _lib
    rng = np.random.default_rng(5)
    B, dims = 2, (64, 32, 48)
    X, Y, Z = (n // 4 for n in dims)
    active = rng.random((B, X, Y, Z)) < 0.3
    index_vol = np.full((B, X, Y, Z), -1, np.int32)
    n = int(active.sum())
    index_vol[active] = np.arange(n, dtype=np.int32)
    row_bits = rng.integers(0, 2**63, size=n, dtype=np.int64) ^ rng.integers(0, 2, size=n, dtype=np.int64) << 63
    dense = np.zeros((B,) + dims, bool)
    b, cx, cy, cz = np.nonzero(active)
    rb = row_bits.view(np.uint64)
    for k in range(64):
        lx, ly, lz = k % 4, (k // 4) % 4, k // 16
        on = ((rb >> np.uint64(k)) & np.uint64(1)).astype(bool)
        dense[b[on], 4 * cx[on] + lx, 4 * cy[on] + ly, 4 * cz[on] + lz] = True
    ref = np.concatenate([FroxelGrid.from_dense(dense[i]).bits for i in range(B)])
    out = torch.full((ref.size,), 0x5A, dtype=torch.uint8, device="cuda")
    rbt = torch.from_numpy(row_bits).cuda()
    ivt = torch.from_numpy(index_vol.ravel()).cuda()
    _lib.call("fpvs_rowbits_to_grid", _lib.ptr(rbt), _lib.ptr(ivt), B, *dims, 4, _lib.ptr(out), _lib.stream_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), ref)
    # the dataflow writer (every producer tile already published) writes the same words
    done = torch.full(((n + 127) // 128,), 4, dtype=torch.int32, device="cuda")
    out2 = torch.full_like(out, 0xA5)
    _lib.call("fpvs_rowbits_to_grid_flow", _lib.ptr(rbt), _lib.ptr(ivt), B, *dims, 4, _lib.ptr(out2), _lib.ptr(done),
              _lib.stream_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(out2.cpu().numpy(), ref)
    # argument checks: d != 4 and N_x % 32 != 0 are rejected
    with pytest.raises(Exception):
        _lib.call("fpvs_rowbits_to_grid", _lib.ptr(rbt), _lib.ptr(ivt), B, *dims, 2, _lib.ptr(out), _lib.stream_ptr())
    with pytest.raises(Exception):
        _lib.call("fpvs_rowbits_to_grid", _lib.ptr(rbt), _lib.ptr(ivt), B, 48, 32, 48, 4, _lib.ptr(out),
                  _lib.stream_ptr())


def test_up_blocks_equal_sorted_up_conv():
    """up21 / up10 as one dense GEMM over the coarse rows with the column-block
    scatter (fpvs_spconv_tc_upblocks) write exactly the rows of the
    parity-sorted gather-GEMM (same operands, same K order), and the frame's
    bits are unchanged."""
    import os
    import torch
    from paper_2509_24677_b200.unet import PvsUNet
    occ = synth.box_grid((128, 128, 128), 600, 1, 12, 2)
    bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
    res = []
    for flag in ("1", "0"):
        os.environ["FPVS_UPBLOCKS"] = flag
        try:
            plan = PvsUNet(seed=1, precision="bf16").plan(1, occ.shape)
        finally:
            os.environ.pop("FPVS_UPBLOCKS", None)
        assert plan.use_upblocks == (flag == "1")
        out = torch.empty(occ.size // 8, dtype=torch.uint8, device="cuda")
        stages = plan.stages(bits, out, 0.5)
        for name, fn in stages:
            fn()
            if name == "up10":
                torch.cuda.synchronize()
                n0, n1 = plan.L0.count(), plan.L1.count()
                snap = (plan.buf1[:n1].clone(), plan.buf0[:n0].clone())
        torch.cuda.synchronize()
        res.append((snap, out.clone()))
    (a1, a0), ab = res[0]
    (b1, b0), bb = res[1]
    assert torch.equal(a1, b1) and torch.equal(a0, b0)
    assert torch.equal(ab, bb)


def test_unet_batch_of_two_equals_two_single_frames():
    """A B = 2 U-Net plan (fused maps over both grids, batch-coordinate rows,
    column-block up convs, fused head + grid writer per batch plane) gives each
    grid exactly the bits of its own B = 1 frame."""
    import torch
    from paper_2509_24677_b200.unet import PvsUNet
    dims = (128, 128, 128)
    occs = [synth.box_grid(dims, 600, 1, 12, s) for s in (11, 12)]
    net = PvsUNet(seed=1, precision="bf16")
    singles = []
    for occ in occs:
        plan = net.plan(1, dims)
        bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
        out = torch.full((occ.size // 8,), 0xA5, dtype=torch.uint8, device="cuda")
        plan.run(bits, out, 0.5)
        torch.cuda.synchronize()
        singles.append(out.cpu().numpy())
    plan2 = net.plan(2, dims)
    bits2 = torch.from_numpy(np.concatenate([FroxelGrid.from_dense(o).bits for o in occs])).cuda()
    out2 = torch.full((2 * occs[0].size // 8,), 0x5A, dtype=torch.uint8, device="cuda")
    plan2.run(bits2, out2, 0.5)
    torch.cuda.synchronize()
    got = out2.cpu().numpy().reshape(2, -1)
    assert np.array_equal(got[0], singles[0]) and np.array_equal(got[1], singles[1])
    assert int(np.unpackbits(got).sum()) > 0


def test_dataflow_pairs_equal_grid_wide_waits():
    """Tile-level dataflow between the two convs of a level (per-tile done
    flags, fpvs_spconv_halo_flow) gives the frame of grid-wide waits bit for
    bit, eagerly and replayed from a CUDA graph."""
    import os
    import torch
    from paper_2509_24677_b200.pipeline import FramePipeline
    from paper_2509_24677_b200.unet import PvsUNet
    for dims, boxes in (((256, 256, 256), 4000), ((128, 128, 128), 600)):
        occ = synth.box_grid(dims, boxes, 1, 12, 5)
        bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
        outs = []
        # level-0 halo pairs (default), + the down conv as a gather-GEMM consumer, off
        for flag, tc in (("1", "0"), ("1", "1"), ("0", "0")):
            os.environ["FPVS_FLOW"], os.environ["FPVS_FLOW_TC"] = flag, tc
            try:
                pipe = FramePipeline(PvsUNet(seed=1), 1, occ.shape)
            finally:
                os.environ.pop("FPVS_FLOW", None)
                os.environ.pop("FPVS_FLOW_TC", None)
            assert pipe.plan.flow == (flag == "1") and bool(pipe.plan.flow_tc) == (tc == "1")
            pipe.load(bits)
            pipe.capture()
            for _ in range(3):
                pipe.run_device()
            torch.cuda.synchronize()
            outs.append(pipe.out_bits.clone())
            eager = torch.full_like(pipe.out_bits, 0xA5)
            pipe.plan.run(bits, eager, 0.5)
            torch.cuda.synchronize()
            assert torch.equal(eager, outs[-1])
        assert torch.equal(outs[0], outs[2]) and torch.equal(outs[1], outs[2]), dims


def test_empty_and_single_cell_frames():
    """Frames with no active cell (every kernel runs on zero rows: the dataflow
    pairs wait for nothing, the grid writer writes zeros) and with one active
    cell run through the captured graph without hanging and give the eager
    bits."""
    import torch
    from paper_2509_24677_b200.pipeline import FramePipeline
    from paper_2509_24677_b200.unet import PvsUNet
    dims = (256, 256, 256)
    one = np.zeros(dims, bool)
    one[100:102, 50:53, 7] = True
    pipe = FramePipeline(PvsUNet(seed=1), 1, dims)
    pipe.load(torch.from_numpy(FroxelGrid.from_dense(synth.config2_grid(1)).bits).cuda())
    pipe.capture()
    for occ in (np.zeros(dims, bool), one):
        bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
        pipe.in_bits.copy_(bits)
        pipe.out_bits.fill_(0xA5)
        pipe.run_device()
        torch.cuda.synchronize()
        graph_out = pipe.out_bits.clone()
        eager = torch.full_like(graph_out, 0x5A)
        pipe.plan.run(bits, eager, 0.5)
        torch.cuda.synchronize()
        assert torch.equal(graph_out, eager)
        if not occ.any():
            assert int(graph_out.count_nonzero()) == 0


@pytest.mark.slow
def test_unet_non_cubic_bits_only_frame_matches_oracle():
    """A non-cubic grid (256 x 128 x 256) through the bits-only frame — the
    head fused into dec0b, the grid writer, the level-0 dataflow pairs and the
    column-block up convs all active — against the oracle's bf16 emulation:
    no mask difference outside the threshold band."""
    import torch
    from paper_2509_24677_b200.unet import PvsUNet
    dims = (256, 128, 256)
    occ = synth.box_grid(dims, 3000, 1, 12, 9)
    net = PvsUNet(seed=1, precision="bf16")
    plan = net.plan(1, dims)
    bits = torch.from_numpy(FroxelGrid.from_dense(occ).bits).cuda()
    plan.tune(bits)
    out = torch.full((occ.size // 8,), 0xA5, dtype=torch.uint8, device="cuda")
    names = [n for n, _ in plan.stages(bits, out, 0.5)]
    plan.run(bits, out, 0.5)
    torch.cuda.synchronize()
    assert "head" not in names, "expected the fused head at this size"
    assert plan.flow and plan.halo_cfg["dec0b"] == (64, 1)
    cells = osp.interleave(occ.astype(np.float64), 4)[None]
    coords, z = osp.unet_forward(cells, osp.unet_init(1), bf16=True, return_logits=True)
    assert plan.L0.count() == len(coords)
    prob = osp.sigmoid(z)
    dense = osp.deinterleave(osp.scatter_cells(coords, prob, (1,) + plan.L0.dims)[0], 4)
    got = FroxelGrid(occ.shape, bits=out.cpu().numpy()).to_dense()
    diff = got != (dense >= 0.5)
    hard = int((diff & (np.abs(dense - 0.5) >= BAND)).sum())
    assert hard == 0, (hard, int(diff.sum()))
    assert int(got.sum()) > 0
