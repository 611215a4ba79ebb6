"""fpvs_froxelize (csrc/froxelize.cu) vs the reference froxelizer.

Pinned on tests/golden/froxelize.npz — grids written by the reference's own
``froxelize`` (froxel.py:387-394, perspective mode) on its scene generator's
scenes and on near-plane-clipping cases (tests/golden/make_froxelize_golden.py).
Linear depth is bit-exact.  Log depth goes through ``log``, whose last bit
differs between numpy's SIMD kernel and CUDA's, so a froxel whose depth sits
exactly on a layer boundary may move; the test allows a handful.
The reference's own froxelize tests (pkg/tests/test_froxel.py:133-215) are
mirrored: empty scene, N_x % 8, full-cross-section quad -> one layer,
s=1 coverage inside s=3 coverage, triangles behind the origin.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import froxelize as ofz

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "froxelize.npz")


def _cases():
    g = np.load(GOLDEN)
    out = []
    for i in range(int(g["ncases"])):
        p = f"c{i}_"
        out.append({k[len(p):]: g[k] for k in g.files if k.startswith(p)})
    return out


CASES = _cases()


def _frustum(c):
    from paper_2509_24677_b200.froxelize import Frustum
    h, n, f = (float(v) for v in c["lens"])
    return Frustum(c["origin"], c["basis"], h, n, f)


def _mode(c):
    return "ortho" if int(c.get("mode", 0)) == 1 else "perspective"


@pytest.mark.parametrize("idx", range(len(CASES)), ids=[str(c["name"]) for c in CASES])
def test_golden(idx):
    from paper_2509_24677_b200.froxelize import FroxelizeConfig, Froxelizer
    c = CASES[idx]
    cfg = FroxelizeConfig(supersample=int(c["ss"]), depth_mode="linear" if int(c["depth"]) == 0 else "log",
                          mode=_mode(c))
    fz = Froxelizer(c["verts"], c["tris"])
    got = fz.run(_frustum(c), tuple(int(v) for v in c["dims"]), cfg).cpu().numpy()
    ref = c["bits"]
    diff = np.unpackbits(got ^ ref).sum()
    if int(c["depth"]) == 0:
        assert diff == 0, f"{c['name']}: {diff} froxels differ"
    else:
        assert diff <= max(4, np.unpackbits(ref).sum() // 1000), diff


def test_drop_in_api_matches_golden():
    """froxelize(scene, frustum, dims, cfg) -> FroxelGrid, as froxel.py:387."""
    from types import SimpleNamespace
    from paper_2509_24677_b200.froxelize import FroxelizeConfig, froxelize
    c = next(c for c in CASES if str(c["name"]) == "scene1")
    scene = SimpleNamespace(vertices=c["verts"], triangles=c["tris"])
    ref_frustum = SimpleNamespace(_o=c["origin"], _basis=c["basis"], half_extent=float(c["lens"][0]),
                                  near=float(c["lens"][1]), far=float(c["lens"][2]))
    grid = froxelize(scene, ref_frustum, tuple(int(v) for v in c["dims"]), FroxelizeConfig(supersample=4))
    assert grid.role == "geometry" and grid.supersample == 4
    assert np.array_equal(grid.bits, c["bits"])


def _soup(seed, n, frustum, spread=6.0, size=1.5):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-spread, spread, size=(n, 1, 3)) + frustum._o + 8.0 * frustum._basis[2]
    return (c + rng.normal(scale=size, size=(n, 3, 3))).reshape(-1, 3), np.arange(3 * n).reshape(-1, 3)


def _random_frustum(seed):
    from paper_2509_24677_b200.froxelize import Frustum
    rng = np.random.default_rng(seed)
    f = rng.normal(size=3)
    f /= np.linalg.norm(f)
    r = np.cross(f, [0.0, 1.0, 0.0])
    r /= np.linalg.norm(r)
    u = np.cross(r, f)
    return Frustum.from_vectors(rng.uniform(-2, 2, size=3), f, u, r, rng.uniform(40, 100),
                                rng.uniform(0.2, 1.0), rng.uniform(15, 30))


@pytest.mark.parametrize("seed,dims,ss", [(0, (64, 64, 64), 4), (1, (32, 48, 16), 3), (2, (128, 64, 96), 2),
                                          (3, (8, 8, 8), 1), (4, (256, 128, 64), 4)])
def test_random_scenes_vs_oracle(seed, dims, ss):
    from paper_2509_24677_b200.froxelize import FroxelizeConfig, Froxelizer
    fr = _random_frustum(seed)
    v, t = _soup(seed, 600, fr)
    got = Froxelizer(v, t).run(fr, dims, FroxelizeConfig(supersample=ss)).cpu().numpy()
    ref = ofz.froxelize(v, t, fr._o, fr._basis, fr.half_extent, fr.near, fr.far, dims, ss)
    assert np.array_equal(got, ref), np.unpackbits(got ^ ref).sum()


def test_empty_scene_and_bad_dims():
    from paper_2509_24677_b200.froxelize import Froxelizer
    fr = _random_frustum(0)
    fz = Froxelizer(np.zeros((0, 3)), np.zeros((0, 3), dtype=np.int64))
    out = fz.run(fr, (16, 16, 16))
    assert int(out.sum()) == 0
    with pytest.raises(ValueError):
        fz.run(fr, (15, 16, 16))


def test_behind_origin_contributes_nothing():
    from paper_2509_24677_b200.froxelize import Froxelizer, Frustum
    fr = Frustum.from_vectors([0, 0, 0], [0, 0, 1], [0, 1, 0], [1, 0, 0], 90.0, 2.0, 18.0)
    v = np.array([[-3.0, -3.0, -5.0], [3.0, -3.0, -5.0], [3.0, 3.0, -5.0], [-3.0, 3.0, -5.0]])
    out = Froxelizer(v, [[0, 1, 2], [0, 2, 3]]).run(fr, (16, 16, 16))
    assert int(out.sum()) == 0


def test_supersample_coverage_nests():
    """s=1 sample centres reappear at s=3, so coverage only grows (test_froxel.py:183-205)."""
    from paper_2509_24677_b200.froxelize import FroxelizeConfig, Froxelizer
    for seed in range(6):
        fr = _random_frustum(10 + seed)
        v, t = _soup(seed, 80, fr, size=0.8)
        fz = Froxelizer(v, t)
        lo = fz.run(fr, (16, 16, 16), FroxelizeConfig(supersample=1)).cpu().numpy()
        hi = fz.run(fr, (16, 16, 16), FroxelizeConfig(supersample=3)).cpu().numpy()
        assert not np.any(lo & ~hi), seed


def test_unaligned_output_and_graph_replay():
    import torch
    from paper_2509_24677_b200.froxelize import FroxelizeConfig, Froxelizer
    fr = _random_frustum(7)
    v, t = _soup(7, 300, fr)
    dims = (24, 8, 7)  # 168 bytes: word-aligned size, but placed at an odd offset below
    ref = ofz.froxelize(v, t, fr._o, fr._basis, fr.half_extent, fr.near, fr.far, dims, 2)
    fz = Froxelizer(v, t)
    buf = torch.full((ref.size + 1,), 0xAA, dtype=torch.uint8, device="cuda")
    fz.run(fr, dims, FroxelizeConfig(supersample=2), out=buf[1:])
    assert np.array_equal(buf[1:].cpu().numpy(), ref) and int(buf[0]) == 0xAA
    # graph capture: one replay per frustum reproduces the eager result
    out = torch.empty(ref.size, dtype=torch.uint8, device="cuda")
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    from paper_2509_24677_b200.pipeline import no_gc
    with torch.cuda.stream(s), no_gc():
        fz.run(fr, dims, FroxelizeConfig(supersample=2), out=out)
        with torch.cuda.graph(g, stream=s):
            fz.run(fr, dims, FroxelizeConfig(supersample=2), out=out)
    torch.cuda.current_stream().wait_stream(s)
    out.fill_(0x55)
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), ref)
    assert fz.samples() > 0


def test_feeds_the_pvs_pipeline():
    """Froxelized grid -> FramePipeline.in_bits on the device (no host hop)."""
    import torch
    from paper_2509_24677_b200.froxelize import Froxelizer
    from paper_2509_24677_b200.neural import ModelConfig, PvsNet
    from paper_2509_24677_b200.pipeline import FramePipeline
    fr = _random_frustum(3)
    v, t = _soup(3, 400, fr)
    dims = (64, 64, 64)
    net = PvsNet(ModelConfig.config1(), np.random.Generator(np.random.PCG64(0)), precision="bf16")
    pipe = FramePipeline(net, 1, dims, graph=False)
    Froxelizer(v, t).run(fr, dims, out=pipe.in_bits)
    pipe.capture(tune=False)
    ref = ofz.froxelize(v, t, fr._o, fr._basis, fr.half_extent, fr.near, fr.far, dims, 4)
    assert np.array_equal(pipe.in_bits.cpu().numpy(), ref)
    out = pipe.run_device()
    torch.cuda.synchronize()
    assert out.numel() == ref.size


@pytest.mark.parametrize("seed,dims,ss,depth", [(0, (32, 32, 32), 2, "linear"), (1, (24, 40, 16), 3, "linear"),
                                                (2, (64, 32, 48), 1, "linear"), (3, (16, 16, 16), 4, "log")])
def test_ortho_random_scenes_vs_oracle(seed, dims, ss, depth):
    """mode="ortho" (froxel.py:351-376) on random soups and frusta vs the oracle."""
    from paper_2509_24677_b200.froxelize import FroxelizeConfig, Froxelizer
    fr = _random_frustum(100 + seed)
    v, t = _soup(seed, 300, fr)
    got = Froxelizer(v, t).run(fr, dims, FroxelizeConfig(supersample=ss, mode="ortho", depth_mode=depth)).cpu().numpy()
    ref = ofz.froxelize_ortho(v, t, fr._o, fr._basis, fr.half_extent, fr.near, fr.far, dims, ss, depth)
    diff = int(np.unpackbits(got ^ ref).sum())
    assert np.unpackbits(ref).sum() > 0
    if depth == "linear":
        assert diff == 0, diff
    else:
        assert diff <= 4, diff


def _boxes(seed, n, frustum):
    """Axis-aligned boxes (12 triangles each): faces edge-on in two of the
    three ortho passes (zero-area, dropped by the degeneracy test) and
    edges on lattice lines."""
    rng = np.random.default_rng(seed)
    corners = np.array([[x, y, z] for z in (0, 1) for y in (0, 1) for x in (0, 1)], dtype=np.float64)
    faces = np.array([[0, 1, 3], [0, 3, 2], [4, 6, 7], [4, 7, 5], [0, 4, 5], [0, 5, 1],
                      [2, 3, 7], [2, 7, 6], [0, 2, 6], [0, 6, 4], [1, 5, 7], [1, 7, 3]])
    vs, ts = [], []
    for k in range(n):
        lo = frustum._o + 8.0 * frustum._basis[2] + rng.uniform(-5, 5, size=3)
        vs.append(lo + corners * rng.uniform(0.2, 3.0, size=3))
        ts.append(faces + 8 * k)
    return np.concatenate(vs), np.concatenate(ts)


@pytest.mark.parametrize("seed,dims,ss", [(0, (8, 8, 8), 1), (1, (32, 32, 32), 2), (2, (16, 40, 24), 3)])
def test_axis_aligned_boxes_vs_oracle(seed, dims, ss):
    from paper_2509_24677_b200.froxelize import FroxelizeConfig, Froxelizer
    fr = _random_frustum(200 + seed)
    v, t = _boxes(seed, 60, fr)
    fz = Froxelizer(v, t)
    for mode, fn in (("ortho", ofz.froxelize_ortho), ("perspective", ofz.froxelize)):
        got = fz.run(fr, dims, FroxelizeConfig(supersample=ss, mode=mode)).cpu().numpy()
        ref = fn(v, t, fr._o, fr._basis, fr.half_extent, fr.near, fr.far, dims, ss)
        assert np.unpackbits(ref).sum() > 0, mode
        assert np.array_equal(got, ref), (mode, int(np.unpackbits(got ^ ref).sum()))


def test_ortho_drop_in_and_graph_replay():
    """froxelize(..., FroxelizeConfig(mode="ortho")) and a captured replay give the golden grid."""
    import torch
    from types import SimpleNamespace
    from paper_2509_24677_b200.froxelize import FroxelizeConfig, Froxelizer, froxelize
    c = next(c for c in CASES if str(c["name"]) == "ortho_scene1")
    scene = SimpleNamespace(vertices=c["verts"], triangles=c["tris"])
    ref_frustum = SimpleNamespace(_o=c["origin"], _basis=c["basis"], half_extent=float(c["lens"][0]),
                                  near=float(c["lens"][1]), far=float(c["lens"][2]))
    dims = tuple(int(v) for v in c["dims"])
    cfg = FroxelizeConfig(supersample=int(c["ss"]), mode="ortho")
    grid = froxelize(scene, ref_frustum, dims, cfg)
    assert np.array_equal(grid.bits, c["bits"])
    fz = Froxelizer(c["verts"], c["tris"])
    out = torch.zeros(int(np.prod(dims)) // 8, dtype=torch.uint8, device="cuda")
    fz.run(_frustum(c), dims, cfg, out=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            fz.run(_frustum(c), dims, cfg, out=out)
    out.fill_(0)
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), c["bits"])


_ALT_CHECK = r"""
import os, sys, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2509_24677_b200.froxelize import FroxelizeConfig, Froxelizer, Frustum
g = np.load("tests/golden/froxelize.npz")
bad = 0
for i in range(int(g["ncases"])):
    c = {k[len(f"c{i}_"):]: g[k] for k in g.files if k.startswith(f"c{i}_")}
    if int(c["depth"]) != 0:
        continue
    h, n, f = (float(v) for v in c["lens"])
    got = Froxelizer(c["verts"], c["tris"]).run(Frustum(c["origin"], c["basis"], h, n, f),
        tuple(int(v) for v in c["dims"]), FroxelizeConfig(supersample=int(c["ss"]),
        mode="ortho" if int(c.get("mode", 0)) == 1 else "perspective")).cpu().numpy()
    bad += int(np.unpackbits(got ^ c["bits"]).sum())
print("BAD", bad)
"""


@pytest.mark.parametrize("env", [{"FPVS_FROX_SPANS": "0"}, {"FPVS_FROX_EXACT": "1"}, {"FPVS_FROX_SEG": "8"},
                                 {"FPVS_FROX_SEG": "256"}])
def test_alternative_raster_paths_match_golden(env):
    """The whole-box raster, the exact-only evaluation and other span segment
    widths (env switches read once per process, hence the subprocess)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _ALT_CHECK], cwd=root, env={**os.environ, **env},
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "BAD 0" in r.stdout, r.stdout
