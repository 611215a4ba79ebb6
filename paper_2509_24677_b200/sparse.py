"""Sparse active-cell sets and kernel maps on the device (row KM).

A ``Level`` is one resolution of a batch of interleaved grids: the active
cells of a (B, X, Y, Z) cell grid in canonical C-order, the direct-mapped
index volume (row of each cell or -1), the submanifold neighbour table, and —
between levels — the k2s2 down / up tables.  Counts live on the device
(``n``, int32[1]) and every buffer is sized by a host capacity, so building a
frame's maps issues only kernels: no host round trip, CUDA-graph capturable.

The canonical form is the one the oracle pins (oracle/sparse.py): rows in
np.nonzero order, nbr[i][j] for o_j = (a-1, b-1, c-1), j = 9a + 3b + c
(the tap order of pkg/src/froxelpvs/neural.py:187-199).
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import _lib


def _torch():
    import torch
    return torch


@dataclass
class Level:
    B: int
    dims: tuple               # (X, Y, Z) cells
    cap: int
    coords: object = None      # int32 [cap, 4] (b, x, y, z)
    index_vol: object = None   # int32 [B*X*Y*Z]
    n: object = None           # int32 [1] on device
    nbr: object = None         # int32 [cap, 27]
    nbr_masks: object = None   # uint32 [ceil(cap/128)] offsets present per 128-row tile
    active: object = None      # u8 [B*X*Y*Z]
    hash_keys: object = None
    hash_vals: object = None
    extra: dict = field(default_factory=dict)

    @property
    def ncells(self) -> int:
        X, Y, Z = self.dims
        return self.B * X * Y * Z

    def count(self) -> int:
        """Active row count (host sync — for tests and reporting only)."""
        return min(int(self.n.item()), self.cap)


def new_level(B: int, dims, cap: int | None = None, device="cuda") -> Level:
    torch = _torch()
    X, Y, Z = dims
    ncell = B * X * Y * Z
    cap = ncell if cap is None else min(cap, ncell)
    lv = Level(B, (X, Y, Z), cap)
    lv.coords = torch.empty((cap, 4), dtype=torch.int32, device=device)
    lv.index_vol = torch.empty(ncell, dtype=torch.int32, device=device)
    lv.n = torch.zeros(1, dtype=torch.int32, device=device)
    lv.nbr = torch.empty((cap, 27), dtype=torch.int32, device=device)
    lv.active = torch.empty(ncell, dtype=torch.uint8, device=device)
    lv.extra["ws"] = torch.empty(_lib.size("fpvs_kmap_workspace_size", B, X, Y, Z), dtype=torch.uint8,
                                 device=device)
    return lv


def compact(lv: Level, stream=None):
    s = _lib.stream_ptr(stream)
    X, Y, Z = lv.dims
    ws = lv.extra["ws"]
    _lib.call("fpvs_kmap_compact", _lib.ptr(lv.active), lv.B, X, Y, Z, _lib.ptr(lv.coords), _lib.ptr(lv.index_vol),
              _lib.ptr(lv.n), lv.cap, _lib.ptr(ws), ws.numel(), s)


def new_masks(cap: int, device="cuda"):
    torch = _torch()
    return torch.empty(max(1, (cap + 127) // 128), dtype=torch.int32, device=device)


def tile_masks(table, K: int, n, cap: int, out=None, stream=None):
    """Per 128-row tile: bit j set iff any live row has table[row][j] >= 0."""
    if out is None:
        out = new_masks(cap, table.device)
    _lib.call("fpvs_kmap_tile_masks", _lib.ptr(table), K, _lib.ptr(n), cap, _lib.ptr(out), _lib.stream_ptr(stream))
    return out


def build_subm(lv: Level, stream=None):
    X, Y, Z = lv.dims
    _lib.call("fpvs_kmap_subm", _lib.ptr(lv.coords), _lib.ptr(lv.n), lv.cap, _lib.ptr(lv.index_vol), lv.B, X, Y, Z,
              _lib.ptr(lv.nbr), _lib.stream_ptr(stream))
    if lv.nbr_masks is None:
        lv.nbr_masks = new_masks(lv.cap, lv.nbr.device)
    tile_masks(lv.nbr, 27, lv.n, lv.cap, lv.nbr_masks, stream)


HALO_MAX = 512  # FPVS_HALO_MAX


def pair_lists(table, K: int, n, cap: int, stream=None):
    """Per-offset (in_row, out_row) pair lists of a neighbour table, sorted by
    out_row within each offset, and their int64 offsets [K+1] (row KM).
    Returns device tensors (pair_in, pair_out, pair_off); one host sync sizes
    the outputs (the pair count is data-dependent)."""
    torch = _torch()
    dev = table.device
    ws = torch.empty(_lib.size("fpvs_kmap_pairs_workspace_size", K, cap), dtype=torch.uint8, device=dev)
    off = torch.empty(K + 1, dtype=torch.int64, device=dev)
    s = _lib.stream_ptr(stream)
    _lib.call("fpvs_kmap_pairs", _lib.ptr(table), K, _lib.ptr(n), cap, None, None, _lib.ptr(off), 0, _lib.ptr(ws),
              ws.numel(), s)
    total = int(off[K].item())
    pin = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    pout = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    _lib.call("fpvs_kmap_pairs", _lib.ptr(table), K, _lib.ptr(n), cap, _lib.ptr(pin), _lib.ptr(pout), _lib.ptr(off),
              total, _lib.ptr(ws), ws.numel(), s)
    return pin[:total], pout[:total], off


def _halo_tables(lv: Level) -> dict:
    h = lv.extra.get("halo")
    if h is None:
        torch = _torch()
        tiles = max(1, (lv.cap + 127) // 128)
        dev = lv.nbr.device
        h = {"rows": torch.empty((tiles, HALO_MAX), dtype=torch.int32, device=dev),
             "n": torch.zeros(tiles, dtype=torch.int32, device=dev),
             "lnbr": torch.empty((tiles, 128 * 27), dtype=torch.int16, device=dev)}
        lv.extra["halo"] = h
    return h


def build_halo(lv: Level, stream=None) -> dict:
    """Per 128-row tile: distinct neighbour rows of the level's K = 27 table and
    the tile-local table (fpvs_kmap_halo) that the halo-cached conv reads."""
    h = _halo_tables(lv)
    _lib.call("fpvs_kmap_halo", _lib.ptr(lv.nbr), _lib.ptr(lv.n), lv.cap, _lib.ptr(h["rows"]), _lib.ptr(h["n"]),
              _lib.ptr(h["lnbr"]), _lib.stream_ptr(stream))
    return h


class HaloBuilder:
    """Halo tables of several levels in one launch (fpvs_kmap_halo_multi)."""

    def __init__(self, levels):
        import ctypes as C
        self.levels = list(levels)
        arr = (_lib.HaloJob * len(self.levels))()
        for i, lv in enumerate(self.levels):
            h = _halo_tables(lv)
            arr[i].nbr, arr[i].n_dev, arr[i].cap = _lib.ptr(lv.nbr), _lib.ptr(lv.n), lv.cap
            arr[i].halo_rows, arr[i].halo_n, arr[i].lnbr = _lib.ptr(h["rows"]), _lib.ptr(h["n"]), _lib.ptr(h["lnbr"])
        self._arr = arr
        self._ptr = C.addressof(arr)

    def run(self, stream=None):
        _lib.call("fpvs_kmap_halo_multi", self._ptr, len(self.levels), _lib.stream_ptr(stream))


def _up_sorted(fine: Level, up) -> dict:
    u = fine.extra.get("upsort")
    if u is None:
        torch = _torch()
        dev = up.device
        cap_pad = _lib.size("fpvs_up_sort_cap", fine.cap)
        u = {"cap": cap_pad,
             "table": torch.empty((cap_pad, 8), dtype=torch.int32, device=dev),
             "perm": torch.empty(cap_pad, dtype=torch.int32, device=dev),
             "masks": torch.empty(max(1, cap_pad // 128), dtype=torch.int32, device=dev),
             "n": torch.zeros(1, dtype=torch.int32, device=dev),
             "ws": torch.empty(_lib.size("fpvs_up_sort_workspace_size", fine.cap), dtype=torch.uint8, device=dev),
             "up": up}
        fine.extra["upsort"] = u
    return u


class UpSorter:
    """Parity-sorted up tables of several (fine level, up table) pairs
    (fpvs_up_sort_multi): each 128-row tile of the sorted order has one class."""

    def __init__(self, pairs):
        import ctypes as C
        self.pairs = list(pairs)
        arr = (_lib.UpSortJob * len(self.pairs))()
        for i, (fine, up) in enumerate(self.pairs):
            u = _up_sorted(fine, up)
            e = arr[i]
            e.up, e.n_fine_dev, e.cap_fine = _lib.ptr(up), _lib.ptr(fine.n), fine.cap
            e.sorted_table, e.perm, e.masks, e.n_pad_dev = (_lib.ptr(u["table"]), _lib.ptr(u["perm"]),
                                                            _lib.ptr(u["masks"]), _lib.ptr(u["n"]))
            e.workspace, e.workspace_bytes = _lib.ptr(u["ws"]), u["ws"].numel()
        self._arr = arr
        self._ptr = C.addressof(arr)

    def run(self, stream=None):
        _lib.call("fpvs_up_sort_multi", self._ptr, len(self.pairs), _lib.stream_ptr(stream))


def build_subm_hash(lv: Level, hash_capacity: int | None = None, stream=None):
    """Same table through the open-addressing hash instead of the index volume."""
    torch = _torch()
    X, Y, Z = lv.dims
    if hash_capacity is None:
        hash_capacity = 1 << max(4, (2 * lv.cap - 1).bit_length())
    keys = torch.empty(hash_capacity, dtype=torch.int64, device=lv.coords.device)
    vals = torch.empty(hash_capacity, dtype=torch.int32, device=lv.coords.device)
    s = _lib.stream_ptr(stream)
    _lib.call("fpvs_hash_build", _lib.ptr(lv.coords), _lib.ptr(lv.n), lv.cap, lv.B, X, Y, Z, _lib.ptr(keys),
              _lib.ptr(vals), hash_capacity, s)
    nbr = torch.empty((lv.cap, 27), dtype=torch.int32, device=lv.coords.device)
    _lib.call("fpvs_kmap_subm_hash", _lib.ptr(lv.coords), _lib.ptr(lv.n), lv.cap, _lib.ptr(keys), _lib.ptr(vals),
              hash_capacity, lv.B, X, Y, Z, _lib.ptr(nbr), s)
    lv.hash_keys, lv.hash_vals = keys, vals
    return nbr


def fill_level_from_bits(lv: Level, bits, grid_dims, d: int, stream=None, with_nbr: bool = True) -> Level:
    """Level 0 of a batch of packed grids: active cells = blocks with any bit set."""
    nx, ny, nz = grid_dims
    if nx % 8:
        raise ValueError(f"N_x must be divisible by 8, got {nx}")
    if d < 1 or nx % d or ny % d or nz % d:
        raise ValueError(f"grid dims {tuple(grid_dims)} not divisible by interleave factor {d}")
    if lv.dims != (nx // d, ny // d, nz // d):
        raise ValueError("level dims do not match the grid")
    _lib.call("fpvs_cell_active_from_bits", _lib.ptr(bits), lv.B, nx, ny, nz, d, _lib.ptr(lv.active),
              _lib.stream_ptr(stream))
    compact(lv, stream)
    if with_nbr:
        build_subm(lv, stream)
    return lv


def level_from_bits(bits, B: int, grid_dims, d: int, cap: int | None = None, stream=None,
                    with_nbr: bool = True) -> Level:
    nx, ny, nz = grid_dims
    if d < 1 or nx % d or ny % d or nz % d:
        raise ValueError(f"grid dims {tuple(grid_dims)} not divisible by interleave factor {d}")
    lv = new_level(B, (nx // d, ny // d, nz // d), cap, device=bits.device)
    return fill_level_from_bits(lv, bits, grid_dims, d, stream, with_nbr)


def new_coarse(fine: Level, cap: int | None = None):
    """Allocate the next level plus its (down, up) tables."""
    torch = _torch()
    X, Y, Z = fine.dims
    if X % 2 or Y % 2 or Z % 2:
        raise ValueError(f"k2s2 needs even cell dims, got {fine.dims}")
    coarse = new_level(fine.B, (X // 2, Y // 2, Z // 2), cap, device=fine.coords.device)
    down = torch.empty((coarse.cap, 8), dtype=torch.int32, device=fine.coords.device)
    up = torch.empty((fine.cap, 8), dtype=torch.int32, device=fine.coords.device)
    coarse.extra["down_masks"] = new_masks(coarse.cap, fine.coords.device)
    coarse.extra["up_masks"] = new_masks(fine.cap, fine.coords.device)
    return coarse, down, up


def fill_coarse(fine: Level, coarse: Level, down, up, stream=None, with_nbr: bool = True):
    """Active set of a k2s2 down-conv (parents of active cells) and its maps."""
    X, Y, Z = fine.dims
    s = _lib.stream_ptr(stream)
    coarse.active.zero_()
    _lib.call("fpvs_kmap_coarsen", _lib.ptr(fine.coords), _lib.ptr(fine.n), fine.cap, fine.B, X, Y, Z,
              _lib.ptr(coarse.active), s)
    compact(coarse, stream)
    if with_nbr:
        build_subm(coarse, stream)
    _lib.call("fpvs_kmap_down", _lib.ptr(coarse.coords), _lib.ptr(coarse.n), coarse.cap, _lib.ptr(fine.index_vol),
              fine.B, X, Y, Z, _lib.ptr(down), s)
    _lib.call("fpvs_kmap_up", _lib.ptr(fine.coords), _lib.ptr(fine.n), fine.cap, _lib.ptr(coarse.index_vol),
              fine.B, X, Y, Z, _lib.ptr(up), s)
    tile_masks(down, 8, coarse.n, coarse.cap, coarse.extra["down_masks"], stream)
    tile_masks(up, 8, fine.n, fine.cap, coarse.extra["up_masks"], stream)


class LevelMaps:
    """A frame's level hierarchy built by one fused call (fpvs_levels_from_bits).

    ``levels[0]`` comes from the packed bits, ``levels[l]`` (l > 0) is the k2s2
    parent set of ``levels[l-1]`` with ``downs[l-1]`` / ``ups[l-1]`` between
    them (allocated by ``new_coarse``).  Three launches replace the granular
    sequence fill_level_from_bits -> fill_coarse -> ... and produce the same
    tables and tile masks bit for bit.
    """

    def __init__(self, levels, downs, ups, grid_dims, d: int, with_nbr: bool = True, halo_levels=(),
                 with_up: bool = True):
        """``halo_levels``: indices of levels whose halo tables (the halo-cached
        conv's, ``_halo_tables``) are built in the same launch as their maps;
        ``with_up`` False skips the up tables (the column-block up convs,
        fpvs_spconv_tc_upblocks, read the down tables instead)."""
        import ctypes as C
        torch = _torch()
        self.levels, self.grid_dims, self.d = list(levels), tuple(grid_dims), d
        lv0 = self.levels[0]
        nx, ny, nz = self.grid_dims
        nlev = len(self.levels)
        ws = _lib.size("fpvs_levels_workspace_size", lv0.B, nx, ny, nz, d, nlev)
        if ws == 0:
            raise ValueError(f"fused level build does not support grid {self.grid_dims}, d={d}, {nlev} levels")
        self.ws = torch.zeros(ws, dtype=torch.uint8, device=lv0.coords.device)  # must start zeroed
        arr = (_lib.Level * nlev)()
        for i, lv in enumerate(self.levels):
            if with_nbr and lv.nbr_masks is None:
                lv.nbr_masks = new_masks(lv.cap, lv.coords.device)
            e = arr[i]
            e.coords, e.index_vol, e.n, e.cap = _lib.ptr(lv.coords), _lib.ptr(lv.index_vol), _lib.ptr(lv.n), lv.cap
            if with_nbr:
                e.nbr, e.nbr_masks = _lib.ptr(lv.nbr), _lib.ptr(lv.nbr_masks)
            if i > 0:
                e.down, e.down_masks = _lib.ptr(downs[i - 1]), _lib.ptr(lv.extra["down_masks"])
                if with_up:
                    e.up, e.up_masks = _lib.ptr(ups[i - 1]), _lib.ptr(lv.extra["up_masks"])
            if i in halo_levels and with_nbr:
                h = _halo_tables(lv)
                e.halo_rows, e.halo_n, e.halo_lnbr = _lib.ptr(h["rows"]), _lib.ptr(h["n"]), _lib.ptr(h["lnbr"])
        self._arr = arr
        self._arr_ptr = C.addressof(arr)

    def run(self, bits, feat=None, ldf: int = 0, clear=None, stream=None):
        """Build every level; optionally gather level-0 features into ``feat`` and zero ``clear``."""
        nx, ny, nz = self.grid_dims
        lv0 = self.levels[0]
        fdt = 0
        if feat is not None:
            torch = _torch()
            fdt = _lib.BF16 if feat.dtype == torch.bfloat16 else _lib.F32
            ldf = ldf or feat.shape[1]
        _lib.call("fpvs_levels_from_bits", _lib.ptr(bits), lv0.B, nx, ny, nz, self.d, len(self.levels),
                  self._arr_ptr, _lib.ptr(self.ws), self.ws.numel(), _lib.ptr(feat), fdt, ldf,
                  _lib.ptr(clear), 0 if clear is None else clear.numel(), _lib.stream_ptr(stream))


def coarsen(fine: Level, cap: int | None = None, stream=None, with_nbr: bool = True):
    coarse, down, up = new_coarse(fine, cap)
    fill_coarse(fine, coarse, down, up, stream, with_nbr)
    return coarse, down, up


def gather_features(bits, lv: Level, grid_dims, d: int, dtype, ld: int | None = None, out=None, stream=None):
    """Sparse interleave: (cap, ld) features of the active cells straight from packed bits."""
    torch = _torch()
    d3 = d ** 3
    ld = ld or d3
    if out is None:
        out = torch.zeros((lv.cap, ld), dtype=dtype, device=bits.device)
    nx, ny, nz = grid_dims
    dt = _lib.BF16 if dtype == torch.bfloat16 else _lib.F32
    _lib.call("fpvs_gather_cells_bits", _lib.ptr(bits), lv.B, nx, ny, nz, d, _lib.ptr(lv.coords), _lib.ptr(lv.n),
              lv.cap, _lib.ptr(out), ld, dt, _lib.stream_ptr(stream))
    return out
