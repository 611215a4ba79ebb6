"""numpy restatement of the NeuralPVS hot path (float64; test infrastructure).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU legs (cpu_baseline, --impl reference) as the checker / CPU
baseline — never by the product package, which has no CPU fallback.

Submanifold ("masked") semantics: a layer's output exists only on the active
cells of its input set and inactive cells read as zero.
shows this equals ``where(active, Conv3d.forward(h), 0)`` of the reference
dense layer (pkg/src/froxelpvs/neural.py:201-219) applied layer by layer;
``tests/test_oracle.py`` checks that identity against the reference itself.

Conventions followed from the reference
* interleave channel ``k = lx + d*(ly + d*lz)`` (interleave.py:54-65);
* conv weight rows ``((a*k + b)*k + c)*Cin + ci`` (neural.py:163-166), tap
  (a, b, c) reads ``x[p + (a-1, b-1, c-1)]`` (neural.py:187-199) — so kernel
  offset ``j = 9a + 3b + c`` is z-fastest;
* relu backward uses ``z > 0`` (neural.py:227-228), sigmoid' = y(1-y)
  (neural.py:229-230);
* loss algebra of neural.py:130-144, 353-399.

Pinned here (not in the reference): canonical kernel maps, k2s2 down/up convs,
the U-Net of BASELINE config 2, Kaiming-uniform init, bf16 emulation.
"""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# numerics helpers
# ---------------------------------------------------------------------------


def bf16_round(x) -> np.ndarray:
    """Round to the nearest bf16 (ties to even); returns float64 values."""
    f = np.ascontiguousarray(np.asarray(x, np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def sigmoid(z: np.ndarray) -> np.ndarray:
    """Split-branch stable sigmoid (neural.py:151-157)."""
    z = np.asarray(z, np.float64)
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


# ---------------------------------------------------------------------------
# interleave (interleave.py:54-85)
# ---------------------------------------------------------------------------


def interleave(dense: np.ndarray, d: int) -> np.ndarray:
    """(Nx,Ny,Nz) -> (Nx/d,Ny/d,Nz/d,d^3), channel k = lx + d*(ly + d*lz)."""
    nx, ny, nz = dense.shape
    if d < 1 or nx % d or ny % d or nz % d:
        raise ValueError("interleave factor must divide grid dims")
    b = dense.reshape(nx // d, d, ny // d, d, nz // d, d)
    return np.ascontiguousarray(b.transpose(0, 2, 4, 5, 3, 1).reshape(nx // d, ny // d, nz // d, d ** 3))


def deinterleave(cells: np.ndarray, d: int) -> np.ndarray:
    """(X,Y,Z,d^3) -> (X*d, Y*d, Z*d), the exact inverse index map."""
    bx, by, bz, c = cells.shape
    if c != d ** 3:
        raise ValueError("channel count does not match d^3")
    t = cells.reshape(bx, by, bz, d, d, d).transpose(0, 5, 1, 4, 2, 3)
    return np.ascontiguousarray(t.reshape(bx * d, by * d, bz * d))


# ---------------------------------------------------------------------------
# kernel maps (row KM); coords are (b, x, y, z) int64 rows
# ---------------------------------------------------------------------------

SUBM_OFFSETS = np.array([(a - 1, b - 1, c - 1) for a in range(3) for b in range(3) for c in range(3)],
                        np.int64)                      # j = 9a + 3b + c
DOWN_OFFSETS = np.array([(a, b, c) for a in range(2) for b in range(2) for c in range(2)],
                        np.int64)                      # j = 4a + 2b + c


def active_coords(cells: np.ndarray) -> np.ndarray:
    """Active cells of a (B,X,Y,Z,C) tensor in C-order: any nonzero channel."""
    act = np.any(cells != 0, axis=-1)
    return np.argwhere(act).astype(np.int64)


def _lin(coords, dims):
    b, x, y, z = coords.T
    X, Y, Z = dims
    return ((b * X + x) * Y + y) * Z + z


def lookup(coords_q, coords_set, dims) -> np.ndarray:
    """Row of each query coordinate in ``coords_set`` (C-order sorted) or -1."""
    X, Y, Z = dims
    ok = ((coords_q[:, 1] >= 0) & (coords_q[:, 1] < X) & (coords_q[:, 2] >= 0) & (coords_q[:, 2] < Y)
          & (coords_q[:, 3] >= 0) & (coords_q[:, 3] < Z))
    keys = _lin(coords_set, dims)
    q = _lin(np.where(ok[:, None], coords_q, 0), dims)
    pos = np.searchsorted(keys, q)
    pos_c = np.minimum(pos, len(keys) - 1) if len(keys) else pos
    hit = ok & (len(keys) > 0) & (keys[pos_c] == q) if len(keys) else np.zeros(len(q), bool)
    return np.where(hit, pos_c, -1).astype(np.int64)


def subm_offsets(k: int) -> np.ndarray:
    """Tap offsets of an odd k^3 kernel, j = (a*k + b)*k + c -> (a-p, b-p, c-p), p = k//2
    (the im2col order of neural.py:187-199)."""
    p = k // 2
    return np.array([(a - p, b - p, c - p) for a in range(k) for b in range(k) for c in range(k)], np.int64)


def kmap_subm(coords: np.ndarray, dims, k: int = 3) -> np.ndarray:
    """nbr[i, j] = row of coords[i] + o_j, or -1 (o_j z-fastest, j = 9a+3b+c for k = 3)."""
    a = len(coords)
    offs = SUBM_OFFSETS if k == 3 else subm_offsets(k)
    nbr = np.empty((a, len(offs)), np.int64)
    for j, o in enumerate(offs):
        q = coords.copy()
        q[:, 1:] += o
        nbr[:, j] = lookup(q, coords, dims)
    return nbr


def coarsen(coords: np.ndarray) -> np.ndarray:
    """Parent active set of a k2s2 down-conv: unique (b, x>>1, y>>1, z>>1), C-order."""
    par = coords.copy()
    par[:, 1:] >>= 1
    return np.unique(par, axis=0) if len(par) else par


def kmap_down(fine: np.ndarray, fine_dims, coarse: np.ndarray) -> np.ndarray:
    """down[p, j] = fine row of child 2*parent + (a,b,c), j = 4a+2b+c, or -1."""
    out = np.empty((len(coarse), 8), np.int64)
    for j, o in enumerate(DOWN_OFFSETS):
        q = coarse.copy()
        q[:, 1:] = 2 * q[:, 1:] + o
        out[:, j] = lookup(q, fine, fine_dims)
    return out


def kmap_up(fine: np.ndarray, coarse: np.ndarray, coarse_dims):
    """(parent row, parity j) of every fine cell; the transpose of kmap_down."""
    par = fine.copy()
    par[:, 1:] >>= 1
    rows = lookup(par, coarse, coarse_dims)
    j = 4 * (fine[:, 1] & 1) + 2 * (fine[:, 2] & 1) + (fine[:, 3] & 1)
    return rows, j


def pair_lists(nbr: np.ndarray):
    """Per-offset (in_row, out_row) lists, sorted by out_row, and offsets.

    pairs for offset j are all (nbr[i, j], i) with nbr[i, j] >= 0; ``pair_off``
    is the exclusive prefix over j (row KM).
    """
    ins, outs, off = [], [], [0]
    for j in range(nbr.shape[1]):
        i = np.nonzero(nbr[:, j] >= 0)[0]
        ins.append(nbr[i, j])
        outs.append(i)
        off.append(off[-1] + len(i))
    return np.concatenate(ins), np.concatenate(outs), np.array(off, np.int64)


# ---------------------------------------------------------------------------
# sparse convs (gather-GEMM-scatter restatement of neural.py:187-219)
# ---------------------------------------------------------------------------


def _act(z, act):
    if act == "relu":
        return np.maximum(z, 0.0)
    if act == "sigmoid":
        return sigmoid(z)
    return z


def gather_conv(x: np.ndarray, nbr: np.ndarray, w: np.ndarray, b: np.ndarray) -> np.ndarray:
    """z[i] = b + sum_j x[nbr[i,j]] @ W_j with W_j = w[j*Cin:(j+1)*Cin] (neural.py:208)."""
    cin = x.shape[1]
    z = np.broadcast_to(np.asarray(b, np.float64), (nbr.shape[0], w.shape[1])).copy()
    for j in range(nbr.shape[1]):
        m = nbr[:, j] >= 0
        if m.any():
            z[m] += x[nbr[m, j]] @ w[j * cin:(j + 1) * cin]
    return z


def up_conv(x_coarse: np.ndarray, parent: np.ndarray, parity: np.ndarray, w: np.ndarray, b) -> np.ndarray:
    """Transposed k2s2: z[child] = b + x[parent] @ W_parity."""
    cin = x_coarse.shape[1]
    z = np.broadcast_to(np.asarray(b, np.float64), (len(parent), w.shape[1])).copy()
    for j in range(8):
        m = parity == j
        if m.any():
            z[m] += x_coarse[parent[m]] @ w[j * cin:(j + 1) * cin]
    return z


# ---------------------------------------------------------------------------
# init (row INIT)
# ---------------------------------------------------------------------------


def kaiming_uniform(rng: np.random.Generator, taps: int, cin: int, cout: int, act: str):
    """U(+-sqrt(3*gain/fan_in)), fan_in = taps*Cin, gain 2 for relu else 1; bias 0.

    Follows the reference's He-normal rule (neural.py:168-176) with the
    uniform distribution BASELINE.json asks for, drawn in (taps*Cin, Cout) order.
    """
    fan_in = taps * cin
    bound = np.sqrt(3.0 * (2.0 if act == "relu" else 1.0) / fan_in)
    return rng.uniform(-bound, bound, size=(fan_in, cout)), np.zeros(cout)


# ---------------------------------------------------------------------------
# networks
# ---------------------------------------------------------------------------


def chain_forward(cells: np.ndarray, layers, bf16: bool = False, return_logits: bool = False):
    """Linear stack of submanifold convs over a (B,X,Y,Z,C) interleaved tensor.

    ``layers`` = list of (kernel, w, b, act).  Returns (coords, out rows) where
    the last layer's sigmoid probabilities (or logits) are per active cell.
    Inactive cells are p = 0 by definition.
    """
    dims = cells.shape[1:4]
    coords = active_coords(cells)
    x = cells[tuple(coords.T)].astype(np.float64)
    tabs = {k: kmap_subm(coords, dims, k) for k in {layer[0] for layer in layers}}
    rnd = bf16_round if bf16 else (lambda v: v)
    x = rnd(x)
    for li, (k, w, b, act) in enumerate(layers):
        w = rnd(w)
        z = gather_conv(x, tabs[k], w, b)
        if li == len(layers) - 1:
            return coords, (z if return_logits else _act(z, act))
        x = rnd(_act(z, act))
    raise ValueError("empty layer list")


def unet_init(seed: int, widths=(64, 128, 256), d3: int = 64):
    """Kaiming-uniform U-Net parameters from Generator(PCG64(seed)), layer order."""
    rng = np.random.Generator(np.random.PCG64(seed))
    params = {}
    for name, kind, cin, cout in unet_layer_table(widths, d3):
        taps = {"subm": 27, "down": 8, "up": 8, "head": 1}[kind]
        params[name] = kaiming_uniform(rng, taps, cin, cout, "sigmoid" if kind == "head" else "relu")
    return params


def unet_layer_table(widths=(64, 128, 256), d3: int = 64):
    c0, c1, c2 = widths
    return (("enc0a", "subm", d3, c0), ("enc0b", "subm", c0, c0), ("down01", "down", c0, c1),
            ("enc1a", "subm", c1, c1), ("enc1b", "subm", c1, c1), ("down12", "down", c1, c2),
            ("enc2a", "subm", c2, c2), ("enc2b", "subm", c2, c2), ("up21", "up", c2, c1),
            ("dec1a", "subm", 2 * c1, c1), ("dec1b", "subm", c1, c1), ("up10", "up", c1, c0),
            ("dec0a", "subm", 2 * c0, c0), ("dec0b", "subm", c0, c0), ("head", "head", c0, d3))


def unet_forward(cells: np.ndarray, params, bf16: bool = True, return_logits: bool = False,
                 widths=(64, 128, 256)):
    """3-level sparse U-Net (row UNET) over (B,X,Y,Z,C) cells.

    Returns (coords0, out rows on the level-0 active set).  bf16=True rounds
    weights and every stored activation to bf16 and accumulates in float64,
    emulating a bf16-in / fp32-accumulate device path.
    """
    rnd = bf16_round if bf16 else (lambda v: v)
    d0 = cells.shape[1:4]
    c0 = active_coords(cells)
    c1 = coarsen(c0)
    c2 = coarsen(c1)
    d1 = tuple(v // 2 for v in d0)
    d2 = tuple(v // 2 for v in d1)
    n0, n1, n2 = kmap_subm(c0, d0), kmap_subm(c1, d1), kmap_subm(c2, d2)
    dn01, dn12 = kmap_down(c0, d0, c1), kmap_down(c1, d1, c2)
    up10, up21 = kmap_up(c0, c1, d1), kmap_up(c1, c2, d2)

    def conv(name, x, nbr):
        w, b = params[name]
        return rnd(np.maximum(gather_conv(x, nbr, rnd(w), b), 0.0))

    def upc(name, x, up):
        w, b = params[name]
        return rnd(np.maximum(up_conv(x, up[0], up[1], rnd(w), b), 0.0))

    x = rnd(cells[tuple(c0.T)].astype(np.float64))
    e0 = conv("enc0b", conv("enc0a", x, n0), n0)
    h = conv("down01", e0, dn01)
    e1 = conv("enc1b", conv("enc1a", h, n1), n1)
    h = conv("down12", e1, dn12)
    h = conv("enc2b", conv("enc2a", h, n2), n2)
    u1 = upc("up21", h, up21)
    h = conv("dec1b", conv("dec1a", np.concatenate([e1, u1], 1), n1), n1)
    u0 = upc("up10", h, up10)
    h = conv("dec0b", conv("dec0a", np.concatenate([e0, u0], 1), n0), n0)
    w, b = params["head"]
    z = rnd(h) @ rnd(w) + b
    return c0, (z if return_logits else sigmoid(z))


def scatter_cells(coords, rows, dims_bxyz, fill=0.0) -> np.ndarray:
    """Dense (B,X,Y,Z,C) from per-active-cell rows; inactive cells = fill."""
    out = np.full(tuple(dims_bxyz) + (rows.shape[1],), fill, np.float64)
    out[tuple(coords.T)] = rows
    return out


def predict_bits(cells_prob: np.ndarray, d: int, tau: float) -> np.ndarray:
    """Deinterleave + threshold ``>= tau`` (interleave.py:85) of one (X,Y,Z,d^3) grid."""
    return deinterleave(cells_prob, d) >= tau


# ---------------------------------------------------------------------------
# losses (neural.py:130-144, 353-399)
# ---------------------------------------------------------------------------


def counts(pred, gt):
    tp = float((pred * gt).sum())
    fp = float((pred * (1.0 - gt)).sum())
    fn = float(((1.0 - pred) * gt).sum())
    return tp, fp, fn, float(gt.sum())


def dice_loss(pred, gt, alpha):
    tp, fp, fn, _ = counts(pred, gt)
    num = 2.0 * tp
    den = 2.0 * tp + alpha * fp + (1.0 - alpha) * fn
    if den == 0.0:
        return 0.0, np.zeros_like(pred, dtype=np.float64)
    dden = 2.0 * gt + alpha * (1.0 - gt) - (1.0 - alpha) * gt
    return (den - num) / den, -(2.0 * gt * den - num * dden) / (den * den)


def rvl_loss(pred, gt):
    tp, fp, _, gtp = counts(pred, gt)
    if gtp == 0.0:
        return 0.0, np.zeros_like(pred, dtype=np.float64)
    return (1.0 - tp / gtp) + fp / gtp, (1.0 - 2.0 * gt) / gtp


def combined_loss(pred, gt, alpha=0.1, lam=0.99):
    dv, dg = dice_loss(pred, gt, alpha)
    rv, rg = rvl_loss(pred, gt)
    return lam * dv + (1.0 - lam) * rv, lam * dg + (1.0 - lam) * rg


# ---------------------------------------------------------------------------
# backward of the sparse chain (restates neural.py:221-249 on the active set)
# ---------------------------------------------------------------------------


def chain_forward_cached(x0, nbr, layers, tables=None):
    """``nbr`` is the k = 3 table; ``tables`` maps other kernel sizes to their k^3 tables."""
    centre = np.arange(len(x0))[:, None]
    caches, x = [], x0
    for k, w, b, act in layers:
        tab = nbr if k == 3 else centre if k == 1 else tables[k]
        z = gather_conv(x, tab, w, b)
        y = _act(z, act)
        caches.append((x, tab, z, y))
        x = y
    return x, caches


def chain_backward(dy, layers, caches):
    """Per-layer (dw, db) and dx on the active set.

    dgrad uses mirrored offsets: dx[n] += dz[i] @ W_j^T for every pair
    (n = nbr[i, j], i), exactly the col2im of neural.py:240-248 restricted to
    active cells.
    """
    grads = [None] * len(layers)
    for li in reversed(range(len(layers))):
        k, w, b, act = layers[li]
        x, tab, z, y = caches[li]
        if act == "relu":
            dz = dy * (z > 0)
        elif act == "sigmoid":
            dz = dy * y * (1.0 - y)
        else:
            dz = dy
        cin = x.shape[1]
        dw = np.zeros_like(w)
        dx = np.zeros_like(x)
        for j in range(tab.shape[1]):
            m = tab[:, j] >= 0
            src = tab[m, j]
            dw[j * cin:(j + 1) * cin] += x[src].T @ dz[m]
            np.add.at(dx, src, dz[m] @ w[j * cin:(j + 1) * cin].T)
        grads[li] = (dw, dz.sum(0))
        dy = dx
    return grads, dy


def chain_train_step_bf16(cells, gts, layers, alpha=0.1, lam=0.99):
    """bf16-emulating restatement of the device's bf16 training step
    (TrainStep with the tcgen05 backward, BASELINE config 5).

    Rounding points follow the device: weights and every stored activation are
    RNE-rounded to bf16; products accumulate exactly here (float64; the device
    accumulates in fp32 in TMEM); the head's logits and probabilities stay
    unrounded; dL/dlogit (the per-sample combined loss of neural.py:353-399
    times sigmoid', over the batch size) is rounded to bf16 before the
    backward; each lower layer's dz is rounded to bf16 after the relu' mask
    (the dgrad epilogue, z > 0 <=> the kept bf16 output > 0, neural.py:227-228);
    dW and db accumulate exactly from those bf16 operands.
    Returns (batch-mean loss, [(dw, db)] per layer, coords, probs)."""
    dims = cells.shape[1:4]
    B = cells.shape[0]
    coords = active_coords(cells)
    x = cells[tuple(coords.T)].astype(np.float64)
    tabs = {k: (np.arange(len(coords))[:, None] if k == 1 else kmap_subm(coords, dims, k))
            for k in {layer[0] for layer in layers}}
    wb = [bf16_round(w) for _, w, _, _ in layers]
    acts = [bf16_round(x)]
    for (k, _, b, act), w in zip(layers[:-1], wb[:-1]):
        acts.append(bf16_round(_act(gather_conv(acts[-1], tabs[k], w, b), act)))
    kh, _, bh, _ = layers[-1]
    probs = sigmoid(gather_conv(acts[-1], tabs[kh], wb[-1], bh))
    loss, dp = 0.0, np.zeros_like(probs)
    for bi in range(B):
        rows = coords[:, 0] == bi
        pd = np.zeros(dims + (probs.shape[1],))
        pd[tuple(coords[rows, 1:].T)] = probs[rows]
        lv, lg = combined_loss(pd, gts[bi], alpha, lam)
        loss += lv
        dp[rows] = lg[tuple(coords[rows, 1:].T)] / B
    dz = bf16_round(dp * probs * (1.0 - probs))
    grads = [None] * len(layers)
    for li in reversed(range(len(layers))):
        k = layers[li][0]
        tab, xin = tabs[k], acts[li]
        cin = xin.shape[1]
        dw = np.zeros_like(wb[li])
        dx = np.zeros_like(xin)
        for j in range(tab.shape[1]):
            m = tab[:, j] >= 0
            src = tab[m, j]
            dw[j * cin:(j + 1) * cin] += xin[src].T @ dz[m]
            if li > 0:
                np.add.at(dx, src, dz[m] @ wb[li][j * cin:(j + 1) * cin].T)
        grads[li] = (dw, dz.sum(0))
        if li > 0:
            dz = bf16_round(dx * (xin > 0))
    return loss / B, grads, coords, probs
