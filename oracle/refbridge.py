"""Import the real reference package (``froxelpvs``) when it is present.

Only this container has /root/reference; the GPU box does not.  Callers must
treat ``load()`` returning None as "reference unavailable" and fall back to the
committed golden fixtures under tests/golden/.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = os.environ.get("FPVS_REFERENCE_SRC", "/root/reference/pkg/src")


def load():
    """Namespace of ``froxelpvs.{froxel,interleave,neural}`` modules, or None when the reference is absent."""
    if not os.path.isdir(os.path.join(REF_SRC, "froxelpvs")):
        return None
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import importlib
    import types
    mods = {m: importlib.import_module(f"froxelpvs.{m}") for m in ("froxel", "interleave", "neural")}
    return types.SimpleNamespace(**mods)


def masked_reference_forward(neural, net, x, mask):
    """Layer-by-layer reference ``Conv3d.forward`` with inactive cells zeroed.

    This is the reference's own arithmetic (neural.py:201-219) plus the
    submanifold mask of SURVEY.md §8(c)(1); it is the parity anchor for the
    sparse restatement.  Returns (outputs per layer, caches per layer).
    """
    m = mask[..., None].astype(np.float64)
    outs, caches = [], []
    for layer in net.layers:
        y, cache = layer.forward(x, keep_cache=True)
        y = y * m
        outs.append(y)
        caches.append(cache)
        x = y
    return outs, caches

