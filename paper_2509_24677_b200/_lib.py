"""ctypes binding of libfpvs.so (include/fpvs.h) — the only way into the kernels.

There is no CPU fallback: importing a compute entry point without the built
library, or calling it without a CUDA device, raises.  Status codes map to
the reference's exceptions: FPVS_EINVAL / FPVS_ESHAPE -> ValueError (as
pkg/src/froxelpvs/interleave.py:58-59, neural.py:203-205 raise), FPVS_ECUDA
-> RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FPVS_LIB", os.path.join(HERE, "libfpvs.so"))

F32, BF16, F64 = 0, 1, 2
IN_PACKED, IN_U8, IN_F32, IN_F64 = 0, 1, 2, 3
EXCHANGE_TAIL = 10  # FPVS_EXCHANGE_TAIL
ACT = {"none": 0, "relu": 1, "sigmoid": 2}
TABLES_SETTLED = 0x100  # FPVS_TABLES_SETTLED (fpvs_spconv_halo act flag)

_i, _f, _d, _p, _z = C.c_int, C.c_float, C.c_double, C.c_void_p, C.c_size_t

# name -> (restype, argtypes); mirrors include/fpvs.h one to one
SIGNATURES = {
    "fpvs_last_error": (C.c_char_p, []),
    "fpvs_abi_version": (_i, []),
    "fpvs_interleave": (_i, [_p, _i, _i, _i, _i, _i, _i, _p, _i, _p, _p]),
    "fpvs_deinterleave": (_i, [_p, _i, _i, _i, _i, _i, _i, _d, _p, _p]),
    "fpvs_kmap_workspace_size": (_z, [_i, _i, _i, _i]),
    "fpvs_cell_active_from_bits": (_i, [_p, _i, _i, _i, _i, _i, _p, _p]),
    "fpvs_kmap_compact": (_i, [_p, _i, _i, _i, _i, _p, _p, _p, _i, _p, _z, _p]),
    "fpvs_kmap_subm": (_i, [_p, _p, _i, _p, _i, _i, _i, _i, _p, _p]),
    "fpvs_kmap_subm_k": (_i, [_p, _p, _i, _p, _i, _i, _i, _i, _i, _p, _p]),
    "fpvs_kmap_coarsen": (_i, [_p, _p, _i, _i, _i, _i, _i, _p, _p]),
    "fpvs_kmap_down": (_i, [_p, _p, _i, _p, _i, _i, _i, _i, _p, _p]),
    "fpvs_kmap_up": (_i, [_p, _p, _i, _p, _i, _i, _i, _i, _p, _p]),
    "fpvs_kmap_tile_masks": (_i, [_p, _i, _p, _i, _p, _p]),
    "fpvs_levels_workspace_size": (_z, [_i, _i, _i, _i, _i, _i]),
    "fpvs_levels_from_bits": (_i, [_p, _i, _i, _i, _i, _i, _i, _p, _p, _z, _p, _i, _i, _p, _z, _p]),
    "fpvs_hash_build": (_i, [_p, _p, _i, _i, _i, _i, _i, _p, _p, _i, _p]),
    "fpvs_kmap_subm_hash": (_i, [_p, _p, _i, _p, _p, _i, _i, _i, _i, _i, _p, _p]),
    "fpvs_gather_cells_bits": (_i, [_p, _i, _i, _i, _i, _i, _p, _p, _i, _p, _i, _i, _p]),
    "fpvs_spconv_simt": (_i, [_p, _i, _i, _p, _i, _p, _i, _p, _p, _i, _i, _i, _p, _i, _i, _i, _p]),
    "fpvs_pack_weights_tc_size": (_z, [_i, _i, _i, _i]),
    "fpvs_pack_weights_tc": (_i, [_p, _i, _i, _i, _i, _p, _p]),
    "fpvs_spconv_tc": (_i, [_p, _i, _i, _p, _i, _p, _p, _i, _p, _i, _p, _i, _i, _i, _p, _i, _i, _p]),
    "fpvs_kmap_halo_size": (_z, [_i]),
    "fpvs_kmap_halo": (_i, [_p, _p, _i, _p, _p, _p, _p]),
    "fpvs_kmap_halo_multi": (_i, [_p, _i, _p]),
    "fpvs_spconv_halo_workspace_size": (_z, [_i, _i, _i, _i]),
    "fpvs_spconv_halo": (_i, [_p, _i, _i, _p, _p, _p, _p, _p, _p, _i, _p, _i, _i, _p, _i, _i, _i, _p, _i, _i, _p,
                              _z, _p]),
    "fpvs_spconv_halo_head": (_i, [_p, _i, _i, _p, _p, _p, _p, _p, _p, _i, _p, _p, _i, _p, _z, _p, _p, _f, _p, _i, _p,
                                   _p]),
    "fpvs_spconv_halo_flow": (_i, [_p, _i, _i, _p, _p, _p, _p, _p, _p, _i, _p, _i, _i, _p, _i, _i, _i, _p, _i, _i, _p,
                                   _z, _p, _p, _p]),
    "fpvs_spconv_brick_workspace_size": (_z, [_i, _i, _i, _i, _i, _i, _i]),
    "fpvs_spconv_brick": (_i, [_p, _i, _i, _p, _i, _i, _i, _i, _p, _i, _i, _p, _i, _i, _i, _p, _i, _i, _p, _z,
                               _p]),
    "fpvs_rowbits_to_grid": (_i, [_p, _p, _i, _i, _i, _i, _i, _p, _p]),
    "fpvs_rowbits_to_grid_flow": (_i, [_p, _p, _i, _i, _i, _i, _i, _p, _p, _p]),
    "fpvs_spconv_halo_head_flow": (_i, [_p, _i, _i, _p, _p, _p, _p, _p, _p, _i, _p, _p, _i, _p, _z, _p, _p, _f, _p, _i,
                                        _p, _p, _p]),
    "fpvs_pack_weights_tc_dgrad": (_i, [_p, _i, _i, _i, _i, _p, _p]),
    "fpvs_pack_weights_tc_multi": (_i, [_p, _i, _p]),
    "fpvs_spconv_tc_dgrad": (_i, [_p, _i, _i, _p, _i, _p, _p, _i, _p, _i, _i, _i, _p, _i, _p, _i, _p]),
    "fpvs_wgrad_tc_workspace_size": (_z, [_i, _i, _i, _i]),
    "fpvs_spconv_wgrad_tc": (_i, [_p, _i, _p, _i, _p, _i, _p, _i, _i, _i, _p, _p, _p, _z, _p]),
    "fpvs_cast_bf16": (_i, [_p, C.c_longlong, _p, _p]),
    "fpvs_up_sort_cap": (_i, [_i]),
    "fpvs_up_sort_workspace_size": (_z, [_i]),
    "fpvs_up_sort": (_i, [_p, _p, _i, _p, _p, _p, _p, _p, _z, _p]),
    "fpvs_up_sort_multi": (_i, [_p, _i, _p]),
    "fpvs_spconv_tc_scatter": (_i, [_p, _i, _i, _p, _i, _p, _p, _i, _p, _p, _i, _p, _i, _i, _i, _p, _i, _i, _p]),
    "fpvs_spconv_tc_flow": (_i, [_p, _i, _i, _p, _i, _p, _p, _i, _p, _i, _p, _i, _i, _i, _p, _i, _i, _p, _p, _p]),
    "fpvs_spconv_tc_upblocks": (_i, [_p, _i, _i, _p, _i, _p, _i, _p, _i, _i, _i, _p, _p, _i, _i, _p]),
    "fpvs_head_simt": (_i, [_p, _i, _i, _p, _p, _i, _p, _p, _i, _i, _i, _i, _i, _i, _f, _p, _p, _p, _p]),
    "fpvs_head_tc": (_i, [_p, _i, _i, _p, _p, _i, _p, _p, _i, _i, _i, _i, _i, _i, _f, _p, _p, _p, _p]),
    "fpvs_loss_sums_size": (_z, [_i, _i]),
    "fpvs_loss_counts": (_i, [_p, _i, _p, _p, _i, _p, _i, _i, _i, _i, _i, _p, _p]),
    "fpvs_loss_grad": (_i, [_p, _i, _p, _p, _i, _p, _i, _i, _i, _i, _i, _p, _d, _d, _p, _p, _p]),
    "fpvs_head_rows": (_i, [_p, _i, _p, _p, _i, _i, _i, _i, _i, _i, _f, _p, _p, _p]),
    "fpvs_act_backward": (_i, [_p, _i, _p, _i, _i, _p, _i, _i, _i, _p, _i, _p]),
    "fpvs_spconv_dgrad_simt": (_i, [_p, _i, _p, _i, _p, _i, _p, _i, _i, _p, _i, _i, _p, _i, _p]),
    "fpvs_wgrad_workspace_size": (_z, [_i, _i, _i, _i]),
    "fpvs_spconv_wgrad_simt": (_i, [_p, _i, _i, _p, _i, _p, _i, _p, _i, _i, _i, _p, _p, _p, _z, _p]),
    "fpvs_exchange_pack": (_i, [_p, _z, _f, _p, _p, _i, _p]),
    "fpvs_exchange_accumulate": (_i, [_p, _p, _i, _p]),
    "fpvs_sgd_step": (_i, [_p, _p, _z, _f, _p]),
    "fpvs_adamw_step": (_i, [_p, _p, _p, _p, _z, _f, _f, _f, _f, _f, _i, _p]),
    "fpvs_bits_confusion_workspace_size": (_z, [_i]),
    "fpvs_bits_confusion": (_i, [_p, _p, _i, C.c_longlong, _p, _p, _z, _p]),
    "fpvs_first_hit_labels": (_i, [_p, _i, _i, _i, _i, _i, _p, _p, _p]),
    "fpvs_froxelize_workspace_size": (_z, [C.c_longlong, _i, _i, _i, _i]),
    "fpvs_froxelize": (_i, [_p, C.c_longlong, _p, C.c_longlong, _p, _i, _i, _i, _i, _i, _p, _p, _z, _p]),
    "fpvs_froxelize_samples": (C.c_longlong, [_p, _p]),
    "fpvs_froxelize_ortho_workspace_size": (_z, [C.c_longlong, _i, _i, _i, _i]),
    "fpvs_froxelize_ortho": (_i, [_p, C.c_longlong, _p, C.c_longlong, _p, _i, _i, _i, _i, _i, _p, _p, _z, _p]),
    "fpvs_gt_pvs_workspace_size": (_z, [C.c_longlong, _i, _i, _i, _i]),
    "fpvs_cast_bf16_rows": (_i, [_p, _i, _p, _i, _p, _p]),
    "fpvs_kmap_pairs_workspace_size": (_z, [_i, _i]),
    "fpvs_kmap_pairs": (_i, [_p, _i, _p, _i, _p, _p, _p, C.c_longlong, _p, _z, _p]),
    "fpvs_wgrad_halo_workspace_size": (_z, [_i]),
    "fpvs_spconv_wgrad_halo": (_i, [_p, _i, _p, _i, _p, _p, _i, _p, _p, _p, _i, _i, _p, _p, _p, _z, _p]),
    "fpvs_froxel_cull": (_i, [_p, C.c_longlong, _p, C.c_longlong, _p, _i, _i, _i, _i, _i, _p, _p, _p, _z, _p]),
    "fpvs_froxel_pairs": (_i, [_p, C.c_longlong, _p, C.c_longlong, _p, _i, _i, _i, _i, _i, _p, C.c_longlong, _p, _p,
                               _z, _p]),
    "fpvs_froxel_cull_ortho": (_i, [_p, C.c_longlong, _p, C.c_longlong, _p, _i, _i, _i, _i, _i, _p, _p, _p, _z, _p]),
    "fpvs_froxel_pairs_ortho": (_i, [_p, C.c_longlong, _p, C.c_longlong, _p, _i, _i, _i, _i, _i, _p, C.c_longlong, _p,
                                     _p, _z, _p]),
    "fpvs_render_depth": (_i, [_p, C.c_longlong, _p, C.c_longlong, _p, _p, _i, _i, _i, _p, _p, _p, _z, _p]),
    "fpvs_gt_pvs": (_i, [_p, C.c_longlong, _p, C.c_longlong, _p, _p, _i, _i, _i, _p, _i, _i, _i, _i, _i, _p, _p, _p,
                         _z, _p]),
}



class Level(C.Structure):
    """struct fpvs_level (include/fpvs.h)."""
    _fields_ = [("coords", _p), ("index_vol", _p), ("n", _p), ("cap", _i), ("nbr", _p), ("nbr_masks", _p),
                ("down", _p), ("down_masks", _p), ("up", _p), ("up_masks", _p), ("halo_rows", _p), ("halo_n", _p),
                ("halo_lnbr", _p)]


class PackJob(C.Structure):
    """struct fpvs_pack_job (include/fpvs.h)."""
    _fields_ = [("w", _p), ("K", _i), ("cin", _i), ("cout", _i), ("bn", _i), ("dgrad", _i), ("packed", _p)]


class Frustum(C.Structure):
    """fpvs_frustum (include/fpvs.h)."""
    _fields_ = [("origin", C.c_double * 3), ("basis", C.c_double * 9), ("half_extent", C.c_double),
                ("near_z", C.c_double), ("far_z", C.c_double)]


class HaloJob(C.Structure):
    """struct fpvs_halo_job (include/fpvs.h)."""
    _fields_ = [("nbr", _p), ("n_dev", _p), ("cap", _i), ("halo_rows", _p), ("halo_n", _p), ("lnbr", _p)]


class UpSortJob(C.Structure):
    """struct fpvs_up_sort_job (include/fpvs.h)."""
    _fields_ = [("up", _p), ("n_fine_dev", _p), ("cap_fine", _i), ("sorted_table", _p), ("perm", _p),
                ("masks", _p), ("n_pad_dev", _p), ("workspace", _p), ("workspace_bytes", _z)]


_LIB = None


def load():
    """dlopen libfpvs.so once; raise loudly when it is missing."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libfpvs.so not built at {LIB_PATH}; run python -m paper_2509_24677_b200.build")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


def exported_symbols():
    return list(SIGNATURES)


class FpvsError(RuntimeError):
    pass


def call(name: str, *args):
    """Invoke a status-returning entry point; map status to Python errors."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.fpvs_last_error().decode(errors="replace")
        if rc in (1, 2):
            raise ValueError(msg)
        raise FpvsError(f"{name}: {msg}")
    return rc


def size(name: str, *args) -> int:
    return int(getattr(load(), name)(*args))


# ---- torch plumbing --------------------------------------------------------

def ptr(t) -> int | None:
    """Device pointer of a CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("fpvs kernels take CUDA tensors")
    return t.data_ptr()


def stream_ptr(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2509_24677_b200 runs on a CUDA (sm_100a) device; none is visible")
    load()
