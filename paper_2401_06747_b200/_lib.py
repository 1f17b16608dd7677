"""ctypes binding of libsparsepaint_b200.so (include/sparsepaint_b200.h).

The product path has no CPU fallback: if the library or a CUDA device is
missing, every entry point raises immediately.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# SP_B200_LIB overrides the in-tree library (A/B runs of two builds)
LIB_PATH = os.environ.get("SP_B200_LIB") or os.path.join(_HERE, "libsparsepaint_b200.so")

c_int, c_long, c_double, c_void_p = ctypes.c_int, ctypes.c_long, ctypes.c_double, ctypes.c_void_p
P = c_void_p

# name -> argtypes (restype is always int)
_SIGS = {
    "sp_abi_version": [],
    "sp_negated_laplacian": [c_int, P, P, c_int, c_int, c_int, c_double, P],
    "sp_inpaint_matvec": [c_int, P, P, P, c_int, c_int, c_int, c_double, P],
    "sp_sym_matvec": [c_int, P, P, P, c_int, c_int, c_int, c_double, P],
    "sp_sym_rhs": [c_int, P, P, P, c_int, c_int, c_int, c_double, P],
    "sp_ct_apply": [c_int, P, P, P, c_int, c_int, c_int, c_double, P],
    "sp_sym_residual": [c_int, P, P, P, P, P, c_int, c_int, c_int, c_double, P],
    "sp_oras_apply": [c_int, P, P, P, P, c_int, P, c_int, c_int, c_int, c_double, P, c_long,
                      P, c_double, c_int, c_int, c_int, P],
    "sp_restrict_values": [c_int, P, P, c_int, c_int, c_int, P],
    "sp_restrict_mask": [c_int, P, P, P, P, c_int, c_int, c_int, P],
    "sp_prolongate": [c_int, P, P, c_int, c_int, c_int, c_int, c_int, P],
    "sp_jfa_run": [P, P, P, c_long, P, c_int, c_int, c_int, P],
    "sp_jfa_dist2": [P, P, c_long, P, c_int, c_int, P, P],
    "sp_fs_dither": [P, P, c_int, c_int, P],
    "sp_assign_triangles": [P, c_long, P, P, c_int, c_int, P, P],
    "sp_fallback_assign": [P, P, P, P, c_int, c_int, P],
    "sp_reduce_cells": [P, P, c_long, P, P, P, c_int, c_int, P],
    "sp_masked_sym_rhs": [c_int, P, P, P, c_int, c_int, c_int, P],
    "sp_enforce": [c_int, P, P, P, c_int, c_int, c_int, c_int, P],
    "sp_chan_reduce": [c_int, c_int, P, P, P, c_long, c_int, P, P],
    "sp_error_map": [c_int, P, P, P, c_int, c_long, P],
    "sp_error_map_sum": [c_int, P, P, P, c_int, c_long, P, P],
    "sp_hier_create": [P, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int,
                       c_double, c_double, c_int, c_int],
    "sp_hier_destroy": [P],
    "sp_hier_levels": [P, P, P, c_int],
    "sp_hier_use_graphs": [P, c_int],
    "sp_hier_set_mask": [P, P, P, P],
    "sp_hier_level_mask": [P, c_int, P, P],
    "sp_hier_solve": [P, P, P, c_int, c_double, c_int, c_int, P, P],
    "sp_hier_solve_ex": [P, P, c_int, P, P, c_int, c_double, c_int, c_int, P, P],
    "sp_hier_vcycle": [P, P, P, P],
    "sp_hier_solve_tiles": [P, P, P, c_int, c_double, c_int, c_int, P, P, P, P],
    "sp_nccl_unique_id": [P],
    "sp_nccl_comm_create": [P, P, c_int, c_int],
    "sp_nccl_comm_destroy": [P],
    "sp_strip_create": [P, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_int, c_double,
                        c_double, c_int, c_int, c_int, c_int, c_int, P, P, P],
    "sp_strip_destroy": [P],
    "sp_strip_set_mask": [P, P, P, P],
    "sp_strip_solve": [P, P, P, c_int, c_double, c_int, c_int, P, P],
    "sp_strip_levels": [P, P, P, c_int],
    "sp_strip_set_host_transport": [P, P, P, P, P],
    "sp_geo_create": [P, c_int, c_int],
    "sp_geo_destroy": [P],
    "sp_geo_voronoi": [P, P, c_double, P, P, P, P],
    "sp_geo_delaunay": [P, P, P],
    "sp_geo_accumulate": [P, P, c_int, P],
    "sp_geo_corner_keys": [P, c_int, c_int, P, P],
    "sp_geo_wide_threshold": [c_long],
    "sp_geo_keys_copy": [P, P, c_long, P],
    "sp_geo_delaunay_from_keys": [P, P, c_long, P, P],
    "sp_geo_raster_rows": [P, c_int, c_int, P],
    "sp_geo_assign_rows": [P, P, c_int, c_int, c_int, P],
    "sp_geo_reduce_range": [P, P, c_long, c_long, P],
    "sp_geo_set_buckets": [P, P, P, P, c_long, c_long, P],
    "sp_geo_accumulate_mode": [c_int],
    "sp_pdl_from_level": [c_int],
    "sp_geo_select": [P, P, c_long, c_long, P, P],
    "sp_geo_fill_highest_error": [P, P, P, c_long, P],
    "sp_geo_load": [P, P, P, P, c_long, P],
    "sp_stats": [c_int, P],
    "sp_hier_bench": [P, c_int, c_int, P, P, P],
    "sp_cell_index": [P, c_int, c_int, c_long, P, P, P, P],
    "sp_vi_weights": [P, P, P, P, P, P, c_int, c_int, c_long, c_int, P, P],
    "sp_cell_sum": [P, P, P, P, c_long, P, P],
    "sp_vi_step": [c_int, P, P, P, P, P, P, P, P, c_long, c_int, c_int, c_int, c_double, P, P],
    "sp_plane_dot": [c_int, P, P, c_long, c_long, c_int, P, P, P],
    "sp_plane_axpy": [c_int, P, P, P, P, c_double, c_long, c_long, c_int, P, P],
    "sp_gather_tiles": [c_int, P, P, P, c_int, c_int, c_int, c_int, c_int, c_int, P, P],
    "sp_gather_mask_tiles": [P, P, P, c_int, c_int, c_int, c_int, c_int, P, P],
    "sp_ras_scatter": [c_int, P, P, P, P, P, P, P, P, P, c_int, c_int, c_int, c_int, c_int,
                       c_int, P],
    "sp_where_mask": [c_int, P, P, P, c_int, c_int, c_int, P],
    "sp_neighbor_balance": [c_int, P, P, P, P, c_int, c_int, c_int, P],
    "sp_pack_mask_bits": [P, c_int, c_int, P, P],
    "sp_unpack_mask_bits": [P, c_int, c_int, P, P],
    "sp_encode_pnm": [c_int, P, P, c_int, c_int, c_int, c_int, P, P],
    "sp_masked_sym_rhs_tiles": [c_int, P, P, P, c_int, c_int, c_int, c_int, P, P],
    "sp_ct_apply_tiles": [c_int, P, P, P, c_int, c_int, c_int, c_int, P, P],
    "sp_density_map": [P, c_int, c_int, c_int, c_double, P, c_int, P, P, P],
    "sp_init_mask_random": [P, c_int, c_int, c_int, c_long, c_double, P, c_int, P, P, P, P],
    "sp_pcg64_doubles": [P, ctypes.c_longlong, ctypes.c_longlong, P, P],
    "sp_pairwise_sum": [P, ctypes.c_longlong, P, P],
    "sp_oras_variant": [c_int],
    "sp_march_variant": [c_int],
    "sp_ws_variant": [c_int],
    "sp_ws_prefetch": [c_int],
    "sp_ws_stages": [c_int],
    "sp_oras_offbits": [c_int],
    "sp_tile_list": [c_int],
    "sp_fused_bnorm": [c_int],
    "sp_tma_min_pixels": [c_long],
    "sp_jfa_short4": [c_int],
    "sp_blend_packed": [c_int],
    "sp_tile_fused": [c_int],
    "sp_channel_parallel": [c_int],
    "sp_graph_loop": [c_int],
    "sp_hier_residual": [P, c_int, P, P, P],
    "sp_geo_export": [P, P, P, P, P, P, P, P, c_long, P],
}

_lib = None


class SolveReport(ctypes.Structure):
    _fields_ = [("iterations", c_int), ("converged", c_int), ("nres", c_int),
                ("pad", c_int), ("residuals", c_double * 256)]


def load(require_cuda: bool = True):
    """Load the library (no GPU needed just to load); raise loudly if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: run `python -m paper_2401_06747_b200.build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = c_int
        lib.sp_launch_count.restype = ctypes.c_longlong
        lib.sp_launch_count.argtypes = [c_int]
        lib.sp_work_count.restype = ctypes.c_longlong
        lib.sp_work_count.argtypes = [c_int, c_int]
        lib.sp_geo_wide_threshold.restype = c_long
        lib.sp_tma_min_pixels.restype = c_long
        lib.sp_last_error.restype = ctypes.c_char_p
        lib.sp_last_error.argtypes = []
        _lib = lib
    if require_cuda and not torch.cuda.is_available():
        raise RuntimeError("paper_2401_06747_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    return _lib


def exported_symbols():
    return list(_SIGS) + ["sp_last_error", "sp_launch_count", "sp_work_count"]


def call(name, *args):
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.sp_last_error().decode(errors="replace")
        if rc == -3:
            raise ValueError(msg)
        raise RuntimeError(f"{name} failed ({rc}): {msg}")
    return rc


def stream():
    return c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return c_void_p(t.data_ptr())
    if isinstance(t, np.ndarray):
        return t.ctypes.data_as(c_void_p)
    raise TypeError(type(t))


DTYPE_CODE = {torch.float32: 0, torch.float64: 1}
NP_TO_TORCH = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
               np.dtype(np.uint8): torch.uint8, np.dtype(np.int32): torch.int32,
               np.dtype(np.int64): torch.int64}


def dcode(t):
    try:
        return DTYPE_CODE[t.dtype]
    except KeyError:
        raise TypeError(f"unsupported dtype {t.dtype}: float32 or float64") from None


def device():
    return torch.device("cuda", torch.cuda.current_device())


def to_dev(a, dtype=None):
    """numpy / tensor -> contiguous CUDA tensor (optionally cast)."""
    if isinstance(a, torch.Tensor):
        t = a
    else:
        arr = np.ascontiguousarray(a)
        t = torch.from_numpy(arr)
    if dtype is not None and t.dtype != dtype:
        t = t.to(dtype)
    if not t.is_cuda:
        t = t.to(device(), non_blocking=False)
    return t.contiguous()
