"""ctypes loader for the in-tree libasot.so (C ABI in include/asot.h).

Fails loudly when the library is missing: there is no CPU fallback anywhere in the product
path.  Build it with ``python -c "import __graft_entry__ as g; g.build()"``.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libasot.so")

c_f32p = ctypes.c_void_p  # device / host pointers are passed as integers
c_i64 = ctypes.c_int64
c_i32 = ctypes.c_int32
c_f32 = ctypes.c_float
c_size = ctypes.c_size_t
c_vp = ctypes.c_void_p

# name: (restype, [argtypes])
_SIGS = {
    "asot_abi_version": (c_i32, []),
    "asot_last_error": (ctypes.c_char_p, []),
    "asot_last_launch_count": (c_i32, []),
    "asot_num_tiles": (c_i64, [c_i64]),
    "asot_effective_precision": (c_i32, [c_i32, c_i32]),
    "asot_map_to_anchors": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_i32, c_vp, c_vp,
                                    c_vp, c_vp]),
    "asot_pairwise_sinkhorn": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_f32, c_f32, c_i32, c_i32, c_vp,
                                       c_vp, c_i64, c_vp, c_vp, c_vp, c_size, c_vp]),
    "asot_pairwise_workspace_bytes": (c_size, [c_i64, c_i32, c_i32]),
    "asot_pairwise_list_workspace_bytes": (c_size, [c_i64, c_i32, c_i32, c_i64]),
    "asot_distance_matrix": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_i32, c_vp, c_f32,
                                     c_f32, c_i32, c_i32, c_vp, c_i64, c_i64, c_vp, c_vp, c_vp,
                                     c_vp, c_vp, c_vp, c_size, c_vp]),
    "asot_distance_matrix_workspace_bytes": (c_size, [c_i64, c_i64, c_i32, c_i32]),
    "asot_distance_matrix_host": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_i32, c_vp, c_f32,
                                          c_i32, c_i32, c_vp, c_vp, c_vp, c_size, c_vp]),
    "asot_distance_matrix_host_workspace_bytes": (c_size, [c_i64, c_i64, c_i32, c_i32, c_i32]),
    "asot_unpack_tiles": (c_i32, [c_vp, c_i64, c_i64, c_i64, c_vp, c_i32, c_vp]),
    "asot_tile_pairs_host": (c_i32, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "asot_map_soft_ml": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_i32, c_i32, c_vp, c_vp, c_vp,
                                 c_vp, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "asot_map_soft_ml_workspace_bytes": (c_size, [c_i32, c_i32, c_i32]),
    "asot_sinkhorn_path_kind": (c_i32, [c_i32, c_i32, c_i32]),
    "asot_distance_matrix_partition": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_f32, c_f32, c_i32, c_i32, c_i64,
                                               c_i64, c_vp, c_vp, c_vp, c_size, c_vp]),
    "asot_map_soft_dl": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_i32, c_i32, c_i32, c_vp,
                                 c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_size, c_vp]),
    "asot_map_soft_dl_workspace_bytes": (c_size, [c_i32, c_i32, c_i64]),
    "asot_mahalanobis_cost": (c_i32, [c_vp, c_i32, c_i32, c_vp, c_i32, c_i32, c_vp, c_vp, c_size, c_vp]),
    "asot_mahalanobis_workspace_bytes": (c_size, [c_i32, c_i32]),
    "asot_kmeans_minibatch": (c_i32, [c_vp, c_i64, c_i32, c_i32, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp,
                                      c_vp, c_vp, c_vp]),
    "asot_sqeuclid_cost": (c_i32, [c_vp, c_i32, c_i32, c_i32, c_vp, c_vp]),
    "asot_eot_pairs": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_f32, c_f32, c_i32, c_vp, c_vp,
                               c_i64, c_vp, c_vp, c_vp, c_size, c_vp]),
    "asot_eot_workspace_bytes": (c_size, [c_i64, c_vp, c_i64]),
    "asot_sinkhorn_kernel_kind": (c_i32, [c_i32, c_i32]),
    "asot_exact_asot_pairs": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp,
                                      c_size, c_vp]),
    "asot_exact_asot_workspace_bytes": (c_size, [c_i64, c_i32]),
    "asot_exact_w1_points": (c_i32, [c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "asot_bound_terms": (c_i32, [c_vp, c_vp, c_i64, c_i32, c_vp, c_i32, c_vp, c_vp, c_vp, c_vp, c_i64,
                                 c_vp, c_vp, c_vp, c_vp, c_vp]),
    "asot_map_to_anchors_bcast": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_i32, c_vp, c_vp,
                                          c_vp, c_i32, c_i64, c_vp, c_vp]),
    "asot_map_workspace_bytes": (c_size, [c_i64, c_i32]),
    "asot_map_to_anchors_ws": (c_i32, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_i32, c_vp, c_vp,
                                       c_vp, c_i32, c_i64, c_vp, c_vp, c_size, c_vp]),
    "asot_profile_enable": (c_i32, [c_i32]),
    "asot_profile_read": (c_i32, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(c_i64), c_i32]),
    "asot_profile_clock": (c_i32, [c_i32, ctypes.POINTER(ctypes.c_double)]),
    "asot_profile_read_kernel": (c_i32, [c_i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(c_i64),
                                         c_i32]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libasot.so not found at {LIB_PATH}: the CUDA extension is required (no CPU "
            "fallback). Build it with __graft_entry__.build().")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
