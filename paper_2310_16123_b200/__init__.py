"""B200-native ASOT pairwise distance matrix (arXiv 2310.16123 hot path).

C ABI: include/asot.h (libasot.so, built in-tree for sm_100a).  Python: asot.py (binding),
distributed.py (multi-GPU tile partition + NCCL gathers).
"""
from .asot import (FP32, TF32, TILE_SLOTS, Workspace, bound_terms, check_status, distance_matrix,  # noqa: F401
                   distance_matrix_host, distance_matrix_partition, sinkhorn_path_kind, exact_w1_points, effective_precision, eot_pairs, exact_asot_pairs, kmeans_minibatch, last_launch_count,
                   mahalanobis_cost, sqeuclid_cost, map_soft_dl, map_soft_ml, map_to_anchors, num_tiles,
                   pairwise_sinkhorn, tile_pairs, unpack_tiles)
