"""fp64 CPU oracle for the NEXT-4 comparison baseline: entropic OT on the ORIGINAL point sets,
one pair at a time (the paper's "eOT" / BDS-eOT comparison systems).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu_baseline / ``--impl reference`` legs may import this module; the product path never imports
it and shares no code with it.

Per pair (i, j): C = s * ||x_r - y_c||^2 over the n_i x n_j point pairs (the same normalised
squared-Euclidean ground cost as the anchors' C_s, with s = 1 / max_{u,v} ||w_u - w_v||^2, so
ASOT and OT values are comparable -- R#32), then the pinned entropic Sinkhorn of asot_oracle
(v0 = 1, exactly L iterations, linear cost <T, C>) with a = w_i, b = w_j.
"""
from __future__ import annotations

import numpy as np

from .asot_oracle import sinkhorn


def sqeuclid_point_cost(X: np.ndarray, Y: np.ndarray, scale: float) -> np.ndarray:
    """C[r, c] = scale * sum_k (x_rk - y_ck)^2 in fp64."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    diff = X[:, None, :] - Y[None, :, :]
    return float(scale) * np.sum(diff * diff, axis=-1)


def eot_pair_costs(points, offsets, weights, eps, iters, pi, pj, scale) -> np.ndarray:
    out = np.empty(len(pi), dtype=np.float64)
    for q, (i, j) in enumerate(zip(pi, pj)):
        si, ei = int(offsets[i]), int(offsets[i + 1])
        sj, ej = int(offsets[j]), int(offsets[j + 1])
        C = sqeuclid_point_cost(points[si:ei], points[sj:ej], scale)
        out[q], _ = sinkhorn(weights[si:ei], weights[sj:ej], C, eps, iters)
    return out
