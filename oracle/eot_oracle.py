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


# ------------------------------------------------------------------------------------------
# The block-diagonal stacking strategy (BDS, Sec. 2.4; S:123-131 bds_sinkhorn): the
# pairs' Gibbs kernels K_q = exp(-C_q / eps) placed along the diagonal of ONE sparse matrix
# K_bd, the marginals and scalings stacked vertically, and ONE update sequence
# u = a / (K_bd v), v = b / (K_bd^T u) run on the stacked system (v0 = 1, exactly L iterations);
# pair q's cost is the sum over its block of u_r K_rc C_rc v_c.  Written independently of
# eot_pair_costs (no shared helper beyond the input slicing), so the pins below can compare the
# two.  Denominators are not clamped (the S:62 floor is the per-pair form's; BDS inputs in the
# pins keep every denominator far above it).
# ------------------------------------------------------------------------------------------
def bds_eot_costs(points, offsets, weights, eps, iters, pi, pj, scale) -> np.ndarray:
    import scipy.sparse as sp

    blocks_K, blocks_C, a_parts, b_parts, rows, cols = [], [], [], [], [], []
    for i, j in zip(pi, pj):
        si, ei = int(offsets[i]), int(offsets[i + 1])
        sj, ej = int(offsets[j]), int(offsets[j + 1])
        X = np.asarray(points[si:ei], dtype=np.float64)
        Y = np.asarray(points[sj:ej], dtype=np.float64)
        C = float(scale) * ((X[:, None, :] - Y[None, :, :]) ** 2).sum(-1)
        blocks_C.append(C)
        blocks_K.append(np.exp(-C / float(eps)))
        a_parts.append(np.asarray(weights[si:ei], dtype=np.float64))
        b_parts.append(np.asarray(weights[sj:ej], dtype=np.float64))
        rows.append(ei - si)
        cols.append(ej - sj)
    Kbd = sp.block_diag(blocks_K, format="csr")
    KCbd = sp.block_diag([k * c for k, c in zip(blocks_K, blocks_C)], format="csr")
    a = np.concatenate(a_parts)
    b = np.concatenate(b_parts)
    v = np.ones(b.shape[0])
    u = np.zeros(a.shape[0])
    for _ in range(iters):
        u = a / (Kbd @ v)
        v = b / (Kbd.T @ u)
    per_row = u * (KCbd @ v)                       # u_r sum_c K_rc C_rc v_c, stacked rows
    ends = np.cumsum(rows)
    return np.add.reduceat(per_row, np.concatenate([[0], ends[:-1]])) if len(rows) else np.zeros(0)
