"""fp64 CPU oracle for ASOT-k anchor learning: mini-batch k-means.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu_baseline / ``--impl reference`` legs may import this module; the product path never imports it
and shares no code with it (common module: ``asot_inputs``, draws only).

What it computes ("W is the set of cluster centers and P_o is the clustering operator";
Table 4 P:577 "Mini-batch k-means [sculley2010web]"):
  state: centers C (fp64) and per-center counts v (integers), initial centers and the batch
  draws are seeded inputs (R#30: Forgy initialisation -- K distinct points -- instead of the
  SPEC's k-means++, and the random draws are passed in);
  every iteration t with batch B_t (point indices):
    1. assignment: j*(x) = argmin_j ||x - c_j||^2 over the f32 copy of the centers, with the
       pinned fp64 op order and lowest-index ties of the hot path's mapping (R#8, R#31);
    2. per-center batch sums S_j = sum_{x in B_t, j*(x) = j} x, accumulated in batch order in
       fp64, and counts m_j;
    3. Sculley's per-center learning rate 1/v_j applied to the m_j points one after another is
       the running mean, so c_j <- (v_j c_j + S_j) / (v_j + m_j), v_j <- v_j + m_j (R#31; pinned
       against the point-by-point update in exact rational arithmetic); centers without points
       stay put (no empty-cluster repair in the cited algorithm).
  The final anchors are the f32 copy of C; their cost C_s is the normalised squared Euclidean
  distance (R#7), computed here in fp64.
"""
from __future__ import annotations

import numpy as np

from .asot_oracle import map_assign


def kmeans_minibatch(points: np.ndarray, init_centers: np.ndarray, batch_idx: np.ndarray):
    """points [T, d] f32, init_centers [K, d], batch_idx [iters, b] int64.
    Returns (centers fp64 [K, d], anchors f32 [K, d], counts int64 [K])."""
    X = np.asarray(points)
    C = np.asarray(init_centers, dtype=np.float64).copy()
    K, d = C.shape
    v = np.zeros(K, dtype=np.int64)
    for t in range(batch_idx.shape[0]):
        idx = batch_idx[t]
        anchors32 = C.astype(np.float32)                      # what the assignment reads
        a = map_assign(X[idx], anchors32)                     # step 1 (pinned argmin)
        S = np.zeros((K, d), dtype=np.float64)
        m = np.zeros(K, dtype=np.int64)
        for b in range(idx.shape[0]):                         # step 2, batch order
            j = a[b]
            S[j] = S[j] + X[idx[b]].astype(np.float64)
            m[j] += 1
        for j in range(K):                                    # step 3
            if m[j] > 0:
                vn = v[j] + m[j]
                C[j] = (np.float64(v[j]) * C[j] + S[j]) / np.float64(vn)
                v[j] = vn
    return C, C.astype(np.float32), v


def sculley_pointwise(points, init_centers, batch_idx):
    """Reference form of Sculley's algorithm, one point at a time with eta = 1/v_j, in exact
    rational arithmetic (fractions) -- used only to pin the batched running-mean form."""
    from fractions import Fraction
    X = [[Fraction(float(t)) for t in row] for row in np.asarray(points, dtype=np.float64)]
    C = [[Fraction(float(t)) for t in row] for row in np.asarray(init_centers, dtype=np.float64)]
    K = len(C)
    v = [0] * K
    for t in range(batch_idx.shape[0]):
        snap = [row[:] for row in C]                          # assignment uses the pre-batch centers
        assign = []
        for b in batch_idx[t]:
            x = X[b]
            dist = [sum((x[k] - snap[j][k]) ** 2 for k in range(len(x))) for j in range(K)]
            best = min(range(K), key=lambda j: (dist[j], j))
            assign.append(best)
        for b, j in zip(batch_idx[t], assign):
            v[j] += 1
            eta = Fraction(1, v[j])
            C[j] = [(1 - eta) * C[j][k] + eta * X[b][k] for k in range(len(C[j]))]
    return C, v


def inertia(points: np.ndarray, anchors: np.ndarray) -> float:
    """sum_x min_j ||x - w_j||^2 in fp64 (the k-means objective)."""
    X = np.asarray(points, dtype=np.float64)
    W = np.asarray(anchors, dtype=np.float64)
    D = ((X[:, None, :] - W[None, :, :]) ** 2).sum(-1)
    return float(D.min(axis=1).sum())


def sqeuclid_cost(anchors: np.ndarray, normalize: bool = True) -> np.ndarray:
    """C_s(u, v) = ||w_u - w_v||^2 (/ max) in fp64 from the f32 anchors (R#7)."""
    W = np.asarray(anchors, dtype=np.float64)
    K = W.shape[0]
    C = np.zeros((K, K))
    for u in range(K):
        diff = W[u][None, :] - W
        C[u] = np.sum(diff * diff, axis=1)
    if normalize and C.max() > 0:
        C = C / C.max()
    return C
