"""fp64 CPU oracle for the soft / near-one-hot mappings.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu_baseline / ``--impl reference`` legs may import this module.  The product path never
imports it and shares no code with it (the common module is ``asot_inputs``: seeded inputs and
model parameters, none of the method's arithmetic).

Plain numpy in float64, step by step in the paper's order and notation.  ``P:n`` = PAPER.md
line n, ``S:n`` = SPEC.md line n; readings ``R#n`` are listed in DESIGN.md §3.

What the soft mappings compute (inference only -- training needs the paper's datasets and is
out of scope; the parameters are seeded inputs, ``asot_inputs.soft``):

  ASOT-ML (Table 4): P(x) = MLP(x) normalised by its l1 norm, with the MLP
    (d -> 2d -> K) (R#24) and |.| before the normalisation (R#25); the anchor cost is the
    Mahalanobis distance d_AS(w_u, w_v) = ||M w_u - M w_v||_2, M in R^{h x d} (R#19, R#29).
  ASOT-DL (Eqs. (8)(9), appendix, Table 4): L near-one-hot layers
    z <- S_lambda(z - W^T (W z - x)), S_theta(a) = max(0, a - theta), W = [w_1 .. w_k] in
    R^{d x k}, lambda = softplus(MLP(x)) with the MLP (d -> d/2 -> 1) (R#24, R#26), z^(0) = 0
    and a final l1 normalisation onto the simplex (R#27).
  Mapped marginals a' = Z^T a (Eq. (5) P:100 with the 1/n factor dropped, R#1), as a
    segmented sum over each distribution's points.

Parity status: every function is pinned in ``tests/test_soft_oracle_pins.py`` (SPEC worked
examples, closed forms for orthonormal dictionaries, the Eq. (8) minimiser from an independent
bound-constrained solver, objective monotonicity, reduction to the pinned one-hot histograms,
Euclidean special cases of the Mahalanobis cost, the soft Lemma-1 inequality).
"""
from __future__ import annotations

import numpy as np


# ------------------------------------------------------------------------------------------
# MLP forward (Table 4 P:568-569 "(5d, 10d, k)", "(5d, 2.5d, 1)"; hidden activation ReLU, R#24).
# layers = [(W [in, out], b [out]), ...]; ReLU on every layer but the last.
# ------------------------------------------------------------------------------------------
def mlp_forward(X: np.ndarray, layers) -> np.ndarray:
    h = np.asarray(X, dtype=np.float64)
    for li, (W, b) in enumerate(layers):
        h = h @ np.asarray(W, dtype=np.float64) + np.asarray(b, dtype=np.float64)
        if li + 1 < len(layers):
            h = np.maximum(h, 0.0)
    return h


# ------------------------------------------------------------------------------------------
# ASOT-ML mapping ("the outputs of the MLP for P are normalized by dividing their l1
# norms"; R#25: |.| first, an all-zero row falls back to the uniform row, flagged).
# ------------------------------------------------------------------------------------------
def ml_encode(X: np.ndarray, layers) -> tuple[np.ndarray, np.ndarray]:
    """Returns (Z [n, K] rows on the simplex, fallback flags [n])."""
    O = np.abs(mlp_forward(X, layers))
    s = O.sum(axis=1)
    K = O.shape[1]
    zero = s == 0.0
    Z = np.empty_like(O)
    Z[~zero] = O[~zero] / s[~zero, None]
    Z[zero] = 1.0 / K
    return Z, zero


# ------------------------------------------------------------------------------------------
# Mahalanobis anchor cost ("d_AS(w_u, w_v) = ||M w_u - M w_v||_2"; R#29:
# optionally divided by its max, as the configs normalise C_s, R#7).
# ------------------------------------------------------------------------------------------
def mahalanobis_cost(anchors: np.ndarray, M: np.ndarray, normalize: bool = False) -> np.ndarray:
    W = np.asarray(anchors, dtype=np.float64)          # [K, d], row u = w_u
    Mm = np.asarray(M, dtype=np.float64)               # [h, d]
    K = W.shape[0]
    C = np.zeros((K, K), dtype=np.float64)
    for u in range(K):
        for v in range(K):
            diff = Mm @ W[u] - Mm @ W[v]
            C[u, v] = np.sqrt(np.sum(diff * diff))
    if normalize and C.max() > 0:
        C = C / C.max()
    return C


# ------------------------------------------------------------------------------------------
# ASOT-DL near-one-hot encoder (Eq. (9); appendix derivation P:500-538 "fixed step
# size as 1", prox = max(0, a - lambda)).
# ------------------------------------------------------------------------------------------
def simplex_shrink(a: np.ndarray, theta) -> np.ndarray:
    """S_theta(a) = max(0, a - theta)."""
    return np.maximum(0.0, np.asarray(a, dtype=np.float64) - theta)


def near_onehot_layer(z: np.ndarray, x: np.ndarray, W: np.ndarray, lam) -> np.ndarray:
    """One layer z <- S_lambda(z - W^T (W z - x)) (Eq. (9)); W is d x k (columns = anchors)."""
    z = np.asarray(z, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    r = W @ z - np.asarray(x, dtype=np.float64)     # W z - x           (d)
    g = W.T @ r                                      # W^T (W z - x)     (k)
    return simplex_shrink(z - g, lam)


def eq8_objective(z: np.ndarray, x: np.ndarray, W: np.ndarray, lam) -> float:
    """Eq. (8) with the constant dropped: 1/2 ||W z - x||^2 + lambda 1^T z (z >= 0)."""
    r = np.asarray(W, dtype=np.float64) @ z - x
    return 0.5 * float(r @ r) + float(lam) * float(np.sum(z))


def softplus(t):
    t = np.asarray(t, dtype=np.float64)
    return np.where(t > 30.0, t, np.log1p(np.exp(np.minimum(t, 30.0))))


def dl_lambda(X: np.ndarray, lam_layers) -> np.ndarray:
    """lambda(x) = softplus(MLP(x)) > 0 ("an MLP to evaluate lambda for each input";
    P:510 assumes lambda > 0; R#26)."""
    return softplus(mlp_forward(X, lam_layers)[:, 0])


def dl_encode(X: np.ndarray, dictionary: np.ndarray, lam_layers, n_layers: int):
    """Near-one-hot encoder: z^(0) = 0, n_layers x Eq. (9), then z / sum(z) (R#27); an all-zero
    code falls back to the uniform row, flagged.  ``dictionary`` is [K, d] (row u = w_u), so the
    paper's W = dictionary^T.  Returns (Z [n, K], flags [n], lambda [n])."""
    X = np.asarray(X, dtype=np.float64)
    W = np.asarray(dictionary, dtype=np.float64).T      # d x K
    K = W.shape[1]
    lam = dl_lambda(X, lam_layers)
    Z = np.zeros((X.shape[0], K), dtype=np.float64)
    flags = np.zeros(X.shape[0], dtype=bool)
    for p in range(X.shape[0]):
        z = np.zeros(K, dtype=np.float64)
        for _ in range(n_layers):
            z = near_onehot_layer(z, X[p], W, lam[p])
        s = z.sum()
        if s > 0.0:
            Z[p] = z / s
        else:
            Z[p] = 1.0 / K
            flags[p] = True
    return Z, flags, lam


# ------------------------------------------------------------------------------------------
# Mapped marginals a' = Z^T a per distribution (Eq. (5), 1/n dropped R#1).
# ------------------------------------------------------------------------------------------
def soft_histograms(Z: np.ndarray, weights: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    Z = np.asarray(Z, dtype=np.float64)
    w = np.asarray(weights, dtype=np.float64)
    N = offsets.shape[0] - 1
    H = np.zeros((N, Z.shape[1]), dtype=np.float64)
    for i in range(N):
        s, e = int(offsets[i]), int(offsets[i + 1])
        H[i] = Z[s:e].T @ w[s:e]
    return H
