"""fp64 CPU oracle for the ASOT pairwise-distance hot path (arxiv 2310.16123).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this module.
The product path (``paper_2310_16123_b200``) never imports it and shares no code
with it: the only common module is ``asot_inputs`` (seeded inputs, no method
arithmetic).

Plain, slow, obviously correct numpy in float64, written step by step in the
paper's order and notation.  Citations: ``P:n`` = PAPER.md line n, ``S:n`` =
SPEC.md line n, readings ``R#n`` = SURVEY.md §8(c) table / DESIGN.md "Readings".

Hot path (what the CUDA path must reproduce):
  1. map_assign      one-hot nearest anchor P_o
  2. histograms      a' = Z^T a, 1/n factor dropped (R#1)
  3. gibbs           K = exp(-C_s / eps) and K (.) C_s for the cost
  4. sinkhorn_batch  U = A/(K V), V = B/(K^T U), v0 = 1, exactly L iterations
                     (R#4, R#5, R#11, R#12)
  5. cost            <diag(u) K diag(v), C_s> = u^T ((K (.) C_s) v) (R#3, R#6)
  6. distance_matrix all pairs i<j, a = H[i] on the u side, mirrored, zero diagonal
                     (Def. 1; R#9, R#10)

Pin-only helpers (never on the hot path): exact LP (scipy HiGHS), log-domain
converged Sinkhorn, brute-force permutation OT, reconstructed cost / Prop. 1 /
Prop. 2 bounds.

Parity status: every hot-path function above is pinned by tests in
``tests/test_oracle_pins.py`` (closed forms, LP, brute force, exact rational
arithmetic, invariants).  The intermediate, non-converged L-iteration values
have no closed form; they are pinned at convergence (LP / brute force /
log-domain) and at finite L by the one-hot closed form, the 2x2 closed form,
batching and invariance pins (SURVEY §8(c) last row).
"""
from __future__ import annotations

import itertools
from typing import Optional

import numpy as np

UNDERFLOW_FLOOR = 1e-300  # S:79 "underflow_floor default 1e-300"


# --------------------------------------------------------------------------------------
# Step 1. Mapping P_o: one-hot nearest anchor ("one-hot mapping function";
# P:246 "P_o is the clustering operator"; S:378 argmin with lowest-index ties).
# Distance formula pinned for bit-exact parity (R#8): D_pj = sum_k (x_pk - w_jk)^2,
# accumulated sequentially in k in fp64, each subtract / square / add individually
# rounded (no fused multiply-add).
# --------------------------------------------------------------------------------------
def point_anchor_sqdist(points: np.ndarray, anchors: np.ndarray) -> np.ndarray:
    """[n, K] fp64 squared distances in the pinned op order (R#8)."""
    X = np.asarray(points, dtype=np.float64)
    W = np.asarray(anchors, dtype=np.float64)
    acc = np.zeros((X.shape[0], W.shape[0]), dtype=np.float64)
    for k in range(X.shape[1]):
        t = X[:, k, None] - W[None, :, k]   # one rounding
        sq = t * t                          # one rounding
        acc = acc + sq                      # one rounding, sequential in k
    return acc


def map_assign(points: np.ndarray, anchors: np.ndarray, chunk: int = 4096) -> np.ndarray:
    """j*(p) = smallest j with D_pj = min_j D_pj. Returns int32 [T]."""
    T = points.shape[0]
    out = np.empty(T, dtype=np.int32)
    for s in range(0, T, chunk):
        D = point_anchor_sqdist(points[s:s + chunk], anchors)
        out[s:s + chunk] = np.argmin(D, axis=1)  # numpy argmin returns the first minimum
    return out


# --------------------------------------------------------------------------------------
# Step 2. Mapped marginals a' = Z_x^T a (Eq. (5) P:100 with the 1/n factor dropped,
# R#1; Lemma 1 proof "T_s 1_k = Z_x^T T 1_m" P:145; "mass = Z^T (D.mass)").
# With one-hot Z this is a histogram: H[i, j] = sum_{p in i, j*(p) = j} w_p, summed in
# fp64 in point order.
# --------------------------------------------------------------------------------------
def histograms(assign: np.ndarray, weights: np.ndarray, offsets: np.ndarray,
               n_anchors: int) -> np.ndarray:
    N = offsets.shape[0] - 1
    H = np.zeros((N, n_anchors), dtype=np.float64)
    row = np.repeat(np.arange(N, dtype=np.int64), np.diff(offsets))
    flat = H.reshape(-1)
    # np.add.at is unbuffered and visits indices in order: per bin, point order.
    np.add.at(flat, row * n_anchors + assign.astype(np.int64), weights.astype(np.float64))
    return H


def map_distribution(Z: np.ndarray, a: np.ndarray) -> np.ndarray:
    """General (soft or one-hot) a' = Z^T a. Pins only."""
    return np.asarray(Z, dtype=np.float64).T @ np.asarray(a, dtype=np.float64)


# --------------------------------------------------------------------------------------
# Step 3. Gibbs kernel K := exp(-C_s / eps), and K (.) C_s for the cost.
# --------------------------------------------------------------------------------------
def gibbs(cost: np.ndarray, eps: float) -> tuple[np.ndarray, np.ndarray]:
    C = np.asarray(cost, dtype=np.float64)
    e = float(np.float64(eps))        # eps is the fp32 value as passed (0.05f = 0.0500000007...)
    G = np.exp(-C / e)
    return G, G * C


# --------------------------------------------------------------------------------------
# Steps 4-5. Batched Sinkhorn on the shared kernel:
#   U^(j+1) = A / (K V^(j)),  V^(j+1) = B / (K^T U^(j+1)),  V^(0) = 1 (R#4)
# exactly L iterations, no tolerance stop (R#5).  0/x = 0 (R#11); a zero denominator
# is clamped to the floor and flagged (R#12).
# Cost = <T, C_s>, T = diag(u) K diag(v) (R#3), linear part only (R#6):
#   d = sum_{r,c} u_r K_rc C_rc v_c = u^T ((K (.) C_s) v).
# Columns are independent, so a batch is just many columns at once.
# --------------------------------------------------------------------------------------
def _scaled_div(num: np.ndarray, den: np.ndarray, flags: np.ndarray) -> np.ndarray:
    small = den < UNDERFLOW_FLOOR
    if small.any():
        flags |= small.any(axis=0)
    out = num / np.maximum(den, UNDERFLOW_FLOOR)
    out[num == 0] = 0.0
    return out


def sinkhorn_batch(A: np.ndarray, B: np.ndarray, G: np.ndarray, GC: np.ndarray, iters: int,
                   V0: Optional[np.ndarray] = None):
    """A, B: [K, P] columns (a_p, b_p).  Returns (cost[P], U, V, clamp_flags[P])."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    K, P = A.shape
    V = np.ones((K, P), dtype=np.float64) if V0 is None else np.array(V0, dtype=np.float64)
    flags = np.zeros(P, dtype=bool)
    U = None
    for _ in range(iters):
        U = _scaled_div(A, G @ V, flags)
        V = _scaled_div(B, G.T @ U, flags)
    cost = np.sum(U * (GC @ V), axis=0)
    return cost, U, V, flags


def sinkhorn(a: np.ndarray, b: np.ndarray, C: np.ndarray, eps: float, iters: int):
    """Single-pair entropic OT with a general (possibly rectangular) cost.
    Returns (cost, plan)."""
    C = np.asarray(C, dtype=np.float64)
    K = np.exp(-C / float(eps))
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    v = np.ones(C.shape[1])
    u = None
    flags = np.zeros(1, dtype=bool)
    for _ in range(iters):
        u = _scaled_div(a[:, None], (K @ v)[:, None], flags)[:, 0]
        v = _scaled_div(b[:, None], (K.T @ u)[:, None], flags)[:, 0]
    T = u[:, None] * K * v[None, :]
    return float(np.sum(T * C)), T


# --------------------------------------------------------------------------------------
# Step 6. The pairwise matrix (Def. 1, pair set i != j; S:132-140 each unordered
# pair once, symmetric, zero diagonal; R#9 diagonal never computed; R#10 a = H[i] on the
# u side for i < j, mirrored to D[j, i]).
# --------------------------------------------------------------------------------------
def upper_pairs(n_dist: int) -> tuple[np.ndarray, np.ndarray]:
    i, j = np.triu_indices(n_dist, k=1)
    return i.astype(np.int64), j.astype(np.int64)


def pair_costs(H: np.ndarray, cost: np.ndarray, eps: float, iters: int,
               pi: np.ndarray, pj: np.ndarray, batch: int = 2048):
    """eASOT cost for explicit pairs (i, j): a = H[i], b = H[j]."""
    G, GC = gibbs(cost, eps)
    out = np.empty(len(pi), dtype=np.float64)
    flags = np.zeros(len(pi), dtype=bool)
    for s in range(0, len(pi), batch):
        A = H[pi[s:s + batch]].T
        B = H[pj[s:s + batch]].T
        c, _, _, f = sinkhorn_batch(A, B, G, GC, iters)
        out[s:s + batch] = c
        flags[s:s + batch] = f
    return out, flags


def map_and_histogram(points, offsets, weights, anchors):
    assign = map_assign(points, anchors)
    return assign, histograms(assign, weights, offsets, anchors.shape[0])


def distance_matrix(points, offsets, weights, anchors, cost, eps, iters):
    """Full pipeline (steps 1-6) on every pair i < j.  Returns (D[N,N], assign, H)."""
    assign, H = map_and_histogram(points, offsets, weights, anchors)
    N = offsets.shape[0] - 1
    pi, pj = upper_pairs(N)
    c, _ = pair_costs(H, cost, eps, iters, pi, pj)
    D = np.zeros((N, N), dtype=np.float64)
    D[pi, pj] = c
    D[pj, pi] = c
    return D, assign, H


# ======================================================================================
# Pin-only helpers (tests): exact OT, converged entropic OT, brute force, bounds.
# ======================================================================================
def euclidean_cost(X: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """C(i,j) = ||x_i - y_j||_2 (Eq. (2))."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    if X.shape[1] != Y.shape[1]:
        raise ValueError("dimension mismatch")
    diff = X[:, None, :] - Y[None, :, :]
    return np.sqrt(np.sum(diff * diff, axis=-1))


def solve_exact(a: np.ndarray, b: np.ndarray, C: np.ndarray) -> float:
    """Exact OT LP (Eq. (1)) by scipy HiGHS on fp64-renormalised marginals (R#14)."""
    from scipy.optimize import linprog

    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    a = a / a.sum()
    b = b / b.sum()
    n, m = C.shape
    Aeq = np.zeros((n + m, n * m))
    for i in range(n):
        Aeq[i, i * m:(i + 1) * m] = 1.0
    for j in range(m):
        Aeq[n + j, j::m] = 1.0
    res = linprog(np.asarray(C, dtype=np.float64).reshape(-1), A_eq=Aeq,
                  b_eq=np.concatenate([a, b]), bounds=(0, None), method="highs",
                  options={"primal_feasibility_tolerance": 1e-10,
                           "dual_feasibility_tolerance": 1e-10})
    if not res.success:
        raise RuntimeError(res.message)
    return float(res.fun)


def sinkhorn_log_converged(a, b, C, eps: float, tol: float = 1e-12, max_iter: int = 200000,
                           anneal: bool = True):
    """Converged entropic OT by log-domain Sinkhorn with eps-annealing (pins only).
    Returns (linear cost <T, C>, plan, marginal residual)."""
    from scipy.special import logsumexp

    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    C = np.asarray(C, dtype=np.float64)
    la, lb = np.log(np.where(a > 0, a, 1e-300)), np.log(np.where(b > 0, b, 1e-300))
    f = np.zeros(C.shape[0])
    g = np.zeros(C.shape[1])
    schedule = [eps]
    if anneal:
        e = max(1.0, eps)
        schedule = []
        while e > eps:
            schedule.append(e)
            e *= 0.5
        schedule.append(eps)
    res = np.inf
    for e in schedule:
        for _ in range(max_iter):
            f = e * la - e * logsumexp((g[None, :] - C) / e, axis=1)
            g = e * lb - e * logsumexp((f[:, None] - C) / e, axis=0)
            T = np.exp((f[:, None] + g[None, :] - C) / e)
            res = np.abs(T.sum(axis=1) - a).sum()
            if res < tol:
                break
    T = np.exp((f[:, None] + g[None, :] - C) / eps)
    return float(np.sum(T * C)), T, float(res)


def brute_force_perm_ot(C: np.ndarray) -> float:
    """Uniform n = m OT: the LP optimum sits at a permutation matrix (Birkhoff), so
    W = min_sigma (1/n) sum_i C[i, sigma(i)]."""
    n = C.shape[0]
    best = np.inf
    for perm in itertools.permutations(range(n)):
        best = min(best, sum(C[i, perm[i]] for i in range(n)) / n)
    return float(best)


def reconstructed_cost(Zx: np.ndarray, Cs: np.ndarray, Zy: np.ndarray) -> np.ndarray:
    """C_hat = Z_x C_s Z_y^T (Lemma 1, Prop. 1)."""
    return np.asarray(Zx, np.float64) @ np.asarray(Cs, np.float64) @ np.asarray(Zy, np.float64).T


def prop1_bound(C_hat: np.ndarray, C: np.ndarray) -> float:
    """||C_hat - C||_1, entrywise (Eq. (7))."""
    return float(np.abs(np.asarray(C_hat) - np.asarray(C)).sum())


def prop2_bound(res_x: np.ndarray, res_y: np.ndarray) -> float:
    """m sum_i ||eps_i^x|| + n sum_j ||eps_j^y|| (Prop. 2)."""
    res_x = np.asarray(res_x, np.float64)
    res_y = np.asarray(res_y, np.float64)
    if (res_x < 0).any() or (res_y < 0).any():
        raise ValueError("negative residual")
    n, m = res_x.shape[0], res_y.shape[0]
    return float(m * res_x.sum() + n * res_y.sum())


def one_hot(assign: np.ndarray, k: int) -> np.ndarray:
    Z = np.zeros((assign.shape[0], k))
    Z[np.arange(assign.shape[0]), assign] = 1.0
    return Z
