"""Pins for the fp64 oracle against what the paper and the mathematics fix.

Every hot-path oracle function is checked here against something other than
itself: closed forms, the exact LP (scipy HiGHS), brute-force permutation OT,
exact rational arithmetic, and invariants the paper states.  A plausible
mistake (dropped term, wrong sign/index, transposed operand, wrong tie rule,
1/n kept in Eq. (5), cost taken on the wrong plan) fails at least one test.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

from oracle import asot_oracle as O

pytestmark = pytest.mark.filterwarnings("ignore::RuntimeWarning")


# ------------------------------------------------------------------ golden (SPEC examples)
def test_golden_euclidean(golden):
    g = golden["euclidean_cost_345"]
    np.testing.assert_allclose(O.euclidean_cost(np.array(g["X"]), np.array(g["Y"])), g["C"], rtol=0, atol=1e-15)


def test_golden_exact_lp(golden):
    for key in ("solve_exact_forced", "solve_exact_zero"):
        g = golden[key]
        assert abs(O.solve_exact(np.array(g["a"]), np.array(g["b"]), np.array(g["C"], float)) - g["cost"]) < 1e-9


def test_golden_sinkhorn(golden):
    g = golden["sinkhorn_2x2"]
    c, _ = O.sinkhorn(np.array(g["a"]), np.array(g["b"]), np.array(g["C"], float), g["eps"], g["iters"])
    assert abs(c - g["cost"]) < g["tol"]
    g = golden["sinkhorn_zero_cost"]
    c, _ = O.sinkhorn(np.array(g["a"]), np.array(g["b"]), np.array(g["C"], float), g["eps"], g["iters"])
    assert c == g["cost"]


def test_golden_anchor_cost_and_mapping(golden):
    g = golden["anchor_cost_345"]
    np.testing.assert_allclose(O.euclidean_cost(np.array(g["anchors"], float), np.array(g["anchors"], float)),
                               g["C_s"], atol=1e-15)
    g = golden["map_distribution_112"]
    assign = np.array(g["assign"], np.int32)
    Z = O.one_hot(assign, g["k"])
    np.testing.assert_allclose(O.map_distribution(Z, np.array(g["mass"])), g["a_prime"], atol=1e-15)
    H = O.histograms(assign, np.array(g["mass"]), np.array([0, 3]), g["k"])
    np.testing.assert_allclose(H[0], g["a_prime"], atol=1e-15)


def test_golden_asot_exact_and_bounds(golden):
    g = golden["asot_exact_forced"]
    Cs = np.array([[0, g["c"]], [g["c"], 0]], float)
    assert abs(O.solve_exact(np.array(g["ax"]), np.array(g["bx"]), Cs) - g["cost"]) < 1e-9
    g = golden["prop1_bound_shift"]
    C = np.array(g["C"])
    assert abs(O.prop1_bound(C + g["shift"], C) - g["bound"]) < 1e-12
    g = golden["prop2_bound_simple"]
    assert abs(O.prop2_bound(np.array(g["res_x"]), np.array(g["res_y"])) - g["bound"]) < 1e-15


# ------------------------------------------------------------------ Sinkhorn closed forms
def test_sinkhorn_symmetric_2x2_closed_form_batch():
    """a = b = [.5,.5], C = [[0,1],[1,0]], eps = .1 -> e^-10 / (1 + e^-10) for any L >= 1."""
    exact = math.exp(-10) / (1 + math.exp(-10))
    C = np.array([[0.0, 1.0], [1.0, 0.0]])
    G, GC = O.gibbs(C, 0.1)
    A = np.array([[0.5], [0.5]])
    for L in (1, 2, 50):
        c, _, _, flags = O.sinkhorn_batch(A, A, G, GC, L)
        assert abs(c[0] - exact) <= 1e-15 * exact * 10
        assert not flags.any()


def _twobytwo_converged_x(p, q, C, eps):
    # T = [[x, p-x], [q-x, 1-p-q+x]], T = diag(u) K diag(v) =>
    # x (1-p-q+x) / ((p-x)(q-x)) = exp((C12 + C21 - C11 - C22)/eps) =: kappa
    kappa = math.exp((C[0, 1] + C[1, 0] - C[0, 0] - C[1, 1]) / eps)
    a2 = 1.0 - kappa
    a1 = (1.0 - p - q) + kappa * (p + q)
    a0 = -kappa * p * q
    lo, hi = max(0.0, p + q - 1.0), min(p, q)
    if abs(a2) < 1e-300:
        return -a0 / a1
    disc = math.sqrt(a1 * a1 - 4 * a2 * a0)
    for x in ((-a1 + disc) / (2 * a2), (-a1 - disc) / (2 * a2)):
        if lo - 1e-12 <= x <= hi + 1e-12:
            return x
    raise AssertionError("no root in range")


def test_sinkhorn_general_2x2_converged_closed_form():
    rng = np.random.default_rng(7)
    for _ in range(20):
        p, q = rng.uniform(0.1, 0.9, 2)
        C = rng.uniform(0, 1, (2, 2))
        eps = 0.5
        x = _twobytwo_converged_x(p, q, C, eps)
        T_exact = np.array([[x, p - x], [q - x, 1 - p - q + x]])
        # batch form (asymmetric C: use the general single-pair routine, which takes C)
        c, T = O.sinkhorn(np.array([p, 1 - p]), np.array([q, 1 - q]), C, eps, 3000)
        np.testing.assert_allclose(T, T_exact, atol=1e-12)
        assert abs(c - float(np.sum(T_exact * C))) < 1e-12
    # symmetric cost through the batched hot-path routine
    for _ in range(10):
        p, q = rng.uniform(0.1, 0.9, 2)
        off = rng.uniform(0, 1)
        C = np.array([[0.0, off], [off, 0.0]])
        eps = 0.3
        x = _twobytwo_converged_x(p, q, C, eps)
        G, GC = O.gibbs(C, eps)
        c, U, V, _ = O.sinkhorn_batch(np.array([[p], [1 - p]]), np.array([[q], [1 - q]]), G, GC, 3000)
        T = U[:, 0][:, None] * G * V[:, 0][None, :]
        np.testing.assert_allclose(T[0, 0], x, atol=1e-12)
        assert abs(c[0] - off * (p - x + q - x)) < 1e-12


def test_sinkhorn_separable_cost_any_L():
    """Finite-L pin (not a convergence statement).  C_s(i, j) = f_i + f_j makes the Gibbs kernel
    rank one, G = g g^T with g = exp(-f / eps), so the first u-update already gives
    T = diag(u) G diag(v) = a b^T after the first v-update: for every L >= 1 the plan is the
    product coupling and d = sum_i a_i f_i + sum_j b_j f_j exactly (up to rounding)."""
    rng = np.random.default_rng(21)
    K, P = 7, 5
    f = rng.uniform(0.0, 1.0, K)
    Cs = f[:, None] + f[None, :]
    A = rng.dirichlet(np.ones(K), P).T
    B = rng.dirichlet(np.ones(K), P).T
    A[2, 0] = 0.0
    A[:, 0] /= A[:, 0].sum()
    for eps in (0.1, 0.5):
        G, GC = O.gibbs(Cs, eps)
        for L in (1, 2, 9):
            c, U, V, flags = O.sinkhorn_batch(A, B, G, GC, L)
            assert not flags.any()
            for p in range(P):
                T = U[:, p][:, None] * G * V[:, p][None, :]
                np.testing.assert_allclose(T, np.outer(A[:, p], B[:, p]), atol=1e-14)
                assert abs(c[p] - (A[:, p] @ f + B[:, p] @ f)) <= 1e-13


def test_sinkhorn_2x2_one_iteration_closed_form():
    """Finite-L pin away from convergence.  C = [[0, c], [c, 0]], G = [[1, k], [k, 1]] with
    k = exp(-c / eps); a = (p, 1-p), b = (q, 1-q), v0 = 1.  One iteration by hand:
    u = a / (1 + k), v_1 = q (1 + k) / (p + k (1-p)), v_2 = (1-q)(1 + k) / (k p + 1 - p), and the
    cost <T, C> = c k (u_1 v_2 + u_2 v_1) =
        c k [ p (1-q) / (k p + 1 - p) + (1-p) q / (p + k (1-p)) ]."""
    rng = np.random.default_rng(22)
    for _ in range(20):
        p, q = rng.uniform(0.05, 0.95, 2)
        cst = rng.uniform(0.1, 2.0)
        eps = rng.uniform(0.2, 2.0)
        k = math.exp(-cst / eps)
        G, GC = O.gibbs(np.array([[0.0, cst], [cst, 0.0]]), eps)
        c, U, V, _ = O.sinkhorn_batch(np.array([[p], [1 - p]]), np.array([[q], [1 - q]]), G, GC, 1)
        exact = cst * k * (p * (1 - q) / (k * p + 1 - p) + (1 - p) * q / (p + k * (1 - p)))
        assert abs(c[0] - exact) <= 1e-14 * max(exact, 1.0)
        np.testing.assert_allclose(U[:, 0], [p / (1 + k), (1 - p) / (1 + k)], rtol=1e-14)
        # the row marginals are NOT met after one iteration unless p = q (a non-converged value)
        T = U[:, 0][:, None] * G * V[:, 0][None, :]
        if abs(p - q) > 0.05:
            assert abs(T.sum(1)[0] - p) > 1e-6


def test_sinkhorn_one_hot_marginals_exact():
    """a = e_u, b = e_v  =>  the plan is the single entry (u, v) => d = C_s(u, v) for any eps, L."""
    rng = np.random.default_rng(3)
    K = 9
    W = rng.normal(size=(K, 3))
    Cs = O.euclidean_cost(W, W) ** 2
    Cs /= Cs.max()
    for eps in (0.05, 0.2, 1.0):
        G, GC = O.gibbs(Cs, eps)
        for L in (1, 3, 17):
            for (u, v) in [(0, 5), (4, 4), (8, 1)]:
                a = np.zeros((K, 1)); a[u] = 1
                b = np.zeros((K, 1)); b[v] = 1
                c, _, _, _ = O.sinkhorn_batch(a, b, G, GC, L)
                assert abs(c[0] - Cs[u, v]) <= 1e-13 * max(Cs[u, v], 1e-300) + 1e-300


def test_sinkhorn_invariants():
    rng = np.random.default_rng(11)
    K, P = 12, 6
    W = rng.normal(size=(K, 4))
    Cs = O.euclidean_cost(W, W) ** 2
    Cs /= Cs.max()
    A = rng.dirichlet(np.ones(K), P).T
    B = rng.dirichlet(np.ones(K), P).T
    A[rng.uniform(size=A.shape) < 0.3] = 0
    A /= A.sum(0)
    G, GC = O.gibbs(Cs, 0.05)
    L = 40
    c, U, V, _ = O.sinkhorn_batch(A, B, G, GC, L)
    # v0 -> s * v0 leaves the cost unchanged (R#4)
    c2, _, _, _ = O.sinkhorn_batch(A, B, G, GC, L, V0=np.full((K, P), 3.7))
    np.testing.assert_allclose(c2, c, rtol=1e-12)
    # column marginals of T after the final v-update equal b
    for p in range(P):
        T = U[:, p][:, None] * G * V[:, p][None, :]
        np.testing.assert_allclose(T.sum(0), B[:, p], atol=1e-14)
        assert abs(c[p] - np.sum(T * Cs)) < 1e-14
        # zero-mass bins carry u = 0 (R#11)
        assert np.all(U[A[:, p] == 0, p] == 0)
    # anchor permutation applied to C_s and to both histograms leaves d unchanged
    perm = rng.permutation(K)
    Gp, GCp = O.gibbs(Cs[np.ix_(perm, perm)], 0.05)
    c3, _, _, _ = O.sinkhorn_batch(A[perm], B[perm], Gp, GCp, L)
    np.testing.assert_allclose(c3, c, rtol=1e-11)
    # C = 0 -> 0
    G0, GC0 = O.gibbs(np.zeros((K, K)), 0.05)
    c0, _, _, _ = O.sinkhorn_batch(A, B, G0, GC0, L)
    assert np.all(c0 == 0)
    # swapping the roles (a <-> b) is NOT an identity at finite L (R#10) but is at convergence
    cs, _, _, _ = O.sinkhorn_batch(B, A, G, GC, 4000)
    cl, _, _, _ = O.sinkhorn_batch(A, B, G, GC, 4000)
    np.testing.assert_allclose(cs, cl, rtol=1e-9)


def test_sinkhorn_underflow_floor_branch():
    """S:62 / S:79 (R#12): a denominator below underflow_floor = 1e-300 is clamped to the floor and
    flagged.  K = 2, C = [[0, 1], [1, 0]], a = 1e-200 e_0, b = e_1, G off-diagonal g, v0 = 1.
    Hand computation of one iteration: G v0 = (1 + g, 1 + g) -> u = (1e-200 / (1 + g), 0);
    G^T u = (u_0, g u_0).
      g = 1e-120: (G^T u)_1 = 1e-320 < 1e-300 -> clamped: v_1 = 1 / 1e-300 (unclamped it would be
        1e320 = inf in fp64), flag set, cost = u_0 g C_01 v_1 = 1e-20;
      g = 1e-90: (G^T u)_1 = 1e-290 >= floor -> v_1 = 1 / (g u_0), no flag, and the cost is the
        one-hot closed form C_01 = 1 (the plan moves all of b's mass across)."""
    C = np.array([[0.0, 1.0], [1.0, 0.0]])
    A = np.array([[1e-200], [0.0]])
    B = np.array([[0.0], [1.0]])
    for g, flagged, v1, cost in ((1e-120, True, 1e300, 1e-20), (1e-90, False, 1e290, 1.0)):
        G = np.array([[1.0, g], [g, 1.0]])
        c, U, V, fl = O.sinkhorn_batch(A, B, G, G * C, 1)
        assert bool(fl[0]) is flagged
        assert V[0, 0] == 0.0                      # b_0 = 0 -> v_0 = 0 (0/x = 0, R#11)
        assert math.isclose(V[1, 0], v1, rel_tol=1e-12)
        assert np.isfinite(c[0]) and math.isclose(c[0], cost, rel_tol=1e-12)
    assert O.UNDERFLOW_FLOOR == 1e-300             # S:79 default


def test_batched_equals_per_pair():
    """batched column p == single-pair Sinkhorn on (a_p, b_p)."""
    rng = np.random.default_rng(5)
    K, P = 10, 8
    W = rng.normal(size=(K, 2))
    Cs = O.euclidean_cost(W, W)
    A = rng.dirichlet(np.ones(K), P).T
    B = rng.dirichlet(np.ones(K), P).T
    G, GC = O.gibbs(Cs, 0.1)
    c, _, _, _ = O.sinkhorn_batch(A, B, G, GC, 30)
    for p in range(P):
        cp, _ = O.sinkhorn(A[:, p], B[:, p], Cs, 0.1, 30)
        assert abs(cp - c[p]) <= 1e-12
    c1, _, _, _ = O.sinkhorn_batch(A[:, :1], B[:, :1], G, GC, 30)
    assert abs(c1[0] - c[0]) <= 1e-14


def test_sinkhorn_converges_to_exact_lp():
    """S:66 / acceptance #5: random 5x7, eps = .01, 2000 iterations within 1e-3 of the LP,
    and never below it by more than 1e-9."""
    rng = np.random.default_rng(21)
    for _ in range(10):
        a = rng.dirichlet(np.ones(5))
        b = rng.dirichlet(np.ones(7))
        C = rng.uniform(0, 1, (5, 7))
        lp = O.solve_exact(a, b, C)
        c, _ = O.sinkhorn(a, b, C, 0.01, 2000)
        assert abs(c - lp) <= 1e-3
        assert c >= lp - 1e-9


# ------------------------------------------------------------------ eps -> 0 vs brute force
def _pooled_support_instance(rng, n):
    X = rng.uniform(0, 1, (n, 2))
    Y = rng.uniform(0, 1, (n, 2))
    pts = np.concatenate([X, Y]).astype(np.float32)
    anchors = pts.copy()                          # anchors = pooled support
    C = O.euclidean_cost(pts, pts)                # Euclidean ground metric
    C = C / C.max()
    offsets = np.array([0, n, 2 * n])
    w = np.full(2 * n, 1.0 / n)
    return pts, anchors, C, offsets, w


@pytest.mark.parametrize("n", [3, 4, 5, 6])
def test_easot_pooled_support_vs_brute_force(n):
    """north star: anchors = pooled support + identity mapping => ASOT = OT (Lemma 1);
    converged eASOT satisfies 0 <= W_eps - W <= eps log n vs brute-force permutation OT."""
    rng = np.random.default_rng(100 + n)
    pts, anchors, C, offsets, w = _pooled_support_instance(rng, n)
    assign, H = O.map_and_histogram(pts, offsets, w, anchors)
    np.testing.assert_array_equal(assign, np.arange(2 * n))        # identity mapping
    W_bf = O.brute_force_perm_ot(C[:n, n:])
    W_lp_ot = O.solve_exact(w[:n], w[n:], C[:n, n:])
    W_lp_asot = O.solve_exact(H[0], H[1], C)                        # K x K anchor problem
    assert abs(W_lp_ot - W_bf) < 1e-9
    assert abs(W_lp_asot - W_bf) < 1e-9
    # plain fixed-L hot-path recurrence, run to convergence at eps = .05
    eps = 0.05
    G, GC = O.gibbs(C, eps)
    c, U, V, _ = O.sinkhorn_batch(H[0][:, None], H[1][:, None], G, GC, 20000)
    T = U[:, 0][:, None] * G * V[:, 0][None, :]
    resid = np.abs(T.sum(1) - H[0]).sum()
    assert resid < 1e-10
    assert -1e-9 <= c[0] - W_bf <= eps * math.log(n) + 1e-9
    # converged eASOT == converged eOT on the original n x m problem
    ce, _, r = O.sinkhorn_log_converged(w[:n], w[n:], C[:n, n:], eps, tol=1e-12, max_iter=20000)
    assert r < 1e-10
    assert abs(ce - c[0]) < 1e-9
    # smaller eps (log domain): the gap shrinks within eps log n
    for e in (0.01, 0.003):
        cl, _, r = O.sinkhorn_log_converged(w[:n], w[n:], C[:n, n:], e, tol=1e-11, max_iter=6000)
        assert r < 1e-5                  # marginal residual; costs are <= 1, so |dW| <= r
        assert -r - 1e-9 <= cl - W_bf <= e * math.log(n) + r + 1e-9


# ------------------------------------------------------------------ Lemma 1, Prop. 1, Prop. 2
def _random_one_hot_instance(rng):
    n, m, k, d = rng.integers(2, 8), rng.integers(2, 8), rng.integers(2, 6), 2
    X = rng.normal(size=(n, d))
    Y = rng.normal(size=(m, d))
    Wa = rng.normal(size=(k, d))
    a = rng.dirichlet(np.ones(n))
    b = rng.dirichlet(np.ones(m))
    return X, Y, Wa, a, b


def test_lemma1_one_hot_equivalence():
    """LP(a', b', C_s) = LP(a, b, Z_x C_s Z_y^T) for one-hot Z (R#17)."""
    rng = np.random.default_rng(31)
    worst = 0.0
    for _ in range(40):
        X, Y, Wa, a, b = _random_one_hot_instance(rng)
        Cs = O.euclidean_cost(Wa, Wa)
        zx = O.map_assign(X, Wa)
        zy = O.map_assign(Y, Wa)
        k = Wa.shape[0]
        ap = O.histograms(zx, a, np.array([0, len(a)]), k)[0]
        bp = O.histograms(zy, b, np.array([0, len(b)]), k)[0]
        Chat = O.reconstructed_cost(O.one_hot(zx, k), Cs, O.one_hot(zy, k))
        w_as = O.solve_exact(ap, bp, Cs)
        w_rec = O.solve_exact(a, b, Chat)
        worst = max(worst, abs(w_as - w_rec))
    assert worst < 1e-8


def test_lemma1_fails_for_soft_mapping():
    """R#17 counterexample: n = m = 1, z = [1/2, 1/2], C_s = [[0,1],[1,0]]: LP(C_hat) = 1/2,
    W_AS = 0.  Only W_AS <= LP(C_hat) survives for soft P."""
    Cs = np.array([[0.0, 1.0], [1.0, 0.0]])
    Z = np.array([[0.5, 0.5]])
    a = np.array([1.0])
    Chat = O.reconstructed_cost(Z, Cs, Z)
    assert abs(O.solve_exact(a, a, Chat) - 0.5) < 1e-12
    ap = O.map_distribution(Z, a)
    assert abs(O.solve_exact(ap, ap, Cs)) < 1e-12


def test_prop1_bound():
    """Eq. (7) P:157 (tested as <=, R#16) and the tighter max|C_hat - C| the proof gives."""
    rng = np.random.default_rng(41)
    for _ in range(40):
        X, Y, Wa, a, b = _random_one_hot_instance(rng)
        k = Wa.shape[0]
        Cs = O.euclidean_cost(Wa, Wa)
        C = O.euclidean_cost(X, Y)
        zx, zy = O.map_assign(X, Wa), O.map_assign(Y, Wa)
        Chat = O.reconstructed_cost(O.one_hot(zx, k), Cs, O.one_hot(zy, k))
        ap = O.histograms(zx, a, np.array([0, len(a)]), k)[0]
        bp = O.histograms(zy, b, np.array([0, len(b)]), k)[0]
        gap = abs(O.solve_exact(ap, bp, Cs) - O.solve_exact(a, b, C))
        assert gap <= O.prop1_bound(Chat, C) + 1e-9
        assert gap <= np.abs(Chat - C).max() + 1e-9


def test_prop2_bound_euclidean():
    """Prop. 2 P:212-218 with Euclidean C_s and C, one-hot nearest-anchor P_o."""
    rng = np.random.default_rng(51)
    for _ in range(40):
        X, Y, Wa, a, b = _random_one_hot_instance(rng)
        k = Wa.shape[0]
        Cs = O.euclidean_cost(Wa, Wa)
        zx, zy = O.map_assign(X, Wa), O.map_assign(Y, Wa)
        ap = O.histograms(zx, a, np.array([0, len(a)]), k)[0]
        bp = O.histograms(zy, b, np.array([0, len(b)]), k)[0]
        gap = abs(O.solve_exact(ap, bp, Cs) - O.solve_exact(a, b, O.euclidean_cost(X, Y)))
        rx = np.linalg.norm(Wa[zx] - X, axis=1)
        ry = np.linalg.norm(Wa[zy] - Y, axis=1)
        assert gap <= O.prop2_bound(rx, ry) + 1e-9
    # zero residuals (anchors = samples) => bound 0 and W_AS = W_1 (acceptance #6)
    X = rng.normal(size=(4, 2)); Y = rng.normal(size=(5, 2))
    Wa = np.concatenate([X, Y])
    a = rng.dirichlet(np.ones(4)); b = rng.dirichlet(np.ones(5))
    zx, zy = O.map_assign(X, Wa), O.map_assign(Y, Wa)
    ap = O.histograms(zx, a, np.array([0, 4]), 9)[0]
    bp = O.histograms(zy, b, np.array([0, 5]), 9)[0]
    assert abs(O.solve_exact(ap, bp, O.euclidean_cost(Wa, Wa)) - O.solve_exact(a, b, O.euclidean_cost(X, Y))) < 1e-9


# ------------------------------------------------------------------ mapping
def test_map_special_cases():
    W = np.array([[0, 0], [2, 0], [0, 2], [2, 0]], np.float32)      # anchor 3 duplicates anchor 1
    X = np.array([[0, 0], [2, 0], [0, 2], [1, 0], [1, 1]], np.float32)
    # exact anchor -> itself; duplicate -> lower index; midpoint (1,0) between 0 and 1 -> 0;
    # (1,1) equidistant from 0,1,2,3 -> 0
    np.testing.assert_array_equal(O.map_assign(X, W), [0, 1, 2, 0, 0])


def test_map_matches_exact_rational_argmin():
    """Brute force in exact rational arithmetic: the fp64 pinned formula must pick the exact
    argmin (lowest index on exact ties) wherever the exact gap exceeds fp64 error."""
    rng = np.random.default_rng(61)
    X = rng.normal(size=(60, 5)).astype(np.float32)
    W = rng.normal(size=(17, 5)).astype(np.float32)
    W[5] = W[3]                                                     # exact duplicate
    X[7] = W[11]
    got = O.map_assign(X, W)
    for p in range(X.shape[0]):
        xs = [Fraction(float(v)) for v in X[p]]
        dist = [sum((xs[k] - Fraction(float(W[j, k]))) ** 2 for k in range(5)) for j in range(W.shape[0])]
        best = min(dist)
        assert got[p] == dist.index(best)


# ------------------------------------------------------------------ histograms
def test_histogram_properties():
    rng = np.random.default_rng(71)
    N, K = 9, 6
    sizes = rng.integers(1, 12, N)
    offsets = np.concatenate([[0], np.cumsum(sizes)])
    T = offsets[-1]
    assign = rng.integers(0, K, T).astype(np.int32)
    w = np.concatenate([rng.dirichlet(np.ones(s)) for s in sizes])
    H = O.histograms(assign, w, offsets, K)
    for i in range(N):
        s, e = offsets[i], offsets[i + 1]
        assert abs(H[i].sum() - w[s:e].sum()) < 1e-14              # mass preserved
        np.testing.assert_allclose(H[i], O.map_distribution(O.one_hot(assign[s:e], K), w[s:e]), atol=1e-15)
        # sequential point-order fp64 accumulation per bin
        ref = [0.0] * K
        for p in range(s, e):
            ref[assign[p]] += float(w[p])
        assert list(H[i]) == ref
    # Z = I => a' = a; 1/n NOT applied (R#1): a uniform 3-point set keeps total mass 1
    a = rng.dirichlet(np.ones(K))
    np.testing.assert_array_equal(O.histograms(np.arange(K, dtype=np.int32), a, np.array([0, K]), K)[0], a)


# ------------------------------------------------------------------ matrix
def test_distance_matrix_properties():
    from asot_inputs import make_inputs

    inp = make_inputs("c1", n_dist=14)
    D, assign, H = O.distance_matrix(inp.points, inp.offsets, inp.weights, inp.anchors,
                                     inp.cost, inp.eps, inp.iters)
    N = inp.n_dist
    assert np.all(np.diag(D) == 0)
    np.testing.assert_array_equal(D, D.T)
    assert np.all(D >= 0)
    off = D[~np.eye(N, dtype=bool)]
    assert np.all(off > 0) and np.all(off <= 1.0)        # costs normalised to [0, 1]
    # permuting distributions permutes D
    perm = np.random.default_rng(0).permutation(N)
    pi, pj = O.upper_pairs(N)
    Hp = H[perm]
    c, _ = O.pair_costs(Hp, inp.cost, inp.eps, inp.iters, pi, pj)
    Dp = np.zeros_like(D); Dp[pi, pj] = c; Dp[pj, pi] = c
    # entries (perm[i], perm[j]) of D equal Dp[i, j] up to orientation (finite L: R#10)
    for i, j in zip(pi, pj):
        a, b = perm[i], perm[j]
        ref = D[a, b]
        assert abs(Dp[i, j] - ref) <= 5e-2 * ref        # orientation changes d slightly at finite L
        if a < b:
            assert abs(Dp[i, j] - ref) <= 1e-12
