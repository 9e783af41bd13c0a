"""Pins for the soft-mapping oracle (oracle/soft_oracle.py) against what the
paper and the mathematics fix: SPEC worked examples, closed forms for orthonormal dictionaries,
the Eq. (8) minimiser from an independent bound-constrained solver, the monotone decrease of the
Eq. (8) objective (proximal gradient with step 1 <= 1/||W||_2^2), reduction to the pinned one-hot
histograms, Euclidean special cases of the Mahalanobis cost and the soft Lemma-1 inequality."""
import numpy as np
import pytest
from scipy.optimize import minimize

from asot_inputs.soft import make_dl_inputs, make_ml_model
from oracle import asot_oracle as O
from oracle import soft_oracle as S


def test_golden_simplex_shrink(golden):
    for key in ("simplex_shrink_theta0", "simplex_shrink_theta03"):
        g = golden[key]
        np.testing.assert_array_equal(S.simplex_shrink(np.array(g["a"]), g["theta"]), g["out"])
    a = np.random.default_rng(0).normal(size=50)
    once = S.simplex_shrink(a, 0.3)   # idempotence S_0(S_theta(a)) = S_theta(a)
    np.testing.assert_array_equal(S.simplex_shrink(once, 0.0), once)
    assert np.all(once >= 0)


def test_golden_near_onehot_layer(golden):
    g = golden["near_onehot_identity_step"]
    out = S.near_onehot_layer(np.array(g["z"], float), np.array(g["x"], float), np.array(g["W"], float),
                              g["lambda"])
    np.testing.assert_array_equal(out, g["out"])


def test_layer_fixed_point_is_eq8_minimiser():
    """Iterating Eq. (9) with a fixed lambda converges to argmin_{z>=0} 1/2||Wz-x||^2 + lambda 1^T z
    (appendix); the minimiser comes from scipy's L-BFGS-B, which shares nothing
    with the layer.  A wrong sign on lambda, a transposed W or a missing clamp moves the limit."""
    rng = np.random.default_rng(1)
    for trial in range(4):
        d, k = 6, 9
        W = rng.normal(size=(d, k))
        W /= np.linalg.norm(W, 2) * 1.05          # ||W||_2 < 1: step size 1 is stable (R#28)
        x = rng.normal(size=d)
        lam = 0.05 * (trial + 1)
        z = np.zeros(k)
        for _ in range(20000):
            z = S.near_onehot_layer(z, x, W, lam)
        f = lambda v: S.eq8_objective(v, x, W, lam)
        grad = lambda v: W.T @ (W @ v - x) + lam
        res = minimize(f, np.full(k, 0.1), jac=grad, method="L-BFGS-B", bounds=[(0, None)] * k,
                       options=dict(ftol=1e-15, gtol=1e-13, maxiter=10000))
        assert f(z) <= res.fun + 1e-10
        np.testing.assert_allclose(z, res.x, atol=2e-5)


def test_layer_objective_non_increasing():
    """Proximal gradient with step 1 <= 1/||W||_2^2 never increases Eq. (8)."""
    rng = np.random.default_rng(2)
    d, k = 10, 30
    W = rng.normal(size=(d, k))
    W /= np.linalg.norm(W, 2)
    x = rng.normal(size=d)
    z = np.abs(rng.normal(size=k))
    prev = S.eq8_objective(z, x, W, 0.02)
    for _ in range(200):
        z = S.near_onehot_layer(z, x, W, 0.02)
        cur = S.eq8_objective(z, x, W, 0.02)
        assert cur <= prev + 1e-12
        prev = cur


def test_dl_encode_orthonormal_dictionary_closed_form():
    """Orthonormal W (k = d), x = w_j: z^1 = max(0, e_j - lambda) = (1 - lambda) e_j, and e_j is
    a fixed direction of every later layer, so the normalised code is exactly e_j."""
    rng = np.random.default_rng(3)
    d = 8
    Q, _ = np.linalg.qr(rng.normal(size=(d, d)))
    dictionary = Q.T                                     # rows = anchors = columns of W = Q
    lam_layers = [(np.zeros((d, 4)), np.zeros(4)), (np.zeros((4, 1)), np.array([np.log(np.expm1(0.1))]))]
    for j in range(d):
        Z, flags, lam = S.dl_encode(dictionary[j][None, :], dictionary, lam_layers, 20)
        np.testing.assert_allclose(lam, [0.1], rtol=1e-14)
        assert not flags[0]
        e = np.zeros(d); e[j] = 1.0
        np.testing.assert_allclose(Z[0], e, atol=1e-12)


def test_dl_encode_total_suppression_fallback():
    """lambda larger than every |W^T x| suppresses every layer -> the uniform fallback row."""
    inp, m = make_dl_inputs("c2", n_dist=3)
    big = [(m.V1, m.c1), (np.zeros_like(m.v2), np.array([50.0], np.float32))]
    Z, flags, _ = S.dl_encode(inp.points[:5], m.dictionary, big, 20)
    assert flags.all()
    np.testing.assert_allclose(Z, 1.0 / inp.n_anchors)


def test_dl_encode_rows_on_simplex_and_lambda_positive():
    inp, m = make_dl_inputs("c2", n_dist=4)
    Z, flags, lam = S.dl_encode(inp.points, m.dictionary, m.lam_layers, m.n_layers)
    assert np.all(lam > 0) and not flags.any()
    assert np.all(Z >= 0)
    np.testing.assert_allclose(Z.sum(1), 1.0, atol=1e-12)


def test_mlp_forward_hand_computed():
    """2 -> 3 -> 1 network evaluated by hand:
    h = relu([1, -2] @ [[1, 0, 2], [1, 1, -1]] + [0.5, 0, -1]) = relu([-0.5, -2, 3]) = [0, 0, 3];
    o = [0, 0, 3] @ [[1], [2], [-0.5]] + 0.25 = -1.25.  Zero weights and biases give 0."""
    layers = [(np.array([[1.0, 0, 2], [1, 1, -1]]), np.array([0.5, 0, -1])),
              (np.array([[1.0], [2], [-0.5]]), np.array([0.25]))]
    np.testing.assert_array_equal(S.mlp_forward(np.array([[1.0, -2.0]]), layers), [[-1.25]])
    zero = [(np.zeros((2, 3)), np.zeros(3)), (np.zeros((3, 1)), np.zeros(1))]
    np.testing.assert_array_equal(S.mlp_forward(np.ones((4, 2)), zero), np.zeros((4, 1)))


def test_ml_encode_simplex_fallback_and_one_hot():
    m = make_ml_model(8, 12)
    X = np.random.default_rng(4).normal(size=(50, 8))
    Z, flags = S.ml_encode(X, m.layers)
    assert not flags.any() and np.all(Z >= 0)
    np.testing.assert_allclose(Z.sum(1), 1.0, atol=1e-12)
    # zero mapper -> uniform rows, flagged
    zero = [(np.zeros((8, 16)), np.zeros(16)), (np.zeros((16, 12)), np.zeros(12))]
    Z0, f0 = S.ml_encode(X, zero)
    assert f0.all()
    np.testing.assert_allclose(Z0, 1.0 / 12)
    # a mapper whose output is -3 e_j (abs then l1: e_j), j chosen by the sign of x_0:
    # first layer relu(+x0), relu(-x0); second layer sends them to anchors 2 and 5
    W1 = np.zeros((8, 2)); W1[0, 0] = 1.0; W1[0, 1] = -1.0
    W2 = np.zeros((2, 12)); W2[0, 2] = -3.0; W2[1, 5] = 7.0
    Zh, fh = S.ml_encode(X, [(W1, np.zeros(2)), (W2, np.zeros(12))])
    assign = np.where(X[:, 0] > 0, 2, 5)
    np.testing.assert_array_equal(Zh, O.one_hot(assign.astype(np.int32), 12))


def test_soft_histograms_reduce_to_pinned_one_hot_histograms():
    """One-hot Z: a' = Z^T a equals the pinned point-order histogram; Z = I gives
    a' = a; the mass is preserved for any simplex rows."""
    rng = np.random.default_rng(5)
    offsets = np.array([0, 7, 7 + 13, 20 + 4])
    w = rng.random(24); 
    for i in range(3):
        w[offsets[i]:offsets[i + 1]] /= w[offsets[i]:offsets[i + 1]].sum()
    assign = rng.integers(0, 10, size=24).astype(np.int32)
    np.testing.assert_allclose(S.soft_histograms(O.one_hot(assign, 10), w, offsets),
                               O.histograms(assign, w, offsets, 10), atol=1e-15)
    a = w[:7]
    np.testing.assert_allclose(S.soft_histograms(np.eye(7), a, np.array([0, 7]))[0], a, atol=1e-15)
    Z = rng.random((24, 10)); Z /= Z.sum(1, keepdims=True)
    np.testing.assert_allclose(S.soft_histograms(Z, w, offsets).sum(1), 1.0, atol=1e-14)


def test_golden_mahalanobis(golden):
    for key in ("mahalanobis_identity_345", "mahalanobis_diag2_345"):
        g = golden[key]
        np.testing.assert_allclose(S.mahalanobis_cost(np.array(g["anchors"], float), np.array(g["M"], float)),
                                   g["C_s"], atol=1e-14)


def test_mahalanobis_orthogonal_invariance_and_normalisation():
    """M orthogonal: ||M(w_u - w_v)|| = ||w_u - w_v|| -- equals the (independently pinned) Euclidean
    cost; normalisation divides by the max so the largest entry is exactly 1."""
    rng = np.random.default_rng(6)
    A = rng.normal(size=(9, 5))
    Q, _ = np.linalg.qr(rng.normal(size=(5, 5)))
    np.testing.assert_allclose(S.mahalanobis_cost(A, Q), O.euclidean_cost(A, A), atol=1e-12)
    Cn = S.mahalanobis_cost(A, rng.normal(size=(5, 5)), normalize=True)
    assert Cn.max() == 1.0 and np.all(np.diag(Cn) == 0) and np.allclose(Cn, Cn.T)


def test_soft_lemma1_inequality():
    """For soft P only W_AS <= LP(a, b, Z_x C_s Z_y^T) holds: every plan T of
    the original problem maps to the feasible anchor plan Z_x^T T Z_y of the same cost."""
    rng = np.random.default_rng(7)
    for _ in range(20):
        n, m, k = 4, 5, 3
        Zx = rng.random((n, k)); Zx /= Zx.sum(1, keepdims=True)
        Zy = rng.random((m, k)); Zy /= Zy.sum(1, keepdims=True)
        A = rng.normal(size=(k, 2))
        Cs = O.euclidean_cost(A, A)
        a = rng.random(n); a /= a.sum()
        b = rng.random(m); b /= b.sum()
        ap, bp = S.soft_histograms(Zx, a, np.array([0, n]))[0], S.soft_histograms(Zy, b, np.array([0, m]))[0]
        w_as = O.solve_exact(ap / ap.sum(), bp / bp.sum(), Cs)
        lp_hat = O.solve_exact(a, b, O.reconstructed_cost(Zx, Cs, Zy))
        assert w_as <= lp_hat + 1e-9
