"""Pins for the NEXT-2 mini-batch k-means oracle (oracle/kmeans_oracle.py): the SPEC's worked
example, exact agreement of the batched running-mean update with Sculley's point-by-point
eta = 1/v update in rational arithmetic, the first full batch = one Lloyd step, zero inertia with
k = #distinct samples, and convergence near scikit-learn's full-batch Lloyd on blobs."""
import numpy as np
import pytest

from asot_inputs import normalized_sqeuclid_cost
from asot_inputs.soft import make_kmeans_draws
from oracle import kmeans_oracle as KM


def test_spec_separable_example():
    """{(0,0),(0,0),(10,10)}, k = 2 -> centers {(0,0),(10,10)}, zero inertia."""
    X = np.array([[0, 0], [0, 0], [10, 10]], np.float32)
    C, A, v = KM.kmeans_minibatch(X, X[[0, 2]], np.array([[0, 1, 2], [2, 1, 0]]))
    np.testing.assert_array_equal(A, [[0, 0], [10, 10]])
    assert KM.inertia(X, A) == 0.0 and list(v) == [4, 2]


def test_batched_update_equals_pointwise_sculley_exactly():
    rng = np.random.default_rng(0)
    centres = np.array([[0, 0, 0], [20, 0, 5], [0, 25, -10]], np.float64)
    X = (centres[rng.integers(0, 3, size=60)] + rng.integers(-3, 4, size=(60, 3))).astype(np.float32)
    init = X[[0, 1, 2]].copy()
    init[:] = centres.astype(np.float32) + 1.0
    batches = rng.integers(0, 60, size=(5, 17))
    C, _, v = KM.kmeans_minibatch(X, init, batches)
    Cq, vq = KM.sculley_pointwise(X, init, batches)
    assert list(v) == vq
    np.testing.assert_allclose(C, np.array([[float(t) for t in row] for row in Cq]), rtol=1e-14, atol=1e-14)


def test_first_full_batch_is_a_lloyd_step():
    rng = np.random.default_rng(1)
    X = rng.normal(size=(200, 4)).astype(np.float32)
    init = X[:5].copy()
    C, _, v = KM.kmeans_minibatch(X, init, np.arange(200)[None, :])
    d = ((X[:, None, :].astype(np.float64) - init[None].astype(np.float64)) ** 2).sum(-1)
    a = d.argmin(1)
    for j in range(5):
        assert v[j] == (a == j).sum()
        np.testing.assert_allclose(C[j], X[a == j].astype(np.float64).mean(0), rtol=1e-13, atol=1e-14)


def test_k_equals_distinct_samples_zero_inertia():
    X = np.repeat(np.array([[1, 2], [5, 5], [-3, 7], [9, -1]], np.float32), 5, axis=0)
    init = X[[0, 5, 10, 15]]
    _, A, _ = KM.kmeans_minibatch(X, init, np.random.default_rng(2).integers(0, 20, size=(4, 8)))
    assert KM.inertia(X, A) == 0.0


def test_blobs_inertia_near_full_batch_lloyd():
    """3 Gaussian blobs, 300 points, k = 3 -> inertia within 5% of Lloyd's algorithm
    (scikit-learn KMeans from the same initial centers, run to convergence; shares nothing with
    the oracle)."""
    sklearn = pytest.importorskip("sklearn.cluster")
    rng = np.random.default_rng(3)
    means = np.array([[0, 0], [6, 1], [2, 7]], np.float64)
    X = (means[np.repeat(np.arange(3), 100)] + rng.normal(size=(300, 2))).astype(np.float32)
    init, batches = make_kmeans_draws(X, 3, iters=60, batch=64, seed=4)
    _, A, _ = KM.kmeans_minibatch(X, init, batches)
    ref = sklearn.KMeans(3, init=init.astype(np.float64), n_init=1).fit(X.astype(np.float64)).inertia_
    assert KM.inertia(X, A) <= 1.05 * ref


def test_sqeuclid_cost():
    A = np.array([[0, 0], [3, 4]], np.float32)
    np.testing.assert_array_equal(KM.sqeuclid_cost(A, normalize=False), [[0, 25], [25, 0]])
    B = np.random.default_rng(5).normal(size=(12, 3)).astype(np.float32)
    np.testing.assert_allclose(KM.sqeuclid_cost(B), normalized_sqeuclid_cost(B), rtol=1e-6)
