"""Pins for the NEXT-4 eOT baseline oracle (oracle/eot_oracle.py): one-point distributions give
the ground cost exactly, identical one-point distributions give 0, and with small eps / many
iterations uniform n = m problems approach the brute-force permutation OT (Birkhoff) from above
within eps log n (entropic bound)."""
import numpy as np

from oracle import asot_oracle as O
from oracle import eot_oracle as E


def test_single_point_distributions_exact():
    X = np.array([[0.0, 0.0], [3.0, 4.0], [1.0, 1.0]], np.float32)
    offs = np.array([0, 1, 2, 3])
    w = np.ones(3, np.float32)
    d = E.eot_pair_costs(X, offs, w, np.float32(0.05), 7, [0, 0, 1, 2], [1, 2, 2, 2], 0.04)
    np.testing.assert_allclose(d[:3], [0.04 * 25, 0.04 * 2, 0.04 * 13], rtol=1e-14)
    assert d[3] == 0.0


def test_small_eps_approaches_permutation_ot():
    rng = np.random.default_rng(0)
    for n in (3, 4, 5):
        X = rng.normal(size=(2 * n, 3)).astype(np.float32)
        offs = np.array([0, n, 2 * n])
        w = np.full(2 * n, 1.0 / n)
        eps = 0.02
        d = E.eot_pair_costs(X, offs, w, eps, 20000, [0], [1], 0.1)[0]
        W = O.brute_force_perm_ot(E.sqeuclid_point_cost(X[:n], X[n:], 0.1))
        assert W - 1e-9 <= d <= W + eps * np.log(n) + 1e-6


def test_bds_two_pairs_of_sizes_2x3_and_4x2():
    """two pairs of sizes (2, 3) and (4, 2) through ONE stacked block-diagonal update
    sequence equal the per-pair Sinkhorn within 1e-10 (Sec. 2.4)."""
    rng = np.random.default_rng(3)
    X = rng.normal(size=(11, 3)).astype(np.float32)
    offs = np.array([0, 2, 5, 9, 11])                 # distributions of sizes 2, 3, 4, 2
    w = np.concatenate([rng.dirichlet(np.ones(n)) for n in (2, 3, 4, 2)]).astype(np.float32)
    pi, pj = [0, 2], [1, 3]
    d_bds = E.bds_eot_costs(X, offs, w, 0.1, 60, pi, pj, 0.3)
    d_one = E.eot_pair_costs(X, offs, w, 0.1, 60, pi, pj, 0.3)
    np.testing.assert_allclose(d_bds, d_one, rtol=0, atol=1e-10)


def test_bds_single_pair_and_ragged_batch():
    """S:128 one pair degenerates to the single Sinkhorn; a ragged batch of 12 pairs (sizes 1-9,
    repeated and reversed pairs) agrees pair by pair; S:129 a distribution against itself gives a
    cost below eps log(n m) (the entropic bound around the zero OT cost)."""
    rng = np.random.default_rng(4)
    sizes = rng.integers(1, 10, size=8)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    X = rng.normal(size=(offs[-1], 4)).astype(np.float32)
    w = np.concatenate([rng.dirichlet(np.ones(n)) for n in sizes]).astype(np.float32)
    d1 = E.bds_eot_costs(X, offs, w, 0.2, 30, [1], [5], 0.5)
    np.testing.assert_allclose(d1, E.eot_pair_costs(X, offs, w, 0.2, 30, [1], [5], 0.5), atol=1e-12)
    pi = [0, 1, 2, 3, 4, 5, 6, 7, 0, 3, 7, 2]
    pj = [1, 2, 3, 4, 5, 6, 7, 0, 1, 0, 6, 2]
    d_bds = E.bds_eot_costs(X, offs, w, 0.2, 30, pi, pj, 0.5)
    d_one = E.eot_pair_costs(X, offs, w, 0.2, 30, pi, pj, 0.5)
    np.testing.assert_allclose(d_bds, d_one, rtol=0, atol=1e-10)
    n2 = int(sizes[2])
    assert 0.0 <= d_bds[-1] <= 0.2 * np.log(max(n2, 2) ** 2) + 1e-9   # W = 0, eps log(n m)
