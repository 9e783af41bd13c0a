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
