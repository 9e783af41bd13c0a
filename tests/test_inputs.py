"""The seeded input generator (shared by oracle and CUDA path) follows the BASELINE.json recipes."""
import numpy as np
import pytest

from asot_inputs import CONFIGS, make_inputs, random_pairs


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_recipe_shapes_and_invariants(cfg):
    p = CONFIGS[cfg]
    inp = make_inputs(cfg, n_dist=12)
    assert inp.points.dtype == np.float32 and inp.points.shape[1] == p["d"]
    assert inp.anchors.shape == (p["K"], p["d"])
    assert inp.offsets[0] == 0 and inp.offsets[-1] == inp.points.shape[0]
    sizes = np.diff(inp.offsets)
    assert sizes.min() >= p["n_lo"] and sizes.max() <= p["n_hi"]
    for i in range(inp.n_dist):
        w = inp.weights[inp.offsets[i]:inp.offsets[i + 1]].astype(np.float64)
        assert np.all(w >= 0) and abs(w.sum() - 1.0) <= 1e-5
    C = inp.cost
    assert C.dtype == np.float32 and C.shape == (p["K"], p["K"])
    np.testing.assert_array_equal(C, C.T)
    assert np.all(np.diag(C) == 0) and C.max() == np.float32(1.0) and C.min() >= 0
    assert inp.eps == np.float32(0.05) and inp.iters == p["L"]
    # max(C)/eps = 20 <= 80 keeps the fp32 Gibbs kernel above FLT_MIN (R#12)
    assert float(C.max()) / float(inp.eps) <= 80


def test_determinism():
    a = make_inputs("c2", n_dist=20)
    b = make_inputs("c2", n_dist=20)
    np.testing.assert_array_equal(a.points, b.points)
    np.testing.assert_array_equal(a.cost, b.cost)
    c = make_inputs("c2", n_dist=20, seed=99)
    assert not np.array_equal(a.points, c.points)


def test_random_pairs():
    i, j = random_pairs(50, 300, seed=3)
    assert len(i) == 300 and np.all(i < j) and np.all(j < 50)
    assert len(set(zip(i.tolist(), j.tolist()))) == 300
