"""GPU parity of NEXT-3 (exact anchor-space OT per pair, fp64 min-cost flow on the histogram
supports) against the oracle's exact LP (scipy HiGHS on the same renormalised marginals,
oracle.asot_oracle.solve_exact), through the C ABI."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from asot_inputs import make_inputs, random_pairs  # noqa: E402
from oracle import asot_oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def asot():
    import paper_2310_16123_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("cfg,n,npairs", [("c1", 64, 300), ("c2", 120, 150), ("c3", 200, 200),
                                          ("c4", 150, 60)])
def test_exact_asot_vs_lp(asot, cfg, n, npairs):
    inp = make_inputs(cfg, n_dist=n)
    _, H = O.map_and_histogram(inp.points, inp.offsets, inp.weights, inp.anchors)
    H32 = H.astype(np.float32)
    pi, pj = random_pairs(n, npairs, seed=11)
    pi = np.concatenate([pi, pj[:3], pi[:2]]).astype(np.int32)   # + reversed and self pairs
    pj = np.concatenate([pj, pi[:3], pi[:2]]).astype(np.int32)
    st = asot.asot.new_status()
    d = asot.exact_asot_pairs(dev(H32), dev(inp.cost), dev(pi), dev(pj), status=st).cpu().numpy()
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    C = inp.cost.astype(np.float64)
    for q in range(len(pi)):
        a, b = H32[pi[q]].astype(np.float64), H32[pj[q]].astype(np.float64)
        sa, sb = a > 0, b > 0
        ref = O.solve_exact(a[sa], b[sb], C[np.ix_(sa, sb)])
        assert abs(d[q] - ref) <= 1e-9 + 1e-9 * abs(ref), (q, d[q], ref)
    assert np.all(d[-2:] == 0.0) or np.allclose(d[-2:], 0.0, atol=1e-12)   # self pairs


def test_exact_asot_large_supports(asot):
    """c5 (K = 1024, supports of ~380 bins): the CTA-per-pair solver, against the oracle LP, plus
    a mixed list (a K = 1024 histogram pair next to an invalid index)."""
    inp = make_inputs("c5", n_dist=4)
    _, H = O.map_and_histogram(inp.points, inp.offsets, inp.weights, inp.anchors)
    H32 = H.astype(np.float32)
    assert (H32 > 0).sum(1).max() > 128
    pi = np.array([0, 1, 2, 3, -1], np.int32)
    pj = np.array([1, 2, 3, 0, 2], np.int32)
    st = asot.asot.new_status()
    d = asot.exact_asot_pairs(dev(H32), dev(inp.cost), dev(pi), dev(pj), status=st).cpu().numpy()
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    assert np.isnan(d[-1])
    C = inp.cost.astype(np.float64)
    for q in range(4):
        a, b = H32[pi[q]].astype(np.float64), H32[pj[q]].astype(np.float64)
        sa, sb = a > 0, b > 0
        ref = O.solve_exact(a[sa], b[sb], C[np.ix_(sa, sb)])
        assert abs(d[q] - ref) <= 1e-9 + 1e-9 * abs(ref), (q, d[q], ref)
