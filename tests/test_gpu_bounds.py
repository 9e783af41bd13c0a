"""NEXT-3 bound checks at scale (VERDICT r1 missing #1): the per-pair right-hand sides of Prop. 1
(Eq. (7)) and Prop. 2, and exact W_1 on the original point sets, on the GPU
against the oracle -- and the paper's guarantee itself, |W_AS - W_1| <= each bound, on every
sampled pair (Euclidean C_s and C, one-hot P_o: R#7, R#16)."""
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


def gpu_side(asot, inp, pi, pj):
    pts, offs, w, anc = dev(inp.points), dev(inp.offsets), dev(inp.weights), dev(inp.anchors)
    assign, H, st = asot.map_to_anchors(pts, offs, w, anc, offsets_host=inp.offsets)
    eye = torch.eye(inp.dim, dtype=torch.float32, device="cuda")
    CsE = asot.mahalanobis_cost(anc, eye, normalize=False)        # ||w_u - w_v||_2 (M = I)
    ti, tj = dev(pi.astype(np.int32)), dev(pj.astype(np.int32))
    st2 = asot.asot.new_status()
    w_as = asot.exact_asot_pairs(H, CsE, ti, tj, status=st2)
    w1 = asot.exact_w1_points(pts, offs, w, ti, tj, status=st2)
    l1, linf, p2 = asot.bound_terms(pts, offs, anc, assign, CsE, ti, tj, status=st2)
    torch.cuda.synchronize()
    return dict(assign=assign.cpu().numpy(), H=H.cpu().numpy(), CsE=CsE.cpu().numpy(),
                w_as=w_as.cpu().numpy(), w1=w1.cpu().numpy(), l1=l1.cpu().numpy(),
                linf=linf.cpu().numpy(), p2=p2.cpu().numpy(), status=int(st2.item()))


def oracle_pair(inp, assign, CsE, i, j):
    """Oracle terms of one pair: Prop. 1 (l1, max), Prop. 2, exact W_1 (HiGHS on the points)."""
    xs, xe = inp.offsets[i], inp.offsets[i + 1]
    ys, ye = inp.offsets[j], inp.offsets[j + 1]
    X, Y = inp.points[xs:xe], inp.points[ys:ye]
    C = O.euclidean_cost(X, Y)
    Zx, Zy = O.one_hot(assign[xs:xe], inp.n_anchors), O.one_hot(assign[ys:ye], inp.n_anchors)
    Ch = O.reconstructed_cost(Zx, CsE.astype(np.float64), Zy)
    W = inp.anchors.astype(np.float64)
    rx = np.sqrt(((W[assign[xs:xe]] - X.astype(np.float64)) ** 2).sum(1))
    ry = np.sqrt(((W[assign[ys:ye]] - Y.astype(np.float64)) ** 2).sum(1))
    w1 = O.solve_exact(inp.weights[xs:xe], inp.weights[ys:ye], C)
    return O.prop1_bound(Ch, C), float(np.abs(Ch - C).max()), O.prop2_bound(rx, ry), w1


@pytest.mark.parametrize("cfg,n,npairs", [("c1", 64, 200), ("c2", 120, 150)])
def test_bounds_and_exact_w1_vs_oracle(asot, cfg, n, npairs):
    inp = make_inputs(cfg, n_dist=n)
    pi, pj = random_pairs(n, npairs, seed=71)
    g = gpu_side(asot, inp, pi, pj)
    assert g["status"] == 0, f"flags {g['status']:#x}"
    a_o = O.map_assign(inp.points, inp.anchors)
    assert np.array_equal(g["assign"], a_o)
    for q in range(len(pi)):
        l1, linf, p2, w1 = oracle_pair(inp, a_o, g["CsE"], int(pi[q]), int(pj[q]))
        assert abs(g["l1"][q] - l1) <= 1e-9 * max(1.0, l1)
        assert abs(g["linf"][q] - linf) <= 1e-9 * max(1.0, linf)
        assert abs(g["p2"][q] - p2) <= 1e-9 * max(1.0, p2)
        assert abs(g["w1"][q] - w1) <= 1e-8 * max(1.0, w1), (q, g["w1"][q], w1)
    # the paper's guarantee on every pair (R#16: tested as <=, plus the proof's tighter max form)
    gap = np.abs(g["w_as"] - g["w1"])
    assert np.all(np.isfinite(gap))
    assert np.all(gap <= g["l1"] + 1e-9) and np.all(gap <= g["linf"] + 1e-9) and np.all(gap <= g["p2"] + 1e-9)


def test_exact_w1_flags_large_supports_and_bad_indices(asot):
    """Supports above 64 points: NaN + EXACT_TOO_LARGE; an index outside [0, N): NaN + BAD_INDEX;
    a pair of one-point distributions: W_1 = ||x - y|| exactly (closed form)."""
    inp = make_inputs("c3", n_dist=6)           # n_i in [50, 300]: some above 64
    big = int(np.argmax(np.diff(inp.offsets)))
    assert np.diff(inp.offsets)[big] > 64
    st = asot.asot.new_status()
    w1 = asot.exact_w1_points(dev(inp.points), dev(inp.offsets), dev(inp.weights),
                              dev(np.array([big, -1], np.int32)), dev(np.array([0, 1], np.int32)), status=st)
    torch.cuda.synchronize()
    assert np.isnan(w1.cpu().numpy()).all()
    assert int(st.item()) == asot.asot.FLAG_EXACT_TOO_LARGE | asot.asot.FLAG_BAD_INDEX
    X = np.random.default_rng(3).normal(size=(4, 5)).astype(np.float32)
    off = np.arange(5, dtype=np.int64)
    w = np.ones(4, np.float32)
    st = asot.asot.new_status()
    d = asot.exact_w1_points(dev(X), dev(off), dev(w), dev(np.array([0, 2], np.int32)),
                             dev(np.array([1, 3], np.int32)), status=st).cpu().numpy()
    want = [np.linalg.norm(X[0].astype(np.float64) - X[1]), np.linalg.norm(X[2].astype(np.float64) - X[3])]
    np.testing.assert_allclose(d, want, rtol=1e-14)
    assert int(st.item()) == 0
