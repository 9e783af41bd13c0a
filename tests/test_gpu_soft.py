"""GPU parity of the NEXT-1 soft mappings (ASOT-ML / ASOT-DL inference, Mahalanobis cost) against
the fp64 oracle (oracle/soft_oracle.py), through the C ABI, and the soft H fed to the unchanged
Sinkhorn path (asot_distance_matrix with hist_in)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from asot_inputs import make_inputs  # noqa: E402
from asot_inputs.soft import make_dl_inputs, make_ml_model  # noqa: E402
from oracle import asot_oracle as O  # noqa: E402
from oracle import soft_oracle as S  # noqa: E402

# fp32 CUDA-core arithmetic vs fp64: codes and marginals within 1e-5 absolute (rows sum to 1),
# distances within the north star's bars (fp32 1e-4, TF32 2e-3)
CODE_TOL = 1e-5
TOL = {0: 1e-4, 1: 2e-3}


@pytest.fixture(scope="module")
def asot():
    import paper_2310_16123_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def rel_err(Dg, Do, floor=1e-3):
    return np.abs(Dg.astype(np.float64) - Do) / np.maximum(Do, floor)


@pytest.mark.parametrize("cfg,n", [("c1", 30), ("c2", 40), ("c3", 12), ("c5", 4)])
def test_soft_ml_codes_and_histograms(asot, cfg, n):
    inp = make_inputs(cfg, n_dist=n)
    m = make_ml_model(inp.dim, inp.n_anchors)
    H, Z, st = asot.map_soft_ml(dev(inp.points), dev(inp.offsets), dev(inp.weights), dev(m.W1),
                                dev(m.b1), dev(m.W2), dev(m.b2), offsets_host=inp.offsets,
                                want_codes=True)
    torch.cuda.synchronize()
    asot.check_status(st)
    Zo, flags = S.ml_encode(inp.points, m.layers)
    assert not flags.any()
    np.testing.assert_allclose(Z.cpu().numpy(), Zo, rtol=0, atol=CODE_TOL)
    Ho = S.soft_histograms(Zo, inp.weights, inp.offsets)
    np.testing.assert_allclose(H.cpu().numpy(), Ho, rtol=0, atol=CODE_TOL)


@pytest.mark.parametrize("cfg,n", [("c1", 30), ("c2", 30), ("c3", 8), ("c5", 3)])
def test_soft_dl_codes_and_histograms(asot, cfg, n):
    """c5 (K = 1024, d = 128) streams the dictionary through SMEM; the others keep it resident."""
    inp, m = make_dl_inputs(cfg, n_dist=n)
    H, Z, st = asot.map_soft_dl(dev(inp.points), dev(inp.offsets), dev(inp.weights), dev(m.dictionary),
                                dev(m.V1), dev(m.c1), dev(m.v2.reshape(-1)), dev(m.c2), m.n_layers,
                                offsets_host=inp.offsets, want_codes=True)
    torch.cuda.synchronize()
    asot.check_status(st)
    Zo, flags, _ = S.dl_encode(inp.points, m.dictionary, m.lam_layers, m.n_layers)
    assert not flags.any()
    np.testing.assert_allclose(Z.cpu().numpy(), Zo, rtol=0, atol=CODE_TOL)
    Ho = S.soft_histograms(Zo, inp.weights, inp.offsets)
    np.testing.assert_allclose(H.cpu().numpy(), Ho, rtol=0, atol=CODE_TOL)


def test_soft_dl_fallback_flag(asot):
    """lambda above every |W^T x|: every code is suppressed -> uniform rows + SOFT_FALLBACK."""
    inp, m = make_dl_inputs("c2", n_dist=5)
    H, Z, st = asot.map_soft_dl(dev(inp.points), dev(inp.offsets), dev(inp.weights), dev(m.dictionary),
                                dev(m.V1), dev(m.c1), dev(np.zeros(m.v2.size, np.float32)),
                                dev(np.array([50.0], np.float32)), m.n_layers,
                                offsets_host=inp.offsets, want_codes=True)
    torch.cuda.synchronize()
    assert int(st.item()) & asot.asot.FLAG_SOFT_FALLBACK
    np.testing.assert_allclose(Z.cpu().numpy(), 1.0 / inp.n_anchors, rtol=1e-6)


@pytest.mark.parametrize("K,d", [(16, 8), (128, 32), (1024, 128)])
def test_mahalanobis_cost(asot, K, d):
    rng = np.random.default_rng(K)
    A = rng.normal(size=(K, d)).astype(np.float32)
    M = (rng.normal(size=(d, d)) / np.sqrt(d)).astype(np.float32)
    for norm in (False, True):
        C = asot.mahalanobis_cost(dev(A), dev(M), normalize=norm).cpu().numpy()
        Co = S.mahalanobis_cost(A, M, normalize=norm) if K <= 128 else None
        assert np.array_equal(C, C.T) and np.all(np.diag(C) == 0)
        if Co is not None:
            np.testing.assert_allclose(C, Co, rtol=2e-5, atol=1e-6)
        else:  # sampled entries at K = 1024
            for u, v in rng.integers(0, K, size=(200, 2)):
                diff = M.astype(np.float64) @ (A[u].astype(np.float64) - A[v].astype(np.float64))
                ref = np.sqrt(diff @ diff)
                if norm:
                    continue
                assert abs(C[u, v] - ref) <= 2e-5 * ref + 1e-6
        if norm:
            assert C.max() == 1.0


@pytest.mark.parametrize("prec", [0, 1])
def test_soft_distance_matrices_end_to_end(asot, prec):
    """Soft H (ML with its Mahalanobis C_s; DL with the dictionary's C_s) -> the unchanged
    Sinkhorn kernels (hist_in) -> D, vs the oracle chain at identical eps and L."""
    inp = make_inputs("c2", n_dist=36, iters=50)
    m = make_ml_model(inp.dim, inp.n_anchors)
    H, _, st = asot.map_soft_ml(dev(inp.points), dev(inp.offsets), dev(inp.weights), dev(m.W1),
                                dev(m.b1), dev(m.W2), dev(m.b2), offsets_host=inp.offsets)
    C = asot.mahalanobis_cost(dev(inp.anchors), dev(m.M), normalize=True)
    D = asot.distance_matrix(None, None, None, None, C, float(inp.eps), inp.iters, precision=prec,
                             hist=H, cost_max=1.0, status=st)
    torch.cuda.synchronize()
    asot.check_status(st)
    Zo, _ = S.ml_encode(inp.points, m.layers)
    Ho = S.soft_histograms(Zo, inp.weights, inp.offsets)
    Co = S.mahalanobis_cost(inp.anchors, m.M, normalize=True)
    pi, pj = O.upper_pairs(inp.n_dist)
    c, _ = O.pair_costs(Ho, Co, inp.eps, inp.iters, pi, pj)
    Do = np.zeros((inp.n_dist, inp.n_dist)); Do[pi, pj] = c; Do[pj, pi] = c
    eff = asot.effective_precision(inp.n_anchors, prec)
    assert rel_err(D.cpu().numpy(), Do).max() <= TOL[eff]

    dinp, dm = make_dl_inputs("c3", n_dist=20, iters=30)
    H, _, st = asot.map_soft_dl(dev(dinp.points), dev(dinp.offsets), dev(dinp.weights),
                                dev(dm.dictionary), dev(dm.V1), dev(dm.c1), dev(dm.v2.reshape(-1)),
                                dev(dm.c2), dm.n_layers, offsets_host=dinp.offsets)
    D = asot.distance_matrix(None, None, None, None, dev(dinp.cost), float(dinp.eps), dinp.iters,
                             precision=prec, hist=H, cost_max=1.0, status=st)
    torch.cuda.synchronize()
    asot.check_status(st)
    Zo, _, _ = S.dl_encode(dinp.points, dm.dictionary, dm.lam_layers, dm.n_layers)
    Ho = S.soft_histograms(Zo, dinp.weights, dinp.offsets)
    pi, pj = O.upper_pairs(dinp.n_dist)
    c, _ = O.pair_costs(Ho, dinp.cost, dinp.eps, dinp.iters, pi, pj)
    Do = np.zeros((dinp.n_dist, dinp.n_dist)); Do[pi, pj] = c; Do[pj, pi] = c
    eff = asot.effective_precision(dinp.n_anchors, prec)
    assert rel_err(D.cpu().numpy(), Do).max() <= TOL[eff]


@pytest.mark.parametrize("d,h,K", [(32, 64, 64), (64, 128, 256), (64, 192, 128), (128, 256, 1024)])
def test_soft_ml_tensor_core_ragged(asot, d, h, K):
    """The tcgen05 ML kernel (BF16x3 split operands, R#35) on ragged distributions around its
    128-point tile (1, 127, 128, 129, 300 points): codes and H within 1e-5 of the oracle and of
    the CUDA-core kernel (tensor_cores=False), status clean."""
    from asot_inputs.soft import make_ml_model
    rng = np.random.default_rng(d + h + K)
    sizes = np.array([1, 127, 128, 129, 300, 5])
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    X = rng.normal(0.0, 1.0, size=(off[-1], d)).astype(np.float32)
    w = np.concatenate([rng.dirichlet(np.ones(n)) for n in sizes]).astype(np.float32)
    m = make_ml_model(d, K)
    W1 = rng.normal(0.0, np.sqrt(2.0 / d), size=(d, h)).astype(np.float32)
    b1 = rng.normal(0.0, 0.1, size=h).astype(np.float32)
    W2 = rng.normal(0.0, np.sqrt(1.0 / h), size=(h, K)).astype(np.float32)
    b2 = m.b2
    args = (dev(X), dev(off), dev(w), dev(W1), dev(b1), dev(W2), dev(b2))
    assert asot.asot._lib_handle().asot_map_soft_ml_workspace_bytes(d, h, K) > 0
    H, Z, st = asot.map_soft_ml(*args, offsets_host=off, want_codes=True)
    Hc, Zc, stc = asot.map_soft_ml(*args, offsets_host=off, want_codes=True, tensor_cores=False)
    torch.cuda.synchronize()
    asot.check_status(st)
    asot.check_status(stc)
    Zo, flags = S.ml_encode(X, [(W1, b1), (W2, b2)])
    assert not flags.any()
    np.testing.assert_allclose(Z.cpu().numpy(), Zo, rtol=0, atol=CODE_TOL)
    np.testing.assert_allclose(Z.cpu().numpy(), Zc.cpu().numpy(), rtol=0, atol=CODE_TOL)
    Ho = S.soft_histograms(Zo, w, off)
    np.testing.assert_allclose(H.cpu().numpy(), Ho, rtol=0, atol=CODE_TOL)
    np.testing.assert_allclose(H.cpu().numpy(), Hc.cpu().numpy(), rtol=0, atol=CODE_TOL)
