"""GPU parity of NEXT-2 (ASOT-k anchor learning by mini-batch k-means) through the C ABI: the
learned centers and counts are bit-identical to the fp64 oracle's (same draws, pinned argmin,
batch-order fp64 sums, explicitly rounded running-mean update); the learned anchors then drive the
unchanged hot path."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from asot_inputs import make_inputs  # noqa: E402
from asot_inputs.soft import make_kmeans_draws  # noqa: E402
from oracle import asot_oracle as O  # noqa: E402
from oracle import kmeans_oracle as KM  # noqa: E402

TOL = {0: 1e-4, 1: 2e-3}


@pytest.fixture(scope="module")
def asot():
    import paper_2310_16123_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("cfg,n,iters,batch", [("c1", 64, 12, 64), ("c2", 200, 10, 700),
                                               ("c3", 40, 6, 1500), ("c5", 3, 3, 512)])
def test_kmeans_bit_exact(asot, cfg, n, iters, batch):
    inp = make_inputs(cfg, n_dist=n)
    init, bidx = make_kmeans_draws(inp.points, inp.n_anchors, iters, batch)
    C, A, v, st = asot.kmeans_minibatch(dev(inp.points), dev(init), dev(bidx))
    torch.cuda.synchronize()
    asot.check_status(st)
    Co, Ao, vo = KM.kmeans_minibatch(inp.points, init, bidx)
    np.testing.assert_array_equal(v.cpu().numpy(), vo)
    np.testing.assert_array_equal(C.cpu().numpy(), Co)      # fp64 centers, bitwise
    np.testing.assert_array_equal(A.cpu().numpy(), Ao)


def test_kmeans_zero_iterations_and_batch_over_1024(asot):
    inp = make_inputs("c2", n_dist=60)
    init, bidx = make_kmeans_draws(inp.points, inp.n_anchors, 2, 2500)
    C, A, v, _ = asot.kmeans_minibatch(dev(inp.points), dev(init), dev(bidx[:0]))
    np.testing.assert_array_equal(A.cpu().numpy(), init)
    assert int(v.sum()) == 0
    C, A, v, _ = asot.kmeans_minibatch(dev(inp.points), dev(init), dev(bidx))
    Co, Ao, vo = KM.kmeans_minibatch(inp.points, init, bidx)
    np.testing.assert_array_equal(C.cpu().numpy(), Co)
    assert int(v.sum()) == 2 * 2500


@pytest.mark.parametrize("K,d", [(16, 8), (256, 64), (1024, 128)])
def test_sqeuclid_cost(asot, K, d):
    A = np.random.default_rng(K).normal(size=(K, d)).astype(np.float32)
    C = asot.sqeuclid_cost(dev(A)).cpu().numpy()
    assert np.array_equal(C, C.T) and np.all(np.diag(C) == 0) and C.max() == 1.0
    Co = KM.sqeuclid_cost(A)
    np.testing.assert_allclose(C, Co, rtol=1e-5, atol=1e-7)


@pytest.mark.parametrize("prec", [0, 1])
def test_learned_anchors_end_to_end(asot, prec):
    inp = make_inputs("c2", n_dist=40, iters=60)
    init, bidx = make_kmeans_draws(inp.points, inp.n_anchors, 8, 512)
    _, A, _, st = asot.kmeans_minibatch(dev(inp.points), dev(init), dev(bidx))
    Cs = asot.sqeuclid_cost(A)
    D = asot.distance_matrix(dev(inp.points), dev(inp.offsets), dev(inp.weights), A, Cs,
                             float(inp.eps), inp.iters, precision=prec, offsets_host=inp.offsets,
                             cost_max=1.0, status=st)
    torch.cuda.synchronize()
    asot.check_status(st)
    _, Ao, _ = KM.kmeans_minibatch(inp.points, init, bidx)
    Do, _, _ = O.distance_matrix(inp.points, inp.offsets, inp.weights, Ao, KM.sqeuclid_cost(Ao),
                                 inp.eps, inp.iters)
    r = np.abs(D.cpu().numpy().astype(np.float64) - Do) / np.maximum(Do, 1e-3)
    assert r.max() <= TOL[asot.effective_precision(inp.n_anchors, prec)]
