"""GPU parity over the whole accepted eps domain, max(C_s)/eps in {40, 50, 60, 80} (the ABI accepts
<= 80, R#12), on every Sinkhorn kernel family and both precisions, plus the S:62 clamp + flag.

At these ratios the Gibbs kernel spans e^-80 .. 1 and the Sinkhorn denominators of the configs'
data reach 1e-35 .. 1e21 (fp64 oracle, c1-c5): each stays inside fp32's normal range, but the
product of two of them does not -- the paired-reciprocal epilogue (one MUFU per two anchors) must
fall back to per-anchor reciprocals there.  No clamp may fire on real data
(status stays 0); a histogram with a 1e-30 mass drives a denominator below FLT_MIN and must raise
ASOT_FLAG_DENOM_CLAMPED on every family."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from asot_inputs import make_inputs, normalized_sqeuclid_cost, random_pairs  # noqa: E402
from asot_inputs.synth import AsotInputs  # noqa: E402
from oracle import asot_oracle as O  # noqa: E402

TOL = {0: 1e-4, 1: 2e-3}          # north_star bars (R#20)
RATIOS = [40, 50, 60, 80]


@pytest.fixture(scope="module")
def asot():
    import paper_2310_16123_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def eps_for(ratio):
    """eps as the fp32 value with max(C_s)/eps <= ratio (max C_s = 1)."""
    e = np.float32(1.0 / ratio)
    if 1.0 / float(e) > ratio:
        e = np.nextafter(e, np.float32(1.0))
    return float(e)


# (config, N, K) per kernel family: K = 16 lane-per-anchor fp32 (both requests, R#23); K = 64 and
# 128 the 1-SM resident kernels (TF32 tc 4 / 2 slots, fp32 3xTF32 tc3); K = 256 the CTA pair (tc2)
# and streamed 3xTF32 (tc5); K = 512 / 1024 the streamed TF32 kernel (tc4, one / two N passes) and tc5.
FAMILIES = [("c1", 40, 16), ("c2", 26, 64), ("c2", 26, 128), ("c3", 24, 256), ("c5", 12, 512),
            ("c5", 12, 1024)]


def family_inputs(cfg, n, K, ratio):
    base = make_inputs(cfg, n_dist=n)
    if K == base.n_anchors:
        anchors, cost = base.anchors, base.cost
    else:
        anchors = np.ascontiguousarray(base.anchors[:K])
        cost = normalized_sqeuclid_cost(anchors)
    return AsotInputs(base.name, base.points, base.offsets, base.weights, anchors, cost,
                      eps_for(ratio), base.iters)


@pytest.fixture(scope="module")
def oracle_cache():
    return {}


def oracle_D(cache, inp, key):
    if key not in cache:
        cache[key] = O.distance_matrix(inp.points, inp.offsets, inp.weights, inp.anchors, inp.cost,
                                       inp.eps, inp.iters)
    return cache[key]


@pytest.mark.parametrize("ratio", RATIOS)
@pytest.mark.parametrize("cfg,n,K", FAMILIES)
@pytest.mark.parametrize("prec", [0, 1])
def test_large_ratio_tiles(asot, oracle_cache, cfg, n, K, ratio, prec):
    inp = family_inputs(cfg, n, K, ratio)
    assert float(inp.cost.max()) / inp.eps <= 80.0
    Do, _, H_o = oracle_D(oracle_cache, inp, (cfg, n, K, ratio))
    st = asot.asot.new_status()
    D = asot.distance_matrix(dev(inp.points), dev(inp.offsets), dev(inp.weights), dev(inp.anchors),
                             dev(inp.cost), inp.eps, inp.iters, precision=prec, offsets_host=inp.offsets,
                             status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == 0, f"flags {int(st.item()):#x}"     # no clamp, no non-finite output
    Dg = D.cpu().numpy().astype(np.float64)
    assert np.all(np.isfinite(Dg)) and np.all(Dg >= 0)
    eff = asot.effective_precision(K, prec)
    r = np.abs(Dg - Do) / np.maximum(Do, 1e-3)
    assert r.max() <= TOL[eff], f"{cfg} K={K} ratio={ratio} prec={eff}: max rel {r.max():.3e}"


PAIR_FAMILIES = [("c1", 40, 16), ("c2", 26, 128), ("c3", 24, 256)]


@pytest.mark.parametrize("ratio", [50, 80])
@pytest.mark.parametrize("cfg,n,K", PAIR_FAMILIES)
@pytest.mark.parametrize("prec", [0, 1])
def test_large_ratio_pair_lists(asot, cfg, n, K, ratio, prec):
    """The pair-list modes (lane-per-anchor K < 32; 1-SM resident TF32 / 3xTF32 K <= 128; streamed
    TF32 / 3xTF32 K > 128) at the same ratios, reversed orientations included."""
    inp = family_inputs(cfg, n, K, ratio)
    pts, offs, w, anc, cst = (dev(inp.points), dev(inp.offsets), dev(inp.weights), dev(inp.anchors),
                              dev(inp.cost))
    _, H, _ = asot.map_to_anchors(pts, offs, w, anc, offsets_host=inp.offsets)
    pi, pj = random_pairs(n, 150, seed=21)
    pi, pj = np.concatenate([pi, pj[:30]]).astype(np.int32), np.concatenate([pj, pi[:30]]).astype(np.int32)
    st = asot.asot.new_status()
    d = asot.pairwise_sinkhorn(H, cst, inp.eps, inp.iters, dev(pi), dev(pj), precision=prec, status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == 0, f"flags {int(st.item()):#x}"
    c_o, fl = O.pair_costs(H.cpu().numpy().astype(np.float64), inp.cost.astype(np.float64), inp.eps,
                           inp.iters, pi.astype(np.int64), pj.astype(np.int64))
    assert not fl.any()
    r = np.abs(d.cpu().numpy().astype(np.float64) - c_o) / np.maximum(c_o, 1e-3)
    eff = asot.effective_precision(K, prec)
    assert r.max() <= TOL[eff], f"{cfg} K={K} ratio={ratio} prec={eff}: max rel {r.max():.3e}"


@pytest.mark.parametrize("K", [16, 64, 128, 256, 512, 1024])
@pytest.mark.parametrize("prec", [0, 1])
def test_denominator_clamp_is_flagged(asot, K, prec):
    """S:62 / S:79: a denominator below the floor is clamped and flagged.  H row 0 carries a mass of
    1e-30 on anchor 0, row 1 a unit mass on anchor 1, C_s = 1 - I, max(C_s)/eps = 80: after the
    first u-update (G^T u)_1 = e^-80 * 1e-30 ~ 2e-65 underflows fp32 on every kernel family (the
    fp64 oracle stays above its 1e-300 floor).  The run must raise DENOM_CLAMPED -- a warning that
    check_status lets through -- and nothing else; the pair-list mode must raise it too."""
    H = np.zeros((2, K), np.float32)
    H[0, 0] = 1e-30
    H[1, 1] = 1.0
    C = (1.0 - np.eye(K)).astype(np.float32)
    eps = eps_for(80)
    st = asot.asot.new_status()
    D = asot.distance_matrix(None, None, None, None, dev(C), eps, 5, precision=prec, hist=dev(H),
                             cost_max=1.0, status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == asot.asot.FLAG_DENOM_CLAMPED, f"flags {int(st.item()):#x}"
    asot.check_status(st)                      # a warning, not an error
    assert np.isfinite(D.cpu().numpy()).all()
    _, _, _, fl = O.sinkhorn_batch(H[[0]].T.astype(np.float64), H[[1]].T.astype(np.float64),
                                   *O.gibbs(C, eps), 5)
    assert not fl.any()                        # the oracle's fp64 floor (1e-300) is not reached
    st2 = asot.asot.new_status()
    asot.pairwise_sinkhorn(dev(H), dev(C), eps, 5, dev(np.array([0], np.int32)),
                           dev(np.array([1], np.int32)), precision=prec, cost_max=1.0, status=st2)
    torch.cuda.synchronize()
    assert int(st2.item()) == asot.asot.FLAG_DENOM_CLAMPED, f"flags {int(st2.item()):#x}"
