"""GPU parity of the small-support Sinkhorn path (asot_sinkhorn_sparse.cu, DESIGN R#36) against the
fp64 oracle, through the C ABI with the library's default path selection.

The path serves a call when every histogram has at most 16 non-zero bins (c1, c3); it computes
the same L iterations as the dense definition, leaving out the products with exact zeros, in
fp32 -- so both precision requests are held to the fp32 bar (1e-4).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.sparse_path,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from asot_inputs import make_inputs, random_pairs  # noqa: E402
from oracle import asot_oracle as O  # noqa: E402

FP32_TOL = 1e-4


@pytest.fixture(scope="module")
def asot():
    import paper_2310_16123_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def rel_err(Dg, Do, cmax):
    return np.abs(np.asarray(Dg, np.float64) - Do) / np.maximum(Do, 1e-3 * cmax)


_cache = {}


def oracle_full(cfg, n):
    if (cfg, n) not in _cache:
        inp = make_inputs(cfg, n_dist=n)
        D, _, H = O.distance_matrix(inp.points, inp.offsets, inp.weights, inp.anchors, inp.cost,
                                    inp.eps, inp.iters)
        _cache[(cfg, n)] = (inp, D, H)
    return _cache[(cfg, n)]


def run_matrix(asot, inp, prec, **kw):
    st = asot.asot.new_status()
    D = asot.distance_matrix(dev(inp.points), dev(inp.offsets), dev(inp.weights), dev(inp.anchors),
                             dev(inp.cost), float(inp.eps), inp.iters, precision=prec,
                             offsets_host=inp.offsets, status=st, **kw)
    torch.cuda.synchronize()
    return D, st


@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("cfg,n", [("c1", 64), ("c3", 80)])
def test_sparse_matrix_vs_oracle(asot, cfg, n, prec):
    """c3 (K = 256, supports 1-9): the whole matrix within the fp32 bar for both requests,
    symmetric, zero diagonal, status clean; c1 (K = 16 < 64, supports up to 12) keeps the dense
    lane-per-anchor kernel under the default selection, also fp32."""
    inp, Do, H = oracle_full(cfg, n)
    assert (H > 0).sum(1).max() <= 16
    D, st = run_matrix(asot, inp, prec)
    asot.check_status(st)
    Dg = D.cpu().numpy()
    assert np.all(np.diag(Dg) == 0) and np.array_equal(Dg, Dg.T)
    r = rel_err(Dg, Do, float(inp.cost.max()))
    assert r.max() <= FP32_TOL, f"{cfg} prec={prec}: max rel {r.max():.3e}"


def test_sparse_path_is_the_one_taken(asot, monkeypatch):
    """Which path ran: at c3 (N = 400, 79,800 pairs) the default selection and ASOT_SPARSE=0 (the
    CTA-pair TF32 kernel) give different bits (fp32 vs TF32 arithmetic; on such small supports
    the TF32 errors largely cancel, so both meet the fp32 bar) and the default is several times
    faster (CUDA-event timing of the whole call, after a warm-up)."""
    inp = make_inputs("c3", n_dist=400)
    args = (dev(inp.points), dev(inp.offsets), dev(inp.weights), dev(inp.anchors), dev(inp.cost),
            float(inp.eps), inp.iters)

    def timed():
        asot.distance_matrix(*args, precision=asot.TF32, offsets_host=inp.offsets)
        st = asot.asot.new_status()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        D = asot.distance_matrix(*args, precision=asot.TF32, offsets_host=inp.offsets, status=st)
        e1.record()
        torch.cuda.synchronize()
        asot.check_status(st)
        return D, e0.elapsed_time(e1)

    D_auto, t_auto = timed()
    monkeypatch.setenv("ASOT_SPARSE", "0")
    D_tc, t_tc = timed()
    assert not torch.equal(D_auto, D_tc)
    assert t_auto * 3 < t_tc, (t_auto, t_tc)
    r = (D_auto - D_tc).abs() / torch.clamp(D_tc, min=1e-3 * float(inp.cost.max()))
    assert float(r.max()) <= 2e-3


def test_sparse_full_size_c3_sampled(asot):
    """BASELINE.json's c3 at full size (N = 2000, 1,999,000 pairs) in the bench's launch
    configuration: 2,000 seeded sampled pairs against the oracle, within the fp32 bar."""
    inp = make_inputs("c3")
    D, st = run_matrix(asot, inp, asot.TF32)
    asot.check_status(st)
    _, H = O.map_and_histogram(inp.points, inp.offsets, inp.weights, inp.anchors)
    pi, pj = random_pairs(inp.n_dist, 2000, seed=21)
    do, _ = O.pair_costs(H, inp.cost, inp.eps, inp.iters, pi.astype(np.int64), pj.astype(np.int64))
    dg = D.cpu().numpy()[pi, pj]
    r = rel_err(dg, do, float(inp.cost.max()))
    assert r.max() <= FP32_TOL, f"max rel {r.max():.3e}"


def test_sparse_tile_ranges_bitwise(asot):
    """Tile-range partitions with odd cuts (the multi-GPU unit) reassemble the whole matrix
    bitwise: one thread per pair, the same arithmetic in every launch shape."""
    inp, _, _ = oracle_full("c3", 80)
    D, st = run_matrix(asot, inp, asot.TF32)
    n_tiles = asot.num_tiles(inp.n_dist)
    cuts = [0, 3, 17, 18, 23, n_tiles]
    R = torch.zeros_like(D)
    for t0, t1 in zip(cuts[:-1], cuts[1:]):
        packed = torch.empty((t1 - t0) * 128, dtype=torch.float32, device="cuda")
        run_matrix(asot, inp, asot.TF32, tile_range=(t0, t1), packed=packed, want_matrix=False)
        asot.unpack_tiles(packed, inp.n_dist, t0, t1, R, zero_diag=False)
    torch.cuda.synchronize()
    assert torch.equal(R, D)


@pytest.mark.parametrize("npairs", [300, 5000])
def test_sparse_pair_lists(asot, npairs):
    """Explicit lists (reversed orientations, self pairs, an invalid entry -> NaN + BAD_INDEX; 5000
    entries take the bucketed route where whole tiles are covered): each entry equals the
    matrix entry bitwise."""
    inp, _, H = oracle_full("c3", 80)
    D, _ = run_matrix(asot, inp, asot.TF32)
    Dn = D.cpu().numpy()
    Hd = dev(H.astype(np.float32))
    if npairs > 3000:
        iu, ju = np.triu_indices(inp.n_dist, k=1)
        pi, pj = iu.astype(np.int32), ju.astype(np.int32)
    else:
        pi, pj = random_pairs(inp.n_dist, npairs, seed=4)
        pi, pj = pi.astype(np.int32), pj.astype(np.int32)
    pi = np.concatenate([pi, pj[:7], [5, 80]]).astype(np.int32)
    pj = np.concatenate([pj, pi[:7], [5, 3]]).astype(np.int32)
    st = asot.asot.new_status()
    d = asot.pairwise_sinkhorn(Hd, dev(inp.cost), float(inp.eps), inp.iters, dev(pi), dev(pj),
                               precision=asot.TF32, status=st)
    torch.cuda.synchronize()
    d = d.cpu().numpy()
    assert int(st.item()) & asot.asot.FLAG_BAD_INDEX and np.isnan(d[-1])
    up = pi < pj   # (the invalid last entry has pi > pj)
    np.testing.assert_array_equal(d[up], Dn[pi[up], pj[up]])
    # reversed orientations (a = H[j] on the u side, R#10) and the self pair: against the oracle
    other = np.nonzero(~up)[0][:-1]
    do, _ = O.pair_costs(H, inp.cost, inp.eps, inp.iters, pi[other].astype(np.int64), pj[other].astype(np.int64))
    r = rel_err(d[other], do, float(inp.cost.max()))
    assert r.max() <= FP32_TOL


@pytest.mark.parametrize("sizes", [(1, 8, 8, 3), (9, 16, 5, 12), (16, 16, 1, 2), (8, 17, 4, 4)])
def test_sparse_support_boundaries(asot, sizes):
    """Synthetic histograms with supports at the edges of the two forms (8: registers, 9-16: the
    local-memory form) and past the path (17: the whole call runs on the dense kernels), K = 64,
    against the oracle within the fp32 bar (TF32 bar when a support exceeds 16)."""
    rng = np.random.default_rng(sum(sizes))
    K, n = 64, 24
    X = rng.normal(size=(K, 8))
    C = ((X[:, None, :] - X[None, :, :]) ** 2).sum(-1)
    C = (C / C.max()).astype(np.float32)
    H = np.zeros((n, K), np.float32)
    for i in range(n):
        s = sizes[i % len(sizes)]
        idx = rng.choice(K, size=s, replace=False)
        H[i, idx] = rng.dirichlet(np.ones(s)).astype(np.float32)
    eps, L = 0.05, 60
    pi, pj = np.triu_indices(n, k=1)
    st = asot.asot.new_status()
    d = asot.pairwise_sinkhorn(dev(H), dev(C), eps, L, dev(pi.astype(np.int32)), dev(pj.astype(np.int32)),
                               precision=asot.TF32, status=st)
    torch.cuda.synchronize()
    asot.check_status(st)
    do, _ = O.pair_costs(H, C, eps, L, pi.astype(np.int64), pj.astype(np.int64))
    r = rel_err(d.cpu().numpy(), do, 1.0)
    tol = FP32_TOL if max(sizes) <= 16 else 2e-3
    assert r.max() <= tol, f"max rel {r.max():.3e}"


@pytest.mark.parametrize("ratio", [50.0, 80.0])
def test_sparse_large_ratio_and_clamp(asot, ratio):
    """max(C_s)/eps up to the accepted 80 (R#12): c3 histograms with eps = max(C_s)/ratio, against
    the oracle (its S:62 floor branch included) within the fp32 bar; where a denominator leaves
    [FLT_MIN, 2^126] on a bin with mass, DENOM_CLAMPED is raised exactly when the oracle clamps."""
    inp, _, H = oracle_full("c3", 40)
    cmax = float(inp.cost.max())
    eps = cmax / ratio
    pi, pj = np.triu_indices(inp.n_dist, k=1)
    st = asot.asot.new_status()
    d = asot.pairwise_sinkhorn(dev(H.astype(np.float32)), dev(inp.cost), eps, inp.iters,
                               dev(pi.astype(np.int32)), dev(pj.astype(np.int32)), precision=asot.TF32,
                               status=st)
    torch.cuda.synchronize()
    do, flags = O.pair_costs(H, inp.cost, np.float32(eps), inp.iters, pi.astype(np.int64), pj.astype(np.int64))
    r = rel_err(d.cpu().numpy(), do, cmax)
    assert r.max() <= FP32_TOL, f"ratio {ratio}: max rel {r.max():.3e}"
    assert not flags.any()
    asot.check_status(st)   # at most DENOM_CLAMPED (a warning)


def test_sparse_denominator_clamp_is_flagged(asot):
    """S:62 / S:79 on this path: H row 0 carries 1e-30 on anchor 0, row 1 a unit mass on anchor
    1, C_s = 1 - I, max(C_s)/eps = 80; (K^T u)_1 = e^-80 1e-30 underflows fp32 after the first
    u-update, so DENOM_CLAMPED (and nothing else) is raised, in both the matrix and the list form."""
    K = 64
    H = np.zeros((2, K), np.float32)
    H[0, 0] = 1e-30
    H[1, 1] = 1.0
    C = (1.0 - np.eye(K)).astype(np.float32)
    eps = float(np.float32(1.0 / 80.0))
    st = asot.asot.new_status()
    D = asot.distance_matrix(None, None, None, None, dev(C), eps, 5, precision=asot.TF32, hist=dev(H),
                             cost_max=1.0, status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == asot.asot.FLAG_DENOM_CLAMPED, f"flags {int(st.item()):#x}"
    assert np.isfinite(D.cpu().numpy()).all()
    st2 = asot.asot.new_status()
    asot.pairwise_sinkhorn(dev(H), dev(C), eps, 5, dev(np.array([0], np.int32)),
                           dev(np.array([1], np.int32)), precision=asot.FP32, cost_max=1.0, status=st2)
    torch.cuda.synchronize()
    assert int(st2.item()) == asot.asot.FLAG_DENOM_CLAMPED, f"flags {int(st2.item()):#x}"


@pytest.mark.parametrize("cfg,n", [("c3", 80), ("c2", 60)])
def test_partition_union_bitwise(asot, cfg, n):
    """asot_distance_matrix_partition (the multi-GPU unit of distributed.py's NVLink path): parts
    of [0, num_tiles) with odd cuts, run as separate calls into one matrix, reproduce the whole
    matrix bitwise -- in support order on the small-support path (c3) and in the a4 tiling on the
    dense one (c2)."""
    inp, _, H = oracle_full(cfg, n)
    D, _ = run_matrix(asot, inp, asot.TF32)
    Hd = dev(H.astype(np.float32))
    n_tiles = asot.num_tiles(inp.n_dist)
    cuts = sorted({0, 3, n_tiles // 2, n_tiles // 2 + 1, n_tiles - 1, n_tiles})
    R = torch.zeros_like(D)
    st = asot.asot.new_status()
    for p0, p1 in zip(cuts[:-1], cuts[1:]):
        asot.distance_matrix_partition(Hd, dev(inp.cost), float(inp.eps), inp.iters, (p0, p1),
                                       precision=asot.TF32, out=R, status=st)
    torch.cuda.synchronize()
    asot.check_status(st)
    assert torch.equal(R, D)


def test_sparse_asymmetric_cost(asot):
    """C_s need not be symmetric (an input; R#7): K v and K^T u differ.  Supports of 2, 5 and 7
    bins (three support classes, so pairs run with the u side on the rows and on the columns of
    the register forms, which then hold K^T's block): the whole matrix (support-ordered class
    kernels) and an explicit list (the a4 / list traversal) against the oracle, within the fp32
    bar, the list entries bitwise equal to the matrix entries."""
    rng = np.random.default_rng(17)
    K, n = 96, 40
    C = rng.uniform(0.0, 1.0, size=(K, K)).astype(np.float32)
    np.fill_diagonal(C, 0.0)
    H = np.zeros((n, K), np.float32)
    for i in range(n):
        s = (2, 5, 7)[i % 3]
        idx = rng.choice(K, size=s, replace=False)
        H[i, idx] = rng.dirichlet(np.ones(s)).astype(np.float32)
    eps, L = 0.1, 50
    st = asot.asot.new_status()
    D = asot.distance_matrix(None, None, None, None, dev(C), eps, L, precision=asot.TF32, hist=dev(H),
                             cost_max=1.0, status=st)
    pi, pj = np.triu_indices(n, k=1)
    d = asot.pairwise_sinkhorn(dev(H), dev(C), eps, L, dev(pi.astype(np.int32)), dev(pj.astype(np.int32)),
                               precision=asot.TF32, cost_max=1.0, status=st)
    torch.cuda.synchronize()
    asot.check_status(st)
    do, _ = O.pair_costs(H, C, eps, L, pi.astype(np.int64), pj.astype(np.int64))
    Dn = D.cpu().numpy()
    r = rel_err(Dn[pi, pj], do, 1.0)
    assert r.max() <= FP32_TOL, f"matrix: max rel {r.max():.3e}"
    np.testing.assert_array_equal(d.cpu().numpy(), Dn[pi, pj])
