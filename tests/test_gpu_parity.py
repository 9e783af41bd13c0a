"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the same seeded inputs.

Bars (BASELINE.json north_star): anchor assignments bit-exact; histograms equal to the oracle's
fp64 point-order sums rounded to f32; distances within relative error 1e-4 (ASOT_PREC_FP32) or
2e-3 (ASOT_PREC_TF32) with rel = |D_gpu - D_orc| / max(D_orc, 1e-3 max C_s) (R#20).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from asot_inputs import make_inputs, random_pairs  # noqa: E402
from oracle import asot_oracle as O  # noqa: E402

TOL = {0: 1e-4, 1: 2e-3}


@pytest.fixture(scope="module")
def asot():
    import paper_2310_16123_b200 as m
    return m


def dev_inputs(inp):
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t(inp.points), t(inp.offsets), t(inp.weights), t(inp.anchors), t(inp.cost)


def rel_err(Dg, Do, cmax):
    return np.abs(np.asarray(Dg, np.float64) - Do) / np.maximum(Do, 1e-3 * cmax)


_oracle_cache = {}


def oracle_full(cfg, n):
    key = (cfg, n)
    if key not in _oracle_cache:
        inp = make_inputs(cfg, n_dist=n)
        D, assign, H = O.distance_matrix(inp.points, inp.offsets, inp.weights, inp.anchors,
                                         inp.cost, inp.eps, inp.iters)
        _oracle_cache[key] = (inp, D, assign, H)
    return _oracle_cache[key]


def map_via(asot, path, pts, offs, w, anc, offsets_host):
    """The mapping through asot_map_to_anchors ("exact": the CUDA-core kernel on every point) or
    through asot_distance_matrix with an empty tile range ("tc": with a workspace, the tensor-core
    products and the exact kernel on the points they cannot decide, R#37)."""
    if path == "exact":
        return asot.map_to_anchors(pts, offs, w, anc, offsets_host=offsets_host)
    if path == "ws":   # asot_map_to_anchors_ws: the standalone / multi-GPU mapping with a workspace
        return asot.map_to_anchors(pts, offs, w, anc, offsets_host=offsets_host, tensor_core=True)
    N, K = offsets_host.shape[0] - 1, anc.shape[0]
    assign = torch.empty(max(int(offsets_host[-1]), 1), dtype=torch.int32, device=pts.device)
    H = torch.empty((N, K), dtype=torch.float32, device=pts.device)
    st = asot.asot.new_status()
    C = torch.zeros((K, K), dtype=torch.float32, device=pts.device)
    asot.distance_matrix(pts, offs, w, anc, C, 0.05, 1, tile_range=(0, 0), assign_out=assign,
                         hist_out=H, offsets_host=offsets_host, cost_max=0.0, status=st)
    return assign, H, st


# ------------------------------------------------------------------ mapping + histograms
@pytest.mark.parametrize("path", ["exact", "tc", "ws"])
@pytest.mark.parametrize("cfg,n", [("c1", 64), ("c2", 1000), ("c3", 200), ("c4", 8000), ("c5", 40)])
def test_mapping_bit_exact(asot, cfg, n, path):
    inp = make_inputs(cfg, n_dist=n)
    pts, offs, w, anc, _ = dev_inputs(inp)
    assign, H, st = map_via(asot, path, pts, offs, w, anc, inp.offsets)
    torch.cuda.synchronize()
    asot.check_status(st)
    a_o = O.map_assign(inp.points, inp.anchors)
    a_g = assign.cpu().numpy()
    assert np.array_equal(a_g, a_o), f"{(a_g != a_o).sum()} of {a_o.size} assignments differ"
    H_o = O.histograms(a_o, inp.weights, inp.offsets, inp.n_anchors).astype(np.float32)
    np.testing.assert_array_equal(H.cpu().numpy(), H_o)


@pytest.mark.parametrize("path", ["exact", "tc", "ws"])
def test_mapping_adversarial_ties(asot, path):
    rng = np.random.default_rng(5)
    d, K = 32, 64
    W = rng.integers(-3, 4, size=(K, d)).astype(np.float32)
    W[10] = W[3]                                     # duplicate anchor -> lower index
    pts = []
    for _ in range(600):                             # exact midpoints of integer anchors: exact ties
        a, b = rng.choice(K, 2, replace=False)
        pts.append((W[a] + W[b]) / 2)
    for gap in (1e-9, 1e-8, 1e-7, 1e-6, 1e-5, 1e-4):  # near ties at relative gaps
        for _ in range(300):
            a, b = rng.choice(K, 2, replace=False)
            m = (W[a].astype(np.float64) + W[b]) / 2 + gap * (W[b].astype(np.float64) - W[a])
            pts.append(m)
    pts.append(W[3]); pts.append(W[10]); pts.append(W[0])
    X = np.asarray(pts, dtype=np.float32)
    off = np.array([0, X.shape[0]], np.int64)
    w = np.full(X.shape[0], np.float32(1.0 / X.shape[0]))
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    assign, H, st = map_via(asot, path, t(X), t(off), t(w), t(W), off)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(assign.cpu().numpy(), O.map_assign(X, W))
    assert assign.cpu().numpy()[-2] == 3


@pytest.mark.parametrize("path", ["exact", "tc", "ws"])
@pytest.mark.parametrize("case", ["offset", "tiny", "huge", "mixed"])
@pytest.mark.parametrize("d,K", [(16, 64), (64, 256), (128, 1024)])
def test_mapping_extreme_magnitudes(asot, case, d, K, path):
    """The kernel decides in fp32 with the rigorous near-tie bound of R#8 and falls back to the
    fp64 op sequence: a large common offset (|x| >> the distances), coordinates near 1e-20
    (subnormal squares: the absolute slack), near 1e19 (fp32 overflow of the distances: every
    point falls back to fp64) and a mix of scales within one batch.  The decision stays the
    fp64 definition's, bit for bit."""
    rng = np.random.default_rng(d + K + len(case))
    C = max(K // 8, 1)
    means = rng.normal(size=(C, d))
    W = np.repeat(means, K // C, axis=0)[:K] + 0.2 * rng.normal(size=(K, d))
    comp = rng.integers(0, C, size=3000)
    X = means[comp] + 0.3 * rng.normal(size=(3000, d))
    if case == "offset":
        X, W = X + 1000.0, W + 1000.0
    elif case == "tiny":
        X, W = X * 1e-20, W * 1e-20
    elif case == "huge":
        X, W = X * 1e19, W * 1e19
    else:
        X = X * np.repeat(10.0 ** rng.integers(-6, 6, size=300), 10)[:, None]
    X, W = X.astype(np.float32), W.astype(np.float32)
    off = np.array([0, X.shape[0]], np.int64)
    w = np.full(X.shape[0], np.float32(1.0 / X.shape[0]))
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    assign, H, st = map_via(asot, path, t(X), t(off), t(w), t(W), off)
    torch.cuda.synchronize()
    a_o = O.map_assign(X, W)
    a_g = assign.cpu().numpy()
    assert np.array_equal(a_g, a_o), f"{(a_g != a_o).sum()} of {a_o.size} assignments differ"


@pytest.mark.parametrize("d,K", [(7, 40), (13, 300), (100, 9), (100, 400)])
def test_mapping_odd_dims_unaligned(asot, d, K):
    """Dimensions that are not a multiple of 4 and point / anchor buffers that are not 16-byte
    aligned take the mapping kernel's scalar load paths; K > one SMEM chunk re-stages anchors per
    point group.  Assignments bit-exact, H bit-identical."""
    rng = np.random.default_rng(d * 1000 + K)
    sizes = rng.integers(1, 40, size=25)
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    X = rng.normal(size=(off[-1], d)).astype(np.float32)
    W = rng.normal(size=(K, d)).astype(np.float32)
    wts = np.concatenate([np.full(n, 1.0 / n) for n in sizes]).astype(np.float32)
    # one-float offsets make the device buffers 4- but not 16-byte aligned
    Xb = torch.from_numpy(np.concatenate([[0.0], X.ravel()]).astype(np.float32)).cuda()[1:].view(-1, d)
    Wb = torch.from_numpy(np.concatenate([[0.0], W.ravel()]).astype(np.float32)).cuda()[1:].view(-1, d)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    assign, H, st = asot.map_to_anchors(Xb, t(off), t(wts), Wb, offsets_host=off)
    torch.cuda.synchronize()
    a_o, H_o = O.map_and_histogram(X, off, wts, W)
    np.testing.assert_array_equal(assign.cpu().numpy(), a_o)
    np.testing.assert_array_equal(H.cpu().numpy(), H_o.astype(np.float32))


# ------------------------------------------------------------------ distances (whole pipeline)
@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("cfg,n", [("c1", 64), ("c2", 90), ("c3", 36), ("c4", 50), ("c5", 18)])
def test_distance_matrix_parity(asot, cfg, n, prec):
    inp, Do, _, _ = oracle_full(cfg, n)
    pts, offs, w, anc, cst = dev_inputs(inp)
    st = asot.asot.new_status()
    D = asot.distance_matrix(pts, offs, w, anc, cst, float(inp.eps), inp.iters, precision=prec,
                             offsets_host=inp.offsets, status=st)
    torch.cuda.synchronize()
    asot.check_status(st)
    Dg = D.cpu().numpy()
    eff = asot.effective_precision(inp.n_anchors, prec)
    assert np.all(np.diag(Dg) == 0)
    np.testing.assert_array_equal(Dg, Dg.T)
    assert np.all(Dg >= 0)
    r = rel_err(Dg, Do, float(inp.cost.max()))
    assert r.max() <= TOL[eff], f"{cfg} prec={eff}: max rel {r.max():.3e} p99 {np.quantile(r, .99):.3e}"


@pytest.mark.parametrize("cfg,n,npairs", [("c1", 40, 300), ("c2", 90, 700), ("c3", 30, 300), ("c5", 12, 130)])
@pytest.mark.parametrize("prec", [0, 1])
def test_pairwise_explicit_pairs(asot, cfg, n, npairs, prec):
    """SPEC batched_sinkhorn_fixed: arbitrary pair lists (reversed orientations, a ragged last tile
    of 128) through the streamed tensor-core kernel in pair-list mode (CUDA cores for K < 32)."""
    inp, Do, _, H_o = oracle_full(cfg, n)
    pi, pj = random_pairs(inp.n_dist, npairs, seed=9)
    pi = np.concatenate([pi, pj[:50]]).astype(np.int32)  # include reversed orientation (R#10)
    pj2 = np.concatenate([pj, pi[:50]]).astype(np.int32)
    pts, offs, w, anc, cst = dev_inputs(inp)
    _, H, _ = asot.map_to_anchors(pts, offs, w, anc, offsets_host=inp.offsets)
    st = asot.asot.new_status()
    d = asot.pairwise_sinkhorn(H, cst, float(inp.eps), inp.iters, torch.from_numpy(pi).cuda(),
                               torch.from_numpy(pj2).cuda(), precision=prec, status=st)
    torch.cuda.synchronize()
    asot.check_status(st)
    c_o, _ = O.pair_costs(H_o, inp.cost, inp.eps, inp.iters, pi.astype(np.int64), pj2.astype(np.int64))
    r = rel_err(d.cpu().numpy(), c_o, float(inp.cost.max()))
    assert r.max() <= TOL[asot.effective_precision(inp.n_anchors, prec)], r.max()


@pytest.mark.parametrize("K", [32, 50, 64, 96, 128])
def test_pairwise_resident_pair_mode(asot, K):
    """TF32 pair lists with K <= 128 run the resident 1-SM kernel in pair-list mode (2 and 4 slots
    per CTA): every i < j entry equals the tile path's value for that pair bitwise (same kernel
    arithmetic), invalid entries (out-of-range indices) give NaN and raise FLAG_BAD_INDEX, and all values (reversed
    orientations included) are within the TF32 bar of the oracle."""
    inp = make_inputs("c2", n_dist=45)
    A = np.ascontiguousarray(inp.anchors[:K])
    C = (((A[:, None, :].astype(np.float64) - A[None, :, :]) ** 2).sum(-1))
    C = (C / C.max()).astype(np.float32)
    pts, offs, w, _, _ = dev_inputs(inp)
    anc, cst = torch.from_numpy(A).cuda(), torch.from_numpy(C).cuda()
    _, H, _ = asot.map_to_anchors(pts, offs, w, anc, offsets_host=inp.offsets)
    D = asot.distance_matrix(None, None, None, None, cst, float(inp.eps), inp.iters, precision=asot.TF32,
                             hist=H, cost_max=1.0)
    pi, pj = random_pairs(inp.n_dist, 700, seed=11)
    pi = np.concatenate([pi, pj[:40], [-1, 3, inp.n_dist]]).astype(np.int32)   # reversed + invalid
    pj = np.concatenate([pj, pi[:40], [2, inp.n_dist + 5, 1]]).astype(np.int32)
    st = asot.asot.new_status()
    d = asot.pairwise_sinkhorn(H, cst, float(inp.eps), inp.iters, torch.from_numpy(pi).cuda(),
                               torch.from_numpy(pj).cuda(), precision=asot.TF32, status=st, cost_max=1.0)
    torch.cuda.synchronize()
    d = d.cpu().numpy()
    Dn = D.cpu().numpy()
    ok = (pi >= 0) & (pj >= 0) & (pi < inp.n_dist) & (pj < inp.n_dist)
    assert np.all(np.isnan(d[~ok])) and np.all(np.isfinite(d[ok]))
    assert int(st.item()) == asot.asot.FLAG_BAD_INDEX
    with pytest.raises(ValueError):
        asot.check_status(st)
    fwd = ok & (pi < pj)   # the tile path computes i < j with a = H[i] on the u side (R#10)
    np.testing.assert_array_equal(d[fwd], Dn[pi[fwd], pj[fwd]])
    c_o, _ = O.pair_costs(H.cpu().numpy().astype(np.float64), C.astype(np.float64), inp.eps, inp.iters,
                          pi[ok].astype(np.int64), pj[ok].astype(np.int64))
    assert rel_err(d[ok], c_o, 1.0).max() <= TOL[asot.TF32]


@pytest.mark.parametrize("cfg,n", [("c2", 90), ("c3", 70), ("c5", 40)])
def test_tile_ranges_and_determinism(asot, cfg, n):
    """D must be bitwise identical for every rank partition (each pair's arithmetic
    is independent of the tile range that computes it) -- for every resident / streamed kernel
    (c2: 1-SM and 3xTF32 kernels; c3: CTA-pair and streamed 3xTF32; c5: streamed TF32 / 3xTF32),
    with cuts at odd tiles so CTA pairs straddle range boundaries."""
    inp = make_inputs(cfg, n_dist=n)
    pts, offs, w, anc, cst = dev_inputs(inp)
    for prec in (0, 1):
        D1 = asot.distance_matrix(pts, offs, w, anc, cst, float(inp.eps), inp.iters, precision=prec,
                                  offsets_host=inp.offsets)
        D2 = asot.distance_matrix(pts, offs, w, anc, cst, float(inp.eps), inp.iters, precision=prec,
                                  offsets_host=inp.offsets)
        assert torch.equal(D1, D2)                        # bitwise re-run determinism
        nt = asot.num_tiles(inp.n_dist)
        D3 = torch.full_like(D1, -1.0)
        cuts = [0, 3, nt // 2, nt - 1, nt]
        for a, b in zip(cuts[:-1], cuts[1:]):             # rank-style partition + unpack (KN6)
            packed = torch.empty((b - a) * 128, device="cuda")
            asot.distance_matrix(pts, offs, w, anc, cst, float(inp.eps), inp.iters, precision=prec,
                                 offsets_host=inp.offsets, tile_range=(a, b), packed=packed,
                                 want_matrix=False)
            asot.unpack_tiles(packed, inp.n_dist, a, b, D3, zero_diag=(b == nt))
        assert torch.equal(D1, D3)


def test_host_entry_point_matches_device(asot):
    inp, _, _, _ = oracle_full("c1", 64)
    pts, offs, w, anc, cst = dev_inputs(inp)
    for prec in (0, 1):
        Dd = asot.distance_matrix(pts, offs, w, anc, cst, float(inp.eps), inp.iters, precision=prec,
                                  offsets_host=inp.offsets).cpu().numpy()
        Dh, status = asot.distance_matrix_host(inp.points, inp.offsets, inp.weights, inp.anchors,
                                               inp.cost, float(inp.eps), inp.iters, precision=prec)
        assert status == 0
        np.testing.assert_array_equal(Dh, Dd)


def test_one_hot_histograms_exact_cost(asot):
    """Special case: one-hot a', b' => d = C_s(u, v) exactly for any eps, L (oracle pin); on the
    GPU only the fp32 / TF32 rounding of K and K (.) C_s remains."""
    K, N = 128, 40
    rng = np.random.default_rng(2)
    W = rng.normal(size=(K, 8)).astype(np.float32)
    from asot_inputs import normalized_sqeuclid_cost
    C = normalized_sqeuclid_cost(W)
    u = rng.integers(0, K, N)
    H = np.zeros((N, K), np.float32)
    H[np.arange(N), u] = 1.0
    Ht = torch.from_numpy(H).cuda()
    Ct = torch.from_numpy(C).cuda()
    for prec in (0, 1):
        D = asot.distance_matrix(None, None, None, None, Ct, 0.05, 30, precision=prec, hist=Ht).cpu().numpy()
        want = C[u][:, u].astype(np.float64)
        np.fill_diagonal(want, 0)
        r = rel_err(D, want, 1.0)
        assert r.max() <= TOL[asot.effective_precision(K, prec)]


def test_full_size_sampled_parity_c2(asot):
    """BASELINE configs[1] at full size (N = 1000) in the launch configuration bench.py times:
    sampled pairs against the oracle evaluated pair by pair."""
    inp = make_inputs("c2")
    pts, offs, w, anc, cst = dev_inputs(inp)
    st = asot.asot.new_status()
    D = asot.distance_matrix(pts, offs, w, anc, cst, float(inp.eps), inp.iters, precision=asot.TF32,
                             offsets_host=inp.offsets, cost_max=1.0, status=st)
    torch.cuda.synchronize()
    asot.check_status(st)
    assign_o, H_o = O.map_and_histogram(inp.points, inp.offsets, inp.weights, inp.anchors)
    pi, pj = random_pairs(inp.n_dist, 400, seed=17)
    edge_i = np.array([0, 0, 15, 16, 991, 998, 7, 8], np.int32)   # block / tile boundaries, tail
    edge_j = np.array([1, 999, 16, 17, 999, 999, 8, 15], np.int32)
    pi = np.concatenate([pi, edge_i]); pj = np.concatenate([pj, edge_j])
    c_o, _ = O.pair_costs(H_o, inp.cost, inp.eps, inp.iters, pi.astype(np.int64), pj.astype(np.int64))
    Dg = D.cpu().numpy()
    r = rel_err(Dg[pi, pj], c_o, 1.0)
    eff = asot.effective_precision(inp.n_anchors, asot.TF32)
    assert r.max() <= TOL[eff]
    np.testing.assert_array_equal(Dg, Dg.T)
    assert np.all(np.diag(Dg) == 0)


def test_pair_kernel_odd_tile_ranges(asot):
    """K = 256 runs on the CTA-pair kernel, whose unit is a block pair (two tiles); ranges that
    start or end on an odd tile must mask the half outside the range."""
    inp, Do, _, _ = oracle_full("c3", 36)
    pts, offs, w, anc, cst = dev_inputs(inp)
    D1 = asot.distance_matrix(pts, offs, w, anc, cst, float(inp.eps), inp.iters, precision=asot.TF32,
                              offsets_host=inp.offsets)
    nt = asot.num_tiles(inp.n_dist)
    D3 = torch.full_like(D1, -1.0)
    cuts = [0, 1, 4, 7, nt - 3, nt]
    for a, b in zip(cuts[:-1], cuts[1:]):
        packed = torch.full(((b - a) * 128,), -7.0, device="cuda")
        asot.distance_matrix(pts, offs, w, anc, cst, float(inp.eps), inp.iters, precision=asot.TF32,
                             offsets_host=inp.offsets, tile_range=(a, b), packed=packed, want_matrix=False)
        assert not torch.any(packed == -7.0)          # every slot of the range written (0 if invalid)
        asot.unpack_tiles(packed, inp.n_dist, a, b, D3, zero_diag=(b == nt))
    assert torch.equal(D1, D3)
    r = rel_err(D1.cpu().numpy(), Do, 1.0)
    assert r.max() <= 2e-3


def test_full_size_sampled_parity_c3(asot):
    """c3 at full size (N = 2000, the multi-GPU configuration) on the CTA-pair kernel: sampled
    pairs against the oracle evaluated pair by pair."""
    inp = make_inputs("c3")
    pts, offs, w, anc, cst = dev_inputs(inp)
    st = asot.asot.new_status()
    D = asot.distance_matrix(pts, offs, w, anc, cst, float(inp.eps), inp.iters, precision=asot.TF32,
                             offsets_host=inp.offsets, cost_max=1.0, status=st)
    torch.cuda.synchronize()
    asot.check_status(st)
    _, H_o = O.map_and_histogram(inp.points, inp.offsets, inp.weights, inp.anchors)
    pi, pj = random_pairs(inp.n_dist, 300, seed=23)
    pi = np.concatenate([pi, np.array([0, 15, 1984, 1998], np.int32)])
    pj = np.concatenate([pj, np.array([1, 16, 1999, 1999], np.int32)])
    c_o, _ = O.pair_costs(H_o, inp.cost, inp.eps, inp.iters, pi.astype(np.int64), pj.astype(np.int64))
    Dg = D.cpu().numpy()
    assert rel_err(Dg[pi, pj], c_o, 1.0).max() <= 2e-3
    np.testing.assert_array_equal(Dg, Dg.T)


@pytest.mark.parametrize("cfg,n", [("c2", 70), ("c3", 40)])
def test_distributed_path_single_rank_nccl(asot, cfg, n):
    """The multi-GPU orchestration with the CUDA steps (partitioned mapping + NCCL all-gather of H,
    tile-range sharding, NCCL gather of packed tiles, KN6 unpack) on a 1-rank NCCL group: must be
    bitwise identical to the single-call matrix."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2310_16123_b200 import distributed as D_

    inp = make_inputs(cfg, n_dist=n)
    pts, offs, w, anc, cst = dev_inputs(inp)
    D1 = asot.distance_matrix(pts, offs, w, anc, cst, float(inp.eps), inp.iters, precision=asot.TF32,
                              offsets_host=inp.offsets)
    created = False
    if not dist.is_initialized():
        s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        created = True
    try:
        st = asot.asot.new_status()
        steps = D_.cuda_steps(pts, offs, inp.offsets, w, anc, cst, float(inp.eps), inp.iters, asot.TF32,
                              1.0, st)
        D2 = D_.distance_matrix_distributed(inp.n_dist, inp.n_anchors, inp.offsets,
                                            asot.num_tiles(inp.n_dist), steps, device=torch.device("cuda", 0))
        torch.cuda.synchronize()
        assert torch.equal(D1, D2)
        # p2p form: the Sinkhorn epilogue stores into rank 0's symmetric-memory matrix
        res = D_.P2PResult(inp.n_dist, torch.device("cuda", 0), n_anchors=inp.n_anchors)
        res.D.fill_(-1.0)
        res.H.fill_(-1.0)
        D3 = D_.distance_matrix_distributed_p2p(inp.n_dist, inp.n_anchors, inp.offsets,
                                                asot.num_tiles(inp.n_dist), steps, res,
                                                device=torch.device("cuda", 0))
        torch.cuda.synchronize()
        assert torch.equal(D1, D3)
    finally:
        if created:
            dist.destroy_process_group()


@pytest.mark.parametrize("cfg,prec,npairs", [("c4", 1, 200), ("c3", 0, 200), ("c5", 1, 40), ("c5", 0, 24)])
def test_full_size_sampled_parity_more(asot, cfg, prec, npairs):
    """Full-size c4 (N = 8000, Dirichlet weights), c3 at fp32 (3xTF32 streamed kernel) and c5
    (K = 1024, streamed kernels) in bench.py's launch configuration: sampled pairs against the
    oracle evaluated pair by pair on the histograms of the touched distributions."""
    inp = make_inputs(cfg)
    pts, offs, w, anc, cst = dev_inputs(inp)
    st = asot.asot.new_status()
    D = asot.distance_matrix(pts, offs, w, anc, cst, float(inp.eps), inp.iters, precision=prec,
                             offsets_host=inp.offsets, cost_max=1.0, status=st)
    torch.cuda.synchronize()
    asot.check_status(st)
    pi, pj = random_pairs(inp.n_dist, npairs, seed=23)
    n = inp.n_dist
    pi = np.concatenate([pi, [0, 15, n - 2]]).astype(np.int32)     # block boundary, ragged tail
    pj = np.concatenate([pj, [n - 1, 16, n - 1]]).astype(np.int32)
    touched = np.unique(np.concatenate([pi, pj]))
    H_o = np.zeros((n, inp.n_anchors))
    for d in touched:
        s, e = int(inp.offsets[d]), int(inp.offsets[d + 1])
        _, h = O.map_and_histogram(inp.points[s:e], np.array([0, e - s]), inp.weights[s:e], inp.anchors)
        H_o[d] = h[0]
    c_o, _ = O.pair_costs(H_o, inp.cost, inp.eps, inp.iters, pi.astype(np.int64), pj.astype(np.int64))
    Dg = D.cpu().numpy()
    r = rel_err(Dg[pi, pj], c_o, 1.0)
    assert r.max() <= TOL[asot.effective_precision(inp.n_anchors, prec)], r.max()
    assert np.all(np.diag(Dg) == 0) and np.array_equal(Dg[pi, pj], Dg[pj, pi])


@pytest.mark.parametrize("K", [16, 64, 128])
def test_pair_modes_vs_cuda_core_kernel(K):
    """fp32 pair lists: the 3xTF32 1-SM kernel's pair-list mode (32 <= K <= 128) or the fp32
    lane-per-anchor kernel (K < 32) against the independent fp32 CUDA-core GEMM kernel
    (ASOT_PAIR_KERNEL=simt, a separate process) and the oracle, on the same list with reversed and
    invalid entries.  At K < 32 both are fp32 CUDA-core kernels with the same dot-product order;
    they differ only in the divide (rcp.approx vs IEEE, <= 1 ulp per step) and the final
    reduction order."""
    import os
    import subprocess
    import sys
    ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = f"""
import numpy as np, torch, sys
sys.path.insert(0, {ROOT!r})
from asot_inputs import make_inputs, random_pairs
import paper_2310_16123_b200 as asot
inp = make_inputs('c2', n_dist=40)
A = np.ascontiguousarray(inp.anchors[:{K}])
C = (((A[:, None, :].astype(np.float64) - A[None, :, :]) ** 2).sum(-1)); C = (C / C.max()).astype(np.float32)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
_, H, _ = asot.map_to_anchors(t(inp.points), t(inp.offsets), t(inp.weights), t(A), offsets_host=inp.offsets)
pi, pj = random_pairs(inp.n_dist, 300, seed=5)
pi = np.concatenate([pi, pj[:20], [-1]]).astype(np.int32); pj = np.concatenate([pj, pi[:20], [3]]).astype(np.int32)
d = asot.pairwise_sinkhorn(H, t(C), float(inp.eps), inp.iters, t(pi), t(pj), precision=asot.FP32, cost_max=1.0)
np.save(sys.argv[1], d.cpu().numpy()); np.save(sys.argv[2], H.cpu().numpy()); np.save(sys.argv[3], np.stack([pi, pj]))
"""
    import tempfile
    outs = {}
    with tempfile.TemporaryDirectory() as td:
        for mode in ("tc", "simt"):
            env = dict(os.environ)
            env.pop("ASOT_PAIR_KERNEL", None)
            if mode == "simt":
                env["ASOT_PAIR_KERNEL"] = "simt"
            f = [os.path.join(td, f"{mode}_{k}.npy") for k in ("d", "h", "p")]
            r = subprocess.run([sys.executable, "-c", code, *f], env=env, capture_output=True, text=True,
                               timeout=300)
            assert r.returncode == 0, r.stderr[-2000:]
            outs[mode] = [np.load(x) for x in f]
    d_tc, H, (pi, pj) = outs["tc"]
    d_simt = outs["simt"][0]
    inp = make_inputs("c2", n_dist=40)
    A = inp.anchors[:K].astype(np.float64)
    C = ((A[:, None, :] - A[None, :, :]) ** 2).sum(-1)
    C = (C / C.max()).astype(np.float32)
    ok = (pi >= 0) & (pj >= 0)
    assert np.all(np.isnan(d_tc[~ok])) and np.all(np.isnan(d_simt[~ok]))
    c_o, _ = O.pair_costs(H.astype(np.float64), C.astype(np.float64), inp.eps, inp.iters,
                          pi[ok].astype(np.int64), pj[ok].astype(np.int64))
    assert rel_err(d_tc[ok], c_o, 1.0).max() <= TOL[0]      # ASOT_PREC_FP32
    assert rel_err(d_simt[ok], c_o, 1.0).max() <= TOL[0]
    if K < 32:
        assert np.abs(d_tc[ok].astype(np.float64) - d_simt[ok]).max() <= 2e-6 * np.abs(d_simt[ok]).max()


@pytest.mark.parametrize("K,prec", [(128, 1), (64, 0), (16, 1), (256, 1), (256, 0)])
def test_pair_list_writes_stay_in_bounds(asot, K, prec):
    """Pair lists whose length is not a multiple of the 128-entry tile: the kernels must write
    exactly n_pairs results (a guard region after dist_out stays untouched) -- resident pair-list
    modes (K <= 128, TF32 and 3xTF32) and the streamed one (K = 256)."""
    from paper_2310_16123_b200 import _lib
    inp = make_inputs("c5", n_dist=30)
    A = np.ascontiguousarray(inp.anchors[:K])
    C = (((A[:, None, :].astype(np.float64) - A[None, :, :]) ** 2).sum(-1))
    C = (C / C.max()).astype(np.float32)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    _, H, _ = asot.map_to_anchors(t(inp.points), t(inp.offsets), t(inp.weights), t(A), offsets_host=inp.offsets)
    pi, pj = random_pairs(inp.n_dist, 200, seed=3)
    n = 131   # one full tile + 3
    pi, pj = t(pi[:n].astype(np.int32)), t(pj[:n].astype(np.int32))
    guard = 1024
    out = torch.full((n + guard,), -7.0, dtype=torch.float32, device="cuda")
    st = asot.asot.new_status()
    L = _lib.load()
    nbytes = int(L.asot_pairwise_workspace_bytes(inp.n_dist, K, prec))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")
    rc = L.asot_pairwise_sinkhorn(H.data_ptr(), inp.n_dist, K, t(C).data_ptr(), 1.0, float(inp.eps), 20, prec,
                                  pi.data_ptr(), pj.data_ptr(), n, out.data_ptr(), st.data_ptr(),
                                  ws.data_ptr(), ws.numel(), None)
    torch.cuda.synchronize()
    assert rc == 0
    o = out.cpu().numpy()
    assert np.all(o[n:] == -7.0), "write past dist_out[n_pairs]"
    assert np.all(np.isfinite(o[:n])) and np.all(o[:n] >= 0.0)


@pytest.mark.parametrize("cfg,prec,nrand,pool", [("c3", 1, 10000, None), ("c4", 1, 10000, None),
                                                ("c5", 1, 2000, 100)])
def test_survey_parity_subsets(asot, cfg, prec, nrand, pool):
    """SURVEY 8(d)'s parity subset at full size in bench.py's launch configuration: a seeded set of
    random pairs (>= 10,000 for c3 / c4; for c5, whose oracle mapping runs ~2 distributions/s, 2,000
    among the first 100 distributions), every pair inside the first 64 distributions, and the pairs
    of the tiles on both sides of every rank boundary of the 2-, 4- and 8-GPU partitions -- each
    against the oracle evaluated pair by pair."""
    from paper_2310_16123_b200.distributed import partition_even
    inp = make_inputs(cfg)
    n = inp.n_dist
    pts, offs, w, anc, cst = dev_inputs(inp)
    st = asot.asot.new_status()
    D = asot.distance_matrix(pts, offs, w, anc, cst, float(inp.eps), inp.iters, precision=prec,
                             offsets_host=inp.offsets, cost_max=1.0, status=st)
    torch.cuda.synchronize()
    asot.check_status(st)
    pi, pj = random_pairs(n if pool is None else pool, nrand, seed=29)
    fi, fj = np.triu_indices(64, k=1)
    bi, bj = [], []
    nt = asot.num_tiles(n)
    for world in (2, 4, 8):
        for (a, b) in partition_even(nt, world)[1:]:
            i, j, v = asot.tile_pairs(n, max(a - 1, 0), min(a + 1, nt))   # tiles a-1 and a
            bi.append(i[v]); bj.append(j[v])
    pi = np.concatenate([pi, fi, *bi]).astype(np.int64)
    pj = np.concatenate([pj, fj, *bj]).astype(np.int64)
    touched = np.unique(np.concatenate([pi, pj]))
    H_o = np.zeros((n, inp.n_anchors))
    for d in touched:
        s, e = int(inp.offsets[d]), int(inp.offsets[d + 1])
        _, h = O.map_and_histogram(inp.points[s:e], np.array([0, e - s]), inp.weights[s:e], inp.anchors)
        H_o[d] = h[0]
    c_o, _ = O.pair_costs(H_o, inp.cost, inp.eps, inp.iters, pi, pj)
    Dg = D.cpu().numpy()
    r = rel_err(Dg[pi, pj], c_o, 1.0)
    assert r.max() <= TOL[asot.effective_precision(inp.n_anchors, prec)], r.max()
