"""GPU edge cases through the C ABI: padding paths of every Sinkhorn kernel (K not a multiple of
the tile), tiny and degenerate problems, and the data-dependent status flags."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from asot_inputs import make_inputs, normalized_sqeuclid_cost  # noqa: E402
from asot_inputs.synth import AsotInputs  # noqa: E402
from oracle import asot_oracle as O  # noqa: E402

TOL = {0: 1e-4, 1: 2e-3}


@pytest.fixture(scope="module")
def asot():
    import paper_2310_16123_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def with_anchors(inp, K, dim=None):
    """Same point sets, first K anchors (and optionally the first `dim` coordinates)."""
    d = inp.dim if dim is None else dim
    anchors = np.ascontiguousarray(inp.anchors[:K, :d])
    return AsotInputs(inp.name, np.ascontiguousarray(inp.points[:, :d]), inp.offsets, inp.weights,
                      anchors, normalized_sqeuclid_cost(anchors), inp.eps, inp.iters)


def run_both(asot, inp, prec):
    st = asot.asot.new_status()
    D = asot.distance_matrix(dev(inp.points), dev(inp.offsets), dev(inp.weights), dev(inp.anchors),
                             dev(inp.cost), float(inp.eps), inp.iters, precision=prec,
                             offsets_host=inp.offsets, status=st)
    torch.cuda.synchronize()
    Do, _, _ = O.distance_matrix(inp.points, inp.offsets, inp.weights, inp.anchors, inp.cost,
                                 inp.eps, inp.iters)
    return D.cpu().numpy(), Do, int(st.item())


@pytest.mark.parametrize("K", [1, 7, 31, 32, 33, 70, 100, 129, 192, 200, 257, 300, 700])
@pytest.mark.parametrize("prec", [0, 1])
def test_padded_anchor_counts(asot, K, prec):
    """K off the 32 / 256 / 1024 tile grids exercises the padding of every kernel
    (1-SM K<=128, CTA pair K<=256, streamed K<=1024)."""
    base = make_inputs("c5", n_dist=21, iters=12)
    inp = with_anchors(base, K, dim=37)          # also a dimension that is not a multiple of 4
    Dg, Do, st = run_both(asot, inp, prec)
    assert st == 0
    eff = asot.effective_precision(K, prec)
    r = np.abs(Dg.astype(np.float64) - Do) / np.maximum(Do, 1e-3)
    assert r.max() <= TOL[eff], f"K={K} prec={eff} max rel {r.max():.3e}"
    np.testing.assert_array_equal(Dg, Dg.T)


@pytest.mark.parametrize("cfg,n", [("c2", 1), ("c2", 2), ("c2", 3), ("c2", 17), ("c3", 1), ("c3", 2),
                                   ("c3", 17), ("c5", 2), ("c5", 17), ("c1", 2)])
def test_tiny_n(asot, cfg, n):
    """N = 1 (no pairs), 2 (one pair, one tile), 3, 17 (a ragged second block) on every kernel family:
    1-SM (c2), CTA pair (c3), streamed (c5), fp32 lane-per-anchor kernel at K < 32 (c1), both precisions."""
    inp = make_inputs(cfg, n_dist=n, iters=5)
    for prec in (0, 1):
        Dg, Do, st = run_both(asot, inp, prec)
        assert st == 0 and Dg.shape == (n, n)
        assert np.all(np.diag(Dg) == 0)
        r = np.abs(Dg.astype(np.float64) - Do) / np.maximum(Do, 1e-3)
        assert r.max() <= TOL[asot.effective_precision(inp.n_anchors, prec)]


def test_single_point_distributions_and_duplicates(asot):
    """n_i = 1 everywhere (one-hot marginals: d = C_s(u, v) exactly up to K's rounding) and
    duplicated distributions (same histogram on both sides)."""
    base = make_inputs("c2", n_dist=30, iters=20)
    pts = base.points[base.offsets[:-1]]           # first point of each distribution
    pts = np.concatenate([pts, pts[:5]])           # + 5 duplicates
    N = pts.shape[0]
    offs = np.arange(N + 1, dtype=np.int64)
    w = np.ones(N, np.float32)
    inp = AsotInputs("c2", np.ascontiguousarray(pts), offs, w, base.anchors, base.cost, base.eps, base.iters)
    for prec in (0, 1):
        Dg, Do, st = run_both(asot, inp, prec)
        assert st == 0
        a = O.map_assign(pts, base.anchors)
        exact = base.cost.astype(np.float64)[a][:, a]
        np.fill_diagonal(exact, 0)
        np.testing.assert_allclose(Do, exact, rtol=1e-12, atol=1e-15)   # oracle: closed form
        r = np.abs(Dg.astype(np.float64) - exact) / np.maximum(exact, 1e-3)
        assert r.max() <= TOL[asot.effective_precision(inp.n_anchors, prec)]


def test_single_anchor(asot):
    inp = with_anchors(make_inputs("c1", n_dist=9, iters=4), 1)
    for prec in (0, 1):
        Dg, Do, st = run_both(asot, inp, prec)
        assert np.all(Dg == 0) and np.all(Do == 0)


def test_status_flags(asot):
    inp = make_inputs("c1", n_dist=6, iters=3)
    import paper_2310_16123_b200.asot as A
    # empty distribution
    offs = inp.offsets.copy(); offs[3] = offs[2]
    pts = inp.points; w = inp.weights.copy()
    st = A.new_status()
    A.distance_matrix(dev(pts), dev(offs), dev(w), dev(inp.anchors), dev(inp.cost), float(inp.eps),
                      inp.iters, offsets_host=offs, status=st)
    torch.cuda.synchronize()
    assert int(st.item()) & A.FLAG_EMPTY_DIST
    with pytest.raises(ValueError):
        A.check_status(st)
    # mass not summing to one
    w2 = inp.weights.copy(); w2[0] *= 3
    st = A.new_status()
    A.map_to_anchors(dev(pts), dev(inp.offsets), dev(w2), dev(inp.anchors), offsets_host=inp.offsets, status=st)
    torch.cuda.synchronize()
    assert int(st.item()) & A.FLAG_BAD_MASS
    # non-finite coordinate
    p2 = inp.points.copy(); p2[4, 1] = np.nan
    st = A.new_status()
    A.map_to_anchors(dev(p2), dev(inp.offsets), dev(inp.weights), dev(inp.anchors), offsets_host=inp.offsets,
                     status=st)
    torch.cuda.synchronize()
    assert int(st.item()) & A.FLAG_NONFINITE_INPUT
    assert not int(st.item()) & A.FLAG_BAD_MASS   # a NaN coordinate is not a mass error
    with pytest.raises(FloatingPointError):
        A.check_status(st)


def test_rejects_cpu_tensors_and_bad_args(asot):
    inp = make_inputs("c1", n_dist=4, iters=2)
    with pytest.raises(ValueError):
        asot.distance_matrix(torch.from_numpy(inp.points), None, None, None, torch.from_numpy(inp.cost),
                             0.05, 2)
    with pytest.raises(ValueError):   # eps such that max(C)/eps > 80 (R#12)
        asot.distance_matrix(dev(inp.points), dev(inp.offsets), dev(inp.weights), dev(inp.anchors),
                             dev(inp.cost), 0.001, 2, offsets_host=inp.offsets)


@pytest.mark.parametrize("K", [16, 100, 200, 700])
@pytest.mark.parametrize("prec", [0, 1])
@pytest.mark.parametrize("L", [1, 5])
def test_separable_cost_closed_form(asot, K, prec, L):
    """Oracle-free finite-L check through the C ABI: C_s(i, j) = f_i + f_j has a rank-one Gibbs
    kernel, so after one iteration the plan is a b^T and d = a.f + b.f for every L (the pin of
    test_oracle_pins.test_sinkhorn_separable_cost_any_L), on every kernel family (K = 16: 3xTF32
    1-SM, 100: 1-SM, 200 / 700: streamed pair-list kernels)."""
    rng = np.random.default_rng(K + 10 * L + 100 * prec)
    N, n = 40, 300
    f = rng.uniform(0.0, 0.5, K).astype(np.float32)
    C = (f[:, None] + f[None, :]).astype(np.float32)
    H = rng.dirichlet(np.ones(K), N).astype(np.float32)
    H[rng.uniform(size=H.shape) < 0.2] = 0.0
    H[:, 0] += 1e-3
    H /= H.sum(1, keepdims=True)
    H = H.astype(np.float32)
    pi = rng.integers(0, N, n).astype(np.int32)
    pj = rng.integers(0, N, n).astype(np.int32)
    st = asot.asot.new_status()
    d = asot.pairwise_sinkhorn(dev(H), dev(C), 0.25, L, dev(pi), dev(pj), precision=prec, status=st,
                               cost_max=float(C.max()))
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    Hd = H.astype(np.float64)
    fd = f.astype(np.float64)
    exact = Hd[pi] @ fd + Hd[pj] @ fd
    r = np.abs(d.cpu().numpy().astype(np.float64) - exact) / exact
    eff = asot.effective_precision(K, prec)
    assert r.max() <= TOL[eff], f"K={K} prec={eff} L={L} max rel {r.max():.3e}"


@pytest.mark.parametrize("K", [16, 100, 200, 700])
@pytest.mark.parametrize("prec", [0, 1])
def test_separable_cost_closed_form_tiles(asot, K, prec):
    """The same oracle-free closed form through the tile-mode kernels (distance_matrix: 1-SM, CTA
    pair, streamed), L = 3: D[i, j] = H_i.f + H_j.f off the diagonal, with H from the oracle's
    (bit-exact) mapping."""
    base = make_inputs("c5", n_dist=19, iters=3)
    inp = with_anchors(base, K, dim=37)
    rng = np.random.default_rng(K)
    f = rng.uniform(0.0, 0.5, K).astype(np.float32)
    C = (f[:, None] + f[None, :]).astype(np.float32)
    st = asot.asot.new_status()
    D = asot.distance_matrix(dev(inp.points), dev(inp.offsets), dev(inp.weights), dev(inp.anchors),
                             dev(C), 0.25, 3, precision=prec, offsets_host=inp.offsets, status=st)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    _, H = O.map_and_histogram(inp.points, inp.offsets, inp.weights, inp.anchors)
    m = H.astype(np.float64) @ f.astype(np.float64)
    exact = m[:, None] + m[None, :]
    np.fill_diagonal(exact, 0.0)
    Dg = D.cpu().numpy().astype(np.float64)
    eff = asot.effective_precision(K, prec)
    r = np.abs(Dg - exact) / np.maximum(exact, 1e-3)
    assert r.max() <= TOL[eff], f"K={K} prec={eff} max rel {r.max():.3e}"


def test_profile_clock_probe(asot):
    """asot_profile_clock: after a launch of a tensor-core kernel kind its in-kernel clock probe
    gives a plausible SM clock; kind 0 (CUDA cores) has no probe."""
    inp = make_inputs("c2", n_dist=300)
    run = asot.distance_matrix(dev(inp.points), dev(inp.offsets), dev(inp.weights), dev(inp.anchors),
                               dev(inp.cost), float(inp.eps), inp.iters, precision=1,
                               offsets_host=inp.offsets)
    torch.cuda.synchronize()
    assert run.shape == (300, 300)
    kind = asot.asot.sinkhorn_kernel_kind(inp.n_anchors, 1)
    mhz = asot.asot.profile_clock(kind)
    assert 300.0 < mhz < 2500.0, mhz
    with pytest.raises(Exception):
        asot.asot.profile_clock(0)


def test_map_ws_entry_point(asot):
    """asot_map_to_anchors_ws (include/asot.h): the same bits as asot_map_to_anchors, peer stores at
    row_base, the status flags of the exact kernel, ASOT_ERR_WORKSPACE on a short or misaligned
    workspace, an empty distribution and ragged point counts."""
    import ctypes
    import paper_2310_16123_b200.asot as A
    from paper_2310_16123_b200 import _lib
    inp = make_inputs("c3", n_dist=37)
    pts, offs, w, anc = dev(inp.points), dev(inp.offsets), dev(inp.weights), dev(inp.anchors)
    a0, H0, _ = A.map_to_anchors(pts, offs, w, anc, offsets_host=inp.offsets)
    # peers: two full matrices of 50 rows, this call's rows land at row 9
    full = [torch.full((50, inp.n_anchors), -1.0, device="cuda") for _ in range(2)]
    peers = torch.tensor([f.data_ptr() for f in full], dtype=torch.int64, device="cuda")
    a1, H1, st = A.map_to_anchors_bcast(pts, offs, w, anc, peers, 9, offsets_host=inp.offsets,
                                        tensor_core=True)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    assert torch.equal(a0, a1) and torch.equal(H0, H1)
    for f in full:
        assert torch.equal(f[9:9 + 37], H0)
        assert bool((f[:9] == -1).all()) and bool((f[46:] == -1).all())
    # flags: NaN coordinate (no anchor decided on the tensor cores either) and an empty distribution
    p2 = inp.points.copy(); p2[4, 1] = np.nan
    offs2 = inp.offsets.copy(); offs2[3] = offs2[2]
    st = A.new_status()
    A.map_to_anchors(dev(p2), dev(offs2), w, anc, offsets_host=offs2, status=st, tensor_core=True)
    torch.cuda.synchronize()
    assert int(st.item()) & A.FLAG_NONFINITE_INPUT and int(st.item()) & A.FLAG_EMPTY_DIST
    # workspace errors through the C-ABI itself
    lib = _lib.load()
    T, K, d = int(inp.offsets[-1]), inp.n_anchors, inp.points.shape[1]
    need = int(lib.asot_map_workspace_bytes(T, K))
    assert need > 0 and need % 256 == 0
    ws = torch.empty(need + 256, dtype=torch.uint8, device="cuda")
    asg = torch.empty(T, dtype=torch.int32, device="cuda")
    H = torch.empty((37, K), dtype=torch.float32, device="cuda")
    st = A.new_status()
    oh = np.ascontiguousarray(inp.offsets, dtype=np.int64)
    call = lambda wp, wb: lib.asot_map_to_anchors_ws(
        pts.data_ptr(), offs.data_ptr(), oh.ctypes.data, w.data_ptr(), 37, d, anc.data_ptr(), K,
        asg.data_ptr(), H.data_ptr(), None, 0, 0, st.data_ptr(), wp, wb, None)
    assert call(ws.data_ptr(), need - 1) == 6   # ASOT_ERR_WORKSPACE
    assert call(ws.data_ptr() + 16, need) == 6   # ASOT_ERR_WORKSPACE
    assert call(None, need) == 6   # ASOT_ERR_WORKSPACE
    assert call(ws.data_ptr(), need) == 0
    torch.cuda.synchronize()
    assert torch.equal(asg, a0) and torch.equal(H, H0)
