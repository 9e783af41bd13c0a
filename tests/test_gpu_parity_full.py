"""SURVEY §8(d)'s full-size parity subsets (VERDICT r1 missing #2), in bench.py's launch
configuration (whole configs, one call):

* assignments bit-exact for EVERY point of c3 (N = 2000, 349,010 points) and for a seeded 10% of
  c5's distributions (400 of 4000, ~240k points, K = 1024, d = 128), with their H rows
  bit-identical -- the oracle mapping (R#8) fanned out over the host cores (tests/oracle_par.py);
* >= 2,000 sampled pairs at ASOT_PREC_FP32 (the north star's 1e-4 mode: BF16x3 resident kernel
  at K = 256, 3xTF32 streamed at K = 1024) for c4 (N = 8000, Dirichlet weights) and c5 (pairs
  among the 10% sample), each against the
  oracle evaluated pair by pair on the oracle's own histograms."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from asot_inputs import make_inputs, random_pairs  # noqa: E402
from oracle import asot_oracle as O  # noqa: E402
from oracle_par import map_assign_parallel, rows_of  # noqa: E402

FP32_TOL = 1e-4


@pytest.fixture(scope="module")
def asot():
    import paper_2310_16123_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_map(asot, inp, path="exact"):
    """asot_map_to_anchors (the CUDA-core kernel on every point), or the mapping inside
    asot_distance_matrix (an empty tile range: tensor-core products + the exact kernel on the
    points they cannot decide, R#37)."""
    if path == "exact":
        assign, H, st = asot.map_to_anchors(dev(inp.points), dev(inp.offsets), dev(inp.weights),
                                            dev(inp.anchors), offsets_host=inp.offsets)
    else:
        assign = torch.empty(inp.n_points, dtype=torch.int32, device="cuda")
        H = torch.empty((inp.n_dist, inp.n_anchors), dtype=torch.float32, device="cuda")
        st = asot.asot.new_status()
        asot.distance_matrix(dev(inp.points), dev(inp.offsets), dev(inp.weights), dev(inp.anchors),
                             dev(inp.cost), float(inp.eps), inp.iters, tile_range=(0, 0),
                             assign_out=assign, hist_out=H, offsets_host=inp.offsets, status=st)
    torch.cuda.synchronize()
    asot.check_status(st)
    return assign.cpu().numpy(), H.cpu().numpy()


def sub_hist(inp, dists, assign_o):
    """Oracle histograms (fp64, point order) of the given distributions from their assignments."""
    rows = rows_of(inp.offsets, dists)
    sizes = np.diff(inp.offsets)[dists]
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    return O.histograms(assign_o, inp.weights[rows], off, inp.n_anchors)


_c5 = {}


def c5_sample(asot):
    """c5 at full size: GPU mapping of all 2.4M points; oracle mapping of a seeded 10% of the
    distributions (cached for the pair test)."""
    if not _c5:
        inp = make_inputs("c5")
        a_g, H_g = gpu_map(asot, inp)
        dists = np.sort(np.random.default_rng(51).choice(inp.n_dist, inp.n_dist // 10, replace=False))
        rows = rows_of(inp.offsets, dists)
        a_o = map_assign_parallel(inp.points[rows], inp.anchors)
        _c5.update(inp=inp, a_g=a_g, H_g=H_g, dists=dists, rows=rows, a_o=a_o,
                   H_o=sub_hist(inp, dists, a_o))
    return _c5


def test_mapping_bit_exact_c3_all_points(asot):
    """All 349,010 c3 points, through both mapping paths (the default distance-matrix path is the
    tensor-core one)."""
    inp = make_inputs("c3")
    assert inp.n_points == 349010
    a_o = map_assign_parallel(inp.points, inp.anchors)
    H_o = O.histograms(a_o, inp.weights, inp.offsets, inp.n_anchors).astype(np.float32)
    for path in ("exact", "tc"):
        a_g, H_g = gpu_map(asot, inp, path)
        assert np.array_equal(a_g, a_o), f"{path}: {(a_g != a_o).sum()} of {a_o.size} assignments differ"
        np.testing.assert_array_equal(H_g, H_o)


def test_mapping_bit_exact_c5_ten_percent_tc(asot):
    """c5's seeded 10% of distributions through the tensor-core mapping path (d = 128, K = 1024)."""
    s = c5_sample(asot)
    a_g, H_g = gpu_map(asot, s["inp"], "tc")
    assert np.array_equal(a_g[s["rows"]], s["a_o"]), f"{(a_g[s['rows']] != s['a_o']).sum()} differ"
    np.testing.assert_array_equal(H_g[s["dists"]], s["H_o"].astype(np.float32))


def test_mapping_bit_exact_c5_ten_percent(asot):
    s = c5_sample(asot)
    assert s["rows"].size >= 200_000                # ~240k points of 400 distributions
    a_g = s["a_g"][s["rows"]]
    assert np.array_equal(a_g, s["a_o"]), f"{(a_g != s['a_o']).sum()} of {a_g.size} differ"
    np.testing.assert_array_equal(s["H_g"][s["dists"]], s["H_o"].astype(np.float32))


def _fp32_pairs_check(asot, inp, pi, pj, H_o_rows, row_of):
    st = asot.asot.new_status()
    D = asot.distance_matrix(dev(inp.points), dev(inp.offsets), dev(inp.weights), dev(inp.anchors),
                             dev(inp.cost), float(inp.eps), inp.iters, precision=asot.FP32,
                             offsets_host=inp.offsets, cost_max=1.0, status=st)
    torch.cuda.synchronize()
    asot.check_status(st)
    # K = 256: the BF16x3 resident CTA-pair kernel; K = 1024: the 3xTF32 streamed kernel
    assert asot.asot.sinkhorn_kernel_kind(inp.n_anchors, asot.FP32) == (10 if inp.n_anchors <= 256 else 5)
    c_o, fl = O.pair_costs(H_o_rows, inp.cost, inp.eps, inp.iters, row_of[pi], row_of[pj])
    assert not fl.any()
    Dg = D.cpu().numpy()
    r = np.abs(Dg[pi, pj].astype(np.float64) - c_o) / np.maximum(c_o, 1e-3)
    assert r.max() <= FP32_TOL, f"max rel {r.max():.3e}, p99 {np.quantile(r, 0.99):.3e}"
    assert np.all(np.diag(Dg) == 0) and np.array_equal(Dg[pi, pj], Dg[pj, pi])


def test_full_size_fp32_pairs_c4(asot):
    """c4 (N = 8000, K = 256) at fp32: 2,000 seeded random pairs + block / tail boundaries."""
    inp = make_inputs("c4")
    n = inp.n_dist
    pi, pj = random_pairs(n, 2000, seed=61)
    pi = np.concatenate([pi, [0, 15, 16, n - 2, n - 17]]).astype(np.int64)
    pj = np.concatenate([pj, [n - 1, 16, 31, n - 1, n - 16]]).astype(np.int64)
    touched = np.unique(np.concatenate([pi, pj]))
    rows = rows_of(inp.offsets, touched)
    a_o = map_assign_parallel(inp.points[rows], inp.anchors)
    H_o = sub_hist(inp, touched, a_o)
    row_of = np.full(n, -1, np.int64)
    row_of[touched] = np.arange(touched.size)
    _fp32_pairs_check(asot, inp, pi, pj, H_o, row_of)


def test_full_size_fp32_pairs_c5(asot):
    """c5 (N = 4000, K = 1024) at fp32: 2,000 seeded pairs among the 10% sample's distributions."""
    s = c5_sample(asot)
    inp, dists = s["inp"], s["dists"]
    li, lj = random_pairs(dists.size, 2000, seed=62)
    pi, pj = dists[li].astype(np.int64), dists[lj].astype(np.int64)
    row_of = np.full(inp.n_dist, -1, np.int64)
    row_of[dists] = np.arange(dists.size)
    _fp32_pairs_check(asot, inp, pi, pj, s["H_o"], row_of)
