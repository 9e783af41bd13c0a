"""Bucketed explicit pair lists (asot_pairs_bucket.cu): the tiles of the upper
triangle that a list covers completely run on the tile kernels, every other entry on the
pair-list mode.  Checked, through the C ABI, against
  * the tile path (asot_distance_matrix) -- bitwise, for the entries the tiles serve,
  * the plain pair-list path (the smaller asot_pairwise_workspace_bytes workspace) -- bitwise for
    the entries that stay on it (and at K <= 128 for every entry: both are the 1-SM kernel),
  * the fp64 oracle on a sample (TF32 bar 2e-3, R#20),
on lists mixing a complete triangle with reversed, diagonal, repeated and out-of-range entries,
partly covered tiles and no covered tile at all."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

from asot_inputs import make_inputs, random_pairs  # noqa: E402
from oracle import asot_oracle as O  # noqa: E402

TF32, FP32 = 1, 0
TOL = {FP32: 1e-4, TF32: 2e-3}
FLAG_BAD_INDEX = 128


@pytest.fixture(scope="module")
def asot():
    import paper_2310_16123_b200 as m
    return m


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def setup(asot, cfg, n):
    inp = make_inputs(cfg, n_dist=n)
    _, H, _ = asot.map_to_anchors(t(inp.points), t(inp.offsets), t(inp.weights), t(inp.anchors),
                                  offsets_host=inp.offsets)
    torch.cuda.synchronize()
    return inp, H


def run_list(asot, inp, H, pi, pj, bucket, guard=0, prec=TF32):
    """asot_pairwise_sinkhorn with the bucketed (list) or the plain workspace; returns the
    results (guard region after them untouched) and the status word."""
    from paper_2310_16123_b200 import _lib
    L = _lib.load()
    n, K = len(pi), inp.n_anchors
    nbytes = (L.asot_pairwise_list_workspace_bytes(inp.n_dist, K, prec, n) if bucket
              else L.asot_pairwise_workspace_bytes(inp.n_dist, K, prec))
    ws = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device="cuda")
    out = torch.full((n + guard,), -7.0, dtype=torch.float32, device="cuda")
    st = asot.asot.new_status()
    qi, qj, C = t(pi.astype(np.int32)), t(pj.astype(np.int32)), t(inp.cost)
    rc = L.asot_pairwise_sinkhorn(H.data_ptr(), inp.n_dist, K, C.data_ptr(), float(inp.cost.max()),
                                  float(inp.eps), inp.iters, prec, qi.data_ptr(), qj.data_ptr(), n,
                                  out.data_ptr(), st.data_ptr(), ws.data_ptr(), ws.numel(), None)
    torch.cuda.synchronize()
    assert rc == 0, L.asot_last_error()
    o = out.cpu().numpy()
    if guard:
        assert np.all(o[n:] == -7.0), "write past dist_out[n_pairs]"
    return o[:n], int(st.cpu().numpy()[0])


def tile_matrix(asot, inp, H, prec=TF32):
    D = asot.distance_matrix(None, None, None, None, t(inp.cost), float(inp.eps), inp.iters,
                             precision=prec, hist=H, n_dist=inp.n_dist, cost_max=float(inp.cost.max()))
    torch.cuda.synchronize()
    return D.cpu().numpy()


def mixed_list(n, seed):
    """Every i < j pair once (shuffled) + reversed, diagonal, repeated and out-of-range entries."""
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, k=1)
    ri, rj = random_pairs(n, 300, seed=seed + 1)
    lo, hi = np.minimum(ri, rj), np.maximum(ri, rj)
    d = rng.integers(0, n, 20)
    rep = rng.integers(0, iu.size, 300)
    pi = np.concatenate([iu, hi, d, iu[rep], [-1, n, 0, 3, n + 5]])
    pj = np.concatenate([ju, lo, d, ju[rep], [1, 2, -4, n, 0]])
    perm = rng.permutation(pi.size)
    return pi[perm].astype(np.int64), pj[perm].astype(np.int64)


def valid_mask(pi, pj, n):
    return (pi >= 0) & (pj >= 0) & (pi < n) & (pj < n)


@pytest.mark.parametrize("prec", [TF32, FP32])
@pytest.mark.parametrize("cfg,n", [("c2", 150), ("c3", 90), ("c5", 40)])
def test_complete_triangle_plus_extras(asot, cfg, n, prec):
    inp, H = setup(asot, cfg, n)
    pi, pj = mixed_list(n, seed=7)
    ok = valid_mask(pi, pj, n)
    b, sb = run_list(asot, inp, H, pi, pj, bucket=True, guard=512, prec=prec)
    p, sp = run_list(asot, inp, H, pi, pj, bucket=False, prec=prec)
    assert sb & FLAG_BAD_INDEX and sp & FLAG_BAD_INDEX
    assert np.all(np.isnan(b[~ok])) and np.all(np.isnan(p[~ok]))
    D = tile_matrix(asot, inp, H, prec)
    up = ok & (pi < pj)
    tile_val = np.where(up, D[np.where(ok, pi, 0), np.where(ok, pj, 0)], np.nan)
    if inp.n_anchors <= 128 or (inp.n_anchors > 256 and prec == FP32):
        # one kernel serves both paths (the 1-SM kernels; the streamed 3xTF32 kernel's tile and
        # pair-list modes): every entry bitwise the plain path's value
        np.testing.assert_array_equal(b[ok], p[ok])
    # first occurrences of i < j are tile-served, every other entry stays on the list path;
    # which of two repeated entries the tile serves is unspecified: each is one of the two
    either = (b == tile_val) | (b == p)
    assert np.all(either[ok]), f"{(~either[ok]).sum()} entries match neither path"
    uniq = np.unique(np.stack([pi[up], pj[up]]), axis=1)
    assert uniq.shape[1] == n * (n - 1) // 2
    assert np.all(b[up] == tile_val[up]) or 128 < inp.n_anchors
    # the fp64 oracle on a sample of both kinds of entries
    Hd = H.cpu().numpy().astype(np.float64)
    idx = np.random.default_rng(3).choice(np.flatnonzero(ok), 60, replace=False)
    co, fl = O.pair_costs(Hd, inp.cost.astype(np.float64), float(inp.eps), inp.iters, pi[idx], pj[idx])
    cmax = float(inp.cost.max())
    rel = np.abs(b[idx] - co) / np.maximum(co, 1e-3 * cmax)
    assert rel.max() <= TOL[prec], rel.max()


def test_no_tile_covered(asot):
    """A sparse random list covers no tile: everything runs on the pair-list mode, bitwise."""
    inp, H = setup(asot, "c2", 400)
    pi, pj = random_pairs(400, 3000, seed=11)
    b, _ = run_list(asot, inp, H, pi, pj, bucket=True, guard=300)
    p, _ = run_list(asot, inp, H, pi, pj, bucket=False)
    np.testing.assert_array_equal(b, p)


@pytest.mark.parametrize("prec", [TF32, FP32])
@pytest.mark.parametrize("cfg,n", [("c2", 70), ("c3", 70), ("c5", 70)])
def test_partly_covered_tiles(asot, cfg, n, prec):
    """One block pair covered completely, a second one missing a single pair, plus the first
    16 distributions' pairs in both orientations: tile-served entries equal the tile path, the
    rest the list path."""
    inp, H = setup(asot, cfg, n)
    ii, jj = np.meshgrid(np.arange(16, 32), np.arange(48, 64), indexing="ij")     # block (1, 3)
    a_i, a_j = ii.ravel(), jj.ravel()
    ii, jj = np.meshgrid(np.arange(0, 16), np.arange(32, 48), indexing="ij")      # block (0, 2) - 1
    b_i, b_j = ii.ravel()[1:], jj.ravel()[1:]
    iu, ju = np.triu_indices(16, k=1)                                           # block (0, 0)
    xi, xj = np.arange(1200) % n, (np.arange(1200) * 7 + 3) % n                 # scattered extras,
    keep = ~((xi >= 16) & (xi < 32) & (xj >= 48) & (xj < 64))                   # none repeating a
    pi = np.concatenate([a_i, b_i, iu, ju, xi[keep]])                           # block (1, 3) pair
    pj = np.concatenate([a_j, b_j, ju, iu, xj[keep]])
    b, _ = run_list(asot, inp, H, pi, pj, bucket=True, guard=64, prec=prec)
    p, _ = run_list(asot, inp, H, pi, pj, bucket=False, prec=prec)
    D = tile_matrix(asot, inp, H, prec)
    na = a_i.size
    assert np.all(b[:na] == D[a_i, a_j])                  # the covered block pair: the tile path
    rest = np.arange(na, pi.size)
    if inp.n_anchors <= 128:
        np.testing.assert_array_equal(b, p)
    else:
        tile_val = np.where(pi < pj, D[pi, pj], np.nan)
        assert np.all((b[rest] == p[rest]) | (b[rest] == tile_val[rest]))


@pytest.mark.parametrize("prec", [TF32, FP32])
@pytest.mark.parametrize("cfg,n", [("c2", 20), ("c3", 23)])
def test_small_n_repeated_triangle(asot, cfg, n, prec):
    """A small, ragged N whose whole triangle appears six times (shuffled): every tile covered,
    five of six copies of each pair repeats on the list path; all copies of a pair agree with
    the tile path or the list path and, within the precision, with each other."""
    inp, H = setup(asot, cfg, n)
    iu, ju = np.triu_indices(n, k=1)
    perm = np.random.default_rng(17).permutation(6 * iu.size)
    pi, pj = np.tile(iu, 6)[perm], np.tile(ju, 6)[perm]
    assert pi.size >= 1024
    b, _ = run_list(asot, inp, H, pi, pj, bucket=True, guard=128, prec=prec)
    p, _ = run_list(asot, inp, H, pi, pj, bucket=False, prec=prec)
    D = tile_matrix(asot, inp, H, prec)
    tv = D[pi, pj]
    assert np.all((b == tv) | (b == p))
    rel = np.abs(b - tv) / np.maximum(tv, 1e-3 * float(inp.cost.max()))
    assert rel.max() <= TOL[prec]
    if inp.n_anchors <= 128:
        np.testing.assert_array_equal(b, p)
