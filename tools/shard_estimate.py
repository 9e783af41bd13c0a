"""Per-rank work of the N-GPU tile sharding, measured on ONE GPU: for world size W, time each
rank's share (mapping of its distribution range + Sinkhorn on its tile range, p2p-style output
into a full matrix) sequentially on this GPU and report max over ranks vs the 1-GPU step -- the
compute part of strong-scaling efficiency (the exchanges -- a 4NK-byte all-gather and NVLink
stores -- are not included).  Developer tool:  python tools/shard_estimate.py c3 1 2 4 8"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from asot_inputs import make_inputs  # noqa: E402
import paper_2310_16123_b200 as asot  # noqa: E402
from paper_2310_16123_b200.distributed import partition_by_points, partition_even  # noqa: E402

cfg = sys.argv[1]
worlds = [int(w) for w in sys.argv[2:]] or [1, 2, 4, 8]
inp = make_inputs(cfg)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
pts, offs, w, anc, cst = t(inp.points), t(inp.offsets), t(inp.weights), t(inp.anchors), t(inp.cost)
_, H, _ = asot.map_to_anchors(pts, offs, w, anc, offsets_host=inp.offsets)
D = torch.empty((inp.n_dist, inp.n_dist), dtype=torch.float32, device="cuda")
nt = asot.num_tiles(inp.n_dist)


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


base = None
for W in worlds:
    ranks = []
    for r in range(W):
        lo, hi = partition_by_points(inp.offsets, W)[r]
        s, e = int(inp.offsets[lo]), int(inp.offsets[hi])
        sub = inp.offsets[lo:hi + 1] - s
        subd = t(sub)
        t_map = timed(lambda: asot.map_to_anchors(pts[s:e], subd, w[s:e], anc, offsets_host=sub)) if hi > lo else 0.0
        t0, t1 = partition_even(nt, W)[r]
        t_sk = timed(lambda: asot.distance_matrix(None, None, None, None, cst, float(inp.eps), inp.iters,
                                                  hist=H, tile_range=(t0, t1), want_matrix=False,
                                                  out_ptr=D.data_ptr(), cost_max=1.0)) if t1 > t0 else 0.0
        ranks.append(t_map + t_sk)
    worst = max(ranks)
    base = base if base is not None else worst * W
    print(f"{cfg} W={W}: max rank {worst:.2f} ms (min {min(ranks):.2f}), ideal {base / W:.2f} ms, "
          f"compute efficiency {base / W / worst:.3f}")
