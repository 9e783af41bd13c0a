"""Quick TF32 tensor-core path check on small configs (developer tool; uses the oracle)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from asot_inputs import make_inputs  # noqa: E402
from oracle import asot_oracle as O  # noqa: E402
import paper_2310_16123_b200 as asot  # noqa: E402


def run(cfg, n, iters=None):
    inp = make_inputs(cfg, n_dist=n, iters=iters)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    pts, offs, w, anc, cst = t(inp.points), t(inp.offsets), t(inp.weights), t(inp.anchors), t(inp.cost)
    st = asot.asot.new_status()
    D = asot.distance_matrix(pts, offs, w, anc, cst, float(inp.eps), inp.iters, precision=asot.TF32,
                             offsets_host=inp.offsets, status=st)
    torch.cuda.synchronize()
    Dg = D.cpu().numpy().astype(np.float64)
    Do, _, _ = O.distance_matrix(inp.points, inp.offsets, inp.weights, inp.anchors, inp.cost,
                                 inp.eps, inp.iters)
    r = np.abs(Dg - Do) / np.maximum(Do, 1e-3)
    print(f"{cfg} N={n} K={inp.n_anchors} L={inp.iters} eff={asot.effective_precision(inp.n_anchors, 1)} "
          f"status={int(st.item())} max rel {r.max():.3e} p50 {np.median(r):.3e} "
          f"nan={np.isnan(Dg).sum()} sample gpu {Dg[0, 1:4]} orc {Do[0, 1:4]}", flush=True)


if __name__ == "__main__":
    t0 = time.time()
    run("c1", 20, iters=1)
    run("c1", 64)
    run("c2", 90)
    print("elapsed", time.time() - t0)
