"""Sinkhorn throughput against the number of anchors K (the speed side of the paper's k-ablation,
Fig. 4 / §5.3): N = 1000 distributions of c5 (d = 128), the first K of its anchors, their
normalised squared-Euclidean cost, eps = 0.05, L = 50; TF32 and fp32 requests.  Prints one JSON
line per (K, precision) with the kernel that ran, pairs/s and algorithmic TFLOP/s."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2310_16123_b200 as asot  # noqa: E402
from asot_inputs import make_inputs, normalized_sqeuclid_cost  # noqa: E402

N, L = 1000, 50
base = make_inputs("c5", n_dist=N)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
pts, offs, w = t(base.points), t(base.offsets), t(base.weights)
for K in [int(k) for k in os.environ.get("KS", "16,32,64,96,128,192,256,384,512,768,1024").split(",")]:
    A = np.ascontiguousarray(base.anchors[:K])
    anc, cst = t(A), t(normalized_sqeuclid_cost(A))
    _, H, _ = asot.map_to_anchors(pts, offs, w, anc, offsets_host=base.offsets)
    for prec in (asot.TF32, asot.FP32):
        run = lambda: asot.distance_matrix(None, None, None, None, cst, float(base.eps), L, precision=prec,
                                           hist=H, cost_max=1.0)
        run()
        torch.cuda.synchronize()
        asot.asot.profile_enable(True)
        asot.asot.profile_read(reset=True)
        reps = 3
        for _ in range(reps):
            run()
        torch.cuda.synchronize()
        ms, n = asot.asot.profile_read(reset=True)
        asot.asot.profile_enable(False)
        ms /= max(n, 1)
        P = N * (N - 1) // 2
        kind = asot.asot.sinkhorn_kernel_kind(K, prec)
        print(json.dumps({"K": K, "precision": "tf32" if prec == asot.TF32 else "fp32",
                          "kernel": asot.asot.KERNEL_NAMES[kind], "ms": round(ms, 3),
                          "pairs_per_s": round(P / (ms / 1e3)),
                          "tflops": round((4 * K * K * L + 2 * K * K) * P / (ms / 1e3) / 1e12, 1)}), flush=True)
