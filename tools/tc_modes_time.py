"""Kernel time of the Sinkhorn kernel under ASOT_TC_DEBUG_MODE (0 normal, 1 no epilogue math,
2 no MMAs) for one config.  Developer tool: python tools/tc_modes_time.py c3 600 <mode>"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
cfg, n, mode = sys.argv[1], int(sys.argv[2]), sys.argv[3]
os.environ["ASOT_TC_DEBUG_MODE"] = mode
import torch  # noqa: E402
from asot_inputs import make_inputs  # noqa: E402
import paper_2310_16123_b200 as asot  # noqa: E402
inp = make_inputs(cfg, n_dist=n)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
args = (t(inp.points), t(inp.offsets), t(inp.weights), t(inp.anchors), t(inp.cost), float(inp.eps), inp.iters)
for _ in range(3):
    asot.distance_matrix(*args, offsets_host=inp.offsets, cost_max=1.0)
torch.cuda.synchronize()
asot.asot.profile_enable(True)
asot.asot.profile_read(reset=True)
for _ in range(5):
    asot.distance_matrix(*args, offsets_host=inp.offsets, cost_max=1.0)
torch.cuda.synchronize()
ms, nl = asot.asot.profile_read(reset=True)
K, L = inp.n_anchors, inp.iters
P = n * (n - 1) // 2
print(f"{cfg} N={n} mode={mode}: {ms / nl:.3f} ms/launch, {(4*K*K*L + 2*K*K) * P / (ms / nl / 1e3) / 1e12:.1f} TFLOP/s")
