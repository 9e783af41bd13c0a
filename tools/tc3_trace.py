"""Timeline of the 3xTF32 resident kernel (ASOT_TC_DEBUG_MODE=3, CTA 0's first tile, c2 fp32): per
phase when the epilogue woke for D half 0 / 1, when it arrived on the x-half barriers, and when the
MMA warp passed them.  Developer tool."""
import ctypes, os, sys
import numpy as np
os.environ["ASOT_TC_DEBUG_MODE"] = "3"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from asot_inputs import make_inputs  # noqa: E402
import paper_2310_16123_b200 as asot  # noqa: E402
from paper_2310_16123_b200 import _lib  # noqa: E402

inp = make_inputs("c2", n_dist=300)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
D = asot.distance_matrix(t(inp.points), t(inp.offsets), t(inp.weights), t(inp.anchors), t(inp.cost),
                         float(inp.eps), inp.iters, precision=asot.FP32, offsets_host=inp.offsets, cost_max=1.0)
torch.cuda.synchronize()
buf = np.zeros((6, 256), np.int64)
lib = _lib.load()
lib.asot_debug_tc3_trace.argtypes = [ctypes.c_void_p]
print("rc", lib.asot_debug_tc3_trace(buf.ctypes.data))
for f in range(20, 26):
    b = buf[0, f]
    print(f, "wake", buf[0, f] - b, buf[1, f] - b, " x-arrive", buf[2, f] - b, buf[3, f] - b,
          " issuer gates (f+1)", buf[4, f + 1] - b, buf[5, f + 1] - b)
print("period", np.mean(np.diff(buf[0, 10:200])), "ideal (96 MMAs of M128 N64 k8 at 32.3):", 96 * 32.3)
