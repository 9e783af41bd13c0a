"""Timeline of the 1-SM resident kernel (ASOT_TC_DEBUG_MODE=3, CTA 0's first tile per slot): per
slot and phase, when the epilogue woke for D chunk 0 / 1 and when the MMA warp passed the chunk
gates of the next phase.  Developer tool."""
import ctypes, os, sys
import numpy as np
os.environ["ASOT_TC_DEBUG_MODE"] = os.environ.get("ASOT_TC_DEBUG_MODE", "3")  # 4: no epilogue
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from asot_inputs import make_inputs  # noqa: E402
import paper_2310_16123_b200 as asot  # noqa: E402
from paper_2310_16123_b200 import _lib  # noqa: E402

inp = make_inputs("c2")
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
D = asot.distance_matrix(t(inp.points), t(inp.offsets), t(inp.weights), t(inp.anchors), t(inp.cost),
                         float(inp.eps), inp.iters, offsets_host=inp.offsets, cost_max=1.0)
torch.cuda.synchronize()
buf = np.zeros((2, 4, 512), np.int64)
lib = _lib.load()
lib.asot_debug_tc_trace.argtypes = [ctypes.c_void_p]
print("rc", lib.asot_debug_tc_trace(buf.ctypes.data))
t0 = buf[0, 0, 20]
for f in range(20, 26):
    print(f, " | ".join(f"s{s}: wake {buf[s, 0, f] - t0:6d} {buf[s, 1, f] - t0:6d}  gates(f+1) "
                        f"{buf[s, 2, f + 1] - t0:6d} {buf[s, 3, f + 1] - t0:6d}" for s in range(2)))
for s in range(2):
    print("slot", s, "period", np.mean(np.diff(buf[s, 0, 10:300])),
          "ideal (two 16-MMA chains of M128 N128 k8):", 2 * 16 * 64.6)
