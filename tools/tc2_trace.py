"""Timeline of the CTA-pair kernel (ASOT_TC_DEBUG_MODE=3, CTA 0's first tile): per phase and
anchor chunk, when the epilogue woke (D chunk ready) and finished, and when the MMA warp passed
the chunk's epilogue barrier.  Developer tool."""
import ctypes, os, sys
import numpy as np
os.environ["ASOT_TC_DEBUG_MODE"] = os.environ.get("ASOT_TC_DEBUG_MODE", "3")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from asot_inputs import make_inputs  # noqa: E402
import paper_2310_16123_b200 as asot  # noqa: E402
from paper_2310_16123_b200 import _lib  # noqa: E402

inp = make_inputs("c3", n_dist=int(sys.argv[1]) if len(sys.argv) > 1 else 600)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
D = asot.distance_matrix(t(inp.points), t(inp.offsets), t(inp.weights), t(inp.anchors), t(inp.cost),
                         float(inp.eps), inp.iters, offsets_host=inp.offsets, cost_max=1.0)
torch.cuda.synchronize()
buf = np.zeros((4, 256), np.int64)
lib = _lib.load()
lib.asot_debug_tc2_trace.argtypes = [ctypes.c_void_p]
print("rc", lib.asot_debug_tc2_trace(buf.ctypes.data))
wake, done, issue = (buf[r].reshape(64, 4) for r in range(3))
print("phase period (chunk-0 wake to next):", np.mean(np.diff(wake[10:60, 0])))
print("epilogue chunk durations:", np.mean(done[10:60] - wake[10:60], axis=0))
print("ideal MMA cycles per phase (128 x M256 N64 k8 at 32.7):", 128 * 32.7)
for f in range(20, 24):
    base = wake[f, 0]
    print(f, "wake", wake[f] - base, "done", done[f] - base, "| next-phase issue", issue[f + 1] - base)
print("cost section per tile (cycles, CTA 0, first tiles):", buf[3][:8], "phase period x 2L:", np.mean(np.diff(wake[10:60, 0])) * 2 * inp.iters)
