import ctypes, os, sys, numpy as np, torch
os.environ["ASOT_TC_DEBUG_MODE"] = "3"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from asot_inputs import make_inputs
import paper_2310_16123_b200 as asot
from paper_2310_16123_b200 import _lib
inp = make_inputs("c5", n_dist=300)
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
D = asot.distance_matrix(t(inp.points), t(inp.offsets), t(inp.weights), t(inp.anchors), t(inp.cost), float(inp.eps), inp.iters, offsets_host=inp.offsets, cost_max=1.0)
torch.cuda.synchronize()
buf = np.zeros((5, 256), np.int64)
lib = _lib.load()
lib.asot_debug_tc4_trace.argtypes = [ctypes.c_void_p]
print("rc", lib.asot_debug_tc4_trace(buf.ctypes.data))
t0 = buf[4, 0]
for ps in range(0, 24):
    f = buf[:, ps] - t0
    print(ps, f"load0 {f[4]:8d}  mma_first {f[0]:8d}  mma_last {f[1]:8d} (+{f[1]-f[0]:6d})  epi_wake {f[2]:8d} (+{f[2]-f[1]:5d})  epi_done {f[3]:8d} (+{f[3]-f[2]:6d})")
d = np.diff(buf[0, 10:200])
print("mean pass period", d.mean(), "mean mma span", (buf[1,10:200]-buf[0,10:200]).mean(), "mean epi", (buf[3,10:200]-buf[2,10:200]).mean())
