import ctypes, os, sys, numpy as np, torch
os.environ["ASOT_TC_DEBUG_MODE"] = "3"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from asot_inputs import make_inputs
import paper_2310_16123_b200 as asot
from paper_2310_16123_b200 import _lib
inp = make_inputs("c2")
t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
D = asot.distance_matrix(t(inp.points), t(inp.offsets), t(inp.weights), t(inp.anchors), t(inp.cost), float(inp.eps), inp.iters, offsets_host=inp.offsets, cost_max=1.0)
torch.cuda.synchronize()
buf = np.zeros((2, 4, 512), np.int64)
lib = _lib.load()
lib.asot_debug_tc_trace.argtypes = [ctypes.c_void_p]
print("rc", lib.asot_debug_tc_trace(buf.ctypes.data))
t0 = buf[:, 0, 0].min()
# events: 0 wake, 3 after slot barrier, 1 after turn wait, 2 after issue+commit
for f in range(20, 30):
    row = []
    for s_ in range(2):
        w, b, t, i = [buf[s_, k, f] - t0 for k in (0, 3, 1, 2)]
        row.append(f"s{s_}: wake {w:7d} bar +{b-w:5d} turn +{t-b:5d} issue +{i-t:5d}")
    print(f, " | ".join(row))
for s_ in range(2):
    sl = slice(10, 390)
    w, b, t, i = [buf[s_, k, sl] for k in (0, 3, 1, 2)]
    wn = buf[s_, 0, 11:391]
    print("slot", s_, "epi+bar", np.mean(b - w), "turn", np.mean(t - b), "issue", np.mean(i - t), "wait", np.mean(wn - i), "period", np.mean(np.diff(buf[s_, 0, 10:391])))
