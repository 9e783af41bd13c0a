"""Timeline of the CTA-pair kernel (ASOT_TC_DEBUG_MODE=3, CTA 0's first tile): per phase, when
each anchor half's epilogue woke (D half ready) and finished.  Developer tool."""
import ctypes, os, sys
import numpy as np
os.environ["ASOT_TC_DEBUG_MODE"] = os.environ.get("ASOT_TC_DEBUG_MODE", "3")  # 4: no math, 5: no TMEM ld/st
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
buf = np.zeros((18, 256), np.int64)
lib = _lib.load()
lib.asot_debug_tc2_trace.argtypes = [ctypes.c_void_p]
print("rc", lib.asot_debug_tc2_trace(buf.ctypes.data))
w0, w1, e0, e1, i12s, i12e, i34s, i34e = buf[:8]
hd = buf[8:12]
gt = buf[12:16]
sl = slice(20, 190)
print("phase period (wake h0 -> next wake h0):", np.mean(np.diff(w0[20:191])))
print("epilogue h0 duration:", np.mean(e0[sl] - w0[sl]), " h1:", np.mean(e1[sl] - w1[sl]))
print("wake h1 - wake h0:", np.mean(w1[sl] - w0[sl]))
print("next wake h0 - end epi h0:", np.mean(w0[21:191] - e0[20:190]))
print("next wake h0 - end epi h1:", np.mean(w0[21:191] - e1[20:190]))
print("ideal MMA cycles per phase (4 parts x 16 x 64):", 4 * 16 * 64)
for f in range(30, 36):
    print(f, "w0", w0[f] - w0[30], "e0", e0[f] - w0[30], "w1", w1[f] - w0[30], "e1", e1[f] - w0[30],
          "| issue p12(f+1)", i12s[f + 1] - w0[30], "..", i12e[f + 1] - w0[30],
          " p34(f+1)", i34s[f + 1] - w0[30], "..", i34e[f + 1] - w0[30])
print("half_done - own wake (h0 leader, h0 peer, h1 leader, h1 peer):", [float(np.mean(hd[r][sl])) for r in range(4)])
print("globaltimer ns: peer wake h0 - leader wake h0:", float(np.mean(gt[1][sl] - gt[0][sl])),
      " leader wake h1 - leader wake h0:", float(np.mean(gt[2][sl] - gt[0][sl])),
      " peer wake h1 - leader wake h0:", float(np.mean(gt[3][sl] - gt[0][sl])))
print("sample", gt[0][30:34] - gt[0][30], gt[1][30:34] - gt[0][30])
print("p12 wait: enter, leave (rel. w0 of previous phase):", [(int(buf[16][f + 1] - w0[f]), int(buf[17][f + 1] - w0[f])) for f in range(30, 34)])
