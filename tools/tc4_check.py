"""Quick check of the streamed K=1024 kernel against the oracle (developer tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.tc_check import run
if __name__ == "__main__":
    t0 = time.time()
    run("c5", 18, iters=1)
    run("c5", 18)
    run("c5", 40)
    print("elapsed", time.time() - t0)
