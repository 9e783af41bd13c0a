"""Quick check of the K=256 CTA-pair kernel against the oracle (developer tool)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.tc_check import run
if __name__ == "__main__":
    t0 = time.time()
    run("c3", 40, iters=1)
    run("c3", 40)
    run("c4", 50)
    run("c3", 200)
    print("elapsed", time.time() - t0)
